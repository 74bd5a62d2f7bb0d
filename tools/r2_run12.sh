# round-2 GPU run 12: row swaps fused into the shared-memory panel kernel
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_projector.py tests/test_gpu_iterate.py -x -q > gpurun_out/r2_gpu_tests_v12.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_gpu_tests_v12.log
B="python bench.py --timing-only --config C2 --steps 20 --warmup 5"
for ps in 1 0; do
  FEAST_PANEL_SWAP=$ps timeout 300 $B > gpurun_out/r2_ab12_C2_ps$ps.json 2>&1
  FEAST_PANEL_SWAP=$ps timeout 300 $B > gpurun_out/r2_ab12_C2_ps${ps}_b.json 2>&1
done
FEAST_ABLATE=4 timeout 300 $B > gpurun_out/r2_ab12_C2_noswap.json 2>&1
FEAST_ABLATE=4 timeout 300 $B > gpurun_out/r2_ab12_C2_noswap_b.json 2>&1
for ps in 1 0; do FEAST_PANEL_SWAP=$ps timeout 600 python bench.py --timing-only --steps 2 --warmup 3 > gpurun_out/r2_ab12_C4_ps$ps.json 2>&1; done
FEAST_PANEL_SWAP=1 timeout 300 python bench.py --timing-only --config C3 --steps 5 --warmup 3 > gpurun_out/r2_ab12_C3_ps1.json 2>&1
FEAST_PANEL_SWAP=0 timeout 300 python bench.py --timing-only --config C3 --steps 5 --warmup 3 > gpurun_out/r2_ab12_C3_ps0.json 2>&1
tail -n 3 gpurun_out/r2_gpu_tests_v12.log
for f in gpurun_out/r2_ab12_*.json; do echo "$f $(grep -o '"ms_per_step": [0-9.]*' $f) $(grep -o '"reasons": [^]]*]' $f)"; done
