# round-2 GPU run 5: fused block solve (btrsm) correctness and A/B; adaptive outer blocks
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_projector.py tests/test_gpu_iterate.py tests/test_gpu_next3.py -x -q > gpurun_out/r2_gpu_tests_v5.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_gpu_tests_v5.log
B="python bench.py --timing-only"
for v in 1 0; do
  FEAST_BTRSM=$v timeout 600 $B --config C2 --steps 20 --warmup 5 > gpurun_out/r2_ab5_C2_bt$v.json 2>&1
  FEAST_BTRSM=$v timeout 600 $B --steps 2 --warmup 3 > gpurun_out/r2_ab5_C4_bt$v.json 2>&1
done
FEAST_NBO=256 FEAST_SOLVE_NB=256 timeout 600 $B --steps 2 --warmup 3 > gpurun_out/r2_ab5_C4_nbo256.json 2>&1
timeout 600 python tools/phase_breakdown.py C2 > gpurun_out/r2_phase_C2.log 2>&1
FEAST_BTRSM=0 timeout 600 python tools/phase_breakdown.py C2 > gpurun_out/r2_phase_C2_bt0.log 2>&1
timeout 900 python tools/phase_breakdown.py C4 > gpurun_out/r2_phase_C4_v5.log 2>&1
tail -n 3 gpurun_out/r2_gpu_tests_v5.log
for f in gpurun_out/r2_ab5_*.json; do echo "$f $(grep -o '"ms_per_step": [0-9.]*' $f) $(grep -o '"reasons": [^]]*]' $f)"; done
