# round-2 GPU run 4: sparse-swap coalesced kernel, outer-block / substitution block sizes on C3-C5
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_projector.py -x -q -k "swap or substitution or async" > gpurun_out/r2_gpu_tests_v4.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_gpu_tests_v4.log
B="python bench.py --timing-only"
for v in coalesced chain; do
  FEAST_LASWP=$v timeout 600 $B --config C2 --steps 20 --warmup 5 > gpurun_out/r2_ab4_C2_$v.json 2>&1
  FEAST_LASWP=$v FEAST_ABLATE=4 timeout 600 $B --config C2 --steps 20 --warmup 5 > gpurun_out/r2_ab4_C2_${v}_noswap.json 2>&1
done
timeout 600 $B --steps 2 --warmup 3 > gpurun_out/r2_ab4_C4_base.json 2>&1
FEAST_NBO=512 timeout 600 $B --steps 2 --warmup 3 > gpurun_out/r2_ab4_C4_nbo512.json 2>&1
FEAST_NBO=512 FEAST_SOLVE_NB=512 timeout 600 $B --steps 2 --warmup 3 > gpurun_out/r2_ab4_C4_nbo512_snb512.json 2>&1
FEAST_SOLVE_NB=512 timeout 600 $B --steps 2 --warmup 3 > gpurun_out/r2_ab4_C4_snb512.json 2>&1
FEAST_NBO=384 timeout 600 $B --steps 2 --warmup 3 > gpurun_out/r2_ab4_C4_nbo384.json 2>&1
timeout 600 $B --config C3 --steps 5 --warmup 3 > gpurun_out/r2_ab4_C3_base.json 2>&1
FEAST_NBO=512 timeout 600 $B --config C3 --steps 5 --warmup 3 > gpurun_out/r2_ab4_C3_nbo512.json 2>&1
timeout 900 $B --config C5 --steps 1 --warmup 3 > gpurun_out/r2_ab4_C5_base.json 2>&1
FEAST_NBO=512 timeout 900 $B --config C5 --steps 1 --warmup 3 > gpurun_out/r2_ab4_C5_nbo512.json 2>&1
tail -n 3 gpurun_out/r2_gpu_tests_v4.log
for f in gpurun_out/r2_ab4_*.json; do echo "$f $(grep -o '"ms_per_step": [0-9.]*' $f) $(grep -o '"reasons": [^]]*]' $f)"; done
