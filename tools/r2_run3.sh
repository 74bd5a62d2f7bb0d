# round-2 GPU run 3: full GPU suite on the new swap / substitution / tall-panel kernels, C4 phase
# breakdown and A/B of the new kernels, C4 / C2 rank shares (predicted strong scaling), C4 timeline
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_build.log 2>&1
B="python bench.py --timing-only --steps 2 --warmup 3"
for v in 4 2 0; do FEAST_TALL_VARIANT=$v timeout 600 $B > gpurun_out/r2_ab_C4_tall$v.json 2>&1; done
FEAST_SOLVE_NB=64 timeout 600 $B > gpurun_out/r2_ab_C4_nb64.json 2>&1
FEAST_LASWP=chain timeout 600 $B > gpurun_out/r2_ab_C4_chain.json 2>&1
FEAST_NBO=512 timeout 600 $B > gpurun_out/r2_ab_C4_nbo512.json 2>&1
for v in coalesced chain perm; do
  FEAST_LASWP=$v timeout 600 python bench.py --timing-only --config C2 --steps 20 --warmup 5 > gpurun_out/r2_ab_C2_$v.json 2>&1
done
FEAST_SOLVE_NB=64 timeout 600 python bench.py --timing-only --config C2 --steps 20 --warmup 5 > gpurun_out/r2_ab_C2_nb64.json 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gpu_tests_v3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_gpu_tests_v3.log
timeout 900 python tools/phase_breakdown.py C4 --out gpurun_out/r2_phase_C4.json > gpurun_out/r2_phase_C4.log 2>&1
timeout 900 python tools/timeline.py C4 --out gpurun_out/r2_tl_C4.csv > gpurun_out/r2_tl_C4.log 2>&1
python tools/timeline_rate.py gpurun_out/r2_tl_C4.csv 40 > gpurun_out/r2_tl_C4_rate.log 2>&1
timeout 1200 python tools/rank_share_timing.py C4 --out gpurun_out/r2_share_C4.json > gpurun_out/r2_share_C4.log 2>&1
timeout 600 python tools/rank_share_timing.py C2 --steps 5 --out gpurun_out/r2_share_C2.json > gpurun_out/r2_share_C2.log 2>&1
tail -n 4 gpurun_out/r2_gpu_tests_v3.log gpurun_out/r2_phase*.log gpurun_out/r2_share*.log
grep -h ms_per_step gpurun_out/r2_ab_*.json | cut -c1-200
