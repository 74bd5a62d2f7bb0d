# NCCL callback test; panel row cap 128 (2 GEMM CTAs co-resident with a panel CTA) A/B; swap marginal
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r19_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_multirank.py -m gpu -x -q > gpurun_out/r19_tests.log 2>&1
tail -n 3 gpurun_out/r19_tests.log
B="python bench.py --timing-only --config C2 --steps 20 --warmup 5"
for rep in 1 2; do
  timeout 300 $B > gpurun_out/r19_ab_C2_base_$rep.json 2>&1
  FEAST_PANEL_ROWCAP=128 timeout 300 $B > gpurun_out/r19_ab_C2_cap128_$rep.json 2>&1
done
FEAST_ABLATE=4 timeout 300 $B > gpurun_out/r19_ab_C2_ablate4.json 2>&1
FEAST_ABLATE=1 timeout 300 $B > gpurun_out/r19_ab_C2_ablate1.json 2>&1
FEAST_PANEL_ROWCAP=128 FEAST_ABLATE=1 timeout 300 $B > gpurun_out/r19_ab_C2_cap128_ablate1.json 2>&1
timeout 300 python bench.py --timing-only --config C3 --steps 3 --warmup 3 > gpurun_out/r19_ab_C3_base.json 2>&1
FEAST_PANEL_ROWCAP=128 timeout 300 python bench.py --timing-only --config C3 --steps 3 --warmup 3 > gpurun_out/r19_ab_C3_cap128.json 2>&1
for f in gpurun_out/r19_ab_*.json; do echo "$f $(grep -o '"ms_per_step": [0-9.]*' $f) $(grep -o '"reasons": [^]]*]' $f)"; done
