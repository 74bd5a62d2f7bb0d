# C2: 4-column register chunk for <= 256-row panels (experiment); C3 with the new defaults
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r26_build.log 2>&1
B="python bench.py --timing-only --config C2 --steps 20 --warmup 5"
for rep in 1 2; do
  timeout 300 $B > gpurun_out/r26_ab_C2_wc8_$rep.json 2>&1
  FEAST_PANEL_WC=4 timeout 300 $B > gpurun_out/r26_ab_C2_wc4_$rep.json 2>&1
done
FEAST_PANEL_WC=4 timeout 600 python -m pytest tests/test_gpu_projector.py -m gpu -x -q -k "ragged or layouts or swap_variants" > gpurun_out/r26_tests_wc4.log 2>&1
tail -n 2 gpurun_out/r26_tests_wc4.log
timeout 600 python bench.py --timing-only --config C3 --steps 3 --warmup 3 > gpurun_out/r26_ab_C3_new.json 2>&1
for f in gpurun_out/r26_ab_*.json; do echo "$f $(grep -o '"ms_per_step": [0-9.]*' $f) $(grep -o '"reasons": [^]]*]' $f)"; done
