# outer U12 in dot form (FEAST_U12_DOT) A/B on C4 / C3 / C5, parity tests
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r33_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_projector.py -m gpu -x -q -k "u12_dot or substitution_dot or factor_cache" > gpurun_out/r33_tests.log 2>&1
tail -n 2 gpurun_out/r33_tests.log
for v in 0 1; do
  FEAST_U12_DOT=$v timeout 900 python bench.py --timing-only --config C4 --steps 3 --warmup 3 > gpurun_out/r33_ab_C4_u$v.json 2>&1
  FEAST_U12_DOT=$v timeout 600 python bench.py --timing-only --config C3 --steps 3 --warmup 3 > gpurun_out/r33_ab_C3_u$v.json 2>&1
done
for v in 0 1; do
  FEAST_U12_DOT=$v timeout 1200 python bench.py --timing-only --config C5 --steps 2 --warmup 3 > gpurun_out/r33_ab_C5_u$v.json 2>&1
done
for f in gpurun_out/r33_ab_*.json; do echo "$f $(grep -o '"ms_per_step": [0-9.]*' $f) $(grep -o '"reasons": [^]]*]' $f)"; done
