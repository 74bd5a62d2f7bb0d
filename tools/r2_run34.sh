# inner dot-form substitution blocks (FEAST_SUBST_INNER_DOT) A/B on C4 / C3, parity tests
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r34_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_projector.py -m gpu -x -q > gpurun_out/r34_tests.log 2>&1
tail -n 2 gpurun_out/r34_tests.log
for v in 0 1; do
  FEAST_SUBST_INNER_DOT=$v timeout 900 python bench.py --timing-only --config C4 --steps 3 --warmup 3 > gpurun_out/r34_ab_C4_i$v.json 2>&1
  FEAST_SUBST_INNER_DOT=$v timeout 600 python bench.py --timing-only --config C3 --steps 3 --warmup 3 > gpurun_out/r34_ab_C3_i$v.json 2>&1
done
for f in gpurun_out/r34_ab_*.json; do echo "$f $(grep -o '"ms_per_step": [0-9.]*' $f) $(grep -o '"reasons": [^]]*]' $f)"; done
