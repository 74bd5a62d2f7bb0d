# dot-form (left-looking) substitutions: parity tests, then A/B on C2, C3, C4
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r22_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_projector.py -m gpu -x -q -k "dot_form or column_counts or factor_cache or left" > gpurun_out/r22_tests.log 2>&1
tail -n 3 gpurun_out/r22_tests.log
B="python bench.py --timing-only --config C2 --steps 20 --warmup 5"
for rep in 1 2; do for d in 0 1; do FEAST_SUBST_DOT=$d timeout 300 $B > gpurun_out/r22_ab_C2_d${d}_$rep.json 2>&1; done; done
for d in 0 1; do FEAST_SUBST_DOT=$d timeout 600 python bench.py --timing-only --config C3 --steps 3 --warmup 3 > gpurun_out/r22_ab_C3_d$d.json 2>&1; done
for d in 0 1; do FEAST_SUBST_DOT=$d timeout 900 python bench.py --timing-only --config C4 --steps 3 --warmup 3 > gpurun_out/r22_ab_C4_d$d.json 2>&1; done
for f in gpurun_out/r22_ab_*.json; do echo "$f $(grep -o '"ms_per_step": [0-9.]*' $f) $(grep -o '"reasons": [^]]*]' $f)"; done
