# very tall panels with a 2-column register chunk (experiment) on C5; C4 on the session-2 defaults
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r29_build.log 2>&1
FEAST_VTALL=2 timeout 900 python -m pytest tests/test_gpu_projector.py -m gpu -x -q -k "very_tall" > gpurun_out/r29_tests.log 2>&1
tail -n 2 gpurun_out/r29_tests.log
FEAST_VTALL=2 timeout 1500 python bench.py --timing-only --config C5 --steps 2 --warmup 3 > gpurun_out/r29_ab_C5_vtall2.json 2>&1
timeout 900 python bench.py --timing-only --config C4 --steps 3 --warmup 3 > gpurun_out/r29_ab_C4_s2.json 2>&1
for f in gpurun_out/r29_ab_*.json; do echo "$f $(grep -o '"ms_per_step": [0-9.]*' $f) $(grep -o '"reasons": [^]]*]' $f)"; done
