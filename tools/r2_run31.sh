# 32-wide panels for 257..512 rows per CTA (FEAST_MID_WIDE) on C3 and C4
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r31_build.log 2>&1
FEAST_MID_WIDE=1 timeout 900 python -m pytest tests/test_gpu_projector.py -m gpu -x -q -k "tall or ragged" > gpurun_out/r31_tests.log 2>&1
tail -n 2 gpurun_out/r31_tests.log
B3="python bench.py --timing-only --config C3 --steps 3 --warmup 3"
FEAST_MID_WIDE=1 timeout 600 $B3 > gpurun_out/r31_ab_C3_mid.json 2>&1
timeout 600 $B3 > gpurun_out/r31_ab_C3_base.json 2>&1
FEAST_MID_WIDE=1 timeout 900 python bench.py --timing-only --config C4 --steps 3 --warmup 3 > gpurun_out/r31_ab_C4_mid.json 2>&1
for f in gpurun_out/r31_ab_*.json; do echo "$f $(grep -o '"ms_per_step": [0-9.]*' $f) $(grep -o '"reasons": [^]]*]' $f)"; done
