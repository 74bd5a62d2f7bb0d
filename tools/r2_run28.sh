# very tall cluster panels (1025..2048 rows per CTA): tests, panel trace, C5 A/B
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r28_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_projector.py -m gpu -x -q -k "very_tall or tall_panel" > gpurun_out/r28_tests.log 2>&1
tail -n 3 gpurun_out/r28_tests.log
bash tools/build_panel_trace.sh > gpurun_out/r28_ptrace_build.log 2>&1
timeout 120 tools/panel_trace 8 16 32768 4 > gpurun_out/r28_ptrace_vtall.txt 2>&1
B5="python bench.py --timing-only --config C5 --steps 2 --warmup 3"
FEAST_VTALL=1 timeout 1500 $B5 > gpurun_out/r28_ab_C5_vtall.json 2>&1
timeout 1500 $B5 > gpurun_out/r28_ab_C5_base.json 2>&1
for f in gpurun_out/r28_ab_*.json; do echo "$f $(grep -o '"ms_per_step": [0-9.]*' $f) $(grep -o '"reasons": [^]]*]' $f)"; done
grep "end loop" gpurun_out/r28_ptrace_vtall.txt
