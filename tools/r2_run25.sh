# large-batch defaults (2 groups, full first block), tall panel variant 5 (4-column register chunk)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r25_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_projector.py -m gpu -x -q -k "tall or dot_form or register_panel or ragged" > gpurun_out/r25_tests.log 2>&1
tail -n 3 gpurun_out/r25_tests.log
bash tools/build_panel_trace.sh > gpurun_out/r25_ptrace_build.log 2>&1
for v in 4 5; do FEAST_TALL_VARIANT=$v timeout 120 tools/panel_trace 16 16 16384 8 > gpurun_out/r25_ptrace_tall_v$v.txt 2>&1; done
B4="python bench.py --timing-only --config C4 --steps 3 --warmup 3"
timeout 900 $B4 > gpurun_out/r25_ab_C4_v4.json 2>&1
FEAST_TALL_VARIANT=5 timeout 900 $B4 > gpurun_out/r25_ab_C4_v5.json 2>&1
FEAST_TALL_VARIANT=5 timeout 900 python bench.py --timing-only --config C5 --steps 2 --warmup 3 > gpurun_out/r25_ab_C5_v5.json 2>&1
for f in gpurun_out/r25_ab_*.json; do echo "$f $(grep -o '"ms_per_step": [0-9.]*' $f) $(grep -o '"reasons": [^]]*]' $f)"; done
grep -E "end loop" gpurun_out/r25_ptrace_tall_v*.txt
