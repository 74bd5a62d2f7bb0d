# C2 timeline: FLOP rate over the step (where the machine idles), per-group ends
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r20_build.log 2>&1
timeout 300 python tools/timeline.py C2 --out gpurun_out/tl_c2.csv > gpurun_out/r20_tl_c2.log 2>&1
python tools/timeline_rate.py gpurun_out/tl_c2.csv 40 >> gpurun_out/r20_tl_c2.log 2>&1
python tools/timeline_groups.py gpurun_out/tl_c2.csv >> gpurun_out/r20_tl_c2.log 2>&1
cat gpurun_out/r20_tl_c2.log | tail -60
