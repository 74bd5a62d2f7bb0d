mkdir -p gpurun_out
python tools/timeline.py C2 --out gpurun_out/tl_c2.csv > gpurun_out/tl_c2.log 2>&1
python tools/timeline_rate.py gpurun_out/tl_c2.csv 30 >> gpurun_out/tl_c2.log 2>&1
python tools/timeline.py C3 --out gpurun_out/tl_c3.csv > gpurun_out/tl_c3.log 2>&1
python tools/timeline_rate.py gpurun_out/tl_c3.csv 30 >> gpurun_out/tl_c3.log 2>&1
