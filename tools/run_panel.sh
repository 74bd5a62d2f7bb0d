mkdir -p gpurun_out
python -m pytest tests/test_gpu_projector.py -x -q > gpurun_out/ptests.log 2>&1
python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/pbench.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:shift_kernel -c 4 --csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/shift_ncu.csv 2>/dev/null
