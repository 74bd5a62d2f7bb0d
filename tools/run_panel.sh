mkdir -p gpurun_out
python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/pbench.log 2>&1
python -m pytest tests/test_gpu_projector.py tests/test_gpu_fullsize.py -x -q > gpurun_out/ptests.log 2>&1
python tools/rank_share_timing.py C2 > gpurun_out/pshare.log 2>&1
