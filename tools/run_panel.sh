mkdir -p gpurun_out
python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/pbench.log 2>&1
python tools/rank_share_timing.py C2 > gpurun_out/pshare.log 2>&1
python -m pytest tests/test_gpu_projector.py tests/test_gpu_iterate.py -x -q > gpurun_out/ptests.log 2>&1
FEAST_PANEL_1ROW=1 python -m pytest tests/test_gpu_projector.py -x -q -k "ragged or register_panel or parity" > gpurun_out/ptests1.log 2>&1
