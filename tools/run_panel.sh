# scratch driver for one-off GPU checks (edited per experiment)
mkdir -p gpurun_out
python -m pytest tests/test_gpu_projector.py -x -q > gpurun_out/ptests.log 2>&1
python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/pbench.log 2>&1
