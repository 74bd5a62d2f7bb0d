mkdir -p gpurun_out
python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/pbench.log 2>&1
python -m pytest tests/test_gpu_projector.py -x -q > gpurun_out/ptests.log 2>&1
python tools/zgemm_shapes.py C2 > gpurun_out/shapes_c2b.log 2>&1
