mkdir -p gpurun_out
python -m pytest tests/test_gpu_projector.py tests/test_gpu_fullsize.py tests/test_gpu_iterate.py -x -q > gpurun_out/ptests.log 2>&1
python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/pbench.log 2>&1
./tools/zgemm_lab 0 0 > gpurun_out/lab_v0.txt 2>&1
for c in C3; do python tools/run_config.py $c >> gpurun_out/configs4.jsonl 2>gpurun_out/configs4_$c.err; done
