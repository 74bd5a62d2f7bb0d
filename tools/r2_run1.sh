set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gpu_tests_v1.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_gpu_tests_v1.log
timeout 1200 python bench.py --steps 3 --warmup 3 > gpurun_out/r2_bench_c4_v1.json 2> gpurun_out/r2_bench_c4_v1.err
echo bench rc=$?
tail -3 gpurun_out/r2_gpu_tests_v1.log
