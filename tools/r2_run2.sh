# round-2 GPU run 2: new GPU tests, per-config bench lines, C4 launch list + traffic + full capture
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_build.log 2>&1
timeout 1800 python -m pytest tests/test_gpu_next3.py tests/test_gpu_multirank.py "tests/test_gpu_fullsize.py::test_c3_full_node_solutions_vs_oracle" -x -q > gpurun_out/r2_gpu_tests_v2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_gpu_tests_v2.log
for c in C1 C2 C3; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/r2_bench_$c.json 2> gpurun_out/r2_bench_$c.err
done
timeout 1500 python bench.py --config C5 --steps 2 --warmup 3 > gpurun_out/r2_bench_C5.json 2> gpurun_out/r2_bench_C5.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 18000 --csv --log-file gpurun_out/r2_launches_C4.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r2_ncu_launch.log 2>&1
python tools/zgemm_traffic.py alg gpurun_out/zg_alg_C4.json --config=C4 > gpurun_out/zg_alg_C4.log 2>&1
timeout 1500 ncu --replay-mode application --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:zgemm_dmma --profile-from-start off --csv --log-file gpurun_out/zg_ncu_C4.csv python tools/zgemm_traffic.py ncu --config=C4 > gpurun_out/zg_ncu_C4.log 2>&1
python tools/zgemm_traffic.py merge gpurun_out/zg_alg_C4.json gpurun_out/zg_ncu_C4.csv gpurun_out/zgemm_traffic_C4.json --config=C4 > gpurun_out/zg_merge_C4.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:zgemm_dmma --launch-skip 40 --launch-count 6 -o gpurun_out/r2_zgemm_C4_full --profile-from-start off python tools/zgemm_traffic.py ncu --config=C4 --batch=1 > gpurun_out/r2_ncu_full.log 2>&1
tail -n 3 gpurun_out/r2_*.log gpurun_out/zg_*C4.log
