# round-2 GPU run 8: evidence on the current defaults — full GPU suite, smoke, bench lines of every
# config (C4 with the driver's step counts), the reference arm, C4 ncu launch list / zgemm DRAM
# traffic / full capture of a trailing update
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gpu_tests_v8.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_gpu_tests_v8.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1
( time timeout 2400 python bench.py --steps 20 --warmup 5 ) > gpurun_out/r2_bench_C4_final.json 2> gpurun_out/r2_bench_C4_final.err
for c in C1 C2 C3; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/r2_bench_${c}_final.json 2> gpurun_out/r2_bench_${c}_final.err; done
timeout 1500 python bench.py --config C5 --steps 2 --warmup 3 > gpurun_out/r2_bench_C5_final.json 2> gpurun_out/r2_bench_C5_final.err
( time timeout 900 python bench.py --impl reference --steps 3 --warmup 1 ) > gpurun_out/r2_bench_ref_C4.json 2> gpurun_out/r2_bench_ref_C4.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file gpurun_out/r2_launches_C4_final.csv python bench.py --steps 1 --warmup 3 --timing-only > gpurun_out/r2_ncu_launch_final.log 2>&1
python tools/zgemm_traffic.py alg gpurun_out/zg_alg_C4.json --config=C4 > gpurun_out/zg_alg_C4.log 2>&1
timeout 1500 ncu --replay-mode application --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:zgemm_dmma --profile-from-start off --csv --log-file gpurun_out/zg_ncu_C4.csv python tools/zgemm_traffic.py ncu --config=C4 > gpurun_out/zg_ncu_C4.log 2>&1
python tools/zgemm_traffic.py merge gpurun_out/zg_alg_C4.json gpurun_out/zg_ncu_C4.csv gpurun_out/zgemm_traffic_C4.json --config=C4 > gpurun_out/zg_merge_C4.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:zgemm_dmma --launch-skip 30 --launch-count 12 -o gpurun_out/r2_zgemm_C4_full2 --profile-from-start off python tools/zgemm_traffic.py ncu --config=C4 --batch=1 > gpurun_out/r2_ncu_full2.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:panel_smem --launch-skip 40 --launch-count 2 -o gpurun_out/r2_panel_C4_full --profile-from-start off python tools/zgemm_traffic.py ncu --config=C4 --batch=1 > gpurun_out/r2_ncu_panel.log 2>&1
tail -n 3 gpurun_out/r2_gpu_tests_v8.log gpurun_out/r2_smoke.log gpurun_out/r2_bench_C4_final.err gpurun_out/zg_merge_C4.log
