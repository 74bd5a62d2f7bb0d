# round-2 GPU run 14: final evidence on the round-2 defaults
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_build.log 2>&1
bash tools/build_lab.sh > gpurun_out/r2_lab_build.log 2>&1
timeout 2700 python -m pytest tests -m gpu -x -q > gpurun_out/r3_gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r3_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3_smoke.log 2>&1
( time timeout 2400 python bench.py --steps 20 --warmup 5 ) > gpurun_out/r3_bench_C4.json 2> gpurun_out/r3_bench_C4.err
for c in C1 C2 C3; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/r3_bench_$c.json 2> gpurun_out/r3_bench_$c.err; done
timeout 1500 python bench.py --config C5 --steps 2 --warmup 3 > gpurun_out/r3_bench_C5.json 2> gpurun_out/r3_bench_C5.err
( time timeout 900 python bench.py --impl reference --steps 20 --warmup 5 ) > gpurun_out/r3_bench_ref_C4.json 2> gpurun_out/r3_bench_ref_C4.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file gpurun_out/r3_launches_C4.csv python bench.py --steps 1 --warmup 3 --timing-only > gpurun_out/r3_ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:zgemm -c 1 -o gpurun_out/r3_lab_c4_trailing_full tools/zgemm_lab 14 0 > gpurun_out/r3_lab_full.log 2>&1
timeout 900 python tools/phase_breakdown.py C4 --out gpurun_out/r3_phase_C4.json > gpurun_out/r3_phase_C4.log 2>&1
timeout 600 python tools/phase_breakdown.py C2 > gpurun_out/r3_phase_C2.log 2>&1
timeout 1200 python tools/rank_share_timing.py C4 --out gpurun_out/r3_share_C4.json > gpurun_out/r3_share_C4.log 2>&1
timeout 900 python tools/rank_share_timing.py C5 --worlds 1,2,4,8 --steps 1 --out gpurun_out/r3_share_C5.json > gpurun_out/r3_share_C5.log 2>&1
tail -n 3 gpurun_out/r3_gpu_tests.log gpurun_out/r3_smoke.log gpurun_out/r3_bench_C4.err gpurun_out/r3_share_C4.log gpurun_out/r3_share_C5.log
