# final evidence on the session-3 defaults (dot-form outer U12 and inner substitution blocks)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r36_build.log 2>&1
timeout 2700 python -m pytest tests -m gpu -x -q > gpurun_out/r36_gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r36_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r36_smoke.log 2>&1
( time timeout 2400 python bench.py --steps 20 --warmup 5 ) > gpurun_out/r36_bench_C4.json 2> gpurun_out/r36_bench_C4.err
for c in C1 C2 C3; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/r36_bench_$c.json 2> gpurun_out/r36_bench_$c.err; done
timeout 1500 python bench.py --config C5 --steps 2 --warmup 3 > gpurun_out/r36_bench_C5.json 2> gpurun_out/r36_bench_C5.err
( time timeout 900 python bench.py --impl reference --steps 20 --warmup 5 ) > gpurun_out/r36_bench_ref_C4.json 2> gpurun_out/r36_bench_ref_C4.err
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file gpurun_out/r36_launches_C4.csv python bench.py --steps 1 --warmup 3 --timing-only > gpurun_out/r36_ncu_launch.log 2>&1
timeout 1200 python tools/rank_share_timing.py C4 --out gpurun_out/r36_share_C4.json > gpurun_out/r36_share_C4.log 2>&1
timeout 1500 python tools/rank_share_timing.py C5 --worlds 1,2,4,8 --steps 1 --out gpurun_out/r36_share_C5.json > gpurun_out/r36_share_C5.log 2>&1
timeout 900 python tools/phase_breakdown.py C4 > gpurun_out/r36_phase_C4.txt 2>&1
tail -n 3 gpurun_out/r36_gpu_tests.log gpurun_out/r36_smoke.log gpurun_out/r36_bench_C4.err gpurun_out/r36_share_C4.log gpurun_out/r36_share_C5.log
