# session-4 evidence at HEAD, part 2: C5 line, C4 ncu launch list (share of the step), C4 phase breakdown, rank shares
set -x
timeout 1200 python bench.py --config C5 --steps 2 --warmup 3 > gpurun_out/r38_bench_C5.json 2> gpurun_out/r38_bench_C5.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file gpurun_out/r38_launches_C4.csv python bench.py --steps 1 --warmup 3 --timing-only > gpurun_out/r38_ncu_launch.log 2>&1
timeout 600 python tools/phase_breakdown.py C4 > gpurun_out/r38_phase_C4.txt 2>&1
timeout 900 python tools/rank_share_timing.py C4 --out gpurun_out/r38_share_C4.json > gpurun_out/r38_share_C4.log 2>&1
tail -n 3 gpurun_out/r38_bench_C5.err gpurun_out/r38_share_C4.log
