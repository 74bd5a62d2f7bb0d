mkdir -p gpurun_out
python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/pbench.log 2>&1
python -m pytest tests -m gpu -x -q > gpurun_out/ptests.log 2>&1
for c in C3 C4; do python tools/run_config.py $c >> gpurun_out/configs5.jsonl 2>gpurun_out/configs5_$c.err; done
python tools/rank_share_timing.py C2 > gpurun_out/pshare.log 2>&1
