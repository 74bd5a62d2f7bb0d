mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/ptests.log 2>&1
python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/pbench.log 2>&1
for c in C3 C4; do python tools/run_config.py $c >> gpurun_out/configs3.jsonl 2>gpurun_out/configs3_$c.err; done
