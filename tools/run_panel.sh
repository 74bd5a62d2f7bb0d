mkdir -p gpurun_out
for c in C5 C1 C2; do python tools/run_config.py $c >> gpurun_out/configs6.jsonl 2>gpurun_out/configs6_$c.err; done
