mkdir -p gpurun_out
for v in 256 192 320 384 256; do
  r=$(FEAST_NBO=$v timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3))")
  echo "nbo=$v -> $r"
done > gpurun_out/nbo.log 2>&1
