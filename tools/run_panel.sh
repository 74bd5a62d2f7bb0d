mkdir -p gpurun_out
for g in 4 8 6 4; do
  r=$(FEAST_GROUPS=$g timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3))")
  echo "groups=$g -> $r"
done > gpurun_out/groups.log 2>&1
