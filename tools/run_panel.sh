mkdir -p gpurun_out
for cfg in "graph:" "nograph:FEAST_GRAPH=0"; do
  name=${cfg%%:*}; envs=${cfg#*:}
  r=$(env $envs timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3))")
  echo "$name -> $r"
done
