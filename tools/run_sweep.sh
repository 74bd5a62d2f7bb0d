# C2 bench step (ms) under schedule / panel knobs
mkdir -p gpurun_out
for cfg in "default:" "rowcap4:FEAST_ROWCAP=4" "rowcap1:FEAST_ROWCAP=1" "csmax8:FEAST_CS_MAX=8" "csmax4:FEAST_CS_MAX=4" \
           "groups8:FEAST_GROUPS=8" "groups2:FEAST_GROUPS=2" "wide512:FEAST_WIDE_ROWS=512" "wide1024:FEAST_WIDE_ROWS=1024" \
           "wide0:FEAST_WIDE_ROWS=0" "default2:"; do
  name=${cfg%%:*}; envs=${cfg#*:}
  r=$(env $envs timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3), round(d['lu_solve_frac_peak'],3))")
  echo "$name $envs -> $r"
done
