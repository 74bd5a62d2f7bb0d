mkdir -p gpurun_out
for cfg in "default:" "rowcap4:FEAST_ROWCAP=4" "rowcap4cs8:FEAST_ROWCAP=4 FEAST_CS_MAX=8" "default2:"; do
  name=${cfg%%:*}; envs=${cfg#*:}
  r=$(env $envs timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3), round(d['lu_solve_frac_peak'],3))")
  echo "$name $envs -> $r"
  env $envs timeout 300 python tools/rank_share_timing.py C2 2>&1 | tail -4
done
