# C2 bench step and rank shares under the schedule / panel knobs of DESIGN §6 (one line each)
mkdir -p gpurun_out
for cfg in "default:" "groups2:FEAST_GROUPS=2" "nolookahead:FEAST_LOOKAHEAD=0" "csmax8:FEAST_CS_MAX=8" \
           "wide1024:FEAST_WIDE_ROWS=1024" "onerow:FEAST_PANEL_1ROW=1" "default2:"; do
  name=${cfg%%:*}; envs=${cfg#*:}
  r=$(env $envs timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3), round(d['lu_solve_frac_peak'],3))")
  echo "$name $envs -> $r"
  env $envs timeout 300 python tools/rank_share_timing.py C2 2>&1 | tail -3
done
