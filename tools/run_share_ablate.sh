mkdir -p gpurun_out
for cfg in "a0:" "a1:FEAST_ABLATE=1" "a2:FEAST_ABLATE=2" "a4:FEAST_ABLATE=4" "a7:FEAST_ABLATE=7" "a7nolook:FEAST_ABLATE=7 FEAST_LOOKAHEAD=0" "nograph:FEAST_GRAPH=0"; do
  name=${cfg%%:*}; envs=${cfg#*:}
  echo "== $name $envs"; env $envs timeout 300 python tools/rank_share_timing.py C2 2>&1 | tail -3
done
