mkdir -p gpurun_out
for cfg in "default:" "g1:FEAST_GROUPS=1" "g2:FEAST_GROUPS=2" "nolook:FEAST_LOOKAHEAD=0" "cs4:FEAST_CS_MAX=4" "nograph:FEAST_GRAPH=0"; do
  name=${cfg%%:*}; envs=${cfg#*:}
  echo "== $name"; env $envs timeout 300 python tools/rank_share_timing.py C2 2>&1 | tail -4
done > gpurun_out/share.log 2>&1
