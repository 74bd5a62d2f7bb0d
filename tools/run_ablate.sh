# marginal cost of each latency-bound class in the overlapped C2 step (timing only; results invalid)
mkdir -p gpurun_out
for cfg in "a7:FEAST_ABLATE=7" "a7nbo512:FEAST_ABLATE=7 FEAST_NBO=512" "a7g2:FEAST_ABLATE=7 FEAST_GROUPS=2" "a7g1:FEAST_ABLATE=7 FEAST_GROUPS=1" "nbo512:FEAST_NBO=512" "a7nolook:FEAST_ABLATE=7 FEAST_LOOKAHEAD=0"; do
  name=${cfg%%:*}; envs=${cfg#*:}
  r=$(env $envs timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3), round(d['roofline']['achieved'],2))")
  echo "$name ($envs) -> $r"
done
