mkdir -p gpurun_out
for v in 0 64 128 0 192; do
  r=$(FEAST_NBO0=$v timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3))")
  echo "nbo0=$v -> $r"
done > gpurun_out/nbo0.log 2>&1
FEAST_NBO0=128 python -m pytest tests/test_gpu_projector.py -x -q -k "parity or ragged" > gpurun_out/ptests.log 2>&1
