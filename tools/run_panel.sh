mkdir -p gpurun_out
FEAST_TRTRI=1 python -m pytest tests/test_gpu_projector.py -x -q -k "parity or ragged" > gpurun_out/ptests.log 2>&1
for v in 0 1 2 3 0; do
  r=$(FEAST_TRTRI=$v timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3), round(d['roofline']['per_class_ms_per_step']['trsm'],3))")
  echo "trtri=$v -> $r"
done > gpurun_out/trtri.log 2>&1
