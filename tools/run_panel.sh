mkdir -p gpurun_out
for i in 1 2; do for m in 0 1; do echo "mma=$m $(FEAST_PANEL_MMA=$m ./tools/panel_trace 32 8 2048 4 | grep "end loop") | $(FEAST_PANEL_MMA=$m ./tools/panel_trace 32 1 256 4 | grep "end loop") | $(FEAST_PANEL_MMA=$m ./tools/panel_trace 64 2 512 4 | grep "end loop")"; done; done > gpurun_out/mma.log 2>&1
python -m pytest tests/test_gpu_projector.py -x -q > gpurun_out/ptests.log 2>&1
python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/pbench.log 2>&1
FEAST_PANEL_MMA=0 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/pbench0.log 2>&1
python tools/rank_share_timing.py C2 > gpurun_out/pshare.log 2>&1
