# deferred rank-1 update in the cluster panel: bit-identity + panel tests, trace, C2/C3 A/B
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r17_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_projector.py -m gpu -x -q -k "deferred or ragged or panel or swap" > gpurun_out/r17_tests.log 2>&1
tail -n 3 gpurun_out/r17_tests.log
bash tools/build_panel_trace.sh > gpurun_out/r17_ptrace_build.log 2>&1
for d in 0 1; do
  for b in 1 16; do FEAST_PANEL_DEFER=$d timeout 120 tools/panel_trace 32 8 2048 $b > gpurun_out/r17_ptrace_d${d}_b$b.txt 2>&1; done
done
B="python bench.py --timing-only --config C2 --steps 20 --warmup 5"
for rep in 1 2; do for d in 0 1; do FEAST_PANEL_DEFER=$d timeout 300 $B > gpurun_out/r17_ab_C2_d${d}_$rep.json 2>&1; done; done
for d in 0 1; do FEAST_PANEL_DEFER=$d timeout 300 python bench.py --timing-only --config C3 --steps 3 --warmup 3 > gpurun_out/r17_ab_C3_d$d.json 2>&1; done
for f in gpurun_out/r17_ab_*.json; do echo "$f $(grep -o '"ms_per_step": [0-9.]*' $f) $(grep -o '"reasons": [^]]*]' $f)"; done
tail -n 5 gpurun_out/r17_ptrace_*.txt
