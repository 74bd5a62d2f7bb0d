# session-2 re-entry check: GPU suite on the restored tree, panel trace, C2 bench line
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r16_build_smoke.log 2>&1
bash tools/build_panel_trace.sh > gpurun_out/r16_ptrace_build.log 2>&1
for b in 1 16; do timeout 120 tools/panel_trace 32 8 2048 $b > gpurun_out/r16_ptrace_32_8_b$b.txt 2>&1; done
timeout 120 tools/panel_trace 16 16 16384 1 > gpurun_out/r16_ptrace_16_16_16384.txt 2>&1
timeout 600 python bench.py --config C2 --steps 20 --warmup 5 > gpurun_out/r16_bench_C2.json 2> gpurun_out/r16_bench_C2.err
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r16_gpu_tests.log 2>&1
tail -n 3 gpurun_out/r16_gpu_tests.log
cat gpurun_out/r16_bench_C2.json
