# panel per-column trace (current kernel) + C2 bench line with the profiling fix
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_build.log 2>&1
bash tools/build_panel_trace.sh > gpurun_out/r4_ptrace_build.log 2>&1
for b in 1 16; do timeout 120 tools/panel_trace 32 8 2048 $b > gpurun_out/r4_ptrace_32_8_b$b.txt 2>&1; done
timeout 120 tools/panel_trace 16 16 16384 1 > gpurun_out/r4_ptrace_16_16_16384.txt 2>&1
timeout 600 python bench.py --config C2 --steps 20 --warmup 5 > gpurun_out/r4_bench_C2.json 2> gpurun_out/r4_bench_C2.err
tail -n 4 gpurun_out/r4_ptrace_*.txt
