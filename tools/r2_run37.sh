# re-entry evidence at HEAD (session-4): full GPU suite, smoke, driver-argument C4 bench, C2 line, reference arm
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r37_gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r37_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r37_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r37_smoke.log
( time timeout 1200 python bench.py --steps 20 --warmup 5 ) > gpurun_out/r37_bench_C4.json 2> gpurun_out/r37_bench_C4.err
for c in C2 C3 C1; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/r37_bench_$c.json 2> gpurun_out/r37_bench_$c.err; done
( time timeout 600 python bench.py --impl reference --steps 3 --warmup 1 ) > gpurun_out/r37_bench_ref_C4.json 2> gpurun_out/r37_bench_ref_C4.err
tail -n 3 gpurun_out/r37_gpu_tests.log gpurun_out/r37_smoke.log gpurun_out/r37_bench_C4.err
