# round-2 GPU run 13: L-column swaps off the chain
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_projector.py tests/test_gpu_iterate.py tests/test_gpu_multirank.py -x -q > gpurun_out/r2_gpu_tests_v13.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_gpu_tests_v13.log
B="python bench.py --timing-only --config C2 --steps 20 --warmup 5"
for ls in 1 0 1 0; do FEAST_LSWAP_SIDE=$ls timeout 300 $B >> gpurun_out/r2_ab13_C2_ls$ls.jsonl 2>&1; done
FEAST_ABLATE=4 timeout 300 $B > gpurun_out/r2_ab13_C2_noswap.json 2>&1
for ls in 1 0; do FEAST_LSWAP_SIDE=$ls timeout 600 python bench.py --timing-only --steps 2 --warmup 3 > gpurun_out/r2_ab13_C4_ls$ls.json 2>&1; done
tail -n 3 gpurun_out/r2_gpu_tests_v13.log
grep -h -o '"ms_per_step": [0-9.]*' gpurun_out/r2_ab13_C2_ls1.jsonl; echo ---; grep -h -o '"ms_per_step": [0-9.]*' gpurun_out/r2_ab13_C2_ls0.jsonl
for f in gpurun_out/r2_ab13_*.json; do echo "$f $(grep -o '"ms_per_step": [0-9.]*' $f)"; done
