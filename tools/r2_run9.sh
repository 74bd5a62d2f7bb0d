# round-2 GPU run 9: staggered node groups (FEAST_STAGGER) A/B
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_projector.py -x -q -k "stagger or virtual or worst" > gpurun_out/r2_gpu_tests_v9.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_gpu_tests_v9.log
B="python bench.py --timing-only"
for d in 0 1 2 3 4 6; do FEAST_STAGGER=$d timeout 600 $B --config C2 --steps 20 --warmup 5 > gpurun_out/r2_ab9_C2_st$d.json 2>&1; done
for g in 8; do for d in 1 2 3; do FEAST_GROUPS=$g FEAST_STAGGER=$d timeout 600 $B --config C2 --steps 20 --warmup 5 > gpurun_out/r2_ab9_C2_g${g}_st$d.json 2>&1; done; done
for d in 0 2 4 8; do FEAST_STAGGER=$d timeout 600 $B --steps 2 --warmup 3 > gpurun_out/r2_ab9_C4_st$d.json 2>&1; done
for d in 0 2 4; do FEAST_STAGGER=$d timeout 600 $B --config C3 --steps 5 --warmup 3 > gpurun_out/r2_ab9_C3_st$d.json 2>&1; done
tail -n 3 gpurun_out/r2_gpu_tests_v9.log
for f in gpurun_out/r2_ab9_*.json; do echo "$f $(grep -o '"ms_per_step": [0-9.]*' $f) $(grep -o '"reasons": [^]]*]' $f)"; done
