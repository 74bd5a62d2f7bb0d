# C2: outer U12 dot form A/B (default off below n = 8192)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r35_build.log 2>&1
for v in 0 1 0 1; do
  FEAST_U12_DOT=$v timeout 600 python bench.py --timing-only --config C2 --steps 20 --warmup 5 >> gpurun_out/r35_ab_C2_u$v.json 2>&1
done
for f in gpurun_out/r35_ab_*.json; do echo "$f $(grep -o '"ms_per_step": [0-9.]*' $f) $(grep -o '"reasons": [^]]*]' $f)"; done
