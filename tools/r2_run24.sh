# large-n schedule: 2 node groups + 512-wide first block, on C4 / C3 / C5
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r24_build.log 2>&1
B4="python bench.py --timing-only --config C4 --steps 3 --warmup 3"
FEAST_GROUPS=2 FEAST_NBO0=512 timeout 900 $B4 > gpurun_out/r24_ab_C4_g2_nbo0512.json 2>&1
B3="python bench.py --timing-only --config C3 --steps 3 --warmup 3"
timeout 600 $B3 > gpurun_out/r24_ab_C3_base.json 2>&1
FEAST_GROUPS=2 timeout 600 $B3 > gpurun_out/r24_ab_C3_g2.json 2>&1
FEAST_NBO0=512 timeout 600 $B3 > gpurun_out/r24_ab_C3_nbo0512.json 2>&1
FEAST_GROUPS=2 FEAST_NBO0=512 timeout 600 $B3 > gpurun_out/r24_ab_C3_g2_nbo0512.json 2>&1
B5="python bench.py --timing-only --config C5 --steps 2 --warmup 3"
timeout 1200 $B5 > gpurun_out/r24_ab_C5_base.json 2>&1
FEAST_GROUPS=2 FEAST_NBO0=512 timeout 1200 $B5 > gpurun_out/r24_ab_C5_g2_nbo0512.json 2>&1
for f in gpurun_out/r24_ab_*.json; do echo "$f $(grep -o '"ms_per_step": [0-9.]*' $f) $(grep -o '"reasons": [^]]*]' $f)"; done
