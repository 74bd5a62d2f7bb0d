# C4 schedule knobs on the dot-form default: first outer block width, node-group count
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r23_build.log 2>&1
B="python bench.py --timing-only --config C4 --steps 3 --warmup 3"
timeout 900 $B > gpurun_out/r23_ab_C4_base.json 2>&1
FEAST_NBO0=256 timeout 900 $B > gpurun_out/r23_ab_C4_nbo0_256.json 2>&1
FEAST_NBO0=512 timeout 900 $B > gpurun_out/r23_ab_C4_nbo0_512.json 2>&1
FEAST_GROUPS=2 timeout 900 $B > gpurun_out/r23_ab_C4_g2.json 2>&1
FEAST_GROUPS=8 timeout 900 $B > gpurun_out/r23_ab_C4_g8.json 2>&1
for f in gpurun_out/r23_ab_*.json; do echo "$f $(grep -o '"ms_per_step": [0-9.]*' $f) $(grep -o '"reasons": [^]]*]' $f)"; done
