# C3 (pivot-heavy recipe): panel-fused swaps (thread per column) vs a separate coalesced swap launch
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r32_build.log 2>&1
B3="python bench.py --timing-only --config C3 --steps 3 --warmup 3"
FEAST_PANEL_SWAP=0 timeout 600 $B3 > gpurun_out/r32_ab_C3_unfused.json 2>&1
timeout 600 $B3 > gpurun_out/r32_ab_C3_fused.json 2>&1
timeout 900 python tools/phase_breakdown.py C3 > gpurun_out/r32_phase_C3.txt 2>&1
for f in gpurun_out/r32_ab_*.json; do echo "$f $(grep -o '"ms_per_step": [0-9.]*' $f) $(grep -o '"reasons": [^]]*]' $f)"; done
head -20 gpurun_out/r32_phase_C3.txt
