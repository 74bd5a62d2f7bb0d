# round-2 GPU run 11: C2 panel footprint (narrower panels / bigger row caps) and marginal costs
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_build.log 2>&1
B="python bench.py --timing-only --config C2 --steps 20 --warmup 5"
timeout 300 $B > gpurun_out/r2_ab11_base.json 2>&1
for a in 1 2 4 8 15; do FEAST_ABLATE=$a timeout 300 $B > gpurun_out/r2_ab11_ablate$a.json 2>&1; done
FEAST_WP=16 timeout 300 $B > gpurun_out/r2_ab11_wp16.json 2>&1
FEAST_WP=16 FEAST_PANEL_ROWS=512 timeout 300 $B > gpurun_out/r2_ab11_wp16_r512.json 2>&1
FEAST_WP=16 FEAST_PANEL_ROWS=1024 timeout 300 $B > gpurun_out/r2_ab11_wp16_r1024.json 2>&1
FEAST_WP=16 FEAST_PANEL_ROWS=512 FEAST_WIDE_ROWS=512 timeout 300 $B > gpurun_out/r2_ab11_wp16_r512_w512.json 2>&1
FEAST_PANEL_ROWS=384 timeout 300 $B > gpurun_out/r2_ab11_r384.json 2>&1
FEAST_WIDE_ROWS=1024 timeout 300 $B > gpurun_out/r2_ab11_w1024.json 2>&1
FEAST_WIDE_ROWS=512 timeout 300 $B > gpurun_out/r2_ab11_w512.json 2>&1
FEAST_GROUPS=8 timeout 300 $B > gpurun_out/r2_ab11_g8.json 2>&1
FEAST_GROUPS=2 timeout 300 $B > gpurun_out/r2_ab11_g2.json 2>&1
FEAST_PANEL_1ROW=1 timeout 300 $B > gpurun_out/r2_ab11_1row.json 2>&1
for f in gpurun_out/r2_ab11_*.json; do echo "$f $(grep -o '"ms_per_step": [0-9.]*' $f) $(grep -o '"reasons": [^]]*]' $f)"; done
