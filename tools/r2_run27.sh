# phase breakdowns on the new defaults: C4 and C5 (full launch-shape tables)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r27_build.log 2>&1
timeout 900 python tools/phase_breakdown.py C4 --out gpurun_out/r27_phase_C4.json > gpurun_out/r27_phase_C4.txt 2>&1
timeout 1500 python tools/phase_breakdown.py C5 --out gpurun_out/r27_phase_C5.json > gpurun_out/r27_phase_C5.txt 2>&1
head -20 gpurun_out/r27_phase_C5.txt
