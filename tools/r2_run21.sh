# C4 phase breakdown with the time lost per launch shape (LU vs substitutions)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r21_build.log 2>&1
timeout 900 python tools/phase_breakdown.py C4 > gpurun_out/r21_phase_C4.txt 2>&1
timeout 300 python tools/phase_breakdown.py C2 > gpurun_out/r21_phase_C2.txt 2>&1
tail -50 gpurun_out/r21_phase_C4.txt
