# round-2 GPU run 6: register-tile btrsm (2 CTAs / SM) correctness + A/B
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_projector.py -x -q -k "substitution or outer_block or bi or left or cache or csym or complex_symmetric or real" > gpurun_out/r2_gpu_tests_v6.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_gpu_tests_v6.log
B="python bench.py --timing-only"
for v in "1 2" "1 1" "0 2"; do set -- $v
  FEAST_BTRSM=$1 FEAST_BTRSM_MINB=$2 timeout 600 $B --config C2 --steps 20 --warmup 5 > gpurun_out/r2_ab6_C2_bt$1_$2.json 2>&1
  FEAST_BTRSM=$1 FEAST_BTRSM_MINB=$2 timeout 600 $B --steps 2 --warmup 3 > gpurun_out/r2_ab6_C4_bt$1_$2.json 2>&1
done
timeout 600 python tools/phase_breakdown.py C2 > gpurun_out/r2_phase_C2_v6.log 2>&1
FEAST_BTRSM_MINB=1 timeout 600 python tools/phase_breakdown.py C2 > gpurun_out/r2_phase_C2_v6_m1.log 2>&1
tail -n 3 gpurun_out/r2_gpu_tests_v6.log
for f in gpurun_out/r2_ab6_*.json; do echo "$f $(grep -o '"ms_per_step": [0-9.]*' $f) $(grep -o '"reasons": [^]]*]' $f)"; done
