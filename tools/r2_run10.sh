# round-2 GPU run 10: rasterised GEMM tiles (FEAST_SWZ) — correctness, A/B, DRAM traffic
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_build.log 2>&1
bash tools/build_lab.sh > gpurun_out/r2_lab_build.log 2>&1
timeout 1800 python -m pytest tests/test_gpu_projector.py tests/test_gpu_fullsize.py -x -q -k "not c3_full_node" > gpurun_out/r2_gpu_tests_v10.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_gpu_tests_v10.log
B="python bench.py --timing-only"
for z in 16 0 8 32; do FEAST_SWZ=$z timeout 600 $B --steps 2 --warmup 3 > gpurun_out/r2_ab10_C4_swz$z.json 2>&1; done
for z in 16 0; do
  FEAST_SWZ=$z timeout 600 $B --config C2 --steps 20 --warmup 5 > gpurun_out/r2_ab10_C2_swz$z.json 2>&1
  FEAST_SWZ=$z timeout 600 $B --config C3 --steps 5 --warmup 3 > gpurun_out/r2_ab10_C3_swz$z.json 2>&1
done
M="dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct,launch__grid_size"
for z in 16 0; do FEAST_SWZ=$z timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r2_lab_c4_swz$z.csv tools/zgemm_lab 14 0 > /dev/null 2>&1; done
timeout 600 ncu --set full --import-source on --clock-control none -c 1 -o gpurun_out/r2_lab_c4_full tools/zgemm_lab 14 0 > gpurun_out/r2_lab_full.log 2>&1
python tools/zgemm_traffic.py alg gpurun_out/zg_alg_C4.json --config=C4 > gpurun_out/zg_alg_C4.log 2>&1
timeout 1500 ncu --replay-mode application --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:zgemm_dmma --profile-from-start off --csv --log-file gpurun_out/zg_ncu_C4.csv python tools/zgemm_traffic.py ncu --config=C4 > gpurun_out/zg_ncu_C4.log 2>&1
python tools/zgemm_traffic.py merge gpurun_out/zg_alg_C4.json gpurun_out/zg_ncu_C4.csv gpurun_out/zgemm_traffic_C4.json --config=C4 > gpurun_out/zg_merge_C4.log 2>&1
tail -n 3 gpurun_out/r2_gpu_tests_v10.log
cat gpurun_out/zg_merge_C4.log
for f in gpurun_out/r2_ab10_*.json; do echo "$f $(grep -o '"ms_per_step": [0-9.]*' $f) $(grep -o '"reasons": [^]]*]' $f)"; done
