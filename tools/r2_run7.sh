# round-2 GPU run 7: substitutions joined over the batch; swap coalescing metrics
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_projector.py -x -q -k "join or substitution or bi or cache or real or csym or complex" > gpurun_out/r2_gpu_tests_v7.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_gpu_tests_v7.log
B="python bench.py --timing-only"
for j in 1 0; do
  FEAST_SUBST_JOIN=$j timeout 600 $B --config C2 --steps 20 --warmup 5 > gpurun_out/r2_ab7_C2_join$j.json 2>&1
  FEAST_SUBST_JOIN=$j timeout 600 $B --steps 2 --warmup 3 > gpurun_out/r2_ab7_C4_join$j.json 2>&1
  FEAST_SUBST_JOIN=$j timeout 600 $B --config C1 --steps 50 --warmup 5 > gpurun_out/r2_ab7_C1_join$j.json 2>&1
done
M="l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum,l1tex__t_requests_pipe_lsu_mem_global_op_st.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,launch__grid_size"
for v in coalesced chain; do
  FEAST_LASWP=$v timeout 600 python tools/swap_probe.py 2048 > gpurun_out/r2_swap_$v.log 2>&1
  FEAST_LASWP=$v timeout 900 ncu --metrics $M --clock-control none -k regex:laswp -c 60 --csv --log-file gpurun_out/r2_swap_ncu_$v.csv python tools/swap_probe.py 2048 > /dev/null 2>&1
done
tail -n 3 gpurun_out/r2_gpu_tests_v7.log
cat gpurun_out/r2_swap_*.log
for f in gpurun_out/r2_ab7_*.json; do echo "$f $(grep -o '"ms_per_step": [0-9.]*' $f) $(grep -o '"reasons": [^]]*]' $f)"; done
