# Per-kernel ncu evidence for the non-GEMM kernels of the C2 step: HBM kernels'
# DRAM bytes / time, DMMA kernels' tensor-pipe use, the latency-bound kernels' duration.
mkdir -p gpurun_out/kn
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_tensor_subpipe_dmma.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,launch__grid_size,launch__cluster_dim_x,sm__throughput.avg.pct_of_peak_sustained_elapsed
for k in shift_kernel laswp_kernel accum_kernel broadcast_copy_kernel trtri_kernel trsm_warp_kernel panel_smem_kernel zgemm_dmma_kernel splitk_reduce_kernel; do
  ncu --metrics $M --clock-control none -k regex:$k -c 6 --csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/kn/$k.csv 2>/dev/null
done
