mkdir -p gpurun_out
python tools/zgemm_traffic.py alg gpurun_out/zg_alg.json > gpurun_out/zg_alg.log 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:zgemm_dmma --profile-from-start off --csv --log-file gpurun_out/zg_ncu.csv python tools/zgemm_traffic.py ncu > gpurun_out/zg_ncu.log 2>&1
python tools/zgemm_traffic.py merge gpurun_out/zg_alg.json gpurun_out/zg_ncu.csv gpurun_out/zgemm_traffic.json > gpurun_out/zg_merge.log 2>&1
tail -n 3 gpurun_out/*.log
