# DRAM traffic of the dominant kernel at HEAD (session 4): C4 then C2, ncu dram bytes of every zgemm launch of one serialised step
set -x
for c in C4 C2; do
timeout 600 python tools/zgemm_traffic.py alg gpurun_out/r39_zg_alg_$c.json --config=$c > gpurun_out/r39_zg_alg_$c.log 2>&1
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:zgemm_dmma --profile-from-start off --csv --log-file gpurun_out/r39_zg_ncu_$c.csv python tools/zgemm_traffic.py ncu --config=$c > gpurun_out/r39_zg_ncu_$c.log 2>&1
python tools/zgemm_traffic.py merge gpurun_out/r39_zg_alg_$c.json gpurun_out/r39_zg_ncu_$c.csv gpurun_out/r39_zgemm_traffic_$c.json --config=$c > gpurun_out/r39_zg_merge_$c.log 2>&1
rm -f gpurun_out/r39_zg_ncu_$c.csv
done
tail -n 3 gpurun_out/r39_*.log
