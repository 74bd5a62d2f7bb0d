# Round-end evidence: GPU tests, smoke, bench (both arms), ncu launch list + full capture of the
# dominant kernel, DRAM traffic.  Each ncu pass runs only after the same command exited 0 without it.
mkdir -p gpurun_out/final
O=gpurun_out/final
python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo "pytest rc=$?" >> $O/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
python bench.py > $O/bench.json 2> $O/bench.err
python bench.py --impl reference --steps 2 --warmup 0 > $O/bench_ref.json 2> $O/bench_ref.err
python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/bench_small.json 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file $O/launches.csv \
      python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:zgemm_dmma_kernel --launch-skip 20 -c 12 \
    -o $O/zgemm_full python bench.py --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_full.log 2>&1
python tools/zgemm_traffic.py alg $O/zg_alg.json > $O/zg_alg.log 2>&1 && \
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
      -k regex:zgemm_dmma --profile-from-start off --csv --log-file $O/zg_ncu.csv python tools/zgemm_traffic.py ncu \
      > $O/zg_ncu.log 2>&1 && \
  python tools/zgemm_traffic.py merge $O/zg_alg.json $O/zg_ncu.csv $O/zgemm_traffic.json > $O/zg_merge.log 2>&1
echo done > $O/DONE
