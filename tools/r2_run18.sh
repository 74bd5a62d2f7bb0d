# ncu source-level capture of the C2-height cluster panel (2048 rows, 8 CTAs, 32 wide, 16 nodes)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r18_build.log 2>&1
NOTRACE=1 bash tools/build_panel_trace.sh > gpurun_out/r18_pbuild.log 2>&1
timeout 120 tools/panel_notrace 32 8 2048 16 > gpurun_out/r18_plain.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:panel_smem_kernel -s 2 -c 1 \
  -o gpurun_out/r18_panel_c2 tools/panel_notrace 32 8 2048 16 > gpurun_out/r18_ncu.log 2>&1
tail -n 3 gpurun_out/r18_ncu.log
