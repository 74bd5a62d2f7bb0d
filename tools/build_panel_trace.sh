#!/bin/bash
# Build tools/panel_trace (PTRACE timestamps compiled in) against the library objects.
set -e
B=paper_1404_2891_b200/build
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -rdc=false -DFEAST_PANEL_TRACE $EXTRA \
  -Ipaper_1404_2891_b200/csrc -Iinclude --expt-relaxed-constexpr tools/panel_trace_main.cu \
  paper_1404_2891_b200/csrc/panel_smem.cu $B/lu.o $B/trtri.o $B/btrsm.o $B/zgemm_dmma.o $B/feast_api.o \
  -o tools/panel_trace -lcublas -lcusolver
