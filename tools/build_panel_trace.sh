#!/bin/bash
# Build tools/panel_trace (PTRACE timestamps compiled in) against the library objects;
# NOTRACE=1 builds tools/panel_notrace (no instrumentation: for ncu source-level captures).
set -e
B=paper_1404_2891_b200/build
if [ "${NOTRACE:-0}" = 1 ]; then DEF="-DNO_TRACE_READ"; OUT=tools/panel_notrace; else DEF="-DFEAST_PANEL_TRACE"; OUT=tools/panel_trace; fi
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -rdc=false $DEF $EXTRA \
  -Ipaper_1404_2891_b200/csrc -Iinclude --expt-relaxed-constexpr tools/panel_trace_main.cu \
  paper_1404_2891_b200/csrc/panel_smem.cu $B/lu.o $B/trtri.o $B/btrsm.o $B/zgemm_dmma.o $B/feast_api.o \
  -o $OUT -lcublas -lcusolver
