#!/bin/bash
# Build tools/zgemm_lab against the library objects (run from the repo root).
set -e
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Ipaper_1404_2891_b200/csrc -Iinclude \
  tools/zgemm_lab.cu paper_1404_2891_b200/build/*.o -o tools/zgemm_lab -lcublas -lcusolver
