#!/bin/bash
# Sweep LU blocking / overlap knobs on one config (projector time, CUDA events; not the bench).
K=${1:-C2}
for cfg in "default:" "nolookahead:FEAST_LOOKAHEAD=0" "gemm_st3:FEAST_ZGEMM_VARIANT=3" "nbo128:FEAST_NBO=128" \
           "wp16:FEAST_WP=16" "nbo192:FEAST_NBO=192" "gemm_32x64:FEAST_ZGEMM_VARIANT=5" "gemm_64x64:FEAST_ZGEMM_VARIANT=1"; do
  name=${cfg%%:*}; envs=${cfg#*:}
  echo "== $name ($envs)"
  env $envs timeout 300 python tools/timeline.py $K 2>&1 | sed -n '1,6p'
done
