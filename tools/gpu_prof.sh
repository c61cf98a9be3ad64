#!/bin/bash
# ncu capture of the product kernels only: tools/gpu_prof.sh TAG [bench args...]
TAG=${1:-p}; shift
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k 'regex:k_numeric3|k_place' --launch-skip 6 \
  --launch-count 2 -f -o gpurun_out/prof_$TAG python bench.py --steps 1 --warmup 3 --skip-cpu --skip-e2e "$@" \
  > gpurun_out/ncu_$TAG.log 2>&1
tail -3 gpurun_out/ncu_$TAG.log
