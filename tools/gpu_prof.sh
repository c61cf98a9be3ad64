#!/bin/bash
# ncu --set full capture of one kernel (regex) in the bench: tools/gpu_prof.sh TAG REGEX [bench args...]
TAG=${1:-p}; RE=${2:-k_numeric}; shift 2
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:$RE" --launch-skip 2 \
  --launch-count 1 -f -o gpurun_out/prof_$TAG python bench.py --steps 1 --warmup 3 --skip-cpu --skip-e2e --skip-ooc --skip-gcn "$@" \
  > gpurun_out/ncu_$TAG.log 2>&1
tail -2 gpurun_out/ncu_$TAG.log
