#!/bin/bash
# ncu --set full of one k_hw_tc launch (cfg5 layer 2), summarised on the box.
TAG=${1:-hw}
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:${KREGEX:-k_hw}" --launch-skip ${SKIP:-1} --launch-count 1 \
  -f -o /tmp/prof_$TAG python bench.py --steps 1 --warmup 3 --skip-cpu --skip-e2e --skip-ooc --skip-fp64 > gpurun_out/ncu_$TAG.log 2>&1
python tools/ncu_summary.py /tmp/prof_$TAG.ncu-rep > gpurun_out/ncu_$TAG.txt 2>&1
ncu -i /tmp/prof_$TAG.ncu-rep --page source --csv > gpurun_out/src_$TAG.csv 2>/dev/null
