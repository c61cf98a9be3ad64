#!/bin/bash
# ncu --set full of one k_numeric launch of the resident cfg2 bench (fp32), summarised on the box.
# usage: tools/gpu_ncu_num.sh TAG [launch-skip]
TAG=${1:-n}; SKIP=${2:-3}
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k 'regex:k_numeric' --launch-skip $SKIP --launch-count 1 \
  -f -o /tmp/prof_$TAG python bench.py --steps 1 --warmup 3 --skip-cpu --skip-e2e --skip-ooc --skip-gcn --skip-fp64 \
  > gpurun_out/ncu_$TAG.log 2>&1
python tools/ncu_summary.py /tmp/prof_$TAG.ncu-rep > gpurun_out/ncu_$TAG.txt 2>&1
python tools/ncu_wavefronts.py /tmp/prof_$TAG.ncu-rep >> gpurun_out/ncu_$TAG.txt 2>&1
ncu -i /tmp/prof_$TAG.ncu-rep --page source --csv > gpurun_out/src_$TAG.csv 2>/dev/null
ls -la gpurun_out/
