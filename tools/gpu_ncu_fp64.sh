#!/bin/bash
# ncu --set full of one FP64_EXACT k_numeric3 launch (cfg2), summarised on the box.
TAG=${1:-d}
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k 'regex:numeric3<double' \
  --launch-skip 2 --launch-count 1 -f -o /tmp/prof_$TAG python bench.py --steps 1 --warmup 3 --skip-cpu --skip-e2e \
  --skip-ooc --skip-gcn > gpurun_out/ncu_$TAG.log 2>&1
python tools/ncu_summary.py /tmp/prof_$TAG.ncu-rep > gpurun_out/ncu_$TAG.txt 2>&1
python tools/ncu_wavefronts.py /tmp/prof_$TAG.ncu-rep >> gpurun_out/ncu_$TAG.txt 2>&1
ncu -i /tmp/prof_$TAG.ncu-rep --page source --csv > gpurun_out/src_$TAG.csv 2>/dev/null
