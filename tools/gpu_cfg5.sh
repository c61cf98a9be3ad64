#!/bin/bash
# cfg5 check: the GCN/fused-layer GPU tests, the cfg5 bench leg, and its ncu launch list.
# usage: tools/gpu_cfg5.sh TAG
TAG=${1:-cfg5}
mkdir -p gpurun_out
timeout 300 python -m pytest tests -q -m gpu -k "layer or gcn or fused or normalize or combine" 2>&1 | tail -3 > gpurun_out/cfg5_tests_$TAG.txt
timeout 300 python bench.py --steps 5 --warmup 3 --skip-cpu --skip-e2e --skip-ooc --skip-fp64 2>/dev/null | tail -1 > gpurun_out/cfg5_$TAG.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cfg5_launches_$TAG.csv \
  python bench.py --steps 1 --warmup 3 --skip-cpu --skip-e2e --skip-ooc --skip-fp64 > /dev/null 2>&1
