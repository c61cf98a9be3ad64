#!/bin/bash
# Full round check: smoke, every GPU test, the default bench line, the reference arm, the ncu launch list.
# usage: tools/gpu_full.sh TAG
TAG=${1:-full}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu_$TAG.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.txt 2>&1
timeout 1800 python -m pytest tests -q -m gpu 2>&1 | tail -25 > gpurun_out/tests_$TAG.txt
timeout 900 python bench.py 2> gpurun_out/bench_$TAG.err > gpurun_out/bench_$TAG.json
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 2> gpurun_out/ref_$TAG.err > gpurun_out/ref_$TAG.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
  python bench.py --steps 2 --warmup 3 --skip-cpu --skip-e2e --skip-ooc --skip-gcn --skip-fp64 > /dev/null 2>&1
cat gpurun_out/smoke_$TAG.txt gpurun_out/tests_$TAG.txt
