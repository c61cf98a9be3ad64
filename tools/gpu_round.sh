#!/bin/bash
# One GPU session: smoke, parity tests, a bench line, the ncu launch list and one full ncu capture.
# usage: tools/gpu_round.sh TAG [bench args...]
TAG=${1:-r}; shift
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu_$TAG.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.txt 2>&1
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -15 > gpurun_out/tests_$TAG.txt
timeout 600 python bench.py "$@" 2> gpurun_out/bench_$TAG.err | tee gpurun_out/bench_$TAG.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
  python bench.py --steps 2 --warmup 3 --skip-cpu --skip-e2e --skip-ooc --skip-gcn "$@" > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k 'regex:k_numeric|k_place' --launch-skip 6 \
  --launch-count 2 -f -o gpurun_out/prof_$TAG python bench.py --steps 1 --warmup 3 --skip-cpu --skip-e2e --skip-ooc --skip-gcn "$@" \
  > gpurun_out/ncu_$TAG.log 2>&1
cat gpurun_out/smoke_$TAG.txt gpurun_out/tests_$TAG.txt
