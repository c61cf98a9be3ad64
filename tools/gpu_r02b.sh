#!/bin/bash
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu_r02b.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02b.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -25 > gpurun_out/tests_r02b.txt
timeout 900 python bench.py 2> gpurun_out/bench_r02b.err > gpurun_out/bench_r02b.json
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 2> gpurun_out/ref_r02b.err > gpurun_out/ref_r02b.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02b.csv \
  python bench.py --steps 2 --warmup 3 --skip-cpu --skip-e2e --skip-ooc --skip-gcn --skip-fp64 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k 'regex:k_numeric|k_place' --launch-skip 6 \
  --launch-count 2 -f -o gpurun_out/prof_r02b python bench.py --steps 1 --warmup 3 --skip-cpu --skip-e2e --skip-ooc --skip-gcn --skip-fp64 \
  > gpurun_out/ncu_r02b.log 2>&1
cat gpurun_out/smoke_r02b.txt gpurun_out/tests_r02b.txt
