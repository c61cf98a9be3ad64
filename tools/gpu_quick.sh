#!/bin/bash
# Quick GPU check of a kernel change: parity + pipeline tests, a resident cfg2 bench line, one ncu capture of k_numeric.
# usage: tools/gpu_quick.sh TAG
TAG=${1:-q}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pipeline.py -q -m gpu -x 2>&1 | tail -15 > gpurun_out/t_$TAG.txt
timeout 300 python bench.py --steps 5 --warmup 3 --skip-cpu --skip-e2e --skip-ooc --skip-gcn --skip-fp64 > gpurun_out/b_$TAG.json 2> gpurun_out/b_$TAG.err
timeout 600 ncu --set full --import-source on --clock-control none -k 'regex:k_numeric' --launch-skip 3 --launch-count 1 -f -o gpurun_out/prof_$TAG python bench.py --steps 1 --warmup 3 --skip-cpu --skip-e2e --skip-ooc --skip-gcn --skip-fp64 > gpurun_out/ncu_$TAG.log 2>&1
cat gpurun_out/t_$TAG.txt; python -c "import json;d=json.load(open('gpurun_out/b_$TAG.json'));print(d['ms_per_step'],d['roofline'])"
