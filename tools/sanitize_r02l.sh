#!/bin/bash
# compute-sanitizer over the kernels changed late in round 2: the short-row dense cells (every small
# parity product with <= 256 output columns), k_agg_t_cp (cp.async gather), k_hw_tc (hoisted loads).
mkdir -p gpurun_out
SEL="not cfg1_shape and not full_size and not layer_forward_two"
for tool in memcheck synccheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 \
    python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "$SEL" > gpurun_out/san_$tool.txt 2>&1
  echo "== $tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|passed|failed' gpurun_out/san_$tool.txt | tail -2 | tr '\n' ' ')"
done
