#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over the small GPU parity suite.
# usage (on the GPU box): tools/sanitize.sh TAG
TAG=${1:-s}
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 \
    python -m pytest tests/test_gpu_parity.py tests/test_gpu_pipeline.py -q -m gpu -x \
    -k "not cfg1_shape and not layer_forward_two" > gpurun_out/sanitize_${tool}_$TAG.txt 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|passed|failed' gpurun_out/sanitize_${tool}_$TAG.txt | tail -2 | tr '\n' ' ')"
done
