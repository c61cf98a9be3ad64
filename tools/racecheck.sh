#!/bin/bash
# compute-sanitizer racecheck over the parity and pipeline suites.  usage: tools/racecheck.sh TAG
TAG=${1:-s}
mkdir -p gpurun_out
timeout 2400 compute-sanitizer --tool racecheck --print-limit 20 --error-exitcode 9 \
  python -m pytest tests/test_gpu_parity.py tests/test_gpu_pipeline.py -q -m gpu -x \
  -k "not cfg1_shape and not layer_forward_two" > gpurun_out/sanitize_racecheck_$TAG.txt 2>&1
echo "racecheck rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|passed|failed' gpurun_out/sanitize_racecheck_$TAG.txt | tail -3 | tr '\n' ' ')"
