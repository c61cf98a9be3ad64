#!/bin/bash
# Per-tile timeline of the capped streamed run on cfg3 (AB2_TRACE=1), plus the pipeline tests.
TAG=${1:-tr}
mkdir -p gpurun_out
AB2_TRACE=1 timeout 600 python tools/ooc_trace.py cfg3 0.5 0.25 0.125 > gpurun_out/trace_$TAG.txt 2>&1
[ -n "$SKIPT" ] || timeout 900 python -m pytest tests/test_gpu_pipeline.py -q -m gpu -x 2>&1 | tail -5 >> gpurun_out/trace_$TAG.txt
tail -5 gpurun_out/trace_$TAG.txt
