#!/bin/bash
# GPU check of the out-of-core run: pipeline + full-size tests, then the bench's out-of-core legs.
# usage: tools/gpu_ooc.sh TAG
TAG=${1:-o}
mkdir -p gpurun_out
[ -n "$SKIPT" ] || timeout 900 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_scale.py -q -m gpu -x 2>&1 | tail -15 > gpurun_out/t_$TAG.txt
timeout 600 python bench.py --steps 5 --warmup 3 --skip-cpu --skip-e2e --skip-gcn --skip-fp64 > gpurun_out/b_$TAG.json 2> gpurun_out/b_$TAG.err
cat gpurun_out/t_$TAG.txt
python - <<PY
import json
d = json.load(open("gpurun_out/b_$TAG.json"))
for r in d["out_of_core"]["runs"]:
    print(r["label"], r["ms"], "seg", r["segments"], "h2d/alg", r["h2d_over_algorithmic"], "frac", r["roofline"]["frac"],
          "exact", r["exact_protocol"].get("ms"), r["exact_protocol"].get("h2d_over_algorithmic"), "chk", r["checked"],
          "mm", r.get("maxmemory_baseline", {}).get("ms"))
PY
