"""Per-tile timeline of the capped streamed out-of-core run (AB2_TRACE=1) on a bench config.
usage: AB2_TRACE=1 python tools/ooc_trace.py [cfg3|cfg2] [frac ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2507_02006_b200 as ab  # noqa: E402
import torch  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
fracs = [float(f) for f in sys.argv[2:]] or [0.25]
g, st, x = bench.make_inputs(bench.CONFIGS[name])
c_bound = min(g.n_rows * x.n_cols, g.nnz() * 64)
h = bench.HostOperands(ab, torch, g, x, cap=c_bound)
rep0 = h.run(budget=0, c_aware=1, n_buffers=2)
b = 16 * (g.n_rows + 1) + 8 * (g.nnz() + int(rep0.c_nnz)) + 8 * (x.n_rows + 1) + 8 * x.nnz()
for f in fracs:
    for _ in range(2):
        rep = h.run(budget=int(f * b), c_aware=1, n_buffers=3, flags=ab.RUN_STREAM_OUT)
    print(f"{name} @{f}: {rep.total_ms:.3f} ms, phase1 {rep.phase1_ms:.3f} phase2 {rep.phase2_ms:.3f} "
          f"phase3 {rep.phase3_ms:.3f}, parts {rep.segments}, h2d {rep.h2d_bytes}", flush=True)
