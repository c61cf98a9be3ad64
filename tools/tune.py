"""GPU tuning harness: one cfg-shaped input, parity vs the oracle once, then a sweep of
kernel knobs (environment variables read per call) printing the per-stage device times.
usage: python tools/tune.py [cfg2] [KNOB=v1,v2 ...]"""
import itertools
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2507_02006_b200 as ab  # noqa: E402
from oracle import pyoracle as po  # noqa: E402


def main():
    cfgname = sys.argv[1] if len(sys.argv) > 1 and "=" not in sys.argv[1] else "cfg2"
    knobs = [a.split("=") for a in sys.argv[1:] if "=" in a]
    cfg = bench.CONFIGS[cfgname]
    g, st, x = bench.make_inputs(cfg, 0, 1)
    g32 = ab.CsrMatrix(g.n_rows, g.n_cols, g.row_ptr, g.col_idx, g.values.astype(np.float32))
    x32 = ab.CsrMatrix(x.n_rows, x.n_cols, x.row_ptr, x.col_idx, x.values.astype(np.float32))
    op = ab.Operand(x32)
    t = time.time()
    c = ab.spgemm_full(g32, op)
    rc, (wp, wi, wv), macs = po.spgemm_rowwise(g.row_ptr, g.col_idx.astype(np.uint64), g.values, g.n_rows,
                                               g.n_cols, x.n_rows, x.n_cols, x.row_ptr,
                                               x.col_idx.astype(np.uint64), x.values,
                                               nthreads=len(os.sched_getaffinity(0)))
    ok = (np.array_equal(c.row_ptr, wp) and np.array_equal(c.col_idx.astype(np.uint64), wi))
    err = np.abs(c.values.astype(np.float64) - wv) / np.maximum(np.abs(wv), 1e-30)
    print(f"parity: structure {'OK' if ok else 'MISMATCH'} nnz {c.nnz()} vs {wi.shape[0]}, max rel err "
          f"{err.max(initial=0):.3e}, macs {macs} ({time.time() - t:.1f}s)", flush=True)
    names = [k for k, _ in knobs]
    for vals in itertools.product(*[v.split(",") for _, v in knobs]):
        for k, v in zip(names, vals):
            os.environ[k] = v
        op = ab.Operand(x32)  # layout knobs are read when the operand is built
        ts = []
        for it in range(6):
            ab.spgemm_full(g32, op)
            p = ab.last_profile()
            if it >= 2:
                ts.append(p)
        med = {k: float(np.median([q[k] for q in ts])) for k in ts[0]}
        print(" ".join(f"{k}={v}" for k, v in zip(names, vals)),
              " ".join(f"{k}={med[k]:.3f}" for k in ("numeric", "symbolic", "scan", "total")), flush=True)


if __name__ == "__main__":
    main()
