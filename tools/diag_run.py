"""Where the wall time of an aires_b200_run goes (cfg inputs, pinned host buffers).
usage: [AB2_TRACE=1] python tools/diag_run.py [cfg2] [budget_MB] [stream] [name=value ...]
(stream: AIRES_B200_RUN_STREAM_OUT; name=value: aires_b200_set_option, e.g. narrow_cols=0)"""
import ctypes as C
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2507_02006_b200 as ab  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg2"]
g, st, x = bench.make_inputs(cfg)
L = ab.lib()
hA = [torch.from_numpy(g.row_ptr.view(np.int64)).pin_memory(), torch.from_numpy(g.col_idx.view(np.int32)).pin_memory(),
      torch.from_numpy(g.values.astype(np.float32)).pin_memory()]
hX = [torch.from_numpy(x.row_ptr.view(np.int64)).pin_memory(), torch.from_numpy(x.col_idx.view(np.int32)).pin_memory(),
      torch.from_numpy(x.values.astype(np.float32)).pin_memory()]
am = ab._Matrix(g.n_rows, g.n_cols, ab.CSR, ab.HOST, 4, 4, hA[0].data_ptr(), hA[1].data_ptr(), hA[2].data_ptr(), g.nnz())
xm = ab._Matrix(x.n_rows, x.n_cols, ab.CSR, ab.HOST, 4, 4, hX[0].data_ptr(), hX[1].data_ptr(), hX[2].data_ptr(), x.nnz())
hout = {}


def alloc(user, rows, nnz, pp, pi, pv):
    if hout.get("cap", -1) < nnz:
        hout["ptr"] = torch.empty(rows + 1, dtype=torch.int64).pin_memory()
        hout["idx"] = torch.empty(max(nnz, 1), dtype=torch.int32).pin_memory()
        hout["val"] = torch.empty(max(nnz, 1), dtype=torch.float32).pin_memory()
        hout["cap"] = nnz
    pp[0], pi[0], pv[0] = hout["ptr"].data_ptr(), hout["idx"].data_ptr(), hout["val"].data_ptr()
    return 0


afn = ab._ALLOC_FN(alloc)
out = ab._Output(ab.HOST, 4, 4, 0, afn, None, 0, 0, 0, 0)
budget = int(float(sys.argv[2]) * 1e6) if len(sys.argv) > 2 else 0
flags = ab.RUN_STREAM_OUT if "stream" in sys.argv[3:] else 0
nbuf = int(os.environ.get("NBUF", "0" if flags else "3"))
for kv in sys.argv[3:]:
    if "=" in kv:
        k, v = kv.split("=")
        ab.set_option(k, int(v))
for it in range(4):
    rep = ab._RunReport()
    t0 = time.perf_counter()
    ab._check(L.aires_b200_run(C.byref(am), C.byref(xm), C.byref(ab._RunConfig(budget, ab.MODE_FP32, 1, nbuf, flags)),
                               C.byref(out), C.byref(rep)))
    print(f"run {it}: wall {(time.perf_counter() - t0) * 1e3:.2f} ms device {rep.total_ms:.2f} ms "
          f"p1 {rep.phase1_ms:.2f} p2 {rep.phase2_ms:.2f} p3 {rep.phase3_ms:.2f} segs {rep.segments} "
          f"h2d {rep.h2d_bytes / 1e6:.0f} MB d2h {rep.d2h_bytes / 1e6:.0f} MB", flush=True)
