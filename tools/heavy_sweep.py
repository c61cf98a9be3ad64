"""Resident cfg2 product time vs the heavy-row degree threshold (aires_b200_set_option heavy_deg), per
mode.  usage: python tools/heavy_sweep.py [fp64|fp32] [deg ...]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2507_02006_b200 as ab  # noqa: E402

mode = ab.MODE_FP64_EXACT if (sys.argv[1:2] or ["fp64"])[0] == "fp64" else ab.MODE_FP32
degs = [int(v) for v in sys.argv[2:]] or [1024, 4096, 1 << 30]
g, st, x = bench.make_inputs(bench.CONFIGS["cfg2"])
dev = torch.device("cuda", 0)
L = ab.lib()
p = bench.DeviceProduct(ab, torch, dev, g, x, mode)
ref = None
for d in degs:
    ab.set_option("heavy_deg", d)
    for _ in range(3):
        p.step()
    ks = []
    for _ in range(5):
        p.step()
        prof = (C_double := __import__("ctypes").c_double * 8)()
        L.aires_b200_last_profile(prof, 8)
        ks.append(prof[3])
    r = p.result_host()
    same = ref is None or (np.array_equal(r[0], ref[0]) and np.array_equal(r[1], ref[1]) and
                           np.array_equal(np.asarray(r[2]).view(np.uint64 if r[2].itemsize == 8 else np.uint32),
                                          np.asarray(ref[2]).view(np.uint64 if ref[2].itemsize == 8 else np.uint32)))
    ref = ref or r
    print(f"heavy_deg {d}: numeric {np.median(ks):.3f} ms  identical {same}", flush=True)
