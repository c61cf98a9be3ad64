"""Resident cfg2 product time vs a forced X slot width (aires_b200_set_option slot_w).
usage: python tools/slotw_sweep.py [fp64|fp32] [W ...]"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2507_02006_b200 as ab  # noqa: E402

mode = ab.MODE_FP64_EXACT if (sys.argv[1:2] or ["fp64"])[0] == "fp64" else ab.MODE_FP32
ws = [int(v) for v in sys.argv[2:]] or [16, 8]
g, st, x = bench.make_inputs(bench.CONFIGS["cfg2"])
dev = torch.device("cuda", 0)
L = ab.lib()
p = bench.DeviceProduct(ab, torch, dev, g, x, mode)
ref = None
for w in ws:
    ab.set_option("slot_w", w)
    for _ in range(3):
        p.step()
    ks = []
    for _ in range(5):
        p.step()
        prof = (ctypes.c_double * 8)()
        L.aires_b200_last_profile(prof, 8)
        ks.append(prof[3])
    r = p.result_host()
    same = ref is None or all(np.array_equal(np.asarray(a).view(np.uint8), np.asarray(b).view(np.uint8))
                              for a, b in zip(r, ref))
    ref = ref or r
    print(f"slot_w {w}: numeric {np.median(ks):.3f} ms  identical {same}", flush=True)
