"""Resident product kernel time vs one aires_b200_set_option value (results must stay identical).
usage: python tools/option_sweep.py CFG fp32|fp64 OPTION V1 [V2 ...]   e.g. cfg3 fp32 short_pipe 0 1"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2507_02006_b200 as ab  # noqa: E402

cfg, mode_s, name = sys.argv[1], sys.argv[2], sys.argv[3]
vals = [int(v) for v in sys.argv[4:]]
mode = ab.MODE_FP64_EXACT if mode_s == "fp64" else ab.MODE_FP32
g, st, x = bench.make_inputs(bench.CONFIGS[cfg])
dev = torch.device("cuda", 0)
L = ab.lib()
p = bench.DeviceProduct(ab, torch, dev, g, x, mode)
ref = None
for v in vals:
    ab.set_option(name, v)
    for _ in range(3):
        p.step()
    ks, steps = [], []
    for _ in range(7):
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record()
        p.step()
        s1.record()
        torch.cuda.synchronize()
        steps.append(s0.elapsed_time(s1))
        prof = (ctypes.c_double * 8)()
        L.aires_b200_last_profile(prof, 8)
        ks.append(prof[3])
    r = p.result_host()
    same = ref is None or all(np.array_equal(np.asarray(a).view(np.uint8), np.asarray(b).view(np.uint8))
                              for a, b in zip(r, ref))
    ref = ref or r
    print(f"{cfg} {mode_s} {name}={v}: numeric {np.median(ks):.3f} ms  step {np.median(steps):.3f} ms  "
          f"identical {same}", flush=True)
