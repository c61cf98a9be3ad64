"""Pinned cudaMemcpy GB/s vs host / device start offsets (the DMA alignment penalty of writing C tiles at
arbitrary CSR offsets).  usage: python tools/link_align.py"""
import torch
n = 64 << 20
dev = torch.device("cuda:0")
h = torch.empty(n + 4096, dtype=torch.uint8).pin_memory()
d = torch.empty(n + 4096, dtype=torch.uint8, device=dev)
for off_h, off_d in ((0, 0), (4, 0), (0, 4), (4, 4), (8, 0), (16, 0), (64, 0), (128, 0), (512, 0)):
    for name, fn in (("d2h", lambda: h[off_h:off_h + n].copy_(d[off_d:off_d + n], non_blocking=True)),
                     ("h2d", lambda: d[off_d:off_d + n].copy_(h[off_h:off_h + n], non_blocking=True))):
        best = 1e9
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); fn(); e1.record(); e1.synchronize()
            best = min(best, e0.elapsed_time(e1))
        print(f"host+{off_h} dev+{off_d} {name}: {n / best / 1e6:.1f} GB/s")
