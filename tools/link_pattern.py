"""The e2e run's copy pattern without its kernels: 16 tiles, H2D of two arrays per tile on one stream,
D2H of two arrays per tile on another (tile j's D2H after tile j's H2D), pinned buffers; offsets
4-byte aligned (as the run's tiles are) or 4 KiB aligned.  usage: python tools/link_pattern.py"""
import torch

dev = torch.device("cuda:0")
A = 929 << 20
C = 774 << 20
hA = torch.empty(A + (1 << 20), dtype=torch.uint8).pin_memory()
hC = torch.empty(C + (1 << 20), dtype=torch.uint8).pin_memory()
dA = torch.empty(A + (1 << 20), dtype=torch.uint8, device=dev)
dC = torch.empty(C + (1 << 20), dtype=torch.uint8, device=dev)
su, sd = torch.cuda.Stream(dev), torch.cuda.Stream(dev)


def run(align, tiles=16, split=2):
    ta, tc = A // tiles, C // tiles
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e0.record()
    su.wait_event(e0)
    sd.wait_event(e0)
    for j in range(tiles):
        for p in range(split):
            o = (j * ta + p * (ta // split)) // align * align
            n = ta // split
            with torch.cuda.stream(su):
                dA[o:o + n].copy_(hA[o + 4:o + 4 + n] if align == 4 else hA[o:o + n], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(su)
        sd.wait_event(ev)
        for p in range(split):
            o = (j * tc + p * (tc // split)) // align * align
            n = tc // split
            with torch.cuda.stream(sd):
                (hC[o + 4:o + 4 + n] if align == 4 else hC[o:o + n]).copy_(dC[o:o + n], non_blocking=True)
    e1, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e1.record(su)
    e2.record(sd)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1), e0.elapsed_time(e2)


for align in (4, 4096):
    for tiles in (16, 64):
        best = min((run(align, tiles) for _ in range(4)), key=lambda t: max(t))
        print(f"align {align:5d} tiles {tiles:3d}: H2D done {best[0]:.2f} ms ({A / best[0] / 1e6:.1f} GB/s), "
              f"D2H done {best[1]:.2f} ms; total {(A + C) / max(best) / 1e6:.1f} GB/s", flush=True)
