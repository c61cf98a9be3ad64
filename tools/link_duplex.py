"""Host-link bandwidth one way and both ways at once (pinned buffers, CUDA events): what a run that
overlaps the H2D of A with the D2H of C can expect.  usage: python tools/link_duplex.py [MB] [load]   (load: an HBM-bound device copy runs alongside)"""
import sys

import torch

mb = int(sys.argv[1]) if len(sys.argv) > 1 else 512
n = mb << 20
dev = torch.device("cuda:0")
hu, hd = torch.empty(n, dtype=torch.uint8).pin_memory(), torch.empty(n, dtype=torch.uint8).pin_memory()
du, dd = torch.empty(n, dtype=torch.uint8, device=dev), torch.empty(n, dtype=torch.uint8, device=dev)
su, sd = torch.cuda.Stream(dev), torch.cuda.Stream(dev)


def timed(ops):
    best = 1e9
    for _ in range(5):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e0.record()
        ends = []
        for s, fn in ops:
            s.wait_event(e0)
            with torch.cuda.stream(s):
                fn()
                e = torch.cuda.Event(enable_timing=True)
                e.record()
                ends.append(e)
        torch.cuda.synchronize()
        best = min(best, max(e0.elapsed_time(e) for e in ends))
    return best


up = lambda: du.copy_(hu, non_blocking=True)  # noqa: E731
down = lambda: hd.copy_(dd, non_blocking=True)  # noqa: E731
load = "load" in sys.argv[2:]
if load:  # an HBM-bound device-to-device copy loop on a third stream, as the product kernels would be
    sl = torch.cuda.Stream(dev)
    ba, bb = torch.empty(1 << 30, dtype=torch.uint8, device=dev), torch.empty(1 << 30, dtype=torch.uint8, device=dev)

    def up_load():
        with torch.cuda.stream(sl):
            for _ in range(40):
                bb.copy_(ba)
        du.copy_(hu, non_blocking=True)
    t_both_load = timed([(su, up), (sd, down), (sl, lambda: [bb.copy_(ba) for _ in range(20)])])
    print(f"both at once with a device copy loop alongside: {t_both_load:.2f} ms (includes the loop)")
t_up, t_down, t_both = timed([(su, up)]), timed([(sd, down)]), timed([(su, up), (sd, down)])
print(f"H2D {n / t_up / 1e6:.1f} GB/s, D2H {n / t_down / 1e6:.1f} GB/s, both at once {2 * n / t_both / 1e6:.1f} GB/s "
      f"total ({t_both:.2f} ms for {mb} MB each way; serial would be {t_up + t_down:.2f} ms)")
