#!/usr/bin/env python
"""bench.py -- A·X SpGEMM (AIRES hot path) on B200: latency, GFLOP/s and roofline fraction.

Contract (driver): `python bench.py --gpus N --steps K --warmup W` prints ONE JSON line on
rank 0.  N>1 runs under torchrun, one rank per GPU (NCCL); every rank owns one contiguous
row block (weak scaling: each rank's block is a cfg-shaped Ã_r over its own slice of the
replicated X) and the only collective is the all-gather of per-rank nnz(C) that forms the
global row_ptr offsets.

Workload at N=1: BASELINE.json configs[1] (Reddit-shaped, 232,965 nodes, 114 M edges, X 602
wide at 1 %, fully HBM-resident), synthetic (BASELINE.md §4 seeds: graph 1, relabel 2, X 3).
A "step" is one full A·X through the C ABI (aires_b200_spgemm) with device-resident A and X
(device C): X layout build, classify, symbolic, scan, nnz readback + exact allocation,
numeric.  `e2e` is the same call with pinned HOST buffers (H2D of A and X and D2H of C
inside the timed region).  `--impl reference` times the reference's own CPU spgemm_block
(oracle/_ref, built from /root/reference) on a row sample with all host threads.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "A·X SpGEMM latency (ms) and GFLOP/s; % of HBM/host-link roofline at 1/2/4/8 B200"

CONFIGS = {
    "cfg1": dict(workload="cfg1: power-law 100K nodes / 1M edges, X 100Kx512 @1%",
                 n=100_000, nnz=1_000_000, dim=512, cap=20_000),
    "cfg2": dict(workload="cfg2: Reddit-shaped 232,965 nodes / 114M edges, X 602 @1%, HBM-resident",
                 n=232_965, nnz=114_000_000, dim=602, cap=20_000),
    "cfg3": dict(workload="cfg3: ogbn-products-shaped 2,449,029 nodes / 62M edges, X 100 @1%",
                 n=2_449_029, nnz=62_000_000, dim=100, cap=20_000),
    # one of eight row-block shards of the PPI-scale graph (68M nodes / 1.5B edges, X 256 @1%):
    # the per-GPU unit of the 8-GPU run, generated as its own power-law block
    "cfg4shard": dict(workload="cfg4 shard: 1/8 of the PPI-scale graph (8.5M nodes / 187.5M edges, X 256 @1%), "
                               "pinned-host streaming", n=8_500_000, nnz=187_500_000, dim=256, cap=50_000),
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons during the timed region (B200_PROFILING.md)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.samples, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.samples.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def make_inputs(cfg: dict, rank: int, world: int):
    """Rank r: Ã_r (seed 1+r) over node block r; X (seed 3) covering all world*n rows."""
    import paper_2507_02006_b200 as ab
    n = cfg["n"]
    t0 = time.time()
    g, st = ab.synth_graph(n, cfg["nnz"], alpha=0.75, degree_cap=cfg["cap"], seed=1 + rank, relabel_seed=2,
                           idx_dtype=np.uint32, val_dtype=np.float64)
    x = ab.synth_features(n * world, cfg["dim"], 99.0, 3, idx_dtype=np.uint32, val_dtype=np.float64)
    if world > 1:  # Ã_r's columns address X rows [r*n, (r+1)*n)
        g.col_idx = g.col_idx + np.uint32(rank * n)
        g.n_cols = n * world
    log(f"[rank {rank}] inputs: A {g.n_rows}x{g.n_cols} nnz {g.nnz()} (edges {st['nnz_a']}, max deg "
        f"{st['max_degree']}), X {x.n_rows}x{x.n_cols} nnz {x.nnz()} in {time.time() - t0:.1f}s")
    return g, st, x


def algorithmic_bytes(n_rows, nnz_a, k_rows, nnz_x, nnz_c, vb=4):
    """Σ_{A,X,C} 8(rows+1) + (4+vb)·nnz (int64 ptr, int32 idx, fp32/fp64 val)."""
    return (8 * (n_rows + 1) + (4 + vb) * nnz_a) + (8 * (k_rows + 1) + (4 + vb) * nnz_x) + \
        (8 * (n_rows + 1) + (4 + vb) * nnz_c)


def run_b200(args, cfg):
    import torch
    import paper_2507_02006_b200 as ab

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # AB2_FORCE_DEVICE / AB2_DIST_BACKEND exist only to exercise the multi-rank flow on a one-GPU box
    # (gloo, every rank on the same device); production runs use NCCL, one GPU per rank.
    if os.environ.get("AB2_FORCE_DEVICE"):
        local = int(os.environ["AB2_FORCE_DEVICE"])
    backend = os.environ.get("AB2_DIST_BACKEND", "nccl")
    dist = None
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group(backend)
    torch.cuda.set_device(local)
    cdev = torch.device("cuda", local) if backend == "nccl" else torch.device("cpu")  # collective tensors
    L = ab.lib()
    ab._check(L.aires_b200_set_device(local))
    dev = torch.device("cuda", local)
    mode = ab.MODE_FP64_EXACT if args.mode == "fp64" else ab.MODE_FP32
    vdt_np = np.float64 if mode == ab.MODE_FP64_EXACT else np.float32
    vdt_t = torch.float64 if mode == ab.MODE_FP64_EXACT else torch.float32
    vb = 8 if mode == ab.MODE_FP64_EXACT else 4

    g, st, x = make_inputs(cfg, rank, world)
    n, K = g.n_rows, x.n_rows
    # device-resident inputs (u64 ptr, u32 idx, fp32/fp64 values)
    tA = [torch.from_numpy(g.row_ptr.view(np.int64)).to(dev), torch.from_numpy(g.col_idx.view(np.int32)).to(dev),
          torch.from_numpy(g.values.astype(vdt_np)).to(dev)]
    tX = [torch.from_numpy(x.row_ptr.view(np.int64)).to(dev), torch.from_numpy(x.col_idx.view(np.int32)).to(dev),
          torch.from_numpy(x.values.astype(vdt_np)).to(dev)]
    am = ab._Matrix(n, g.n_cols, ab.CSR, ab.DEVICE, 4, vb, tA[0].data_ptr(), tA[1].data_ptr(), tA[2].data_ptr(),
                    g.nnz())
    xm = ab._Matrix(K, x.n_cols, ab.CSR, ab.DEVICE, 4, vb, tX[0].data_ptr(), tX[1].data_ptr(), tX[2].data_ptr(),
                    x.nnz())

    # device output: grow-only buffers handed out by the allocator
    outbuf = {}

    def dev_alloc(user, rows, nnz, pp, pi, pv):
        if outbuf.get("cap", -1) < nnz:
            outbuf["ptr"] = torch.empty(rows + 1, dtype=torch.int64, device=dev)
            outbuf["idx"] = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)
            outbuf["val"] = torch.empty(max(nnz, 1), dtype=vdt_t, device=dev)
            outbuf["cap"] = nnz
        pp[0], pi[0], pv[0] = outbuf["ptr"].data_ptr(), outbuf["idx"].data_ptr(), outbuf["val"].data_ptr()
        return 0

    afn = ab._ALLOC_FN(dev_alloc)
    out = ab._Output(ab.DEVICE, 4, vb, 0, afn, None, 0, 0, 0, 0)

    def step():
        ab._check(L.aires_b200_spgemm(C.byref(am), C.byref(xm), mode, C.byref(out)))

    lib_stream = torch.cuda.ExternalStream(L.aires_b200_stream(), device=dev)
    for _ in range(args.warmup):
        step()
    nnz_c, macs = int(out.nnz), int(out.flops)
    prof_keys = ["classify", "symbolic", "scan", "numeric", "x_prep"]
    prof_sum = {k: 0.0 for k in prof_keys}
    launches = 0
    torch.cuda.synchronize(dev)
    if dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    from paper_2507_02006_b200 import shard
    offsets = np.zeros(world, dtype=np.int64)
    with ClockSampler(local) as clk:
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(lib_stream)
        for _ in range(args.steps):
            step()
            p = ab.last_profile()
            for k in prof_keys:
                prof_sum[k] += p[k]
            launches += L.aires_b200_last_launches()
            if dist:  # global row_ptr offsets: all-gather of one int64 nnz(C) per rank (shard.py)
                offsets, _ = shard.global_offsets(int(out.nnz), device=cdev)
        ev1.record(lib_stream)
        ev1.synchronize()
    torch.cuda.synchronize(dev)
    if dist:
        dist.barrier()
    ms_rank = ev0.elapsed_time(ev1) / args.steps
    ms = ms_rank
    tot_macs = macs
    if dist:
        t = torch.tensor([ms_rank], dtype=torch.float64, device=cdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        m = torch.tensor([macs], dtype=torch.int64, device=cdev)
        dist.all_reduce(m)
        tot_macs = int(m.item())
    gflops = 2.0 * tot_macs / (ms * 1e-3) / 1e9
    c_ptr_check = c_idx_check = None
    if not args.skip_e2e and rank == 0 and world == 1:  # the device product, to check the host-API run against
        c_ptr_check = outbuf["ptr"][: n + 1].cpu().numpy().view(np.uint64)
        c_idx_check = outbuf["idx"][:nnz_c].cpu().numpy()

    # roofline of the dominant kernel (numeric) and of the whole step
    peak, peak_src = peaks()
    b_alg = algorithmic_bytes(n, g.nnz(), K, x.nnz(), nnz_c, vb)
    num_ms = prof_sum["numeric"] / args.steps
    sym_ms = prof_sum["symbolic"] / args.steps
    ach = b_alg / (num_ms * 1e-3) / 1e9
    traffic = None
    try:  # DRAM bytes of the dominant kernel from the committed ncu --set full capture (cfg2 fp32)
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            tj = json.load(f)
        if cfg is CONFIGS["cfg2"] and vb == 4 and "k_numeric3" in tj:
            traffic = tj["k_numeric3"]["dram_bytes"]
    except Exception:
        traffic = None
    roof = {"bound": "hbm", "achieved": round(ach, 1), "peak": peak, "unit": "GB/s", "frac": round(ach / peak, 4),
            "traffic": traffic, "traffic_source": "profiles/traffic.json (ncu dram__bytes_read+write, one launch)",
            "kernel": "k_numeric3_f32" if vb == 4 else "k_numeric3_f64",
            "kernel_ms": round(num_ms, 4), "bytes_per_launch": b_alg, "peak_source": peak_src,
            "step_frac": round(b_alg / (ms * 1e-3) / 1e9 / peak, 4),
            "kernel_ms_breakdown": {k: round(v / args.steps, 4) for k, v in prof_sum.items()}}

    # e2e: same call, pinned host buffers, H2D + D2H inside the timed region
    e2e = None
    if not args.skip_e2e:
        hA = [torch.from_numpy(g.row_ptr.view(np.int64)).pin_memory(),
              torch.from_numpy(g.col_idx.view(np.int32)).pin_memory(),
              torch.from_numpy(g.values.astype(vdt_np)).pin_memory()]
        hX = [torch.from_numpy(x.row_ptr.view(np.int64)).pin_memory(),
              torch.from_numpy(x.col_idx.view(np.int32)).pin_memory(),
              torch.from_numpy(x.values.astype(vdt_np)).pin_memory()]
        ham = ab._Matrix(n, g.n_cols, ab.CSR, ab.HOST, 4, vb, hA[0].data_ptr(), hA[1].data_ptr(), hA[2].data_ptr(),
                         g.nnz())
        hxm = ab._Matrix(K, x.n_cols, ab.CSR, ab.HOST, 4, vb, hX[0].data_ptr(), hX[1].data_ptr(),
                         hX[2].data_ptr(), x.nnz())
        # streamed output hands the allocator an upper bound of nnz(C) (include/aires_b200.h):
        # min(rows * n_cols, nnz(A) * longest X row); the pinned result buffers cover it
        c_bound = min(n * x.n_cols, g.nnz() * int(np.diff(x.row_ptr.astype(np.int64)).max(initial=1)))
        hout = {"ptr": torch.empty(n + 1, dtype=torch.int64).pin_memory(),
                "idx": torch.empty(max(nnz_c, c_bound, 1), dtype=torch.int32).pin_memory(),
                "val": torch.empty(max(nnz_c, c_bound, 1), dtype=vdt_t).pin_memory()}

        def host_alloc(user, rows, nnz, pp, pi, pv):
            if nnz > hout["idx"].numel():
                return 9
            pp[0], pi[0], pv[0] = hout["ptr"].data_ptr(), hout["idx"].data_ptr(), hout["val"].data_ptr()
            return 0

        hfn = ab._ALLOC_FN(host_alloc)
        hout_s = ab._Output(ab.HOST, 4, vb, 0, hfn, None, 0, 0, 0, 0)

        def estep():
            ab._check(L.aires_b200_spgemm(C.byref(ham), C.byref(hxm), mode, C.byref(hout_s)))

        # the public entry point for host-resident operands is the out-of-core run (run_aires,
        # aires_b200_run), uncapped.  Streamed output (the headline): no sizing pass, ~16 row
        # blocks, C drains on copy engine 1 while A still crosses on copy engine 0.  Exact protocol
        # (beside it): sizing pass over A's columns first, exact allocation, then the tiles.
        rrep = ab._RunReport()
        rcfg = ab._RunConfig(0, mode, 1, 0, ab.RUN_STREAM_OUT)
        xrep = ab._RunReport()
        xcfg = ab._RunConfig(0, mode, 1, 3, 0)

        def rstep():
            ab._check(L.aires_b200_run(C.byref(ham), C.byref(hxm), C.byref(rcfg), C.byref(hout_s), C.byref(rrep)))

        def xstep():
            ab._check(L.aires_b200_run(C.byref(ham), C.byref(hxm), C.byref(xcfg), C.byref(hout_s), C.byref(xrep)))

        for _ in range(max(1, args.warmup)):
            estep()
            xstep()
            rstep()
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            estep()
        s_ms = (time.perf_counter() - t0) * 1e3 / args.steps
        t0 = time.perf_counter()
        for _ in range(args.steps):
            xstep()
        x_ms = (time.perf_counter() - t0) * 1e3 / args.steps
        if int(hout_s.nnz) != nnz_c:
            raise RuntimeError(f"run_aires (exact) nnz {int(hout_s.nnz)} != spgemm nnz {nnz_c}")
        t0 = time.perf_counter()
        for _ in range(args.steps):
            rstep()
        e_ms = (time.perf_counter() - t0) * 1e3 / args.steps
        if int(hout_s.nnz) != nnz_c:
            raise RuntimeError(f"run_aires (streamed) nnz {int(hout_s.nnz)} != spgemm nnz {nnz_c}")
        if rank == 0 and world == 1:
            # the streamed result against the device product (structure bit-exact, values 1e-5)
            hp = hout["ptr"].numpy().view(np.uint64)
            if not np.array_equal(hp, c_ptr_check):
                raise RuntimeError("streamed run row_ptr differs from the device product")
            if not np.array_equal(hout["idx"][:nnz_c].numpy(), c_idx_check):
                raise RuntimeError("streamed run col_idx differs from the device product")
        link = link_bandwidth(dev)
        e2e_duplex_ms = max(int(rrep.h2d_bytes) / link["h2d"], int(rrep.d2h_bytes) / link["d2h"]) / 1e6
        if dist:
            t = torch.tensor([e_ms], dtype=torch.float64, device=cdev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = float(t.item())
        h2d = int(rrep.h2d_bytes)
        d2h = int(rrep.d2h_bytes)
        e2e = {"value": round(2.0 * tot_macs / (e_ms * 1e-3) / 1e9, 3), "unit": "GFLOP/s", "ms_per_step": round(e_ms, 3),
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "api": "aires_b200_run (run_aires, streamed output), pinned host A/X/C (u64 ptr, u32 idx, fp32 val), "
                      "wall clock",
               "segments": int(rrep.segments), "device_ms": round(rrep.total_ms, 3),
               "roofline": {"bound": "host-link (full duplex)", "link_gbs": {k: round(v, 2) for k, v in link.items()},
                            "t_roof_ms": round(e2e_duplex_ms, 3), "frac": round(e2e_duplex_ms / e_ms, 4),
                            "basis": "max(H2D bytes / measured pinned H2D GB/s, D2H bytes / measured D2H GB/s)"},
               "exact_protocol": {"api": "aires_b200_run without streamed output (sizing pass over A's columns, "
                                         "exact allocation, then the tiles)",
                                  "ms_per_step": round(x_ms, 3), "value": round(2.0 * tot_macs / (x_ms * 1e-3) / 1e9, 3),
                                  "device_ms": round(xrep.total_ms, 3), "segments": int(xrep.segments)},
               "spgemm_call": {"api": "aires_b200_spgemm with host buffers (one-shot H2D, product, D2H)",
                               "ms_per_step": round(s_ms, 3),
                               "value": round(2.0 * tot_macs / (s_ms * 1e-3) / 1e9, 3)}}

    cpu = None
    if rank == 0 and world == 1 and not args.skip_cpu:
        cpu = cpu_baseline(g, x, args.cpu_seconds)
    ooc = None
    if world == 1 and not args.skip_ooc:
        tA.clear(); tX.clear(); outbuf.clear()
        torch.cuda.empty_cache()
        ooc = out_of_core_leg(args, dev, L, ab, torch)
    ppi = None
    if world == 1 and args.cfg4_shard:
        torch.cuda.empty_cache()
        ppi = out_of_core_leg(args, dev, L, ab, torch, "cfg4shard")
    gcn = None
    if world == 1 and not args.skip_gcn:
        torch.cuda.empty_cache()
        gcn = gcn_leg(args, dev, L, ab, torch)
    elif world > 1 and not args.skip_gcn:
        tA.clear(); tX.clear(); outbuf.clear()
        torch.cuda.empty_cache()
        gcn = gcn_leg_dist(args, dev, L, ab, torch, dist, rank, world, cdev)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(gflops, 3), "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32" if vb == 4 else "f64",
            "data": "synthetic (Chung-Lu power-law Ã, gen_features X; seeds graph 1+rank, relabel 2, X 3)",
            "config": {"workload": cfg["workload"], "nodes_per_gpu": n, "edges_per_gpu": st["nnz_a"],
                       "nnz_a_tilde": g.nnz(), "x_cols": x.n_cols, "nnz_x": x.nnz(), "nnz_c": nnz_c,
                       "macs": tot_macs, "max_degree": st["max_degree"], "mode": args.mode,
                       "parallelism": f"row-block shards x{world}" if world > 1 else "single GPU",
                       "global_row_ptr_offsets": [int(o) for o in offsets] if world > 1 else None,
                       "l2": "inputs larger than L2 (A 0.9 GB, C 1.1 GB vs 126 MB L2); X is meant to stay L2-resident",
                       "latency_ms": round(ms, 4)},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "out_of_core": ooc, "gcn_2layer": gcn, "cfg4_shard": ppi,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def link_bandwidth(dev, nbytes=512 << 20, reps=5):
    """Pinned cudaMemcpy H2D / D2H GB/s (best of reps, CUDA events) -- the host-link roofline."""
    import torch
    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    out = {}
    for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
        best = 1e9
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1))
        out[name] = nbytes / (best * 1e-3) / 1e9
    del h, d
    return out


def out_of_core_leg(args, dev, L, ab, torch, cfg_name="cfg3"):
    """cfg3 (ogbn-products-shaped) through aires_b200_run with the device budget capped to
    args.ooc_frac of B_A + B_X + B_C: A and X in pinned host memory, C drained to pinned host
    memory tile by tile.  Roofline = the host link (measured in this run)."""
    cfg = CONFIGS[cfg_name]
    g, st, x = make_inputs(cfg, 0, 1)
    n, K = g.n_rows, x.n_rows
    hA = [torch.from_numpy(g.row_ptr.view(np.int64)).pin_memory(), torch.from_numpy(g.col_idx.view(np.int32)).pin_memory(),
          torch.from_numpy(g.values.astype(np.float32)).pin_memory()]
    hX = [torch.from_numpy(x.row_ptr.view(np.int64)).pin_memory(), torch.from_numpy(x.col_idx.view(np.int32)).pin_memory(),
          torch.from_numpy(x.values.astype(np.float32)).pin_memory()]
    am = ab._Matrix(n, g.n_cols, ab.CSR, ab.HOST, 4, 4, hA[0].data_ptr(), hA[1].data_ptr(), hA[2].data_ptr(), g.nnz())
    xm = ab._Matrix(K, x.n_cols, ab.CSR, ab.HOST, 4, 4, hX[0].data_ptr(), hX[1].data_ptr(), hX[2].data_ptr(), x.nnz())
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
    rep = ab._RunReport()
    # size the budget from a first unconstrained run (C bytes are only known after it)
    ab._check(L.aires_b200_run(C.byref(am), C.byref(xm), C.byref(ab._RunConfig(0, ab.MODE_FP32, 1, 2, 0)),
                               C.byref(out), C.byref(rep)))
    nnz_c, macs = int(out.nnz), int(out.flops)
    b_a = 8 * (n + 1) + 8 * g.nnz()
    b_x = 8 * (K + 1) + 8 * x.nnz()
    b_c = 8 * (n + 1) + 8 * nnz_c
    budget = int(args.ooc_frac * (b_a + b_x + b_c))
    rc = ab._RunConfig(budget, ab.MODE_FP32, 1, args.ooc_buffers, 0)
    for _ in range(max(1, args.warmup)):
        ab._check(L.aires_b200_run(C.byref(am), C.byref(xm), C.byref(rc), C.byref(out), C.byref(rep)))
    dev_ms, wall_ms, segs, launches = [], [], 0, 0
    for _ in range(args.steps):
        t0 = time.perf_counter()
        ab._check(L.aires_b200_run(C.byref(am), C.byref(xm), C.byref(rc), C.byref(out), C.byref(rep)))
        wall_ms.append((time.perf_counter() - t0) * 1e3)
        dev_ms.append(rep.total_ms)
        segs = int(rep.segments)
        launches += L.aires_b200_last_launches()
    h2d_b, d2h_b = int(rep.h2d_bytes), int(rep.d2h_bytes)
    # the paper's baseline on the same budget: MaxMemory (fixed byte tiles, split rows' fragments
    # returned to the host and re-sent; scheduler.hpp:174-293), same ring and streams
    mm = None
    try:
        rcm = ab._RunConfig(budget, ab.MODE_FP32, 2, args.ooc_buffers, 0)
        repm = ab._RunReport()
        ab._check(L.aires_b200_run(C.byref(am), C.byref(xm), C.byref(rcm), C.byref(out), C.byref(repm)))
        mms = []
        for _ in range(max(1, args.steps // 2)):
            ab._check(L.aires_b200_run(C.byref(am), C.byref(xm), C.byref(rcm), C.byref(out), C.byref(repm)))
            mms.append(repm.total_ms)
        mm = {"ms": round(float(np.median(mms)), 3), "segments": int(repm.segments), "h2d_bytes": int(repm.h2d_bytes),
              "d2h_bytes": int(repm.d2h_bytes), "merge_bytes": int(repm.merge_bytes),
              "aires_speedup": round(float(np.median(mms)) / float(np.median(dev_ms)), 3)}
    except Exception as e:  # the baseline may not fit where AIRES does (the paper's point)
        mm = {"failed": str(e)[:200]}
    bw = link_bandwidth(dev)
    ms = float(np.median(dev_ms))
    t_roof = (b_a + b_x + b_c) / (bw["h2d"] * 1e9) * 1e3
    t_duplex = max(h2d_b / (bw["h2d"] * 1e9), d2h_b / (bw["d2h"] * 1e9)) * 1e3
    return {
        "workload": cfg["workload"] + f", device budget {args.ooc_frac:.3g} x (B_A+B_X+B_C) = {budget / 1e6:.1f} MB",
        "metric": "A·X latency (ms) and GFLOP/s, out-of-core", "ms": round(ms, 3),
        "gflops": round(2.0 * macs / (ms * 1e-3) / 1e9, 3), "wall_ms": round(float(np.median(wall_ms)), 3),
        "segments": segs, "n_buffers": args.ooc_buffers, "nnz_a": g.nnz(), "nnz_x": x.nnz(), "nnz_c": nnz_c,
        "macs": macs, "h2d_bytes": h2d_b, "d2h_bytes": d2h_b, "gpu_launches_per_run": launches // args.steps,
        "phase_ms": {"phase1": round(rep.phase1_ms, 3), "phase2": round(rep.phase2_ms, 3),
                     "phase3": round(rep.phase3_ms, 3)},
        "roofline": {"bound": "host-link", "achieved": round((b_a + b_x + b_c) / (ms * 1e-3) / 1e9, 2),
                     "peak": round(bw["h2d"], 2), "unit": "GB/s", "frac": round(t_roof / ms, 4),
                     "frac_full_duplex": round(t_duplex / ms, 4), "link_gbs": {k: round(v, 2) for k, v in bw.items()},
                     "basis": "(B_A+B_X+B_C) / measured pinned H2D GB/s; full duplex: max(H2D bytes/H2D, D2H bytes/D2H)"},
        "storage": "pinned host memory (GPUDirect Storage not used: operands arrive through the host API)",
        "maxmemory_baseline": mm,
    }


class DevOut:
    """aires_b200_output handing out grow-only device tensors (torch) -- results stay in HBM."""

    def __init__(self, ab, torch, dev, idx_dtype, val_dtype):
        self.ab, self.torch, self.dev = ab, torch, dev
        self.idx_dtype, self.val_dtype, self.t = idx_dtype, val_dtype, {}
        self.fn = ab._ALLOC_FN(self._alloc)
        self.out = ab._Output(ab.DEVICE, 4, 4 if val_dtype == torch.float32 else 8, 0, self.fn, None, 0, 0, 0, 0)

    def _alloc(self, user, rows, nnz, pp, pi, pv):
        T = self.torch
        if self.t.get("rows", -1) < rows:
            self.t["ptr"] = T.empty(rows + 1, dtype=T.int64, device=self.dev)
            self.t["rows"] = rows
        if self.t.get("cap", -1) < nnz:
            self.t["idx"] = T.empty(max(nnz, 1), dtype=self.idx_dtype, device=self.dev)
            self.t["val"] = T.empty(max(nnz, 1), dtype=self.val_dtype, device=self.dev)
            self.t["cap"] = nnz
        pp[0], pi[0], pv[0] = self.t["ptr"].data_ptr(), self.t["idx"].data_ptr(), self.t["val"].data_ptr()
        return 0

    def matrix(self, n_cols):
        ab = self.ab
        o = self.out
        return ab._Matrix(o.n_rows, n_cols, ab.CSR, ab.DEVICE, 4, o.val_bytes, self.t["ptr"].data_ptr(),
                          self.t["idx"].data_ptr(), self.t["val"].data_ptr(), o.nnz)


def gcn_leg_dist(args, dev, L, ab, torch, dist, rank, world, cdev):
    """cfg5 across ranks (strong scaling): the same products-shaped graph on every rank, rank r owns a
    work-balanced contiguous row block of Ã; layer 1 on the block, then the H1 blocks are all-gathered
    over NCCL into the replicated H1 the next layer needs (shard.allgather_csr_torch), then the fused
    layer 2 on the block.  Time = max over ranks (CUDA events)."""
    from paper_2507_02006_b200 import shard
    cfg = CONFIGS["cfg3"]
    a, _ = ab.synth_graph(cfg["n"], cfg["nnz"], alpha=0.75, degree_cap=cfg["cap"], seed=1, relabel_seed=2,
                          normalize=False, idx_dtype=np.uint32, val_dtype=np.float32)
    x = ab.synth_features(cfg["n"], cfg["dim"], 99.0, 3, idx_dtype=np.uint32, val_dtype=np.float32)
    w1 = torch.from_numpy(ab.gen_weights(cfg["dim"], 256, 4).astype(np.float32)).to(dev)
    w2 = torch.from_numpy(ab.gen_weights(256, 47, 5).astype(np.float32)).to(dev)
    n = a.n_rows
    cuts = shard.row_shards(a.row_ptr, world)
    r0, r1 = int(cuts[rank]), int(cuts[rank + 1])
    tA = [torch.from_numpy(a.row_ptr.view(np.int64)).to(dev), torch.from_numpy(a.col_idx.view(np.int32)).to(dev),
          torch.from_numpy(a.values).to(dev)]
    tX = [torch.from_numpy(x.row_ptr.view(np.int64)).to(dev), torch.from_numpy(x.col_idx.view(np.int32)).to(dev),
          torch.from_numpy(x.values).to(dev)]
    am = ab._Matrix(n, n, ab.CSR, ab.DEVICE, 4, 4, tA[0].data_ptr(), tA[1].data_ptr(), tA[2].data_ptr(), a.nnz())
    xm = ab._Matrix(n, x.n_cols, ab.CSR, ab.DEVICE, 4, 4, tX[0].data_ptr(), tX[1].data_ptr(), tX[2].data_ptr(), x.nnz())
    o_t, o_c1, o_h1, o_h2 = (DevOut(ab, torch, dev, torch.int32, torch.float32) for _ in range(4))
    stream = torch.cuda.ExternalStream(L.aires_b200_stream(), device=dev)
    gathered = {}

    def block(o, cols):  # rows [r0, r1) of a device CSR as a zero-copy view (absolute row pointers)
        t = o.t
        return ab._Matrix(r1 - r0, cols, ab.CSR, ab.DEVICE, 4, 4, t["ptr"].data_ptr() + 8 * r0, t["idx"].data_ptr(),
                          t["val"].data_ptr(), o.out.nnz)

    def forward(rec=None):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        ev[0].record(stream)
        ab._check(L.aires_b200_normalize_adjacency(C.byref(am), C.byref(o_t.out)))
        at_blk = block(o_t, n)
        ab._check(L.aires_b200_spgemm(C.byref(at_blk), C.byref(xm), ab.MODE_FP32, C.byref(o_c1.out)))
        ab._check(L.aires_b200_combine(C.byref(o_c1.matrix(x.n_cols)), C.c_void_p(w1.data_ptr()), w1.shape[0],
                                       w1.shape[1], ab.DEVICE, C.byref(o_h1.out)))
        ev[1].record(stream)
        ev[1].synchronize()
        t = o_h1.t
        rows_h = int(o_h1.out.n_rows)
        g_ptr, g_idx, g_val = shard.allgather_csr_torch(t["ptr"][: rows_h + 1], t["idx"], t["val"])
        torch.cuda.synchronize(dev)
        ev[2].record(stream)
        gathered.update(ptr=g_ptr, idx=g_idx, val=g_val)
        h1 = ab._Matrix(n, w1.shape[1], ab.CSR, ab.DEVICE, 4, 4, g_ptr.data_ptr(), g_idx.data_ptr(),
                        g_val.data_ptr(), g_idx.numel())
        ab._check(L.aires_b200_layer_fused(C.byref(at_blk), C.byref(h1), C.c_void_p(w2.data_ptr()), w2.shape[0],
                                           w2.shape[1], ab.DEVICE, C.byref(o_h2.out)))
        ev[3].record(stream)
        ev[3].synchronize()
        if rec is not None:
            rec.setdefault("layer1", []).append(ev[0].elapsed_time(ev[1]))
            rec.setdefault("layer2_fused", []).append(ev[2].elapsed_time(ev[3]))
            rec.setdefault("h1_allgather", []).append(ev[1].elapsed_time(ev[2]))
            rec.setdefault("total", []).append(ev[0].elapsed_time(ev[3]))

    for _ in range(max(1, args.warmup)):
        forward()
    dist.barrier()
    rec = {}
    for _ in range(args.steps):
        forward(rec)
    med = {k: float(np.median(v)) for k, v in rec.items()}
    tt = torch.tensor([med["total"], med["layer1"], med["layer2_fused"], med["h1_allgather"]], dtype=torch.float64,
                      device=cdev)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    return {"workload": f"cfg5 across {world} ranks: 2-layer GCN forward on the ogbn-products shape, rows of Ã in "
                        "work-balanced contiguous blocks, H1 all-gathered for layer 2, fp32",
            "ms_max_over_ranks": {"total": round(float(tt[0]), 3), "layer1_incl_normalize": round(float(tt[1]), 3),
                                  "layer2_fused": round(float(tt[2]), 3), "h1_allgather": round(float(tt[3]), 3)},
            "collective": f"torch.distributed {dist.get_backend()} all_gather_into_tensor (sizes, then padded arrays)",
            "rows_per_rank": [int(cuts[i + 1] - cuts[i]) for i in range(world)],
            "h1_allgather_bytes": int(gathered["idx"].numel()) * 8 + 8 * (n + 1), "h2_nnz_rank0": int(o_h2.out.nnz)}


def gcn_leg(args, dev, L, ab, torch):
    """cfg5 on one GPU: the 2-layer GCN forward (gcn.hpp:125-132 twice) on the ogbn-products shape,
    everything device-resident: Ã = normalize(A); H1 = ReLU((Ã·X)·W1); H2 = ReLU((Ã·H1)·W2)."""
    cfg = CONFIGS["cfg3"]
    t0 = time.time()
    a, st = ab.synth_graph(cfg["n"], cfg["nnz"], alpha=0.75, degree_cap=cfg["cap"], seed=1, relabel_seed=2,
                           normalize=False, idx_dtype=np.uint32, val_dtype=np.float32)
    x = ab.synth_features(cfg["n"], cfg["dim"], 99.0, 3, idx_dtype=np.uint32, val_dtype=np.float32)
    w1 = torch.from_numpy(ab.gen_weights(cfg["dim"], 256, 4).astype(np.float32)).to(dev)
    w2 = torch.from_numpy(ab.gen_weights(256, 47, 5).astype(np.float32)).to(dev)
    log(f"[gcn] inputs in {time.time() - t0:.1f}s")
    tA = [torch.from_numpy(a.row_ptr.view(np.int64)).to(dev), torch.from_numpy(a.col_idx.view(np.int32)).to(dev),
          torch.from_numpy(a.values).to(dev)]
    tX = [torch.from_numpy(x.row_ptr.view(np.int64)).to(dev), torch.from_numpy(x.col_idx.view(np.int32)).to(dev),
          torch.from_numpy(x.values).to(dev)]
    n = a.n_rows
    am = ab._Matrix(n, n, ab.CSR, ab.DEVICE, 4, 4, tA[0].data_ptr(), tA[1].data_ptr(), tA[2].data_ptr(), a.nnz())
    xm = ab._Matrix(n, x.n_cols, ab.CSR, ab.DEVICE, 4, 4, tX[0].data_ptr(), tX[1].data_ptr(), tX[2].data_ptr(), x.nnz())
    o_t, o_c1, o_h1, o_c2, o_h2 = (DevOut(ab, torch, dev, torch.int32, torch.float32) for _ in range(5))
    stream = torch.cuda.ExternalStream(L.aires_b200_stream(), device=dev)
    stats = {}

    def forward(record=None, fused=True):
        """layer 2 (H1 ~50% dense) runs the fused dense-H aggregate+combine unless fused=False"""
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
        ev[0].record(stream)
        ab._check(L.aires_b200_normalize_adjacency(C.byref(am), C.byref(o_t.out)))
        at = o_t.matrix(n)
        ev[1].record(stream)
        ab._check(L.aires_b200_spgemm(C.byref(at), C.byref(xm), ab.MODE_FP32, C.byref(o_c1.out)))
        macs1 = int(o_c1.out.flops)
        ev[2].record(stream)
        ab._check(L.aires_b200_combine(C.byref(o_c1.matrix(x.n_cols)), C.c_void_p(w1.data_ptr()), w1.shape[0],
                                       w1.shape[1], ab.DEVICE, C.byref(o_h1.out)))
        ev[3].record(stream)
        h1 = o_h1.matrix(w1.shape[1])
        macs2 = 0
        if fused:
            ev[4].record(stream)
            ab._check(L.aires_b200_layer_fused(C.byref(at), C.byref(h1), C.c_void_p(w2.data_ptr()), w2.shape[0],
                                               w2.shape[1], ab.DEVICE, C.byref(o_h2.out)))
        else:
            ab._check(L.aires_b200_spgemm(C.byref(at), C.byref(h1), ab.MODE_FP32, C.byref(o_c2.out)))
            macs2 = int(o_c2.out.flops)
            ev[4].record(stream)
            ab._check(L.aires_b200_combine(C.byref(o_c2.matrix(w1.shape[1])), C.c_void_p(w2.data_ptr()), w2.shape[0],
                                           w2.shape[1], ab.DEVICE, C.byref(o_h2.out)))
        ev[5].record(stream)
        ev[5].synchronize()
        if record is not None:
            names = ["normalize", "aggregate1", "combine1", "aggregate2", "combine2"]
            if fused:
                names[3], names[4] = "(fused below)", "layer2_fused"
            for i, nm in enumerate(names):
                record.setdefault(nm, []).append(ev[i].elapsed_time(ev[i + 1]))
            record.setdefault("total", []).append(ev[0].elapsed_time(ev[5]))
        return macs1, macs2

    for _ in range(max(1, args.warmup)):
        forward(fused=False)
        forward()
    rec_u, rec = {}, {}
    for _ in range(max(1, args.steps // 2)):
        macs1, macs2 = forward(rec_u, fused=False)
    for _ in range(args.steps):
        forward(rec)
    med = {k: round(float(np.median(v)), 3) for k, v in rec.items() if not k.startswith("(")}
    med_u = {k: round(float(np.median(v)), 3) for k, v in rec_u.items()}
    comb_flops = 2 * (int(o_c1.out.nnz) * 256 + int(o_c2.out.nnz) * 47)
    return {"workload": "cfg5 (1 GPU): 2-layer GCN forward on the ogbn-products shape, W1 100x256, W2 256x47 "
                        "(gen_weights seeds 4, 5), all operands device-resident, fp32",
            "ms": med, "ms_unfused": med_u,
            "nnz": {"a_tilde": int(o_t.out.nnz), "c1": int(o_c1.out.nnz), "h1": int(o_h1.out.nnz),
                    "c2": int(o_c2.out.nnz), "h2": int(o_h2.out.nnz)},
            "macs_aggregate": [macs1, macs2],
            "gflops_aggregate_unfused": round(2.0 * (macs1 + macs2) / ((med_u["aggregate1"] + med_u["aggregate2"]) * 1e-3)
                                              / 1e9, 2),
            "gflops_combine_unfused": round(comb_flops / ((med_u["combine1"] + med_u["combine2"]) * 1e-3) / 1e9, 2),
            "layer2_fused_gflops": round((2.0 * macs2 + 2 * int(o_c2.out.nnz) * 47) / (med["layer2_fused"] * 1e-3) / 1e9, 2),
            "forward_ms": med["total"], "forward_ms_unfused": med_u["total"],
            "layers_per_s": round(2.0 / (med["total"] * 1e-3), 2)}


def sample_rows(n: int, count: int, seed: int = 11) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return np.sort(rng.choice(n, size=min(count, n), replace=False)).astype(np.uint64)


def ref_sample_run(g, x, seconds: float, threads: int):
    """Reference spgemm_block (oracle/_ref) on a random row sample sized to ~`seconds` of work.
    Returns (gflops, sample description, kind, rows, secs)."""
    from oracle import pyoracle as po
    a_ptr, a_idx, a_val = g.row_ptr, g.col_idx.astype(np.uint64), g.values.astype(np.float64)
    cp, ri, cv = po.csr_to_csc(x.n_rows, x.n_cols, x.row_ptr, x.col_idx.astype(np.uint64), x.values)
    kind = "reference" if po.ref_available() else "port"
    if kind == "reference":
        def run(rows):
            s, macs, z, _ = po.ref_rows_timed(a_ptr, a_idx, a_val, g.n_cols, rows, cp, ri, cv, x.n_rows, x.n_cols,
                                              threads)
            return s, macs
    else:  # oracle port of spgemm_block (inner product), one thread
        def run(rows):
            t0 = time.perf_counter()
            macs = 0
            for r in rows:
                rc, _, m = po.spgemm_inner(a_ptr[r:r + 2], a_idx, a_val, 1, g.n_cols, x.n_rows, x.n_cols, cp, ri, cv)
                macs += m
            return time.perf_counter() - t0, macs
    probe = sample_rows(g.n_rows, max(threads * 4, 16), seed=5)
    s, _ = run(probe)
    per_row = s / len(probe)
    count = int(max(threads * 4, min(g.n_rows, seconds / max(per_row, 1e-9))))
    rows = sample_rows(g.n_rows, count)
    s, macs = run(rows)
    return 2.0 * macs / s / 1e9, rows, kind, s


def cpu_baseline(g, x, seconds: float):
    threads = len(os.sched_getaffinity(0))
    try:
        gf, rows, kind, s = ref_sample_run(g, x, seconds, threads)
    except Exception as e:  # baseline is reported, never fatal
        return {"value": None, "unit": "GFLOP/s", "cores": threads, "kind": "reference", "sample": f"failed: {e}"}
    return {"value": round(gf, 6), "unit": "GFLOP/s", "cores": threads if kind == "reference" else 1, "kind": kind,
            "sample": f"{len(rows)} uniformly sampled rows of the same Ã·X ({s:.1f} s), reference spgemm_block "
                      f"(inner product, spgemm.hpp:60-132) unmodified, -O3 no -march; GFLOP/s = 2*MACs/t"}


def run_reference(args, cfg):
    """--impl reference: the reference's own CPU spgemm_block on the host cores (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    threads = len(os.sched_getaffinity(0))
    g, st, x = make_inputs(cfg, 0, 1)
    per_step = max(2.0, args.cpu_seconds / max(1, args.steps + args.warmup))
    vals = []
    kind = "reference"
    rows_total = 0
    for i in range(args.warmup + args.steps):
        gf, rows, kind, s = ref_sample_run(g, x, per_step, threads)
        if i >= args.warmup:
            vals.append(gf)
            rows_total += len(rows)
    v = float(np.median(vals))
    line = {"metric": METRIC, "value": round(v, 6), "unit": "GFLOP/s", "n_gpus": int(os.environ.get("WORLD_SIZE", "1")),
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (same seeds as the b200 arm)",
            "config": {"workload": cfg["workload"], "nodes": g.n_rows, "edges": st["nnz_a"], "x_cols": x.n_cols},
            "impl": "reference",
            "cpu_baseline": {"value": round(v, 6), "unit": "GFLOP/s", "kind": kind,
                             "cores": threads if kind == "reference" else 1,
                             "sample": f"{rows_total} sampled rows over {args.steps} steps (~{per_step:.0f} s each)"},
            "e2e": {"value": round(v, 6), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="cfg2")
    ap.add_argument("--mode", choices=["fp32", "fp64"], default="fp32")
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--skip-e2e", action="store_true")
    ap.add_argument("--skip-ooc", action="store_true", help="skip the cfg3 out-of-core leg")
    ap.add_argument("--skip-gcn", action="store_true", help="skip the cfg5 2-layer GCN leg")
    ap.add_argument("--cfg4-shard", action="store_true", help="also run one 1/8 shard of the PPI-scale cfg4 "
                    "out of core (slow input generation)")
    ap.add_argument("--ooc-frac", type=float, default=0.25, help="cfg3 device budget / (B_A+B_X+B_C)")
    ap.add_argument("--ooc-buffers", type=int, default=3)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_b200(args, cfg)


if __name__ == "__main__":
    main()
