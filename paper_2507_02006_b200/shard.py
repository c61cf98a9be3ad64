"""Row-block sharding of the A·X path across ranks (one process per GPU).

Rows of C depend only on the same rows of A and on all of X (spgemm.hpp:96-130), and results do not
depend on how rows are blocked (spgemm_test.cpp:97-115).  So each rank owns a contiguous block of
rows, X is replicated, and the only exchange is an all-gather of one int64 nnz(C) per rank, turned
into global row_ptr offsets.  Assembling a replicated C for a next layer is a
variable-size all-gather.  The functions take a torch.distributed process group and work with
NCCL (CUDA tensors) or gloo (CPU tensors, used by the multi-process CPU tests).
"""
from __future__ import annotations

from typing import Optional, Sequence

import numpy as np


def row_shards(row_ptr: np.ndarray, world: int, work: Optional[np.ndarray] = None) -> np.ndarray:
    """Contiguous row cuts (world+1 boundaries) balancing the prefix sum of per-row work.

    work defaults to the A row lengths (nnz); pass the MAC count per row (the X row lengths gathered
    over A's columns) to balance compute instead.  Every rank gets a (possibly empty) block; the cut
    for rank r is the first row whose work prefix reaches r/world of the total.
    """
    rp = np.asarray(row_ptr, dtype=np.int64)
    n = rp.shape[0] - 1
    if world < 1:
        raise ValueError("world must be >= 1")
    w = np.diff(rp) if work is None else np.asarray(work, dtype=np.int64)
    if w.shape[0] != n:
        raise ValueError("work must have one entry per row")
    pref = np.concatenate([[0], np.cumsum(w + 1)])  # +1 per row: empty rows still cost a row
    total = pref[-1]
    targets = (total * np.arange(world + 1, dtype=np.float64) / world)
    cuts = np.searchsorted(pref, targets, side="left").astype(np.int64)
    cuts[0], cuts[-1] = 0, n
    return np.maximum.accumulate(np.minimum(cuts, n))


def global_offsets(local_nnz: int, group=None, device=None) -> tuple:
    """All-gather of one int64 nnz(C) per rank -> (exclusive offsets per rank, total nnz)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    dev = device if device is not None else ("cuda" if dist.get_backend(group) == "nccl" else "cpu")
    mine = torch.tensor([int(local_nnz)], dtype=torch.int64, device=dev)
    allv = torch.zeros(world, dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(allv, mine, group=group)
    counts = allv.cpu().numpy()
    offs = np.concatenate([[0], np.cumsum(counts)[:-1]]).astype(np.int64)
    return offs, int(counts.sum())


def global_row_ptr(local_row_ptr: np.ndarray, offset: int) -> np.ndarray:
    """A rank's slice of the global row_ptr: its local (rebased) row_ptr shifted by its offset."""
    return np.asarray(local_row_ptr, dtype=np.int64) + int(offset)


def allgather_csr(row_ptr: np.ndarray, col_idx: np.ndarray, values: np.ndarray, group=None,
                  device=None) -> tuple:
    """Assembles the replicated global C from each rank's row block (variable-size all-gather,
    padded to the largest block).  Returns (row_ptr, col_idx, values) of the whole matrix."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    dev = device if device is not None else ("cuda" if dist.get_backend(group) == "nccl" else "cpu")
    rp = np.asarray(row_ptr, dtype=np.int64)
    rows, nnz = rp.shape[0] - 1, int(rp[-1] - rp[0])
    # absolute row pointers (e.g. shard_rows' zero-copy blocks) address the block's entries from rp[0]
    col_idx = np.asarray(col_idx)[int(rp[0]): int(rp[0]) + nnz]
    values = np.asarray(values)[int(rp[0]): int(rp[0]) + nnz]
    meta = torch.tensor([rows, nnz], dtype=torch.int64, device=dev)
    metas = torch.zeros(world * 2, dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(metas, meta, group=group)
    metas = metas.view(world, 2).cpu().numpy()
    max_rows, max_nnz = int(metas[:, 0].max()), int(metas[:, 1].max())

    def gather(arr: np.ndarray, length: int, dtype) -> list:
        t = torch.zeros(max(length, 1), dtype=dtype, device=dev)
        a = torch.from_numpy(np.ascontiguousarray(arr)).to(dev)
        t[: a.numel()] = a
        out = torch.zeros(world * max(length, 1), dtype=dtype, device=dev)
        dist.all_gather_into_tensor(out, t, group=group)
        return list(out.view(world, max(length, 1)).cpu().numpy())

    counts = gather(np.diff(rp), max_rows, torch.int64)
    cols = gather(np.asarray(col_idx, dtype=np.int64), max_nnz, torch.int64)
    vals_dt = torch.float64 if np.asarray(values).dtype == np.float64 else torch.float32
    vals = gather(np.asarray(values), max_nnz, vals_dt)
    all_counts = np.concatenate([counts[r][: metas[r, 0]] for r in range(world)])
    g_rp = np.concatenate([[0], np.cumsum(all_counts)]).astype(np.uint64)
    g_col = np.concatenate([cols[r][: metas[r, 1]] for r in range(world)])
    g_val = np.concatenate([vals[r][: metas[r, 1]] for r in range(world)])
    return g_rp, g_col, g_val


def shard_rows(row_ptr: np.ndarray, col_idx: np.ndarray, values: np.ndarray, cuts: Sequence[int], rank: int) -> tuple:
    """Zero-copy row block of rank `rank`: (absolute row_ptr slice, col_idx, values, rows)."""
    r0, r1 = int(cuts[rank]), int(cuts[rank + 1])
    return np.asarray(row_ptr)[r0:r1 + 1], col_idx, values, r1 - r0


def allgather_csr_torch(ptr, idx, val, group=None):
    """Device-side assembly of the replicated C (or H) for the next GCN layer: every rank passes its
    row block as torch tensors (ptr int64 rows+1 rebased or absolute, idx, val); one all-gather of
    the sizes, then one padded all-gather per array (NCCL: the tensors stay on the GPU; gloo: they
    are staged through host memory).  Returns (ptr, idx, val) of the whole matrix on the input
    tensors' device, blocks in rank order."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    nccl = dist.get_backend(group) == "nccl"
    dev = ptr.device
    cdev = dev if nccl else torch.device("cpu")
    rows = ptr.numel() - 1
    base = ptr[0]
    nnz = int((ptr[-1] - base).item())
    meta = torch.tensor([rows, nnz], dtype=torch.int64, device=cdev)
    metas = torch.zeros(2 * world, dtype=torch.int64, device=cdev)
    dist.all_gather_into_tensor(metas, meta, group=group)
    metas = metas.view(world, 2).cpu()
    mr, mn = int(metas[:, 0].max()), max(int(metas[:, 1].max()), 1)

    def gather(t, length):
        pad = torch.zeros(max(length, 1), dtype=t.dtype, device=cdev)
        pad[: t.numel()] = t.to(cdev)
        out = torch.empty(world * max(length, 1), dtype=t.dtype, device=cdev)
        dist.all_gather_into_tensor(out, pad, group=group)
        return out.view(world, max(length, 1))

    counts = gather((ptr[1:] - ptr[:-1]).to(torch.int64), mr)
    cols = gather(idx[int(base): int(base) + nnz], mn)
    vals = gather(val[int(base): int(base) + nnz], mn)
    parts_c = [counts[r, : int(metas[r, 0])] for r in range(world)]
    g_cnt = torch.cat(parts_c).to(dev)
    g_ptr = torch.zeros(g_cnt.numel() + 1, dtype=torch.int64, device=dev)
    torch.cumsum(g_cnt, 0, out=g_ptr[1:])
    g_idx = torch.cat([cols[r, : int(metas[r, 1])] for r in range(world)]).to(dev)
    g_val = torch.cat([vals[r, : int(metas[r, 1])] for r in range(world)]).to(dev)
    return g_ptr, g_idx, g_val
