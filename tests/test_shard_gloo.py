"""CPU tier: the multi-GPU host logic (paper_2507_02006_b200/shard.py) over torch.distributed with
gloo, world size 2 -- row-block cuts, the nnz(C) all-gather that forms global row_ptr offsets, and
assembly of the replicated C -- checked against the single-process oracle product (each rank
computes its block with the oracle; on the GPU box the block product is aires_b200_spgemm)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2507_02006_b200 import shard


def test_row_shards_balanced_and_contiguous():
    rng = np.random.default_rng(0)
    lens = (rng.pareto(1.5, 5000) * 10).astype(np.int64)
    rp = np.concatenate([[0], np.cumsum(lens)])
    for world in (1, 2, 3, 8):
        cuts = shard.row_shards(rp, world)
        assert cuts[0] == 0 and cuts[-1] == 5000 and np.all(np.diff(cuts) >= 0) and len(cuts) == world + 1
        loads = [int(rp[cuts[r + 1]] - rp[cuts[r]] + cuts[r + 1] - cuts[r]) for r in range(world)]
        assert max(loads) <= (rp[-1] + 5000) / world + lens.max() + 1
    c = shard.row_shards(np.array([0, 0, 0]), 4)  # fewer rows than ranks: empty blocks allowed
    assert len(c) == 5 and c[0] == 0 and c[-1] == 2 and np.all(np.diff(c) >= 0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist

    from oracle import pyoracle as po
    from tests._util import random_csr
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(42)  # same matrices on every rank
        a = random_csr(rng, 57, 40, 0.15)
        x = random_csr(rng, 40, 23, 0.2)
        cuts = shard.row_shards(a[0], world)
        rp, ci, va, rows = shard.shard_rows(*a, cuts, rank)
        rc, (lp, li, lv), macs = po.spgemm_rowwise(rp, ci, va, rows, 40, 40, 23, *x)
        assert rc == 0
        offs, total = shard.global_offsets(int(lp[-1]))
        g_rows = shard.global_row_ptr(lp, offs[rank])
        g_rp, g_col, g_val = shard.allgather_csr(lp, li, lv)
        rc, (wp, wi, wv), _ = po.spgemm_rowwise(*a, 57, 40, 40, 23, *x)
        import torch
        # absolute row pointers into the full arrays (shard_rows' zero-copy view) assemble the same C
        base = 1000
        ap = lp.astype(np.int64) + base
        pad_i = np.concatenate([np.zeros(base, li.dtype), li, np.zeros(7, li.dtype)])
        pad_v = np.concatenate([np.zeros(base, lv.dtype), lv, np.zeros(7, lv.dtype)])
        a_rp, a_col, a_val = shard.allgather_csr(ap, pad_i, pad_v)
        ok_abs = (np.array_equal(a_rp, wp) and np.array_equal(a_col.astype(np.uint64), wi)
                  and np.array_equal(a_val.view(np.uint64), wv.view(np.uint64)))
        tp, ti, tv = shard.allgather_csr_torch(torch.from_numpy(lp.astype(np.int64)), torch.from_numpy(li.astype(np.int64)),
                                               torch.from_numpy(lv))
        ok = (total == wi.shape[0] and np.array_equal(g_rp, wp) and np.array_equal(g_col.astype(np.uint64), wi)
              and np.array_equal(g_val.view(np.uint64), wv.view(np.uint64))
              and np.array_equal(g_rows.astype(np.uint64), wp[cuts[rank]:cuts[rank + 1] + 1])
              and np.array_equal(tp.numpy().astype(np.uint64), wp) and np.array_equal(ti.numpy().astype(np.uint64), wi)
              and np.array_equal(tv.numpy().view(np.uint64), wv.view(np.uint64)))
        q.put((rank, bool(ok and ok_abs)))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_gloo_offsets_and_assembly():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(240)
    res = dict(q.get(timeout=5) for _ in range(2))
    assert res == {0: True, 1: True}
    assert all(p.exitcode == 0 for p in procs)
