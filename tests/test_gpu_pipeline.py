"""GPU parity of the out-of-core run (aires_b200_run / run_aires, scheduler.hpp:72-168) against
the oracle: results must not depend on the device budget, tile count or ring depth (the
partition-independence of spgemm_test.cpp:97-115 and acceptance.cpp:66-103, criterion 2)."""
import numpy as np
import pytest

import paper_2507_02006_b200 as ab
from oracle import pyoracle as po

pytestmark = pytest.mark.gpu


def _graph(n, nnz, dim, seed=1):
    g, _ = ab.synth_graph(n, nnz, degree_cap=max(50, n // 10), seed=seed, idx_dtype=np.uint64)
    x = ab.synth_features(n, dim, 99.0 if dim >= 100 else 90.0, 3, idx_dtype=np.uint64)
    return g, x


def _oracle(g, x):
    rc, (p, i, v), macs = po.spgemm_rowwise(g.row_ptr, g.col_idx, g.values, g.n_rows, g.n_cols, x.n_rows, x.n_cols,
                                            x.row_ptr, x.col_idx, x.values, nthreads=8)
    assert rc == 0
    return p, i, v, macs


def _bytes(g, x, want, vb=8):
    a = 8 * (g.n_rows + 1) + (8 + vb) * g.nnz()
    c = 8 * (g.n_rows + 1) + (8 + vb) * want[1].shape[0]
    return a, c


@pytest.mark.parametrize("frac", [1.0, 0.5, 0.25, 0.125])
def test_run_fp64_bit_exact_across_budgets(frac):
    g, x = _graph(20_000, 300_000, 128)
    wp, wi, wv, macs = _oracle(g, x)
    ck = po.checksum(g.n_rows, x.n_cols, wp, wi, wv)
    a_b, c_b = _bytes(g, x, (wp, wi))
    budget = ab.MemoryBudget(int(3e6 + frac * (a_b + c_b)))
    res = ab.run_aires(g, x, budget)
    if frac < 1.0:
        assert res.report.segments >= 2
    assert res.report.c_checksum == ck
    assert res.report.flops == macs
    assert np.array_equal(res.c.row_ptr, wp) and np.array_equal(res.c.col_idx, wi)
    # ledger: A (ptr + one column pass for the symbolic sizing + col/val) and X cross H2D once,
    # C (ptr + col/val) crosses D2H once
    rep = res.report.ledger
    assert rep.d2h.bytes == 8 * (g.n_rows + 1) + 16 * wi.shape[0]
    # A's columns cross once (kept resident after the sizing pass) or twice (sizing + tile)
    base = 8 * (g.n_rows + 1) + 16 * g.nnz() + 8 * (x.n_rows + 1) + 16 * x.nnz()
    assert rep.h2d.bytes in (base, base + 8 * g.nnz())


@pytest.mark.parametrize("n_buffers,resident", [(2, "1"), (3, "0"), (4, "1"), (2, "0")])
def test_run_fp32_tolerance_many_tiles(n_buffers, resident):
    ab.set_option("run_resident_cols", int(resident))  # A columns kept on the device or re-streamed
    g, x = _graph(30_000, 400_000, 100, seed=4)
    wp, wi, wv, macs = _oracle(g, x)
    g32 = ab.CsrMatrix(g.n_rows, g.n_cols, g.row_ptr, g.col_idx.astype(np.uint32), g.values.astype(np.float32))
    x32 = ab.CsrMatrix(x.n_rows, x.n_cols, x.row_ptr, x.col_idx.astype(np.uint32), x.values.astype(np.float32))
    a_b = 8 * (g.n_rows + 1) + 8 * g.nnz()
    c_b = 8 * (g.n_rows + 1) + 8 * wi.shape[0]
    res = ab.run_aires(g32, x32, ab.MemoryBudget(int(3e6 + (a_b + c_b) / 8)), n_buffers=n_buffers,
                       with_checksum=False)
    assert res.report.segments >= 4
    assert np.array_equal(res.c.row_ptr, wp) and np.array_equal(res.c.col_idx.astype(np.uint64), wi)
    err = np.abs(res.c.values.astype(np.float64) - wv) / np.abs(wv)
    assert err.max() <= 1e-5
    assert res.report.flops == macs


def test_run_matches_in_core_product_fp32():
    g, x = _graph(10_000, 200_000, 64, seed=6)
    g32 = ab.CsrMatrix(g.n_rows, g.n_cols, g.row_ptr, g.col_idx.astype(np.uint32), g.values.astype(np.float32))
    x32 = ab.CsrMatrix(x.n_rows, x.n_cols, x.row_ptr, x.col_idx.astype(np.uint32), x.values.astype(np.float32))
    full = ab.spgemm_full(g32, x32)
    res = ab.run_aires(g32, x32, ab.MemoryBudget(int(8e6)), with_checksum=False)
    assert res.report.segments >= 2
    assert np.array_equal(res.c.row_ptr, full.row_ptr) and np.array_equal(res.c.col_idx, full.col_idx)
    np.testing.assert_allclose(res.c.values, full.values, rtol=2e-6)


def test_run_budget_too_small_raises():
    g, x = _graph(5_000, 50_000, 64)
    with pytest.raises(ab.AiresError) as e:
        ab.run_aires(g, x, ab.MemoryBudget(1000))
    assert e.value.code == ab.errc.insufficient_device_memory


def test_run_a_only_tiling_fails_like_the_reference():
    """c_aware=False reproduces the reference admission (A-only RoBW segments, C must fit the rest):
    on a GCN shape with a multi-segment budget it raises insufficient_device_memory."""
    g, x = _graph(20_000, 300_000, 128)
    wp, wi, wv, _ = _oracle(g, x)
    a_b, c_b = _bytes(g, x, (wp, wi))
    with pytest.raises(ab.AiresError) as e:
        ab.run_aires(g, x, ab.MemoryBudget(int(3e6 + 0.25 * (a_b + c_b))), c_aware=False)
    assert e.value.code == ab.errc.insufficient_device_memory


def test_run_empty_and_csc_operand():
    a = ab.CsrMatrix(4, 3, np.zeros(5, np.uint64), np.zeros(0, np.uint64), np.zeros(0))
    b = ab.CsrMatrix(3, 2, np.array([0, 1, 1, 2], np.uint64), np.array([0, 1], np.uint64), np.array([1.0, 2.0]))
    res = ab.run_aires(a, b, ab.MemoryBudget(int(1e7)))
    assert res.c.nnz() == 0 and list(res.c.row_ptr) == [0] * 5
    g, x = _graph(3_000, 30_000, 32)
    cp, ri, cv = po.csr_to_csc(x.n_rows, x.n_cols, x.row_ptr, x.col_idx, x.values)
    res1 = ab.run_aires(g, ab.CscMatrix(x.n_rows, x.n_cols, cp, ri, cv), ab.MemoryBudget(int(2e7)))
    res2 = ab.run_aires(g, x, ab.MemoryBudget(int(2e7)))
    assert res1.report.c_checksum == res2.report.c_checksum


@pytest.mark.parametrize("sizes,mode", [((8, 8), ab.MODE_FP64_EXACT), ((4, 4), ab.MODE_FP32)])
def test_storage_leg_segments_file(tmp_path, sizes, mode):
    """The storage leg: RoBW segments written in the reference's container are read straight to the
    device (cuFile/GDS or pread + pinned H2D), multiplied per segment, and the assembled fragments
    equal the whole product (partition independence, spgemm_test.cpp:97-115)."""
    g, x = _graph(8_000, 100_000, 64, seed=12)
    I, V = sizes
    gi = ab.CsrMatrix(g.n_rows, g.n_cols, g.row_ptr, g.col_idx, g.values)
    segs = ab.robw_partition(gi, 400_000, ab.ElementSizes(I, V))
    assert len(segs) >= 3
    path = str(tmp_path / "a.seg")
    ab.write_segments(path, segs, ab.ElementSizes(I, V))
    xx = x if mode == ab.MODE_FP64_EXACT else ab.CsrMatrix(x.n_rows, x.n_cols, x.row_ptr, x.col_idx,
                                                             x.values.astype(np.float32))
    blocks, rep = ab.spgemm_segments_file(path, ab.ElementSizes(I, V), g.n_cols, xx, mode)
    c = ab.assemble_blocks(blocks, g.n_rows, x.n_cols)
    wp, wi, wv, macs = _oracle(g, x)
    assert rep["segments"] == len(segs) and rep["flops"] == macs
    assert np.array_equal(c.row_ptr, wp) and np.array_equal(c.col_idx, wi)
    if mode == ab.MODE_FP64_EXACT:
        assert np.array_equal(c.values.view(np.uint64), wv.view(np.uint64))
    else:
        # A's values were rounded to fp32 in the file: compare against the fp64 product within 1e-5
        # plus the input rounding (2^-24 relative per operand)
        assert np.max(np.abs(c.values - wv) / np.abs(wv)) < 1e-5 + 2 * 2.0 ** -24
    print("storage leg used GDS:", rep["used_gds"])


@pytest.mark.parametrize("frac", [0.5, 0.25])
def test_maxmemory_baseline_same_result_more_traffic(frac):
    """run_maxmemory (scheduler.hpp:174-293) on the device: fixed byte tiles that split rows, each
    split row's fragment returned to the host and re-sent.  Bit-identical C to run_aires (fp64) and
    the oracle; its ledger carries the fragment round trips (merge_bytes > 0 when rows are split)."""
    g, x = _graph(20_000, 300_000, 128)
    wp, wi, wv, macs = _oracle(g, x)
    a_b, c_b = _bytes(g, x, (wp, wi))
    budget = ab.MemoryBudget(int(3e6 + frac * (a_b + c_b)))
    mm = ab.run_maxmemory(g, x, budget)
    ar = ab.run_aires(g, x, budget)
    assert mm.report.c_checksum == ar.report.c_checksum == po.checksum(g.n_rows, x.n_cols, wp, wi, wv)
    assert mm.report.segments >= 2 and mm.report.ledger.merge_bytes > 0
    assert mm.report.ledger.h2d.bytes > 0 and mm.report.strategy == "maxmemory"


# ---- streamed output (AIRES_B200_RUN_STREAM_OUT): no sizing pass, C drained while A uploads ----

@pytest.mark.parametrize("tiles", ["1", "5", "16", "300"])
def test_stream_out_fp64_bit_exact(tiles):
    ab.set_option("stream_tiles", int(tiles))
    g, x = _graph(20_000, 300_000, 128, seed=8)
    wp, wi, wv, macs = _oracle(g, x)
    res = ab.run_aires(g, x, ab.MemoryBudget(0), stream_out=True)
    assert 1 <= res.report.segments <= int(tiles)
    if int(tiles) > 1:
        assert res.report.segments >= 2
    assert res.report.c_checksum == po.checksum(g.n_rows, x.n_cols, wp, wi, wv)
    assert res.report.flops == macs
    assert np.array_equal(res.c.row_ptr, wp) and np.array_equal(res.c.col_idx, wi)
    # every byte crosses the link once: A (ptr, col, val) and X up, C (ptr, col, val) down
    base = 8 * (g.n_rows + 1) + 16 * g.nnz() + 8 * (x.n_rows + 1) + 16 * x.nnz()
    assert res.report.ledger.h2d.bytes == base
    # C down once: row pointers, fp64 values, and the column indices as u16 on the wire (widened on the host)
    assert res.report.ledger.d2h.bytes >= 8 * (g.n_rows + 1) + 10 * wi.shape[0]
    with ab.options(narrow_cols=0, stream_tiles=int(tiles)):
        wide = ab.run_aires(g, x, ab.MemoryBudget(0), stream_out=True)
    assert wide.report.c_checksum == res.report.c_checksum
    assert wide.report.ledger.d2h.bytes - res.report.ledger.d2h.bytes == 6 * wi.shape[0]


@pytest.mark.parametrize("n_buffers", [2, 3, 4])
def test_stream_out_fp32_matches_exact_protocol(n_buffers):
    ab.set_option("stream_tiles", 12)
    g, x = _graph(30_000, 400_000, 100, seed=4)
    g32 = ab.CsrMatrix(g.n_rows, g.n_cols, g.row_ptr, g.col_idx.astype(np.uint32), g.values.astype(np.float32))
    x32 = ab.CsrMatrix(x.n_rows, x.n_cols, x.row_ptr, x.col_idx.astype(np.uint32), x.values.astype(np.float32))
    exact = ab.run_aires(g32, x32, ab.MemoryBudget(0), with_checksum=False)
    res = ab.run_aires(g32, x32, ab.MemoryBudget(0), n_buffers=n_buffers, with_checksum=False, stream_out=True)
    assert res.report.segments >= 4
    assert np.array_equal(res.c.row_ptr, exact.c.row_ptr)
    assert np.array_equal(res.c.col_idx, exact.c.col_idx)
    np.testing.assert_allclose(res.c.values, exact.c.values, rtol=2e-6)
    assert res.report.flops == exact.report.flops


def test_stream_out_edge_shapes():
    # empty rows at both ends, an all-empty A, and zero rows
    g, x = _graph(4_000, 40_000, 64, seed=9)
    lens = np.diff(g.row_ptr.astype(np.int64))
    row_of = np.repeat(np.arange(g.n_rows), lens)
    keep = (row_of >= 100) & (row_of < g.n_rows - 100)
    lens[:100] = 0
    lens[-100:] = 0
    ptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
    g2 = ab.CsrMatrix(g.n_rows, g.n_cols, ptr, g.col_idx[keep], g.values[keep])
    wp, wi, wv, _ = _oracle(g2, x)
    res = ab.run_aires(g2, x, ab.MemoryBudget(0), stream_out=True)
    assert np.array_equal(res.c.row_ptr, wp) and np.array_equal(res.c.col_idx, wi)
    assert res.report.c_checksum == po.checksum(g2.n_rows, x.n_cols, wp, wi, wv)
    empty = ab.CsrMatrix(g.n_rows, g.n_cols, np.zeros(g.n_rows + 1, np.uint64), np.zeros(0, np.uint64),
                         np.zeros(0, np.float64))
    res = ab.run_aires(empty, x, ab.MemoryBudget(0), stream_out=True)
    assert res.c.nnz() == 0 and not res.c.row_ptr.any()
    none = ab.CsrMatrix(0, g.n_cols, np.zeros(1, np.uint64), np.zeros(0, np.uint64), np.zeros(0, np.float64))
    res = ab.run_aires(none, x, ab.MemoryBudget(0), stream_out=True)
    assert res.c.nnz() == 0 and res.c.row_ptr.shape[0] == 1


@pytest.mark.parametrize("frac", [0.5, 0.25, 0.125, 0.06])
def test_stream_out_capped_single_pass(frac):
    """capped + streamed output: each tile is sized on the device from the columns already in its
    slot (no sizing pass over A), so every byte of A crosses the link exactly once; the tiny budgets
    force tiles whose C is split into several parts.  fp64-exact: C bit-identical to the oracle."""
    g, x = _graph(20_000, 300_000, 128)
    wp, wi, wv, macs = _oracle(g, x)
    a_b, c_b = _bytes(g, x, (wp, wi))
    res = ab.run_aires(g, x, ab.MemoryBudget(int(3e6 + frac * (a_b + c_b))), stream_out=True, n_buffers=3)
    assert res.report.segments >= 2
    assert res.report.c_checksum == po.checksum(g.n_rows, x.n_cols, wp, wi, wv)
    assert res.report.flops == macs
    assert np.array_equal(res.c.row_ptr, wp) and np.array_equal(res.c.col_idx, wi)
    base = 8 * (g.n_rows + 1) + 16 * g.nnz() + 8 * (x.n_rows + 1) + 16 * x.nnz()
    # A once (the exact protocol sends its columns twice); each tile's row pointers include its end row
    assert base <= res.report.ledger.h2d.bytes <= base + 8 * res.report.segments


@pytest.mark.parametrize("n_buffers", [2, 3, 4])
def test_stream_out_capped_fp32_matches_exact_protocol(n_buffers):
    g, x = _graph(30_000, 400_000, 100, seed=4)
    g32 = ab.CsrMatrix(g.n_rows, g.n_cols, g.row_ptr, g.col_idx.astype(np.uint32), g.values.astype(np.float32))
    x32 = ab.CsrMatrix(x.n_rows, x.n_cols, x.row_ptr, x.col_idx.astype(np.uint32), x.values.astype(np.float32))
    a_b, c_b = _bytes(g, x, (None, np.zeros(int(1.5 * g.nnz()))), vb=4)
    budget = ab.MemoryBudget(int(2e6 + 0.2 * (a_b + c_b)))
    exact = ab.run_aires(g32, x32, budget, n_buffers=n_buffers, with_checksum=False)
    res = ab.run_aires(g32, x32, budget, n_buffers=n_buffers, with_checksum=False, stream_out=True)
    assert res.report.segments >= 2
    assert np.array_equal(res.c.row_ptr, exact.c.row_ptr)
    assert np.array_equal(res.c.col_idx, exact.c.col_idx)
    np.testing.assert_allclose(res.c.values, exact.c.values, rtol=2e-6)
    assert res.report.flops == exact.report.flops
    # A crosses the link once; each tile's row pointers include its end row
    base = 8 * (g.n_rows + 1) + 8 * g.nnz() + 8 * (x.n_rows + 1) + 8 * x.nnz()
    assert base <= res.report.ledger.h2d.bytes <= base + 8 * res.report.segments
    assert res.report.ledger.h2d.bytes <= exact.report.ledger.h2d.bytes + 8 * res.report.segments


def test_stream_out_capped_edge_shapes():
    g, x = _graph(4_000, 40_000, 64, seed=9)
    lens = np.diff(g.row_ptr.astype(np.int64))
    row_of = np.repeat(np.arange(g.n_rows), lens)
    keep = (row_of >= 100) & (row_of < g.n_rows - 100)
    lens[:100] = 0
    lens[-100:] = 0
    ptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
    g2 = ab.CsrMatrix(g.n_rows, g.n_cols, ptr, g.col_idx[keep], g.values[keep])
    wp, wi, wv, _ = _oracle(g2, x)
    # (the budget covers X's fp64 layouts, ~1.4 MB, and its raw upload while the layouts are built)
    res = ab.run_aires(g2, x, ab.MemoryBudget(2_600_000), stream_out=True)
    assert res.report.segments >= 2
    assert np.array_equal(res.c.row_ptr, wp) and np.array_equal(res.c.col_idx, wi)
    assert res.report.c_checksum == po.checksum(g2.n_rows, x.n_cols, wp, wi, wv)
    empty = ab.CsrMatrix(g.n_rows, g.n_cols, np.zeros(g.n_rows + 1, np.uint64), np.zeros(0, np.uint64),
                         np.zeros(0, np.float64))
    res = ab.run_aires(empty, x, ab.MemoryBudget(2_600_000), stream_out=True)
    assert res.c.nnz() == 0 and not res.c.row_ptr.any()


def test_stream_out_capped_budget_too_small_raises():
    g, x = _graph(4_000, 40_000, 64, seed=9)
    with pytest.raises(ab.AiresError) as e:
        ab.run_aires(g, x, ab.MemoryBudget(100_000), stream_out=True)
    assert e.value.code == ab.errc.insufficient_device_memory


def test_stream_out_a_only_tiling_keeps_the_exact_protocol():
    # c_aware=False (RoBW by A alone, the reference's admission) is not streamed
    g, x = _graph(20_000, 300_000, 128)
    wp, wi, wv, _ = _oracle(g, x)
    a_b, c_b = _bytes(g, x, (wp, wi))
    res = ab.run_aires(g, x, ab.MemoryBudget(int(3e6 + 2.0 * (a_b + c_b))), stream_out=True, c_aware=False)
    assert res.report.c_checksum == po.checksum(g.n_rows, x.n_cols, wp, wi, wv)


def _audit(res, budget):
    """audit_trace (tiered_sim.hpp:344-420) over the measured trace: per-channel transfer counts and
    bytes equal the ledger, timestamps and phases monotone, frees matched, occupancy within budget."""
    tr = res.trace
    assert tr, "empty trace"
    led = res.report.ledger
    for ch, tot in (("h2d", led.h2d), ("d2h", led.d2h)):
        xs = [e for e in tr if e.kind == "transfer" and e.where == ch]
        assert len(xs) == tot.count and sum(e.bytes for e in xs) == tot.bytes, ch
        assert tot.seconds > 0 and abs(sum(e.duration for e in xs) - tot.seconds) <= 1e-9 + 1e-6 * tot.seconds
    ts = [e.timestamp for e in tr]
    assert ts == sorted(ts)
    ph = [("I", "II", "III").index(e.phase) for e in tr]
    assert ph == sorted(ph)
    live, occ, peak = {}, 0, 0
    for e in tr:
        if e.kind == "alloc" and e.where == "device":
            assert e.buffer not in live
            live[e.buffer] = e.bytes
            occ += e.bytes
            peak = max(peak, occ)
        elif e.kind == "free" and e.where == "device":
            assert live.pop(e.buffer) == e.bytes
            occ -= e.bytes
    assert not live and occ == 0
    if budget:
        assert peak <= budget
    assert sum(e.flops for e in tr if e.kind == "compute") == res.report.flops
    r = res.report
    assert abs(r.total_s - (r.phase1_s + r.phase2_s + r.phase3_s)) <= 1e-6 * max(r.total_s, 1e-9) + 1e-9


@pytest.mark.parametrize("proto", ["exact", "streamed", "capped", "capped_streamed", "maxmemory"])
def test_run_trace_audits(proto):
    g, x = _graph(20_000, 300_000, 128)
    wp, wi, wv, macs = _oracle(g, x)
    a_b, c_b = _bytes(g, x, (wp, wi))
    budget = 0 if proto in ("exact", "streamed") else int(3e6 + 0.3 * (a_b + c_b))
    if proto == "maxmemory":
        res = ab.run_maxmemory(g, x, ab.MemoryBudget(budget), with_checksum=False)
    else:
        res = ab.run_aires(g, x, ab.MemoryBudget(budget), n_buffers=3, with_checksum=False,
                           stream_out=proto in ("streamed", "capped_streamed"))
    assert np.array_equal(res.c.row_ptr, wp) and np.array_equal(res.c.col_idx, wi)
    assert res.report.flops == macs
    _audit(res, budget)
    if proto == "maxmemory" and res.report.ledger.merge_bytes:
        assert res.report.merge_seconds > 0
    elif proto != "maxmemory":
        assert res.report.merge_seconds == 0.0


@pytest.mark.parametrize("budget_frac", [0.0, 0.3])
def test_pageable_arrays_through_bounce_slots(budget_frac):
    """Pageable caller arrays (numpy here, std::vector behind the drop-in) move through pinned bounce
    slots with host copy threads instead of being registered for the call (stage_min_bytes=0 forces
    it at test size): C bit-identical to the oracle, every byte of A up once, C's tiles down in order."""
    g, x = _graph(20_000, 300_000, 128, seed=12)
    wp, wi, wv, macs = _oracle(g, x)
    a_b, c_b = _bytes(g, x, (wp, wi))
    budget = int(3e6 + budget_frac * (a_b + c_b)) if budget_frac else 0
    with ab.options(stage_min_bytes=0, stream_tiles=7):
        res = ab.run_aires(g, x, ab.MemoryBudget(budget), stream_out=True, n_buffers=3)
    assert res.report.segments >= 2
    assert np.array_equal(res.c.row_ptr, wp) and np.array_equal(res.c.col_idx, wi)
    assert res.report.c_checksum == po.checksum(g.n_rows, x.n_cols, wp, wi, wv)
    assert res.report.flops == macs
