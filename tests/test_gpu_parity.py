"""GPU parity: the B200 kernels (through the C ABI) against the CPU oracle.

Known answers follow the reference's own unit tests (spgemm_test.cpp); random cases follow
its property tests.  fp64-exact mode must be bit-identical to the reference (values and
structure); fp32 mode must match structure exactly and values within 1e-5 relative to the
cell's sum of |terms| (north_star tolerance).
"""
import numpy as np
import pytest

import paper_2507_02006_b200 as ab
from oracle import pyoracle as po
from tests._util import (assert_close_fp32, assert_structure_equal, bits_equal, oracle_product, random_csr,
                         to_csc)

pytestmark = pytest.mark.gpu


def csr(nr, nc, ptr, idx, val):
    return ab.CsrMatrix(nr, nc, np.asarray(ptr, np.uint64), np.asarray(idx, np.uint64), np.asarray(val))


def csc_of(nr, nc, ptr, idx, val):
    cp, ri, cv = to_csc(nr, nc, ptr, idx, val)
    return ab.CscMatrix(nr, nc, cp, ri, cv)


def triplets(rows, cols, vals, nr, nc):
    order = np.lexsort((cols, rows))
    rows, cols, vals = np.asarray(rows)[order], np.asarray(cols)[order], np.asarray(vals, float)[order]
    ptr = np.zeros(nr + 1, np.uint64)
    np.add.at(ptr, np.asarray(rows) + 1, 1)
    return np.cumsum(ptr).astype(np.uint64), np.asarray(cols, np.uint64), vals


def test_tiny_hand_product():
    # spgemm_test.cpp:43-53: [[1,2],[0,3]] * [[4,0],[5,6]] = [[14,12],[15,18]]
    a = csr(2, 2, *triplets([0, 0, 1], [0, 1, 1], [1, 2, 3], 2, 2))
    b = csr(2, 2, *triplets([0, 1, 1], [0, 0, 1], [4, 5, 6], 2, 2))
    for bb in (b, csc_of(2, 2, b.row_ptr, b.col_idx, b.values)):
        c = ab.spgemm_full(a, bb)
        assert list(c.row_ptr) == [0, 2, 4]
        assert list(c.col_idx) == [0, 1, 0, 1]
        assert list(c.values) == [14.0, 12.0, 15.0, 18.0]


def test_identity_is_neutral():
    # spgemm_test.cpp:55-60
    rng = np.random.default_rng(3)
    p, i, v = random_csr(rng, 9, 9, 0.4)
    a = csr(9, 9, p, i, v)
    eye = csr(9, 9, np.arange(10, dtype=np.uint64), np.arange(9, dtype=np.uint64), np.ones(9))
    assert ab.spgemm_full(eye, csc_of(9, 9, p, i, v)) == a
    assert ab.spgemm_full(a, csc_of(9, 9, eye.row_ptr, eye.col_idx, eye.values)) == a


def test_keeps_computed_structural_zeros():
    # spgemm_test.cpp:62-70
    a = csr(1, 2, *triplets([0, 0], [0, 1], [1, -1], 1, 2))
    b = csr(2, 1, *triplets([0, 1], [0, 0], [1, 1], 2, 1))
    for mode in (ab.MODE_FP64_EXACT, ab.MODE_FP32):
        c = ab.spgemm_full(a, b, mode=mode)
        assert c.nnz() == 1 and c.values[0] == 0.0


def test_all_negative_zero_contributions_keep_structure():
    # every contribution to cell (0,0) is -0.0: the reference stores +0.0 (sum starts at 0.0)
    a = csr(1, 2, *triplets([0, 0], [0, 1], [-1.0, -2.0], 1, 2))
    b = csr(2, 2, np.array([0, 2, 3], np.uint64), np.array([0, 1, 0], np.uint64), np.array([0.0, 3.0, 0.0]))
    for mode in (ab.MODE_FP64_EXACT, ab.MODE_FP32):
        c = ab.spgemm_full(a, b, mode=mode)
        assert list(c.col_idx) == [0, 1]
        assert np.signbit(c.values[0]) == False and c.values[0] == 0.0  # noqa: E712
        assert c.values[1] == -3.0


def test_flops_count_structural_matches():
    # spgemm_test.cpp:72-83
    rng = np.random.default_rng(7)
    for _ in range(25):
        a = random_csr(rng, 8, 6, 0.5)
        b = random_csr(rng, 6, 7, 0.5)
        want, macs = oracle_product(8, 6, 7, a, b)
        blk = ab.spgemm_block(a[0], a[1], a[2], 8, 6, csc_of(6, 7, *b))
        assert blk.flops == macs


@pytest.mark.parametrize("seed", [13, 14])
def test_matches_oracle_bit_exact_fp64(seed):
    # spgemm_test.cpp:85-95 shapes; fp64-exact must be bit-identical, not just within 1e-12
    rng = np.random.default_rng(seed)
    for _ in range(120):
        nr, ni, nc = (int(x) for x in rng.integers(1, 25, 3))
        d = 0.05 + 0.4 * rng.random()
        a = random_csr(rng, nr, ni, d)
        b = random_csr(rng, ni, nc, d)
        (wp, wi, wv), macs = oracle_product(nr, ni, nc, a, b)
        blk = ab.spgemm_block(a[0], a[1], a[2], nr, ni, csc_of(ni, nc, *b))
        assert_structure_equal(blk.fragment.row_ptr, blk.fragment.col_idx, wp, wi)
        assert bits_equal(blk.fragment.values, wv)
        assert blk.flops == macs


def test_matches_oracle_fp32_tolerance():
    rng = np.random.default_rng(21)
    for _ in range(80):
        nr, ni, nc = (int(x) for x in rng.integers(1, 40, 3))
        d = 0.05 + 0.4 * rng.random()
        a = random_csr(rng, nr, ni, d)
        b = random_csr(rng, ni, nc, d)
        (wp, wi, wv), _ = oracle_product(nr, ni, nc, a, b)
        (_, _, sv), _ = oracle_product(nr, ni, nc, (a[0], a[1], np.abs(a[2])), (b[0], b[1], np.abs(b[2])))
        c = ab.spgemm_full(csr(nr, ni, a[0], a[1], a[2].astype(np.float32)),
                           csr(ni, nc, b[0], b[1], b[2].astype(np.float32)))
        assert c.values.dtype == np.float32
        assert_structure_equal(c.row_ptr, c.col_idx, wp, wi)
        assert_close_fp32(c.values, wv, sv)


def test_csr_and_csc_operands_agree():
    rng = np.random.default_rng(5)
    a = random_csr(rng, 30, 40, 0.2)
    b = random_csr(rng, 40, 50, 0.2)
    c1 = ab.spgemm_full(csr(30, 40, *a), csr(40, 50, *b))
    c2 = ab.spgemm_full(csr(30, 40, *a), csc_of(40, 50, *b))
    assert c1 == c2


def test_absolute_row_pointer_span():
    # spgemm.hpp:79-84: row_ptr need not start at 0; it indexes the spans directly
    rng = np.random.default_rng(9)
    ptr, idx, val = random_csr(rng, 20, 15, 0.3)
    b = random_csr(rng, 15, 12, 0.3)
    full = ab.spgemm_full(csr(20, 15, ptr, idx, val), csr(15, 12, *b))
    blk = ab.spgemm_block(ptr[5:12], idx, val, 7, 15, csr(15, 12, *b), start_row=5)
    lo, hi = int(full.row_ptr[5]), int(full.row_ptr[12])
    assert list(blk.fragment.row_ptr) == list(full.row_ptr[5:13] - full.row_ptr[5])
    assert np.array_equal(blk.fragment.col_idx, full.col_idx[lo:hi])
    assert bits_equal(blk.fragment.values, full.values[lo:hi])
    assert (blk.start_row, blk.end_row) == (5, 12)


def test_partition_independent_bit_exact():
    # spgemm_test.cpp:97-115 with the device RoBW tiler
    rng = np.random.default_rng(19)
    for _ in range(20):
        n = int(rng.integers(4, 24))
        ap = random_csr(rng, n, n, 0.3)
        a = csr(n, n, *ap)
        b = csc_of(n, n, *random_csr(rng, n, n, 0.3))
        whole = ab.spgemm_full(a, b)
        need = max(ab.calc_mem(1, int(ap[0][r + 1] - ap[0][r])) for r in range(n))
        for _ in range(3):
            m_a = need + int(rng.integers(0, 300))
            parts = [ab.spgemm_block(s.row_ptr_local, s.col_idx, s.values, s.rows(), n, b, s.start_row)
                     for s in ab.robw_partition(a, m_a)]
            ptr = np.concatenate([[0], np.cumsum(np.concatenate([np.diff(p.fragment.row_ptr) for p in parts]))])
            assert np.array_equal(ptr.astype(np.uint64), whole.row_ptr)
            assert np.array_equal(np.concatenate([p.fragment.col_idx for p in parts]), whole.col_idx)
            assert bits_equal(np.concatenate([p.fragment.values for p in parts]), whole.values)


def test_mismatched_inner_dimension_raises():
    # spgemm_test.cpp:125-129
    a = csr(3, 3, np.arange(4, dtype=np.uint64), np.arange(3, dtype=np.uint64), np.ones(3))
    b = csr(4, 4, np.arange(5, dtype=np.uint64), np.arange(4, dtype=np.uint64), np.ones(4))
    with pytest.raises(ab.AiresError) as e:
        ab.spgemm_full(a, b)
    assert e.value.code == ab.errc.dimension_mismatch


def test_empty_operands():
    # spgemm_test.cpp:156-169
    a = csr(3, 4, np.zeros(4, np.uint64), np.zeros(0, np.uint64), np.zeros(0))
    b = ab.CscMatrix(4, 2, np.zeros(3, np.uint64), np.zeros(0, np.uint64), np.zeros(0))
    c = ab.spgemm_full(a, b)
    assert (c.n_rows, c.n_cols, c.nnz()) == (3, 2, 0)
    assert list(c.row_ptr) == [0, 0, 0, 0]


def test_robw_cuts_match_reference_greedy():
    # partition_test.cpp:50-62 golden + random agreement with the oracle (incl. row_too_large)
    p, i, v = triplets([0, 0, 1, 1, 1, 2, 3, 3, 3], [0, 1, 0, 1, 2, 3, 1, 2, 3], list(range(1, 10)), 4, 4)
    segs = ab.robw_partition(csr(4, 4, p, i, v), 120)
    assert [(s.start_row, s.end_row, s.byte_size) for s in segs] == [(0, 2, 104), (2, 4, 88)]
    with pytest.raises(ab.AiresError) as e:
        ab.robw_cuts(p, 63)
    assert e.value.code == ab.errc.row_too_large
    rng = np.random.default_rng(23)
    for _ in range(200):
        n = int(rng.integers(1, 300))
        lens = rng.integers(0, 20, n) * (rng.random(n) < 0.7)
        ptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
        I, V = int(rng.integers(1, 9)), int(rng.integers(1, 9))
        m_a = int(rng.integers(1, 4000))
        rc, cuts, bad = po.robw_cuts(ptr, m_a, I, V)
        if rc == 0:
            got = ab.robw_cuts(ptr, m_a, ab.ElementSizes(I, V))
            assert np.array_equal(got, cuts)
        else:
            with pytest.raises(ab.AiresError) as e:
                ab.robw_cuts(ptr, m_a, ab.ElementSizes(I, V))
            assert e.value.code == ab.errc.row_too_large and f"row {bad} " in str(e.value)


@pytest.mark.parametrize("mode", [ab.MODE_FP64_EXACT, ab.MODE_FP32])
def test_power_law_cfg1_shape(mode):
    """cfg1 shape (100K nodes / 1M edges, X 100K x 512 @1%): fp64 bit-exact checksum, fp32 tolerance."""
    g, st = ab.synth_graph(100_000, 1_000_000, degree_cap=20_000, idx_dtype=np.uint64)
    x = ab.synth_features(100_000, 512, 99.0, 3, idx_dtype=np.uint64)
    rc, (wp, wi, wv), macs = po.spgemm_rowwise(g.row_ptr, g.col_idx, g.values, g.n_rows, g.n_cols, x.n_rows,
                                               x.n_cols, x.row_ptr, x.col_idx, x.values, nthreads=8)
    assert rc == 0
    if mode == ab.MODE_FP64_EXACT:
        c = ab.spgemm_full(g, x)
        assert c.values.dtype == np.float64
        assert po.checksum(c.n_rows, c.n_cols, c.row_ptr, c.col_idx, c.values) == \
            po.checksum(g.n_rows, x.n_cols, wp, wi, wv)
    else:
        g32 = ab.CsrMatrix(g.n_rows, g.n_cols, g.row_ptr, g.col_idx.astype(np.uint32), g.values.astype(np.float32))
        x32 = ab.CsrMatrix(x.n_rows, x.n_cols, x.row_ptr, x.col_idx.astype(np.uint32), x.values.astype(np.float32))
        c = ab.spgemm_full(g32, x32)
        assert_structure_equal(c.row_ptr, c.col_idx, wp, wi)
        assert_close_fp32(c.values, wv, wv)  # all terms positive: scale == value
    blk = ab.spgemm_block(g.row_ptr, g.col_idx, g.values, g.n_rows, g.n_cols, x)
    assert blk.flops == macs


@pytest.mark.parametrize("mode", [ab.MODE_FP64_EXACT, ab.MODE_FP32])
def test_wide_operand_column_tiles(mode):
    """X wider than the dense accumulator: the product runs in column tiles of X (the reference's
    B column tiling, spgemm.hpp:94-130) and must still match bit for bit (fp64) / 1e-5 (fp32)."""
    rng = np.random.default_rng(31)
    for nc, tile in ((12000, "2048"), (300, "64"), (97, "32")):
        ab.set_option("wide_tile", int(tile))
        if nc < 4096:
            ab.set_option("wide_at", 64)
        a = random_csr(rng, 40, 50, 0.2)
        b = random_csr(rng, 50, nc, min(0.5, 30.0 / nc + 0.02))
        (wp, wi, wv), macs = oracle_product(40, 50, nc, a, b, inner=False)
        if mode == ab.MODE_FP64_EXACT:
            blk = ab.spgemm_block(a[0], a[1], a[2], 40, 50, csc_of(50, nc, *b))
            assert_structure_equal(blk.fragment.row_ptr, blk.fragment.col_idx, wp, wi)
            assert bits_equal(blk.fragment.values, wv) and blk.flops == macs
        else:
            c = ab.spgemm_full(csr(40, 50, a[0], a[1], a[2].astype(np.float32)),
                               csr(50, nc, b[0], b[1], b[2].astype(np.float32)))
            (_, _, sv), _ = oracle_product(40, 50, nc, (a[0], a[1], np.abs(a[2])), (b[0], b[1], np.abs(b[2])),
                                           inner=False)
            assert_structure_equal(c.row_ptr, c.col_idx, wp, wi)
            assert_close_fp32(c.values, wv, sv)


def _gold_gcn():
    import os
    return np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "gcn.npz"))


@pytest.mark.parametrize("n,nnz,cap", [(60_000, 900_000, 3000), (5_000, 400_000, 5000)])
def test_normalize_adjacency_matches_oracle_at_size(n, nnz, cap):
    """normalize_adjacency on power-law graphs with hub rows (> 256 entries: the warp-summed degree
    path) and warps whose 32 rows span several shared-memory windows: bit-identical to the oracle's
    restatement of gcn.hpp:29-72, weighted edges (every value 1 + a random fraction)."""
    a, _ = ab.synth_graph(n, nnz, degree_cap=cap, normalize=False, idx_dtype=np.uint64)
    rng = np.random.default_rng(5)
    a = ab.CsrMatrix(n, n, a.row_ptr, a.col_idx, 1.0 + rng.random(a.col_idx.size))
    assert int(np.max(np.diff(a.row_ptr.astype(np.int64)))) > 256
    t = ab.normalize_adjacency(a)
    rc, (wp, wi, wv) = po.normalize_adjacency(n, a.row_ptr, a.col_idx, a.values)
    assert rc == 0
    assert np.array_equal(t.row_ptr, wp) and np.array_equal(t.col_idx, wi)
    assert bits_equal(t.values, wv)


def test_normalize_adjacency_matches_reference_goldens():
    """gcn.hpp:29-72 on the device: bit-identical to the reference (inserted and existing self loops,
    weighted edges, a 2-node graph)."""
    g = _gold_gcn()
    for c in range(int(g["n_norm"][0])):
        k = f"n{c}"
        n = int(g[k + "_n"][0])
        a = ab.CsrMatrix(n, n, g[k + "_in_ptr"], g[k + "_in_idx"], g[k + "_in_val"])
        t = ab.normalize_adjacency(a)
        assert np.array_equal(t.row_ptr, g[k + "_out_ptr"]) and np.array_equal(t.col_idx, g[k + "_out_idx"])
        assert bits_equal(t.values, g[k + "_out_val"])
    # errors (gcn_test.cpp:65-80)
    with pytest.raises(ab.AiresError) as e:
        ab.normalize_adjacency(ab.CsrMatrix(2, 3, np.zeros(3, np.uint64), np.zeros(0, np.uint64), np.zeros(0)))
    assert e.value.code == ab.errc.non_square
    with pytest.raises(ab.AiresError) as e:
        ab.normalize_adjacency(csr(2, 2, np.array([0, 1, 1], np.uint64), np.array([1], np.uint64), np.array([-1.0])))
    assert e.value.code == ab.errc.negative_weight


def test_combine_matches_reference_goldens():
    """gcn.hpp:90-116 on the device: ReLU(X·W), non-positives dropped; fp64 bit-identical, fp32 1e-5."""
    g = _gold_gcn()
    for c in range(int(g["n_comb"][0])):
        k = f"c{c}"
        rows, cin, cout, seed = (int(x) for x in g[k + "_dims"])
        x = ab.CsrMatrix(rows, cin, g[k + "_x_ptr"], g[k + "_x_idx"], g[k + "_x_val"])
        h = ab.combine(x, g[k + "_w"])
        assert np.array_equal(h.row_ptr, g[k + "_h_ptr"]) and np.array_equal(h.col_idx, g[k + "_h_idx"])
        assert bits_equal(h.values, g[k + "_h_val"])
        x32 = ab.CsrMatrix(rows, cin, g[k + "_x_ptr"], g[k + "_x_idx"].astype(np.uint32),
                           g[k + "_x_val"].astype(np.float32))
        h32 = ab.combine(x32, g[k + "_w"].astype(np.float32))
        # fp32 may flip entries whose fp64 value is within rounding of zero; compare on the common set
        ref = {(r, int(cc)): vv for r in range(rows) for cc, vv in
               zip(g[k + "_h_idx"][g[k + "_h_ptr"][r]:g[k + "_h_ptr"][r + 1]],
                   g[k + "_h_val"][g[k + "_h_ptr"][r]:g[k + "_h_ptr"][r + 1]])}
        got = {(r, int(cc)): float(vv) for r in range(rows) for cc, vv in
               zip(h32.col_idx[h32.row_ptr[r]:h32.row_ptr[r + 1]], h32.values[h32.row_ptr[r]:h32.row_ptr[r + 1]])}
        for key in set(ref) ^ set(got):
            assert abs(ref.get(key, 0.0) + got.get(key, 0.0)) < 1e-5
        for key in set(ref) & set(got):
            assert abs(ref[key] - got[key]) <= 1e-5 * max(1.0, abs(ref[key]))
    with pytest.raises(ab.AiresError) as e:
        ab.combine(ab.CsrMatrix(1, 3, np.array([0, 0], np.uint64), np.zeros(0, np.uint64), np.zeros(0)), np.ones((2, 2)))
    assert e.value.code == ab.errc.dimension_mismatch


def test_layer_forward_two_layers_match_oracle():
    """gcn.hpp:125-132 chained twice on a power-law graph, every step on the device, against the
    oracle's normalize -> row-wise A·H -> combine (fp64, bit-identical)."""
    a, _ = ab.synth_graph(3000, 30000, degree_cap=300, normalize=False, idx_dtype=np.uint64)
    x = ab.synth_features(3000, 64, 95.0, 3, idx_dtype=np.uint64)
    w1, w2 = ab.gen_weights(64, 32, 4), ab.gen_weights(32, 8, 5)
    h1 = ab.layer_forward(a, x, w1).h_next
    h2 = ab.layer_forward(a, h1, w2).h_next
    rc, (tp, ti, tv) = po.normalize_adjacency(3000, a.row_ptr, a.col_idx, a.values)
    want = (x.row_ptr, x.col_idx, x.values)
    for w in (w1, w2):
        rc, c, _ = po.spgemm_rowwise(tp, ti, tv, 3000, 3000, 3000, w.shape[0], *want, nthreads=4)
        rc, want = po.combine(3000, w.shape[0], *c, w)
        assert rc == 0
    assert np.array_equal(h2.row_ptr, want[0]) and np.array_equal(h2.col_idx, want[1])
    assert bits_equal(h2.values, want[2])


@pytest.mark.parametrize("hcols,wcols", [(256, 47), (100, 128), (64, 8), (33, 40), (200, 20), (160, 48)])
def test_layer_fused_matches_unfused_chain(hcols, wcols):
    """ReLU((Ã·H)·W) fused (dense-ish H gathered as dense rows) against the fp64 oracle chain
    normalize -> row-wise A·H -> combine: values within 1e-5 relative to the cell's scale; entries
    whose exact value is within rounding of zero may flip across the ReLU."""
    a, _ = ab.synth_graph(4000, 40000, degree_cap=400, normalize=True, idx_dtype=np.uint64)
    h = ab.synth_features(4000, hcols, 50.0, 7, idx_dtype=np.uint64)
    w = ab.gen_weights(hcols, wcols, 9)
    got = ab.layer_fused(a, h, w)
    rc, c, _ = po.spgemm_rowwise(a.row_ptr, a.col_idx, a.values, 4000, 4000, 4000, hcols, h.row_ptr, h.col_idx,
                                 h.values, nthreads=4)
    rc, (wp, wi, wv) = po.combine(4000, hcols, *c, w)
    # scale per output cell: sum_c |C[r,c]| * |W[c,j]|
    rc, (sp, si, sv) = po.combine(4000, hcols, c[0], c[1], np.abs(c[2]), np.abs(w))
    scale = {}
    for r in range(4000):
        for cc, vv in zip(si[sp[r]:sp[r + 1]], sv[sp[r]:sp[r + 1]]):
            scale[(r, int(cc))] = vv
    want = {(r, int(cc)): vv for r in range(4000) for cc, vv in zip(wi[wp[r]:wp[r + 1]], wv[wp[r]:wp[r + 1]])}
    have = {(r, int(cc)): float(vv) for r in range(4000) for cc, vv in
            zip(got.col_idx[got.row_ptr[r]:got.row_ptr[r + 1]], got.values[got.row_ptr[r]:got.row_ptr[r + 1]])}
    for key in set(want) | set(have):
        err = abs(want.get(key, 0.0) - have.get(key, 0.0))
        assert err <= 1e-5 * max(scale.get(key, 0.0), 1e-30), (key, want.get(key), have.get(key), scale.get(key))


@pytest.mark.parametrize("wcols", [47, 20, 64])
def test_layer_fused_gather_kernels_agree_on_sparse_blocks(wcols):
    """The cp.async Ã·T gather (k_agg_t_cp: warps own 32-row blocks, entries streamed as chunks across
    row boundaries) against the register gather (k_agg_t, option agg_async=0) on a graph where most
    rows are empty, so warps own several blocks, some blocks have no entries and chunks end short of
    32: same cells, same ascending-entry fmaf order -> bit-identical CSR."""
    n = 300_000
    rng = np.random.default_rng(17)
    lens = np.zeros(n, dtype=np.int64)
    live = np.arange(0, n, 20)
    lens[live] = rng.integers(1, 70, live.size)
    lens[123_456] = 0
    lens[200_000:200_040] = 33  # a run of rows that straddle chunk boundaries
    rp = np.zeros(n + 1, dtype=np.uint64)
    rp[1:] = np.cumsum(lens)
    cols = np.concatenate([np.sort(rng.choice(n, int(k), replace=False)) for k in lens if k]).astype(np.uint64)
    a = ab.CsrMatrix(n, n, rp, cols, rng.random(cols.size) + 0.01)
    h = ab.synth_features(n, 160, 50.0, 7, idx_dtype=np.uint64)
    w = ab.gen_weights(160, wcols, 9)
    got = ab.layer_fused(a, h, w)
    ab.set_option("agg_async", 0)
    want = ab.layer_fused(a, h, w)
    assert np.array_equal(got.row_ptr, want.row_ptr)
    assert np.array_equal(got.col_idx, want.col_idx)
    assert np.array_equal(np.asarray(got.values).view(np.uint32), np.asarray(want.values).view(np.uint32))
    assert got.row_ptr[-1] > 0


@pytest.mark.parametrize("cin,cout,path", [(100, 256, "v4"), (64, 130, "v4"), (40, 100, "v4"), (30, 96, "v4"),
                                           (100, 256, "scalar"), (64, 130, "two-pass"), (20, 300, "auto")])
def test_combine_fp32_kernels_match_oracle(cin, cout, path):
    """fp32 combine through each kernel path (LDS.128 one-pass for 96..256 output columns, the scalar
    one-pass, the two-pass count/fill) against the fp64 oracle: values within 1e-5 of the cell's
    scale sum |X|·|W|; only entries within that rounding of zero may flip across the ReLU."""
    if path == "scalar":
        ab.set_option("combine_v4", 0)
    if path == "two-pass":
        ab.set_option("combine_one_pass", 0)
    rows = 5000
    x = ab.synth_features(rows, cin, 80.0, 11, idx_dtype=np.uint64)
    w = ab.gen_weights(cin, cout, 12)
    x32 = ab.CsrMatrix(rows, cin, x.row_ptr, x.col_idx.astype(np.uint32), x.values.astype(np.float32))
    got = ab.combine(x32, w.astype(np.float32))
    rc, (wp, wi, wv) = po.combine(rows, cin, x.row_ptr, x.col_idx, x.values, w)
    assert rc == 0
    rc, (sp, si, sv) = po.combine(rows, cin, x.row_ptr, x.col_idx, np.abs(x.values), np.abs(w))
    dense = lambda p, i, v: {(r, int(c)): float(vv) for r in range(rows)  # noqa: E731
                             for c, vv in zip(i[p[r]:p[r + 1]], v[p[r]:p[r + 1]])}
    want, have, scale = dense(wp, wi, wv), dense(got.row_ptr, got.col_idx, got.values), dense(sp, si, sv)
    assert len(have) > 0.3 * len(want)
    for key in set(want) | set(have):
        err = abs(want.get(key, 0.0) - have.get(key, 0.0))
        assert err <= 1e-5 * max(scale.get(key, 0.0), 1e-30), (key, want.get(key), have.get(key))
    for r in range(0, rows, 97):  # ascending columns per row
        assert np.all(np.diff(got.col_idx[got.row_ptr[r]:got.row_ptr[r + 1]].astype(np.int64)) > 0)


@pytest.mark.slow
@pytest.mark.parametrize("shape", ["cfg2", "cfg3"])
def test_full_size_parity(shape):
    """BASELINE configs at full size (Reddit- and ogbn-products-shaped): fp32 structure bit-exact and
    values within 1e-5 of the fp64 oracle; fp64-exact checksum equal to the oracle's; MACs equal."""
    import bench
    cfg = bench.CONFIGS[shape]
    g, st, x = bench.make_inputs(cfg)
    gu = ab.CsrMatrix(g.n_rows, g.n_cols, g.row_ptr, g.col_idx.astype(np.uint64), g.values)
    xu = ab.CsrMatrix(x.n_rows, x.n_cols, x.row_ptr, x.col_idx.astype(np.uint64), x.values)
    rc, (wp, wi, wv), macs = po.spgemm_rowwise(gu.row_ptr, gu.col_idx, gu.values, g.n_rows, g.n_cols, x.n_rows,
                                               x.n_cols, xu.row_ptr, xu.col_idx, xu.values, nthreads=16)
    assert rc == 0
    g32 = ab.CsrMatrix(g.n_rows, g.n_cols, g.row_ptr, g.col_idx, g.values.astype(np.float32))
    x32 = ab.CsrMatrix(x.n_rows, x.n_cols, x.row_ptr, x.col_idx, x.values.astype(np.float32))
    blk = ab.spgemm_block(g32.row_ptr, g32.col_idx, g32.values, g.n_rows, g.n_cols, x32)
    c = blk.fragment
    assert blk.flops == macs
    assert np.array_equal(c.row_ptr, wp) and np.array_equal(c.col_idx.astype(np.uint64), wi)
    err = np.abs(c.values.astype(np.float64) - wv) / np.abs(wv)
    assert float(err.max()) <= 1e-5
    c64 = ab.spgemm_full(gu, xu)  # fp64-exact
    assert po.checksum(c64.n_rows, c64.n_cols, c64.row_ptr, c64.col_idx, c64.values) == \
        po.checksum(g.n_rows, x.n_cols, wp, wi, wv)
