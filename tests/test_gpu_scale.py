"""GPU parity at the benchmarked sizes: the out-of-core run
(aires_b200_run / run_aires, scheduler.hpp:72-168) under capped device budgets, the streamed
output and the MaxMemory baseline, each against the CPU oracle's row-wise product
(oracle/aires_oracle.c ao_spgemm_rowwise, pinned to the reference by tests/test_oracle.py).

North_star parity rule: structure (row_ptr, col_idx, nnz) bit-exact; fp32 values within 1e-5
relative (the synthetic operands are positive, so no cell cancels and the value itself is the
cell's Σ|a·x|); FP64_EXACT values bit-identical, i.e. checksum(C) (serialize.hpp:50-59) equal.
These are the checks acceptance.cpp:66-103 (criterion 2: out-of-core == in-core) and
spgemm_test.cpp:97-115 (partition independence) make, at the sizes the bench reports."""
import numpy as np
import pytest

import paper_2507_02006_b200 as ab
from oracle import pyoracle as po

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

SHAPES = {  # bench.py CONFIGS (same seeds: graph 1, relabel 2, X 3)
    "cfg2": (232_965, 114_000_000, 602),
    "cfg3": (2_449_029, 62_000_000, 100),
}
_cache = {}


def _inputs(name):
    if name not in _cache:
        n, nnz, dim = SHAPES[name]
        g, _ = ab.synth_graph(n, nnz, alpha=0.75, degree_cap=20_000, seed=1, relabel_seed=2, idx_dtype=np.uint32,
                              val_dtype=np.float64)
        x = ab.synth_features(n, dim, 99.0, 3, idx_dtype=np.uint32, val_dtype=np.float64)
        rc, (wp, wi, wv), macs = po.spgemm_rowwise(g.row_ptr, g.col_idx, g.values, n, n, n, dim, x.row_ptr, x.col_idx,
                                                   x.values, nthreads=16)
        assert rc == 0
        ck = po.checksum(n, dim, wp, wi, wv)
        _cache[name] = (g, x, (wp, wi, wv), macs, ck)
    return _cache[name]


def _f32(m):
    return ab.CsrMatrix(m.n_rows, m.n_cols, m.row_ptr, m.col_idx, m.values.astype(np.float32))


def _budget(g, x, nnz_c, frac, vb=4):
    """frac x (B_A + B_X + B_C) at device widths (u64 ptr, u32 idx, fp32 / fp64 val) -- bench.py's cap."""
    b_a = 8 * (g.n_rows + 1) + (4 + vb) * g.nnz()
    b_x = 8 * (x.n_rows + 1) + (4 + vb) * x.nnz()
    b_c = 8 * (g.n_rows + 1) + (4 + vb) * nnz_c
    return ab.MemoryBudget(int(frac * (b_a + b_x + b_c)))


def _check_fp32(c, want, macs, flops):
    wp, wi, wv = want
    assert np.array_equal(c.row_ptr, wp), "row_ptr differs from the oracle"
    assert np.array_equal(c.col_idx.astype(np.uint64), wi), "col_idx differs from the oracle"
    err = np.abs(c.values.astype(np.float64) - wv) / wv
    assert float(err.max(initial=0.0)) <= 1e-5, f"max rel err {err.max()}"
    assert flops == macs


@pytest.mark.parametrize("frac,min_tiles", [(0.5, 2), (0.25, 4)])
def test_cfg3_capped_fp32_matches_oracle(frac, min_tiles):
    g, x, want, macs, _ = _inputs("cfg3")
    res = ab.run_aires(_f32(g), _f32(x), _budget(g, x, want[1].shape[0], frac), n_buffers=3, with_checksum=False)
    assert res.report.segments >= min_tiles
    _check_fp32(res.c, want, macs, res.report.flops)


@pytest.mark.parametrize("frac", [0.5, 0.25, 0.125])
def test_cfg3_capped_streamed_fp32_matches_oracle(frac):
    """bench.py's out-of-core sweep: capped, streamed output (A crosses the link once)"""
    g, x, want, macs, _ = _inputs("cfg3")
    res = ab.run_aires(_f32(g), _f32(x), _budget(g, x, want[1].shape[0], frac), n_buffers=3, with_checksum=False,
                       stream_out=True)
    assert res.report.segments >= 2
    _check_fp32(res.c, want, macs, res.report.flops)
    b_a = 8 * (g.n_rows + 1) + 8 * g.nnz()
    b_x = 8 * (x.n_rows + 1) + 8 * x.nnz()
    assert b_a + b_x <= res.report.ledger.h2d.bytes <= b_a + b_x + 8 * res.report.segments  # A crosses once


def test_cfg2_capped_streamed_fp32_matches_oracle():
    g, x, want, macs, _ = _inputs("cfg2")
    res = ab.run_aires(_f32(g), _f32(x), _budget(g, x, want[1].shape[0], 0.25), n_buffers=3, with_checksum=False,
                       stream_out=True)
    assert res.report.segments >= 4
    _check_fp32(res.c, want, macs, res.report.flops)


def test_cfg3_capped_fp64_exact_checksum():
    g, x, want, macs, ck = _inputs("cfg3")
    res = ab.run_aires(g, x, _budget(g, x, want[1].shape[0], 0.25, vb=8), n_buffers=3)  # fp64 -> FP64_EXACT
    assert res.report.segments >= 4
    assert res.report.c_checksum == ck
    assert res.report.flops == macs


def test_cfg3_maxmemory_matches_oracle():
    g, x, want, macs, _ = _inputs("cfg3")
    res = ab.run_maxmemory(_f32(g), _f32(x), _budget(g, x, want[1].shape[0], 0.25), n_buffers=3,
                           with_checksum=False)
    assert res.report.segments >= 4
    _check_fp32(res.c, want, macs, res.report.flops)


def test_cfg2_capped_fp32_matches_oracle():
    """north_star's target sentence: Reddit-shaped, out of core, matching the CPU oracle."""
    g, x, want, macs, _ = _inputs("cfg2")
    res = ab.run_aires(_f32(g), _f32(x), _budget(g, x, want[1].shape[0], 0.25), n_buffers=3, with_checksum=False)
    assert res.report.segments >= 4
    _check_fp32(res.c, want, macs, res.report.flops)


def test_cfg2_capped_fp64_exact_checksum():
    g, x, want, macs, ck = _inputs("cfg2")
    res = ab.run_aires(g, x, _budget(g, x, want[1].shape[0], 0.25, vb=8), n_buffers=3)
    assert res.report.segments >= 4
    assert res.report.c_checksum == ck


def test_cfg2_streamed_output_matches_oracle():
    """the bench's e2e run (streamed output, uncapped), values included"""
    g, x, want, macs, _ = _inputs("cfg2")
    res = ab.run_aires(_f32(g), _f32(x), ab.MemoryBudget(0), stream_out=True, n_buffers=3, with_checksum=False)
    _check_fp32(res.c, want, macs, res.report.flops)


def test_cfg2_resident_fp32_and_fp64_match_oracle():
    """the bench's device-resident step (aires_b200_spgemm) in both arithmetic modes"""
    g, x, want, macs, ck = _inputs("cfg2")
    c32 = ab.spgemm_full(_f32(g), _f32(x))
    _check_fp32(c32, want, macs, macs)
    c64 = ab.spgemm_full(g, x)
    assert po.checksum(c64.n_rows, c64.n_cols, c64.row_ptr, c64.col_idx, c64.values) == ck
