"""Shared test helpers: seeded random operands and comparisons against the oracle."""
import numpy as np

from oracle import pyoracle as po


def random_csr(rng: np.random.Generator, nr: int, nc: int, density: float, lo=-2.0, hi=2.0):
    """Canonical CSR (sorted unique columns, no stored zeros) at API widths (u64/f64),
    like spgemm_test.cpp:18-29's random_matrix."""
    mask = rng.random((nr, nc)) < density
    vals = rng.random((nr, nc)) * (hi - lo) + lo
    vals[vals == 0.0] = 0.5
    ptr = np.zeros(nr + 1, dtype=np.uint64)
    ptr[1:] = np.cumsum(mask.sum(axis=1))
    rr, cc = np.nonzero(mask)
    return ptr, cc.astype(np.uint64), vals[rr, cc].astype(np.float64)


def to_csc(nr, nc, ptr, idx, val):
    cp, ri, cv = po.csr_to_csc(nr, nc, ptr, idx, val)
    return cp, ri, cv


def oracle_product(nr, ni, nc, a, b, inner=True):
    """C = A*B via the oracle; a, b are (ptr, idx, val) CSR triples."""
    if inner:
        cp, ri, cv = to_csc(ni, nc, *b)
        rc, c, macs = po.spgemm_inner(a[0], a[1], a[2], nr, ni, ni, nc, cp, ri, cv)
    else:
        rc, c, macs = po.spgemm_rowwise(a[0], a[1], a[2], nr, ni, ni, nc, b[0], b[1], b[2])
    assert rc == 0
    return c, macs


def bits_equal(x: np.ndarray, y: np.ndarray) -> bool:
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    return x.shape == y.shape and np.array_equal(x.view(np.uint64), y.view(np.uint64))


def assert_structure_equal(got_ptr, got_idx, want_ptr, want_idx):
    np.testing.assert_array_equal(np.asarray(got_ptr, dtype=np.uint64), np.asarray(want_ptr, dtype=np.uint64))
    np.testing.assert_array_equal(np.asarray(got_idx, dtype=np.uint64), np.asarray(want_idx, dtype=np.uint64))


def assert_close_fp32(got_val, want_val, scale, rtol=1e-5):
    """fp32 parity: |got - want| <= rtol * max(1e-30, scale) per cell, where scale is the
    oracle's sum of |a_ik * x_kj| for the cell (cancellation-safe relative tolerance)."""
    got = np.asarray(got_val, dtype=np.float64)
    err = np.abs(got - want_val)
    bound = rtol * np.maximum(scale, 1e-30)
    bad = np.nonzero(err > bound)[0]
    assert bad.size == 0, f"{bad.size} cells exceed tolerance; first {bad[:5]} err {err[bad[:5]]} bound {bound[bad[:5]]}"
