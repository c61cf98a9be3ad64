"""CPU tier: the oracle restatement (oracle/aires_oracle.c) pinned against
  (1) the known answers of the reference's own unit tests (cited per test),
  (2) the committed golden fixtures made by the reference itself (tests/golden/make_golden.py), and
  (3) the live reference build (oracle/_ref) where it exists (this container; skipped elsewhere).
"""
import os
import subprocess

import numpy as np
import pytest

from oracle import pyoracle as po

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
need_ref = pytest.mark.skipif(not po.ref_available(), reason="oracle/_ref not built (no /root/reference)")


def gold(name):
    return np.load(os.path.join(GOLD, name))


def bits(v):
    return np.ascontiguousarray(v, np.float64).view(np.uint64)


def test_fnv_known_vectors():
    # serialize_test.cpp:18-22
    assert po.fnv1a64(b"") == 14695981039346656037
    assert po.fnv1a64(b"a") == 0xaf63dc4c8601ec8c
    assert po.fnv1a64(b"foobar") == 0x85944171f73967e8


def test_checksum_distinguishes_explicit_zero():
    # serialize_test.cpp:36-47
    z = po.checksum(1, 1, [0, 1], [0], [0.0])
    e = po.checksum(1, 1, [0, 0], [], [])
    assert z != e


def test_memory_model_goldens():
    # memory_model_test.cpp:12-50, 87-91
    assert po.estimate_output_memory(800, 90.0, 400, 95.0) == 372
    assert po.estimate_output_memory(0, 100.0, 400, 95.0) == 0
    assert po.estimate_output_memory(100, 70.0, 100, 70.0) == 207
    assert po.block_budget(2272, 372, 900) == (0, 333, 1000)
    assert po.block_budget(1272, 372, 900)[0] == 5  # insufficient_device_memory
    assert po.calc_mem(2, 5) == 104 and po.calc_mem(3, 6) == 128


def test_robw_golden_and_row_too_large():
    # partition_test.cpp:50-62 (nnz [2,3,1,3], m_a=120 -> {0,1},{2,3}) and :90-95 (63 fails, 64 ok)
    ptr = np.array([0, 2, 5, 6, 9], np.uint64)
    rc, cuts, _ = po.robw_cuts(ptr, 120)
    assert rc == 0 and list(cuts) == [0, 2, 4]
    assert po.calc_mem(2, 5) == 104 and po.calc_mem(2, 4) == 88
    one = np.array([0, 3], np.uint64)
    assert po.robw_cuts(one, 63)[0] == 6
    assert po.robw_cuts(one, 64)[0] == 0


def test_hand_product_inner_and_rowwise():
    # spgemm_test.cpp:43-53: [[1,2],[0,3]] * [[4,0],[5,6]] = [[14,12],[15,18]]
    a = (np.array([0, 2, 3], np.uint64), np.array([0, 1, 1], np.uint64), np.array([1.0, 2.0, 3.0]))
    b = (np.array([0, 1, 3], np.uint64), np.array([0, 0, 1], np.uint64), np.array([4.0, 5.0, 6.0]))
    cp, ri, cv = po.csr_to_csc(2, 2, *b)
    rc, (p, i, v), macs = po.spgemm_inner(*a, 2, 2, 2, 2, cp, ri, cv)
    assert rc == 0 and list(p) == [0, 2, 4] and list(i) == [0, 1, 0, 1] and list(v) == [14, 12, 15, 18]
    assert macs == 5
    rc, (p2, i2, v2), m2 = po.spgemm_rowwise(*a, 2, 2, 2, 2, *b)
    assert rc == 0 and np.array_equal(p, p2) and np.array_equal(i, i2) and np.array_equal(bits(v), bits(v2))
    assert m2 == macs


def test_structural_zero_kept():
    # spgemm_test.cpp:62-70
    a = (np.array([0, 2], np.uint64), np.array([0, 1], np.uint64), np.array([1.0, -1.0]))
    b = (np.array([0, 1, 2], np.uint64), np.array([0, 0], np.uint64), np.array([1.0, 1.0]))
    rc, (p, i, v), _ = po.spgemm_rowwise(*a, 1, 2, 2, 1, *b)
    assert rc == 0 and list(i) == [0] and v[0] == 0.0


def _golden_spgemm():
    g = gold("spgemm.npz")
    for c in range(int(g["n_cases"][0])):
        nr, ni, nc, macs, ck = (int(x) for x in g[f"c{c}_dims"])
        a = tuple(g[f"c{c}_a_{k}"] for k in ("ptr", "idx", "val"))
        b = tuple(g[f"c{c}_b_{k}"] for k in ("ptr", "idx", "val"))
        want = tuple(g[f"c{c}_c_{k}"] for k in ("ptr", "idx", "val"))
        yield c, nr, ni, nc, a, b, want, macs, ck


def test_oracle_inner_matches_reference_goldens():
    for c, nr, ni, nc, a, b, want, macs, ck in _golden_spgemm():
        cp, ri, cv = po.csr_to_csc(ni, nc, *b)
        rc, got, m = po.spgemm_inner(*a, nr, ni, ni, nc, cp, ri, cv)
        assert rc == 0, c
        assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1]), c
        assert np.array_equal(bits(got[2]), bits(want[2])), c
        assert m == macs and po.checksum(nr, nc, *got) == ck, c


def test_oracle_rowwise_matches_reference_goldens():
    for c, nr, ni, nc, a, b, want, macs, ck in _golden_spgemm():
        for threads in (1, 3):
            rc, got, m = po.spgemm_rowwise(*a, nr, ni, ni, nc, *b, nthreads=threads)
            assert rc == 0
            assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1]), c
            assert np.array_equal(bits(got[2]), bits(want[2])), c
            assert m == macs and po.checksum(nr, nc, *got) == ck, c


def test_tile_width_invariance_oracle():
    # spgemm_test.cpp:117-123
    for c, nr, ni, nc, a, b, want, macs, ck in _golden_spgemm():
        cp, ri, cv = po.csr_to_csc(ni, nc, *b)
        for tile in (1, 7, 1000):
            rc, got, _ = po.spgemm_inner(*a, nr, ni, ni, nc, cp, ri, cv, tile_cols=tile)
            assert rc == 0 and po.checksum(nr, nc, *got) == ck


def test_csr_csc_round_trip():
    # sparse_test.cpp:56-73
    for c, nr, ni, nc, a, b, want, macs, ck in _golden_spgemm():
        cp, ri, cv = po.csr_to_csc(ni, nc, *b)
        p, i, v = po.csc_to_csr(ni, nc, cp, ri, cv)
        assert np.array_equal(p, b[0]) and np.array_equal(i, b[1]) and np.array_equal(bits(v), bits(b[2]))


def test_oracle_robw_matches_reference_goldens():
    g = gold("robw.npz")
    for r in range(int(g["n_cases"][0])):
        m_a, I, V, rc_ref = (int(x) for x in g[f"r{r}_args"])
        rc, cuts, bad = po.robw_cuts(g[f"r{r}_ptr"], m_a, I, V)
        assert rc == rc_ref, r
        if rc == 0:
            assert np.array_equal(cuts, g[f"r{r}_cuts"]), r


def test_oracle_gen_features_matches_reference_goldens():
    g = gold("features.npz")
    for f in range(int(g["n_cases"][0])):
        n, dim, sp, seed = g[f"f{f}_spec"]
        rc, (p, i, v) = po.gen_features(int(n), int(dim), float(sp), int(seed))
        assert rc == 0
        assert np.array_equal(p, g[f"f{f}_ptr"]) and np.array_equal(i, g[f"f{f}_idx"])
        assert np.array_equal(bits(v), bits(g[f"f{f}_val"]))


@need_ref
def test_oracle_matches_live_reference_random():
    rng = np.random.default_rng(99)
    from tests._util import random_csr
    for _ in range(40):
        nr, ni, nc = (int(x) for x in rng.integers(1, 30, 3))
        a = random_csr(rng, nr, ni, 0.3)
        b = random_csr(rng, ni, nc, 0.3)
        cp, ri, cv = po.csr_to_csc(ni, nc, *b)
        _, want, m1 = po.spgemm_inner(*a, nr, ni, ni, nc, cp, ri, cv, use_ref=True)
        _, got, m2 = po.spgemm_rowwise(*a, nr, ni, ni, nc, *b)
        assert m1 == m2 and po.checksum(nr, nc, *got) == po.checksum(nr, nc, *want, use_ref=True)


@need_ref
def test_oracle_normalize_adjacency_matches_reference():
    rc, g = po.gen_symmetric(200, 0.05, 3)
    assert rc == 0
    _, want = po.normalize_adjacency(200, *g, use_ref=True)
    _, got = po.normalize_adjacency(200, *g)
    assert all(np.array_equal(x, y) for x, y in zip(got[:2], want[:2]))
    assert np.array_equal(bits(got[2]), bits(want[2]))


REF_UNITS = ["spgemm_test", "partition_test", "memory_model_test", "sparse_test", "serialize_test", "gcn_test",
             "scheduler_test"]


@pytest.mark.parametrize("unit", REF_UNITS)
def test_reference_unit_suite_passes(unit):
    """The reference's own GTest files, compiled against the reference headers with the
    GTest-compatible shim (oracle/gtest_shim), pass: the shim is a faithful test runner."""
    exe = os.path.join(os.path.dirname(po.REF_SO), f"ref_unit_{unit}")
    if not os.path.exists(exe):
        pytest.skip("reference unit binaries not built (no /root/reference)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]


@pytest.mark.parametrize("args", [(20_000, 200_000, 0.75, 2_000, 1, 2, True, True),
                                  (5_000, 40_000, 0.6, 500, 7, 3, False, True),
                                  (30_000, 300_000, 0.9, 3_000, 2, 5, True, False),
                                  (100_000, 1_000_000, 0.75, 20_000, 1, 2, True, True)])
def test_synth_graph_restatement(args):
    """The reference arm's input generator (ao_synth_graph) is byte-identical to the B200 library's
    aires_b200_synth_graph, so `bench.py --impl reference` multiplies the same Ã without loading
    libaires_b200.so (host code only: no GPU needed)."""
    import paper_2507_02006_b200 as ab
    n, nnz, alpha, cap, seed, rseed, relabel, norm = args
    g, st = ab.synth_graph(n, nnz, alpha=alpha, degree_cap=cap, seed=seed, relabel_seed=rseed, relabel=relabel,
                           normalize=norm, idx_dtype=np.uint64, val_dtype=np.float64)
    (p, i, v), st2 = po.synth_graph(n, nnz, alpha, cap, seed, rseed, relabel, norm)
    assert np.array_equal(g.row_ptr, p) and np.array_equal(g.col_idx, i)
    assert np.array_equal(bits(g.values), bits(v))
    assert all(st[k] == st2[k] for k in ("nnz_a", "max_degree", "rounds", "i0"))


def test_rows_hash_matches_reference_sampled_rows():
    """ao_rows_hash over a CSR product equals the hash ref_spgemm_rows_timed reports for the same rows,
    so the reference's live sampled rows can be compared with any product read back (bench.py)."""
    if not po.ref_available():
        pytest.skip("oracle/_ref not built")
    (ap, ai, av), _ = po.synth_graph(3_000, 30_000, 0.75, 300, 1, 2, True, True)
    rc, (xp, xi, xv) = po.gen_features(3_000, 64, 90.0, 3)
    assert rc == 0
    rc, (cp_, ci_, cv_), macs = po.spgemm_rowwise(ap, ai, av, 3_000, 3_000, 3_000, 64, xp, xi, xv)
    rows = np.sort(np.random.default_rng(0).choice(3_000, 200, replace=False)).astype(np.uint64)
    cp, ri, cv = po.csr_to_csc(3_000, 64, xp, xi, xv)
    _, m, z, h = po.ref_rows_timed(ap, ai, av, 3_000, rows, cp, ri, cv, 3_000, 64, 2)
    assert h == po.rows_hash(cp_, ci_, cv_, rows)
    assert z == int(sum(int(cp_[r + 1] - cp_[r]) for r in rows))
