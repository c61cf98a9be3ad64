"""Regenerates tests/golden/*.npz from the REFERENCE itself (oracle/_ref/libaires_ref.so, the
unmodified /root/reference/proj/include headers compiled by oracle/Makefile).

Run here (where /root/reference exists):  python tests/golden/make_golden.py
The fixtures are committed so the CPU tests (and the GPU box, which has no /root/reference)
can pin the oracle restatement and the B200 kernels against the reference's own outputs.

  spgemm.npz    : spgemm_block (spgemm.hpp:60-132) on seeded random pairs like
                  spgemm_test.cpp:18-29 (signed values, cancellations, empty rows/cols) and on a
                  normalize_adjacency(gen_symmetric) x gen_features chain (gcn.hpp:29-72,
                  synth.hpp:26-46,73-78); outputs with f64 bits, flops, checksum (serialize.hpp:50-59)
  robw.npz      : robw_partition cuts (partition.hpp:52-74) incl. row_too_large cases
  features.npz  : gen_features (synth.hpp:73-78) outputs for the seeds the benches use
  run_aires.npz : run_aires (scheduler.hpp:72-168) ledgers on single-segment budgets
  segments.npz  : the reference's robw_partition + write_segments byte streams (serialize.hpp:148-174)
                  at ElementSizes {8,8} and {4,4}
  gcn.npz       : normalize_adjacency (gcn.hpp:29-72) incl. graphs with existing diagonals and
                  weighted edges, gen_weights (synth.hpp:81-86) and combine (gcn.hpp:90-116)
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import pyoracle as po  # noqa: E402


def random_csr(rng, nr, nc, density, lo=-2.0, hi=2.0, ints=False):
    mask = rng.random((nr, nc)) < density
    if ints:
        vals = rng.integers(-3, 4, (nr, nc)).astype(np.float64)
        vals[vals == 0] = 1.0
    else:
        vals = rng.random((nr, nc)) * (hi - lo) + lo
        vals[vals == 0.0] = 0.5
    ptr = np.zeros(nr + 1, dtype=np.uint64)
    ptr[1:] = np.cumsum(mask.sum(axis=1))
    rr, cc = np.nonzero(mask)
    return ptr, cc.astype(np.uint64), vals[rr, cc].astype(np.float64)


def spgemm_cases():
    rng = np.random.default_rng(2025)
    out = {}
    cases = []
    for t in range(16):
        nr, ni, nc = (int(v) for v in rng.integers(1, 33, 3))
        d = 0.05 + 0.5 * rng.random()
        cases.append((nr, ni, nc, random_csr(rng, nr, ni, d, ints=t % 4 == 3),
                      random_csr(rng, ni, nc, d, ints=t % 4 == 3)))
    # GCN chain: Ã = normalize_adjacency(gen_symmetric), X = gen_features
    rc, g = po.gen_symmetric(300, 0.03, 7)
    assert rc == 0
    rc, at = po.normalize_adjacency(300, *g, use_ref=True)
    assert rc == 0
    rc, xf = po.gen_features(300, 96, 95.0, 3, use_ref=True)
    assert rc == 0
    cases.append((300, 300, 96, at, xf))
    for i, (nr, ni, nc, a, b) in enumerate(cases):
        cp, ri, cv = po.csr_to_csc(ni, nc, *b, use_ref=True)
        rc, (p, ix, v), macs = po.spgemm_inner(a[0], a[1], a[2], nr, ni, ni, nc, cp, ri, cv, use_ref=True)
        assert rc == 0
        out[f"c{i}_dims"] = np.array([nr, ni, nc, macs, po.checksum(nr, nc, p, ix, v, use_ref=True)], np.uint64)
        for nm, arrs in (("a", a), ("b", b), ("c", (p, ix, v))):
            out[f"c{i}_{nm}_ptr"], out[f"c{i}_{nm}_idx"], out[f"c{i}_{nm}_val"] = arrs
    out["n_cases"] = np.array([len(cases)])
    np.savez_compressed(os.path.join(HERE, "spgemm.npz"), **out)


def robw_cases():
    rng = np.random.default_rng(77)
    out = {}
    n_cases = 60
    for i in range(n_cases):
        n = int(rng.integers(1, 200))
        lens = rng.integers(0, 25, n) * (rng.random(n) < 0.75)
        ptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
        I, V = int(rng.integers(1, 9)), int(rng.integers(1, 9))
        m_a = int(rng.integers(1, 3000))
        rc, cuts, _ = po.robw_cuts(ptr, m_a, I, V, use_ref=True)
        out[f"r{i}_ptr"] = ptr
        out[f"r{i}_args"] = np.array([m_a, I, V, rc], np.uint64)
        out[f"r{i}_cuts"] = cuts if rc == 0 else np.zeros(0, np.uint64)
    out["n_cases"] = np.array([n_cases])
    np.savez_compressed(os.path.join(HERE, "robw.npz"), **out)


def feature_cases():
    out = {}
    specs = [(500, 64, 99.0, 3), (200, 602, 99.0, 3), (300, 100, 90.0, 11), (64, 8, 50.0, 4)]
    for i, (n, dim, sp, seed) in enumerate(specs):
        rc, (p, ix, v) = po.gen_features(n, dim, sp, seed, use_ref=True)
        assert rc == 0
        out[f"f{i}_spec"] = np.array([n, dim, sp, seed], np.float64)
        out[f"f{i}_ptr"], out[f"f{i}_idx"], out[f"f{i}_val"] = p, ix, v
    out["n_cases"] = np.array([len(specs)])
    np.savez_compressed(os.path.join(HERE, "features.npz"), **out)


def run_aires_cases():
    """run_aires ledgers (RunReport / IoLedger, scheduler.hpp:25-43) on budgets that fit one segment."""
    rng = np.random.default_rng(5)
    out = {}
    n_cases = 0
    for t in range(6):
        n = int(rng.integers(5, 40))
        a = random_csr(rng, n, n, 0.2, 0.1, 1.0)
        b = random_csr(rng, n, n, 0.2, 0.1, 1.0)
        cp, ri, cv = po.csr_to_csc(n, n, *b, use_ref=True)
        total = 1 << 22
        rc, c, rep = po.ref_run_aires(a[0], a[1], a[2], n, n, cp, ri, cv, n, n, total)
        if rc:
            continue
        k = f"s{n_cases}"
        out[k + "_a_ptr"], out[k + "_a_idx"], out[k + "_a_val"] = a
        out[k + "_b_ptr"], out[k + "_b_idx"], out[k + "_b_val"] = b
        out[k + "_budget"] = np.array([total], np.uint64)
        out[k + "_report"] = np.array([rep[key] for key in sorted(rep) if not key.endswith("_s")], np.uint64)
        out[k + "_report_keys"] = np.array([key for key in sorted(rep) if not key.endswith("_s")])
        n_cases += 1
    out["n_cases"] = np.array([n_cases])
    np.savez_compressed(os.path.join(HERE, "run_aires.npz"), **out)


def gcn_cases():
    rng = np.random.default_rng(91)
    out = {}
    n_cases = 0
    graphs = []
    for n, d, seed in ((40, 0.1, 1), (300, 0.03, 7), (2, 0.5, 3)):
        rc, g = po.gen_symmetric(n, d, seed)
        assert rc == 0
        graphs.append((n, g))
    # weighted, with some diagonal entries present
    n = 60
    p, i, v = random_csr(rng, n, n, 0.1, 0.1, 2.0)
    graphs.append((n, (p, i, np.abs(v))))
    for n, (p, i, v) in graphs:
        rc, (tp, ti, tv) = po.normalize_adjacency(n, p, i, v, use_ref=True)
        assert rc == 0
        k = f"n{n_cases}"
        out[k + "_in_ptr"], out[k + "_in_idx"], out[k + "_in_val"] = p, i, v
        out[k + "_out_ptr"], out[k + "_out_idx"], out[k + "_out_val"] = tp, ti, tv
        out[k + "_n"] = np.array([n], np.uint64)
        n_cases += 1
    out["n_norm"] = np.array([n_cases])
    n_comb = 0
    for rows, cin, cout, d, seed in ((30, 20, 7, 0.3, 4), (50, 64, 40, 0.2, 5), (10, 5, 300, 0.5, 6)):
        x = random_csr(rng, rows, cin, d, -1.0, 1.0)
        w = po.gen_weights(cin, cout, seed, use_ref=True)
        rc, (hp, hi, hv) = po.combine(rows, cin, *x, w, use_ref=True)
        assert rc == 0
        k = f"c{n_comb}"
        out[k + "_x_ptr"], out[k + "_x_idx"], out[k + "_x_val"] = x
        out[k + "_w"] = w
        out[k + "_h_ptr"], out[k + "_h_idx"], out[k + "_h_val"] = hp, hi, hv
        out[k + "_dims"] = np.array([rows, cin, cout, seed], np.uint64)
        n_comb += 1
    out["n_comb"] = np.array([n_comb])
    np.savez_compressed(os.path.join(HERE, "gcn.npz"), **out)


def segment_cases():
    import tempfile
    rng = np.random.default_rng(17)
    out = {}
    cases = [(50, 40, 0.2, 8, 8, 700), (80, 30, 0.15, 4, 4, 300)]
    for c, (nr, nc, d, I, V, m_a) in enumerate(cases):
        a = random_csr(rng, nr, nc, d, 0.1, 1.0)
        with tempfile.NamedTemporaryFile(suffix=".seg") as f:
            rc = po.ref_write_segments(f.name, nr, nc, *a, m_a, I, V)
            assert rc == 0
            out[f"s{c}_bytes"] = np.fromfile(f.name, dtype=np.uint8)
        out[f"s{c}_a_ptr"], out[f"s{c}_a_idx"], out[f"s{c}_a_val"] = a
        out[f"s{c}_args"] = np.array([nr, nc, I, V, m_a], np.uint64)
    out["n_cases"] = np.array([len(cases)])
    np.savez_compressed(os.path.join(HERE, "segments.npz"), **out)


if __name__ == "__main__":
    if not po.ref_available():
        sys.exit("oracle/_ref/libaires_ref.so missing: run `make -C oracle ref` (needs /root/reference)")
    spgemm_cases()
    robw_cases()
    feature_cases()
    run_aires_cases()
    gcn_cases()
    segment_cases()
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))
