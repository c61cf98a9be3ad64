"""CPU tier: the C-ABI library (libaires_b200.so) loads, exports every entry point that
include/*.h declares, and -- with no GPU visible -- fails loudly (never a CPU fallback)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_2507_02006_b200 as ab

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    syms = set()
    for h in os.listdir(os.path.join(ROOT, "include")):
        if h.endswith(".h"):
            txt = open(os.path.join(ROOT, "include", h)).read()
            txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
            syms |= set(re.findall(r"\b(aires_b200_\w+)\s*\(", txt))
    return sorted(s for s in syms if not s.endswith("_fn"))


def test_library_exports_every_declared_symbol():
    L = ab.lib()
    syms = declared_symbols()
    assert len(syms) >= 15
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing


def test_abi_version_and_status_mapping():
    assert ab.lib().aires_b200_abi_version() == ab.ABI_VERSION == 2
    # status = 1 + errc (error.hpp:9-27)
    e = ab.AiresError(8, "x")
    assert e.code == ab.errc.dimension_mismatch and str(e).startswith("dimension_mismatch")
    assert ab.AiresError(6, "r").code == ab.errc.row_too_large
    assert ab.AiresError(101, "n").code is None


@pytest.mark.skipif(ab.device_count() > 0, reason="a CUDA device is visible")
def test_no_device_fails_loudly():
    a = ab.CsrMatrix(2, 2, np.array([0, 1, 2], np.uint64), np.array([0, 1], np.uint64), np.ones(2))
    with pytest.raises(ab.AiresError) as e:
        ab.spgemm_full(a, a)
    assert e.value.status == 101 and "no CUDA device" in str(e.value)
    with pytest.raises(ab.AiresError):
        ab.robw_cuts(np.array([0, 1, 2], np.uint64), 100)


def test_synth_features_is_reference_gen_features():
    """The host-side generator the bench uses reproduces gen_features (synth.hpp:73-78) byte for
    byte (golden fixture made by the reference)."""
    g = np.load(os.path.join(ROOT, "tests", "golden", "features.npz"))
    for f in range(int(g["n_cases"][0])):
        n, dim, sp, seed = g[f"f{f}_spec"]
        x = ab.synth_features(int(n), int(dim), float(sp), int(seed), idx_dtype=np.uint64)
        assert np.array_equal(x.row_ptr, g[f"f{f}_ptr"]) and np.array_equal(x.col_idx, g[f"f{f}_idx"])
        assert np.array_equal(x.values.view(np.uint64), g[f"f{f}_val"].view(np.uint64))


def test_synth_graph_shape_and_normalization():
    """Chung-Lu Ã: symmetric, self-loops present, values 1/sqrt(d_i d_j) (gcn.hpp:29-72)."""
    g, st = ab.synth_graph(3000, 30000, degree_cap=500, idx_dtype=np.uint64)
    assert g.row_ptr[-1] == g.nnz()
    rows = np.repeat(np.arange(g.n_rows), np.diff(g.row_ptr.astype(np.int64)))
    cols = g.col_idx.astype(np.int64)
    assert np.all(np.diff(cols)[np.diff(rows) == 0] > 0)  # canonical
    import scipy.sparse as sp
    m = sp.csr_matrix((g.values, cols, g.row_ptr.astype(np.int64)), shape=(g.n_rows, g.n_cols))
    assert abs(m - m.T).max() < 1e-15
    assert np.all(m.diagonal() > 0)
    deg = np.diff(g.row_ptr.astype(np.int64)).astype(np.float64)
    np.testing.assert_allclose(g.values, 1.0 / np.sqrt(deg[rows] * deg[cols]), rtol=1e-15)
    assert st["nnz_a"] + g.n_rows == g.nnz()


def test_library_checksum_matches_reference_goldens():
    """aires_b200_checksum (host) == the reference's checksum of every golden C (serialize.hpp:50-59)."""
    g = np.load(os.path.join(ROOT, "tests", "golden", "spgemm.npz"))
    for c in range(int(g["n_cases"][0])):
        nr, ni, nc, macs, ck = (int(x) for x in g[f"c{c}_dims"])
        m = ab.CsrMatrix(nr, nc, g[f"c{c}_c_ptr"], g[f"c{c}_c_idx"], g[f"c{c}_c_val"])
        assert ab.checksum(m) == ck
        m32 = ab.CsrMatrix(nr, nc, g[f"c{c}_c_ptr"], g[f"c{c}_c_idx"].astype(np.uint32), g[f"c{c}_c_val"])
        assert ab.checksum(m32) == ck


def test_dropin_binaries_fail_loudly_without_a_device():
    """The reference's spgemm_test built on the drop-in headers aborts (no CPU fallback) when no
    CUDA device is visible."""
    import subprocess
    exe = os.path.join(ROOT, "oracle", "_ref", "dropin_spgemm_test")
    if not os.path.exists(exe) or ab.device_count() > 0:
        pytest.skip("drop-in binary absent or a device is visible")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode != 0 and "no CUDA device" in (r.stdout + r.stderr)


def test_synth_weights_is_reference_gen_weights():
    g = np.load(os.path.join(ROOT, "tests", "golden", "gcn.npz"))
    for c in range(int(g["n_comb"][0])):
        rows, cin, cout, seed = (int(x) for x in g[f"c{c}_dims"])
        assert np.array_equal(ab.gen_weights(cin, cout, seed).view(np.uint64), g[f"c{c}_w"].view(np.uint64))


def _host_segments(ptr, idx, val, n_rows, m_a, I, V):
    """robw_partition on the host for the CPU tier: the oracle's cuts + slice_rows (partition.hpp:33-74)."""
    from oracle import pyoracle as po
    rc, cuts, _ = po.robw_cuts(ptr, m_a, I, V)
    assert rc == 0
    segs = []
    for j in range(len(cuts) - 1):
        r0, r1 = int(cuts[j]), int(cuts[j + 1])
        b0, b1 = int(ptr[r0]), int(ptr[r1])
        segs.append(ab.RobwSegment(j, r0, r1, (np.asarray(ptr[r0:r1 + 1]) - b0).astype(np.uint64), idx[b0:b1],
                                   val[b0:b1], ab.calc_mem(r1 - r0, b1 - b0, ab.ElementSizes(I, V))))
    return segs


def test_segment_container_bytes_match_reference(tmp_path):
    """write_segments (serialize.hpp:148-174) restated: byte-identical to the reference's file at
    ElementSizes {8,8} and {4,4}."""
    g = np.load(os.path.join(ROOT, "tests", "golden", "segments.npz"))
    for c in range(int(g["n_cases"][0])):
        nr, nc, I, V, m_a = (int(x) for x in g[f"s{c}_args"])
        segs = _host_segments(g[f"s{c}_a_ptr"], g[f"s{c}_a_idx"], g[f"s{c}_a_val"], nr, m_a, I, V)
        path = str(tmp_path / f"s{c}.seg")
        ab.write_segments(path, segs, ab.ElementSizes(I, V))
        assert np.array_equal(np.fromfile(path, dtype=np.uint8), g[f"s{c}_bytes"])


def test_matrix_container_round_trip(tmp_path):
    """ARSM (serialize.hpp:102-142): write/read round trip, magic and version checks."""
    g = np.load(os.path.join(ROOT, "tests", "golden", "spgemm.npz"))
    a = ab.CsrMatrix(int(g["c0_dims"][0]), int(g["c0_dims"][1]), g["c0_a_ptr"], g["c0_a_idx"], g["c0_a_val"])
    p = str(tmp_path / "a.arsm")
    ab.write_matrix(p, a)
    assert ab.read_matrix(p) == a
    raw = np.fromfile(p, dtype=np.uint8)
    raw[0] = ord("X")
    raw.tofile(p)
    with pytest.raises(ab.AiresError) as e:
        ab.read_matrix(p)
    assert e.value.code == ab.errc.parse_error


def test_options_are_explicit_and_validated():
    # tuning options / test hooks go through aires_b200_set_option (no environment variables)
    ab.set_option("heavy_deg", 512)
    ab.clear_options()
    with ab.options(stream_tiles=4, wide_at=64):
        pass
    with pytest.raises(ab.AiresError) as e:
        ab.set_option("no_such_option", 1)
    assert e.value.status == 102  # AIRES_B200_INVALID_ARGUMENT
