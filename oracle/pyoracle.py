"""pyoracle -- ctypes bindings of the CPU oracle.  TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
may import this module.  It binds
  * oracle/liboracle.so          -- the plain-C restatement (aires_oracle.c), and
  * oracle/_ref/libaires_ref.so  -- the reference headers compiled as-is (when built),
and never touches the B200 library.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libaires_ref.so")


class AoCsr(C.Structure):
    _fields_ = [("n_rows", C.c_uint64), ("n_cols", C.c_uint64), ("nnz", C.c_uint64),
                ("ptr", C.POINTER(C.c_uint64)), ("idx", C.POINTER(C.c_uint64)),
                ("val", C.POINTER(C.c_double))]


U64P = C.POINTER(C.c_uint64)
F64P = C.POINTER(C.c_double)
_oracle = None
_ref = None


def oracle() -> C.CDLL:
    global _oracle
    if _oracle is None:
        if not os.path.exists(ORACLE_SO):
            raise RuntimeError(f"{ORACLE_SO} missing; run `make -C oracle oracle`")
        L = C.CDLL(ORACLE_SO)
        L.ao_spgemm_inner.argtypes = [U64P, U64P, F64P, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64,
                                      U64P, U64P, F64P, C.c_uint64, C.POINTER(AoCsr), U64P]
        L.ao_spgemm_rowwise.argtypes = [U64P, U64P, F64P, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64,
                                        U64P, U64P, F64P, C.c_int, C.POINTER(AoCsr), U64P]
        L.ao_csr_to_csc.argtypes = [C.c_uint64, C.c_uint64, U64P, U64P, F64P, C.POINTER(AoCsr)]
        L.ao_csc_to_csr.argtypes = [C.c_uint64, C.c_uint64, U64P, U64P, F64P, C.POINTER(AoCsr)]
        L.ao_calc_mem.restype = C.c_uint64
        L.ao_calc_mem.argtypes = [C.c_uint64] * 4
        L.ao_estimate_output_memory.restype = C.c_uint64
        L.ao_estimate_output_memory.argtypes = [C.c_uint64, C.c_double, C.c_uint64, C.c_double]
        L.ao_sparsity_percent.restype = C.c_double
        L.ao_sparsity_percent.argtypes = [C.c_uint64] * 3
        L.ao_block_budget.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, U64P, U64P]
        L.ao_robw_cuts.argtypes = [U64P, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, U64P, U64P, U64P]
        L.ao_fnv1a64.restype = C.c_uint64
        L.ao_fnv1a64.argtypes = [C.c_void_p, C.c_uint64]
        L.ao_checksum.restype = C.c_uint64
        L.ao_checksum.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, U64P, U64P, F64P]
        L.ao_gen_sparse.argtypes = [C.c_uint64, C.c_uint64, C.c_double, C.c_uint64, C.c_double, C.c_double,
                                    C.POINTER(AoCsr)]
        L.ao_gen_features.argtypes = [C.c_uint64, C.c_uint64, C.c_double, C.c_uint64, C.POINTER(AoCsr)]
        L.ao_normalize_adjacency.argtypes = [C.c_uint64, U64P, U64P, F64P, C.POINTER(AoCsr)]
        L.ao_free.argtypes = [C.POINTER(AoCsr)]
        L.ao_gen_weights.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, F64P]
        L.ao_combine.argtypes = [C.c_uint64, C.c_uint64, U64P, U64P, F64P, F64P, C.c_uint64, C.c_uint64,
                                 C.POINTER(AoCsr)]
        L.ao_synth_graph.argtypes = [C.c_uint64, C.c_uint64, C.c_double, C.c_uint64, C.c_uint64, C.c_uint64,
                                     C.c_int, C.c_int, C.c_int, C.POINTER(AoCsr), C.POINTER(C.c_double)]
        L.ao_rows_hash.restype = C.c_uint64
        L.ao_rows_hash.argtypes = [U64P, U64P, F64P, U64P, C.c_uint64]
        _oracle = L
    return _oracle


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref() -> C.CDLL:
    global _ref
    if _ref is None:
        if not ref_available():
            raise RuntimeError(f"{REF_SO} missing; run `make -C oracle ref` where /root/reference exists")
        L = C.CDLL(REF_SO)
        L.ref_spgemm_block.argtypes = [U64P, U64P, F64P, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64,
                                       C.c_uint64, U64P, U64P, F64P, C.c_uint64, C.c_uint64,
                                       C.POINTER(AoCsr), U64P]
        L.ref_csr_to_csc.argtypes = [C.c_uint64, C.c_uint64, U64P, U64P, F64P, C.POINTER(AoCsr)]
        L.ref_robw_cuts.argtypes = [U64P, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, U64P, U64P, U64P]
        L.ref_checksum.restype = C.c_uint64
        L.ref_checksum.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, U64P, U64P, F64P]
        L.ref_fnv1a64.restype = C.c_uint64
        L.ref_fnv1a64.argtypes = [C.c_void_p, C.c_uint64]
        L.ref_estimate_output_memory.restype = C.c_uint64
        L.ref_estimate_output_memory.argtypes = [C.c_uint64, C.c_double, C.c_uint64, C.c_double]
        L.ref_gen_features.argtypes = [C.c_uint64, C.c_uint64, C.c_double, C.c_uint64, C.POINTER(AoCsr)]
        L.ref_gen_sparse.argtypes = [C.c_uint64, C.c_uint64, C.c_double, C.c_uint64, C.c_double, C.c_double,
                                     C.POINTER(AoCsr)]
        L.ref_gen_symmetric.argtypes = [C.c_uint64, C.c_double, C.c_uint64, C.POINTER(AoCsr)]
        L.ref_normalize_adjacency.argtypes = [C.c_uint64, U64P, U64P, F64P, C.POINTER(AoCsr)]
        L.ref_run_aires.argtypes = [C.c_uint64, C.c_uint64, U64P, U64P, F64P, C.c_uint64, C.c_uint64, U64P, U64P,
                                    F64P, C.c_uint64, C.c_uint64, C.c_uint64, C.POINTER(AoCsr), U64P, F64P]
        L.ref_spgemm_rows_timed.restype = C.c_double
        L.ref_spgemm_rows_timed.argtypes = [U64P, U64P, F64P, C.c_uint64, C.c_uint64, U64P, C.c_uint64,
                                            C.c_uint64, C.c_uint64, U64P, U64P, F64P, C.c_int, U64P, U64P, U64P]
        L.ref_free.argtypes = [C.POINTER(AoCsr)]
        L.ref_write_segments.argtypes = [C.c_char_p, C.c_uint64, C.c_uint64, U64P, U64P, F64P, C.c_uint64, C.c_uint64,
                                         C.c_uint64]
        L.ref_gen_weights.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, F64P]
        L.ref_combine.argtypes = [C.c_uint64, C.c_uint64, U64P, U64P, F64P, F64P, C.c_uint64, C.c_uint64,
                                  C.POINTER(AoCsr)]
        _ref = L
    return _ref


# ---------------------------------------------------------------------------
def _u64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.uint64)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _p64(a: np.ndarray):
    return a.ctypes.data_as(U64P)


def _pf(a: np.ndarray):
    return a.ctypes.data_as(F64P)


def _take(m: AoCsr, nptr: int, free) -> tuple:
    ptr = np.ctypeslib.as_array(m.ptr, shape=(nptr,)).copy() if nptr else np.zeros(0, np.uint64)
    if m.nnz:
        idx = np.ctypeslib.as_array(m.idx, shape=(m.nnz,)).copy()
        val = np.ctypeslib.as_array(m.val, shape=(m.nnz,)).copy()
    else:
        idx = np.zeros(0, np.uint64)
        val = np.zeros(0, np.float64)
    free(C.byref(m))
    return ptr, idx, val


def spgemm_inner(row_ptr, col_idx, values, rows, a_n_cols, b_n_rows, b_n_cols, b_col_ptr, b_row_idx, b_values,
                 tile_cols=256, use_ref=False):
    """spgemm.hpp:60-132 (inner product).  Returns (rc, (ptr, idx, val), macs)."""
    rp, ci, va = _u64(row_ptr), _u64(col_idx), _f64(values)
    cp, ri, bv = _u64(b_col_ptr), _u64(b_row_idx), _f64(b_values)
    m, macs = AoCsr(), C.c_uint64()
    if use_ref:
        L = ref()
        rc = L.ref_spgemm_block(_p64(rp), _p64(ci), _pf(va), ci.shape[0], rows, a_n_cols, b_n_rows, b_n_cols,
                                _p64(cp), _p64(ri), _pf(bv), 0, tile_cols, C.byref(m), C.byref(macs))
        free = L.ref_free
    else:
        L = oracle()
        rc = L.ao_spgemm_inner(_p64(rp), _p64(ci), _pf(va), rows, a_n_cols, b_n_rows, b_n_cols, _p64(cp),
                               _p64(ri), _pf(bv), tile_cols, C.byref(m), C.byref(macs))
        free = L.ao_free
    if rc:
        return rc, None, 0
    return 0, _take(m, rows + 1, free), macs.value


def spgemm_rowwise(row_ptr, col_idx, values, rows, a_n_cols, b_n_rows, b_n_cols, b_row_ptr, b_col_idx, b_values,
                   nthreads=1):
    """Same bits as spgemm_inner, from X in CSR.  Returns (rc, (ptr, idx, val), macs)."""
    L = oracle()
    rp, ci, va = _u64(row_ptr), _u64(col_idx), _f64(values)
    bp, bc, bv = _u64(b_row_ptr), _u64(b_col_idx), _f64(b_values)
    m, macs = AoCsr(), C.c_uint64()
    rc = L.ao_spgemm_rowwise(_p64(rp), _p64(ci), _pf(va), rows, a_n_cols, b_n_rows, b_n_cols, _p64(bp), _p64(bc),
                             _pf(bv), nthreads, C.byref(m), C.byref(macs))
    if rc:
        return rc, None, 0
    return 0, _take(m, rows + 1, L.ao_free), macs.value


def csr_to_csc(n_rows, n_cols, row_ptr, col_idx, values, use_ref=False):
    rp, ci, va = _u64(row_ptr), _u64(col_idx), _f64(values)
    m = AoCsr()
    if use_ref:
        L = ref()
        L.ref_csr_to_csc(n_rows, n_cols, _p64(rp), _p64(ci), _pf(va), C.byref(m))
        return _take(m, n_cols + 1, L.ref_free)
    L = oracle()
    L.ao_csr_to_csc(n_rows, n_cols, _p64(rp), _p64(ci), _pf(va), C.byref(m))
    return _take(m, n_cols + 1, L.ao_free)


def csc_to_csr(n_rows, n_cols, col_ptr, row_idx, values):
    L = oracle()
    cp, ri, va = _u64(col_ptr), _u64(row_idx), _f64(values)
    m = AoCsr()
    L.ao_csc_to_csr(n_rows, n_cols, _p64(cp), _p64(ri), _pf(va), C.byref(m))
    return _take(m, n_rows + 1, L.ao_free)


def robw_cuts(row_ptr, m_a, I=8, V=8, use_ref=False):
    """partition.hpp:52-74.  Returns (rc, cuts, bad_row)."""
    rp = _u64(row_ptr)
    n = rp.shape[0] - 1
    cuts = np.zeros(n + 1, dtype=np.uint64)
    ns, bad = C.c_uint64(), C.c_uint64()
    if use_ref:
        rc = ref().ref_robw_cuts(_p64(rp), n, m_a, I, V, _p64(cuts), C.byref(ns), None)
    else:
        rc = oracle().ao_robw_cuts(_p64(rp), n, m_a, I, V, _p64(cuts), C.byref(ns), C.byref(bad))
    return rc, cuts[: ns.value + 1].copy(), bad.value


def checksum(n_rows, n_cols, row_ptr, col_idx, values, use_ref=False) -> int:
    rp, ci, va = _u64(row_ptr), _u64(col_idx), _f64(values)
    L = ref() if use_ref else oracle()
    f = L.ref_checksum if use_ref else L.ao_checksum
    return int(f(n_rows, n_cols, ci.shape[0], _p64(rp), _p64(ci), _pf(va)))


def fnv1a64(data: bytes, use_ref=False) -> int:
    buf = C.create_string_buffer(data, len(data))
    L = ref() if use_ref else oracle()
    return int((L.ref_fnv1a64 if use_ref else L.ao_fnv1a64)(buf, len(data)))


def gen_features(n, dim, sparsity, seed, use_ref=False):
    m = AoCsr()
    if use_ref:
        L = ref()
        rc = L.ref_gen_features(n, dim, sparsity, seed, C.byref(m))
        return rc, (_take(m, n + 1, L.ref_free) if rc == 0 else None)
    L = oracle()
    rc = L.ao_gen_features(n, dim, sparsity, seed, C.byref(m))
    return rc, (_take(m, n + 1, L.ao_free) if rc == 0 else None)


def gen_sparse(rows, cols, density, seed, lo=0.0, hi=1.0, use_ref=False):
    m = AoCsr()
    L = ref() if use_ref else oracle()
    f = L.ref_gen_sparse if use_ref else L.ao_gen_sparse
    rc = f(rows, cols, density, seed, lo, hi, C.byref(m))
    return rc, (_take(m, rows + 1, L.ref_free if use_ref else L.ao_free) if rc == 0 else None)


def gen_symmetric(n, density, seed):
    L = ref()
    m = AoCsr()
    rc = L.ref_gen_symmetric(n, density, seed, C.byref(m))
    return rc, (_take(m, n + 1, L.ref_free) if rc == 0 else None)


def normalize_adjacency(n, row_ptr, col_idx, values, use_ref=False):
    rp, ci, va = _u64(row_ptr), _u64(col_idx), _f64(values)
    m = AoCsr()
    L = ref() if use_ref else oracle()
    f = L.ref_normalize_adjacency if use_ref else L.ao_normalize_adjacency
    rc = f(n, _p64(rp), _p64(ci), _pf(va), C.byref(m))
    return rc, (_take(m, n + 1, L.ref_free if use_ref else L.ao_free) if rc == 0 else None)


def calc_mem(k, q, I=8, V=8) -> int:
    return int(oracle().ao_calc_mem(k, q, I, V))


def estimate_output_memory(aa, sa, ab, sb, use_ref=False) -> int:
    L = ref() if use_ref else oracle()
    return int((L.ref_estimate_output_memory if use_ref else L.ao_estimate_output_memory)(aa, sa, ab, sb))


def block_budget(device_total, m_c, m_b):
    p, m_a = C.c_uint64(), C.c_uint64()
    rc = oracle().ao_block_budget(device_total, m_c, m_b, C.byref(p), C.byref(m_a))
    return rc, p.value, m_a.value


def ref_run_aires(a_ptr, a_idx, a_val, n_rows, n_cols, b_colptr, b_rowidx, b_val, b_n_rows, b_n_cols,
                  device_total, I=8, V=8):
    """scheduler.hpp:72-168 verbatim; returns (rc, (ptr, idx, val), report dict)."""
    L = ref()
    rp, ci, va = _u64(a_ptr), _u64(a_idx), _f64(a_val)
    cp, ri, bv = _u64(b_colptr), _u64(b_rowidx), _f64(b_val)
    m = AoCsr()
    rep = np.zeros(12, dtype=np.uint64)
    secs = np.zeros(4, dtype=np.float64)
    rc = L.ref_run_aires(n_rows, n_cols, _p64(rp), _p64(ci), _pf(va), b_n_rows, b_n_cols, _p64(cp), _p64(ri),
                         _pf(bv), device_total, I, V, C.byref(m), _p64(rep), _pf(secs))
    if rc:
        return rc, None, None
    keys = ["segments", "gds_count", "gds_bytes", "s2h_count", "s2h_bytes", "h2d_count", "h2d_bytes",
            "d2h_count", "d2h_bytes", "merge_bytes", "peak_device_occupancy", "c_checksum"]
    report = {k: int(v) for k, v in zip(keys, rep)}
    report.update(phase1_s=secs[0], phase2_s=secs[1], phase3_s=secs[2], total_s=secs[3])
    return 0, _take(m, n_rows + 1, L.ref_free), report


def ref_rows_timed(row_ptr, col_idx, values, a_n_cols, rows, b_col_ptr, b_row_idx, b_values, b_n_rows, b_n_cols,
                   nthreads):
    """Reference spgemm_block over a row sample on nthreads host threads: (seconds, macs, c_nnz, hash)."""
    L = ref()
    rp, ci, va = _u64(row_ptr), _u64(col_idx), _f64(values)
    rs = _u64(rows)
    cp, ri, bv = _u64(b_col_ptr), _u64(b_row_idx), _f64(b_values)
    macs, z, h = C.c_uint64(), C.c_uint64(), C.c_uint64()
    s = L.ref_spgemm_rows_timed(_p64(rp), _p64(ci), _pf(va), ci.shape[0], a_n_cols, _p64(rs), rs.shape[0],
                                b_n_rows, b_n_cols, _p64(cp), _p64(ri), _pf(bv), nthreads, C.byref(macs),
                                C.byref(z), C.byref(h))
    return s, macs.value, z.value, h.value


def gen_weights(in_dim, out_dim, seed, use_ref=False) -> np.ndarray:
    """synth.hpp:81-86"""
    w = np.empty((in_dim, out_dim), dtype=np.float64)
    (ref().ref_gen_weights if use_ref else oracle().ao_gen_weights)(in_dim, out_dim, seed, _pf(w))
    return w


def combine(rows, x_cols, row_ptr, col_idx, values, w, use_ref=False):
    """gcn.hpp:90-116.  Returns (rc, (ptr, idx, val))."""
    rp = _u64(np.asarray(row_ptr, dtype=np.uint64) - np.uint64(np.asarray(row_ptr)[0]))
    ci, va = _u64(col_idx), _f64(values)
    wd = _f64(w)
    m = AoCsr()
    L = ref() if use_ref else oracle()
    f = L.ref_combine if use_ref else L.ao_combine
    p0 = int(np.asarray(row_ptr)[0])
    ci, va = _u64(ci[p0:]), _f64(va[p0:])
    rc = f(rows, x_cols, _p64(rp), _p64(ci), _pf(va), _pf(wd), wd.shape[0], wd.shape[1], C.byref(m))
    if rc:
        return rc, None
    return 0, _take(m, rows + 1, L.ref_free if use_ref else L.ao_free)


def ref_write_segments(path, n_rows, n_cols, row_ptr, col_idx, values, m_a, I=8, V=8) -> int:
    """The reference's robw_partition + write_segments to `path` (serialize.hpp:148-174)."""
    rp, ci, va = _u64(row_ptr), _u64(col_idx), _f64(values)
    return int(ref().ref_write_segments(path.encode(), n_rows, n_cols, _p64(rp), _p64(ci), _pf(va), m_a, I, V))


def synth_graph(n, target_nnz, alpha=0.75, degree_cap=20000, seed=1, relabel_seed=2, relabel=True, normalize=True,
                threads=0):
    """Restatement of the B200 library's Chung-Lu generator (reference-arm inputs, no libaires_b200.so).
    Returns ((ptr, idx, val) at u64/u64/f64, stats dict) -- the same arrays and stats keys as
    paper_2507_02006_b200.synth_graph."""
    L = oracle()
    m = AoCsr()
    st = (C.c_double * 8)()
    th = threads if threads > 0 else len(os.sched_getaffinity(0))
    rc = L.ao_synth_graph(n, target_nnz, alpha, degree_cap, seed, relabel_seed, int(relabel), int(normalize), th,
                          C.byref(m), st)
    if rc:
        raise RuntimeError(f"ao_synth_graph failed ({rc})")
    arrs = _take(m, n + 1, L.ao_free)
    stats = dict(nnz_a=int(st[0]), max_degree=int(st[1]), mean_degree=st[2], rounds=int(st[3]), i0=st[5])
    return arrs, stats


def rows_hash(row_ptr, col_idx, values, rows) -> int:
    """Sum of per-row FNV-1a 64 over `rows` (matches ref_rows_timed's hash for the same rows)."""
    rp, ci, va, rs = _u64(row_ptr), _u64(col_idx), _f64(values), _u64(rows)
    return int(oracle().ao_rows_hash(_p64(rp), _p64(ci), _pf(va), _p64(rs), rs.shape[0]))
