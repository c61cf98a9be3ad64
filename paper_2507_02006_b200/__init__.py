"""paper_2507_02006_b200 -- B200-native AIRES out-of-core A·X SpGEMM (arXiv 2507.02006).

Python mirror of the reference's operator API for the hot path (namespace ``aires``,
/root/reference/proj/include/aires/): ``CsrMatrix``/``CscMatrix`` (sparse.hpp:29-52),
``spgemm_block`` (spgemm.hpp:60-139), ``spgemm_full`` (spgemm.hpp:142-151),
``robw_partition`` (partition.hpp:52-74) and ``run_aires``-style out-of-core runs
(scheduler.hpp:72-168), all backed by the C ABI of ``include/aires_b200.h``
(``libaires_b200.so``, hand-written sm_100a kernels).  Errors are raised as
``AiresError`` carrying the reference's ``errc`` code (error.hpp:9-27).

There is no CPU fallback: if the CUDA library is missing or no device is visible,
every compute call raises.
"""
from __future__ import annotations

import contextlib
import ctypes as C
import dataclasses
import enum
import os
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("AB2_LIB") or os.path.join(_HERE, "libaires_b200.so")


class errc(enum.IntEnum):
    """aires::errc (error.hpp:9-27); the C ABI returns 1 + errc."""

    index_out_of_range = 0
    parse_error = 1
    unsupported_format = 2
    dense_too_large = 3
    insufficient_device_memory = 4
    row_too_large = 5
    non_adjacent_fragments = 6
    dimension_mismatch = 7
    capacity_exceeded = 8
    buffer_not_resident = 9
    operand_not_on_device = 10
    same_channel_conflict = 11
    invalid_density = 12
    non_square = 13
    negative_weight = 14
    io_error = 15
    config_error = 16


class AiresError(RuntimeError):
    """aires::error (error.hpp:53-62): what() is "<errc name>: <detail>"."""

    def __init__(self, status: int, detail: str):
        self.status = status
        self.code: Optional[errc] = errc(status - 1) if 1 <= status <= 17 else None
        name = self.code.name if self.code is not None else f"b200_status_{status}"
        super().__init__(f"{name}: {detail}")


HOST, DEVICE = 0, 1
CSR, CSC = 0, 1
MODE_AUTO, MODE_FP32, MODE_FP64_EXACT = 0, 1, 2


class _Matrix(C.Structure):
    _fields_ = [
        ("n_rows", C.c_uint64), ("n_cols", C.c_uint64), ("layout", C.c_uint32),
        ("location", C.c_uint32), ("idx_bytes", C.c_uint32), ("val_bytes", C.c_uint32),
        ("ptr", C.c_void_p), ("idx", C.c_void_p), ("val", C.c_void_p), ("span", C.c_uint64),
    ]


_ALLOC_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_uint64, C.c_uint64, C.POINTER(C.c_void_p),
                        C.POINTER(C.c_void_p), C.POINTER(C.c_void_p))


class _Output(C.Structure):
    _fields_ = [
        ("location", C.c_uint32), ("idx_bytes", C.c_uint32), ("val_bytes", C.c_uint32),
        ("reserved", C.c_uint32), ("alloc", _ALLOC_FN), ("user", C.c_void_p),
        ("n_rows", C.c_uint64), ("n_cols", C.c_uint64), ("nnz", C.c_uint64), ("flops", C.c_uint64),
    ]


ABI_VERSION = 2  # AIRES_B200_ABI_VERSION of include/aires_b200.h


class _TraceEvent(C.Structure):
    _fields_ = [("timestamp_ms", C.c_double), ("duration_ms", C.c_double), ("kind", C.c_uint32),
                ("phase", C.c_uint32), ("where", C.c_uint32), ("buffer", C.c_uint32), ("index", C.c_uint64),
                ("bytes", C.c_uint64), ("flops", C.c_uint64)]


_TRACE_FN = C.CFUNCTYPE(None, C.c_void_p, C.POINTER(_TraceEvent), C.c_uint64)


class _RunConfig(C.Structure):
    _fields_ = [("device_budget", C.c_uint64), ("mode", C.c_uint32), ("c_aware", C.c_uint32),
                ("n_buffers", C.c_uint32), ("flags", C.c_uint32), ("trace", _TRACE_FN), ("trace_user", C.c_void_p)]


class _RunReport(C.Structure):
    _fields_ = [("segments", C.c_uint64), ("h2d_bytes", C.c_uint64), ("d2h_bytes", C.c_uint64),
                ("flops", C.c_uint64), ("c_nnz", C.c_uint64), ("peak_device_bytes", C.c_uint64),
                ("total_ms", C.c_double), ("phase1_ms", C.c_double), ("phase2_ms", C.c_double),
                ("phase3_ms", C.c_double), ("merge_bytes", C.c_uint64), ("h2d_count", C.c_uint64),
                ("d2h_count", C.c_uint64), ("h2d_ms", C.c_double), ("d2h_ms", C.c_double), ("merge_ms", C.c_double)]


_SEG_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, C.POINTER(C.c_uint64),
                      C.c_void_p, C.c_void_p, C.c_uint64)


class _StorageReport(C.Structure):
    _fields_ = [("segments", C.c_uint64), ("bytes_read", C.c_uint64), ("flops", C.c_uint64), ("c_nnz", C.c_uint64),
                ("used_gds", C.c_uint32), ("reserved", C.c_uint32), ("read_ms", C.c_double), ("total_ms", C.c_double)]


class _GraphSpec(C.Structure):
    _fields_ = [("n", C.c_uint64), ("target_nnz", C.c_uint64), ("alpha", C.c_double),
                ("degree_cap", C.c_uint64), ("seed", C.c_uint64), ("relabel_seed", C.c_uint64),
                ("relabel", C.c_int32), ("normalize", C.c_int32), ("threads", C.c_int32),
                ("reserved", C.c_int32)]


_lib = None


def lib() -> C.CDLL:
    """Loads libaires_b200.so; raises (never falls back) if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the B200 path has no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    P = C.POINTER
    L.aires_b200_abi_version.restype = C.c_int
    if L.aires_b200_abi_version() != ABI_VERSION:
        raise RuntimeError(f"{LIB_PATH} has ABI {L.aires_b200_abi_version()}, the bindings expect {ABI_VERSION}: rebuild")
    L.aires_b200_last_error.restype = C.c_char_p
    L.aires_b200_set_option.argtypes = [C.c_char_p, C.c_int64]
    L.aires_b200_device_count.argtypes = [P(C.c_int)]
    L.aires_b200_set_device.argtypes = [C.c_int]
    L.aires_b200_spgemm.argtypes = [P(_Matrix), P(_Matrix), C.c_uint32, P(_Output)]
    L.aires_b200_operand_create.argtypes = [P(_Matrix), C.c_uint32, P(C.c_void_p)]
    L.aires_b200_operand_destroy.argtypes = [C.c_void_p]
    L.aires_b200_operand_info.argtypes = [C.c_void_p, P(C.c_uint64), P(C.c_uint64), P(C.c_uint64),
                                          P(C.c_uint32), P(C.c_uint64)]
    L.aires_b200_spgemm_op.argtypes = [P(_Matrix), C.c_void_p, P(_Output)]
    L.aires_b200_robw_cuts.argtypes = [P(C.c_uint64), C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64,
                                       C.c_uint32, P(C.c_uint64), C.c_uint64, P(C.c_uint64),
                                       P(C.c_uint64)]
    L.aires_b200_run.argtypes = [P(_Matrix), P(_Matrix), P(_RunConfig), P(_Output), P(_RunReport)]
    L.aires_b200_last_kernel_ms.restype = C.c_double
    L.aires_b200_stream.restype = C.c_void_p
    L.aires_b200_last_launches.restype = C.c_int
    L.aires_b200_last_profile.argtypes = [P(C.c_double), C.c_int]
    L.aires_b200_synth_graph.argtypes = [P(_GraphSpec), P(_Output), P(C.c_double)]
    L.aires_b200_synth_features.argtypes = [C.c_uint64, C.c_uint64, C.c_double, C.c_uint64, P(_Output)]
    L.aires_b200_synth_last_error.restype = C.c_char_p
    L.aires_b200_normalize_adjacency.argtypes = [P(_Matrix), P(_Output)]
    L.aires_b200_combine.argtypes = [P(_Matrix), C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint32, P(_Output)]
    L.aires_b200_layer_fused.argtypes = [P(_Matrix), P(_Matrix), C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint32,
                                         P(_Output)]
    L.aires_b200_spgemm_segments.argtypes = [C.c_char_p, C.c_uint32, C.c_uint32, C.c_uint64, P(_Matrix), C.c_uint32,
                                             _SEG_FN, C.c_void_p, P(_StorageReport)]
    L.aires_b200_synth_weights.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, P(C.c_double)]
    L.aires_b200_checksum.restype = C.c_uint64
    L.aires_b200_checksum.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, P(C.c_uint64), C.c_void_p, C.c_uint32,
                                      C.c_void_p, C.c_uint32]
    _lib = L
    return L


def _check(rc: int, synth: bool = False) -> None:
    if rc != 0:
        L = lib()
        msg = (L.aires_b200_synth_last_error() if synth else L.aires_b200_last_error()) or b""
        raise AiresError(rc, msg.decode(errors="replace"))


# ---------------------------------------------------------------------------
# containers (sparse.hpp:29-52), numpy-backed at API widths by default
# ---------------------------------------------------------------------------

@dataclasses.dataclass
class CsrMatrix:
    n_rows: int
    n_cols: int
    row_ptr: np.ndarray  # uint64, n_rows+1
    col_idx: np.ndarray  # uint64 (or uint32)
    values: np.ndarray   # float64 (or float32)

    def nnz(self) -> int:
        return int(self.col_idx.shape[0])

    def __eq__(self, o) -> bool:  # operator== (sparse.hpp:38): bit equality of every array
        return (self.n_rows == o.n_rows and self.n_cols == o.n_cols
                and np.array_equal(self.row_ptr.astype(np.uint64), o.row_ptr.astype(np.uint64))
                and np.array_equal(self.col_idx.astype(np.uint64), o.col_idx.astype(np.uint64))
                and self.values.dtype == o.values.dtype
                and np.array_equal(self.values.view(np.uint8), o.values.view(np.uint8)))


@dataclasses.dataclass
class CscMatrix:
    n_rows: int
    n_cols: int
    col_ptr: np.ndarray
    row_idx: np.ndarray
    values: np.ndarray

    def nnz(self) -> int:
        return int(self.row_idx.shape[0])


@dataclasses.dataclass
class CsrBlockResult:
    """spgemm.hpp:47-52"""
    start_row: int
    end_row: int
    fragment: CsrMatrix
    flops: int


@dataclasses.dataclass
class ElementSizes:
    """sparse.hpp:21-24"""
    index_bytes: int = 8
    value_bytes: int = 8


def _np_view(arr: np.ndarray) -> int:
    return arr.ctypes.data if arr.size else 0


def _matrix_from_np(n_rows, n_cols, layout, ptr, idx, val) -> tuple:
    ptr = np.ascontiguousarray(ptr, dtype=np.uint64)
    idx = np.ascontiguousarray(idx)
    val = np.ascontiguousarray(val)
    if idx.dtype not in (np.uint32, np.uint64, np.int32, np.int64):
        idx = idx.astype(np.uint64)
    if val.dtype not in (np.float32, np.float64):
        val = val.astype(np.float64)
    m = _Matrix(n_rows, n_cols, layout, HOST, idx.dtype.itemsize, val.dtype.itemsize,
                _np_view(ptr), _np_view(idx), _np_view(val), idx.shape[0])
    return m, (ptr, idx, val)


class _HostAlloc:
    """Output allocator handing out numpy arrays (the exact allocation, spgemm.hpp:111-112)."""

    def __init__(self, idx_dtype, val_dtype):
        self.idx_dtype, self.val_dtype = idx_dtype, val_dtype
        self.ptr = self.idx = self.val = None
        self.fn = _ALLOC_FN(self._alloc)

    def _alloc(self, user, n_rows, nnz, pptr, pidx, pval):
        try:
            self.ptr = np.zeros(n_rows + 1, dtype=np.uint64)
            self.idx = np.empty(max(nnz, 1), dtype=self.idx_dtype)
            self.val = np.empty(max(nnz, 1), dtype=self.val_dtype)
            self.nnz = nnz
            pptr[0] = self.ptr.ctypes.data
            pidx[0] = self.idx.ctypes.data
            pval[0] = self.val.ctypes.data
            return 0
        except MemoryError:
            return 9  # 1 + capacity_exceeded

    def output(self, location=HOST) -> _Output:
        return _Output(location, np.dtype(self.idx_dtype).itemsize, np.dtype(self.val_dtype).itemsize, 0,
                       self.fn, None, 0, 0, 0, 0)


def _mode_for(values: np.ndarray, mode: int) -> int:
    if mode != MODE_AUTO:
        return mode
    return MODE_FP64_EXACT if values.dtype == np.float64 else MODE_FP32


def spgemm_rows(row_ptr, col_idx, values, rows: int, a_n_cols: int, b, mode: int = MODE_AUTO,
                idx_dtype=None) -> tuple:
    """Raw-span product (spgemm.hpp:60-132).  ``b`` is a CscMatrix, CsrMatrix or Operand.
    Returns (CsrMatrix fragment with rebased row_ptr, flops)."""
    L = lib()
    a, keep_a = _matrix_from_np(rows, a_n_cols, CSR, row_ptr, col_idx, values)
    mode = _mode_for(keep_a[2], mode)
    vdt = np.float64 if mode == MODE_FP64_EXACT else np.float32
    al = _HostAlloc(idx_dtype or keep_a[1].dtype, vdt)
    out = al.output()
    if isinstance(b, Operand):
        _check(L.aires_b200_spgemm_op(C.byref(a), b.handle, C.byref(out)))
        bcols = b.n_cols
    else:
        bm, keep_b = _operand_matrix(b)
        _check(L.aires_b200_spgemm(C.byref(a), C.byref(bm), mode, C.byref(out)))
        bcols = b.n_cols
    frag = CsrMatrix(rows, bcols, al.ptr, al.idx[: out.nnz], al.val[: out.nnz])
    return frag, int(out.flops)


def _operand_matrix(b):
    if isinstance(b, CscMatrix):
        return _matrix_from_np(b.n_rows, b.n_cols, CSC, b.col_ptr, b.row_idx, b.values)
    if isinstance(b, CsrMatrix):
        return _matrix_from_np(b.n_rows, b.n_cols, CSR, b.row_ptr, b.col_idx, b.values)
    raise TypeError("operand must be CsrMatrix or CscMatrix")


def spgemm_block(row_ptr, col_idx, values, rows: int, a_n_cols: int, b, start_row: int = 0,
                 tile_cols: int = 256, mode: int = MODE_AUTO) -> CsrBlockResult:
    """spgemm.hpp:60-132 (tile_cols only changes traversal order in the reference; the
    B200 kernels have no column tiling, results are identical by construction)."""
    del tile_cols
    frag, flops = spgemm_rows(row_ptr, col_idx, values, rows, a_n_cols, b, mode)
    return CsrBlockResult(start_row, start_row + rows, frag, flops)


def spgemm_full(a: CsrMatrix, b, tile_cols: int = 256, mode: int = MODE_AUTO) -> CsrMatrix:
    """spgemm.hpp:142-151: one block spanning every row; b is CSC or CSR."""
    return spgemm_block(a.row_ptr, a.col_idx, a.values, a.n_rows, a.n_cols, b, 0, tile_cols, mode).fragment


class Operand:
    """A resident right operand (the device-resident B of run_aires Phase I)."""

    def __init__(self, b, mode: int = MODE_AUTO):
        L = lib()
        bm, self._keep = _operand_matrix(b)
        self.n_rows, self.n_cols = b.n_rows, b.n_cols
        h = C.c_void_p()
        _check(L.aires_b200_operand_create(C.byref(bm), _mode_for(self._keep[2], mode), C.byref(h)))
        self.handle = h
        self._keep = None

    def info(self) -> dict:
        L = lib()
        r, c, z, b = C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_uint64()
        m = C.c_uint32()
        _check(L.aires_b200_operand_info(self.handle, C.byref(r), C.byref(c), C.byref(z), C.byref(m), C.byref(b)))
        return dict(n_rows=r.value, n_cols=c.value, nnz=z.value, mode=m.value, device_bytes=b.value)

    def close(self):
        if getattr(self, "handle", None):
            lib().aires_b200_operand_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def robw_cuts(row_ptr: np.ndarray, m_a: int, sizes: ElementSizes = ElementSizes()) -> np.ndarray:
    """Device RoBW cut search (partition.hpp:52-74); returns the n_segs+1 boundaries."""
    L = lib()
    rp = np.ascontiguousarray(row_ptr, dtype=np.uint64)
    n = rp.shape[0] - 1
    cuts = np.zeros(n + 1, dtype=np.uint64)
    ns, bad = C.c_uint64(), C.c_uint64()
    P = C.POINTER(C.c_uint64)
    rc = L.aires_b200_robw_cuts(rp.ctypes.data_as(P), n, m_a, sizes.index_bytes, sizes.value_bytes, HOST,
                                cuts.ctypes.data_as(P), cuts.shape[0], C.byref(ns), C.byref(bad))
    if rc == 6:
        raise AiresError(rc, f"row {bad.value} needs more than the block budget {m_a}")
    _check(rc)
    return cuts[: ns.value + 1].copy()


@dataclasses.dataclass
class RobwSegment:
    """partition.hpp:20-31"""
    seg_index: int
    start_row: int
    end_row: int
    row_ptr_local: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray
    byte_size: int

    def rows(self) -> int:
        return self.end_row - self.start_row

    def nnz(self) -> int:
        return int(self.col_idx.shape[0])


def calc_mem(k: int, q: int, s: ElementSizes = ElementSizes()) -> int:
    """memory_model.hpp:84-86"""
    return (k + 1) * s.index_bytes + q * (s.index_bytes + s.value_bytes)


def robw_partition(a: CsrMatrix, m_a: int, s: ElementSizes = ElementSizes()) -> list:
    """partition.hpp:52-74: cuts from the device tiler, segments sliced like slice_rows (:33-47)."""
    cuts = robw_cuts(a.row_ptr, m_a, s)
    segs = []
    for i in range(len(cuts) - 1):
        r0, r1 = int(cuts[i]), int(cuts[i + 1])
        base = int(a.row_ptr[r0])
        end = int(a.row_ptr[r1])
        local = (a.row_ptr[r0:r1 + 1] - np.uint64(base)).astype(np.uint64)
        segs.append(RobwSegment(i, r0, r1, local, a.col_idx[base:end].copy(), a.values[base:end].copy(),
                                calc_mem(r1 - r0, end - base, s)))
    return segs


def checksum(c: CsrMatrix) -> int:
    """aires::checksum (serialize.hpp:50-59): FNV-1a 64 of the canonical CSR byte stream."""
    rp = np.ascontiguousarray(c.row_ptr, dtype=np.uint64)
    idx = np.ascontiguousarray(c.col_idx)
    val = np.ascontiguousarray(c.values)
    return int(lib().aires_b200_checksum(c.n_rows, c.n_cols, idx.shape[0], rp.ctypes.data_as(C.POINTER(C.c_uint64)),
                                         _np_view(idx), idx.dtype.itemsize, _np_view(val), val.dtype.itemsize))


# ---------------------------------------------------------------------------
# out-of-core run (scheduler.hpp:25-43, 72-168)
# ---------------------------------------------------------------------------

@dataclasses.dataclass
class MemoryBudget:
    """memory_model.hpp:26-30"""
    device_total: int = 0
    host_total: int = 0
    element_sizes: ElementSizes = dataclasses.field(default_factory=ElementSizes)


@dataclasses.dataclass
class ChannelTotals:
    """tiered_sim.hpp:70-76 (count, bytes, seconds) -- here real copies and CUDA-event time."""
    count: int = 0
    bytes: int = 0
    seconds: float = 0.0


@dataclasses.dataclass
class IoLedger:
    """tiered_sim.hpp:78-98.  gds/s2h stay zero: operands arrive in host memory through the API."""
    gds: ChannelTotals = dataclasses.field(default_factory=ChannelTotals)
    s2h: ChannelTotals = dataclasses.field(default_factory=ChannelTotals)
    h2d: ChannelTotals = dataclasses.field(default_factory=ChannelTotals)
    d2h: ChannelTotals = dataclasses.field(default_factory=ChannelTotals)
    merge_bytes: int = 0
    peak_device_occupancy: int = 0

    def host_device_bytes(self) -> int:
        return self.h2d.bytes + self.d2h.bytes


@dataclasses.dataclass
class RunReport:
    """scheduler.hpp:25-37; times are measured (CUDA events), not simulated."""
    strategy: str = "aires"
    budget_bytes: int = 0
    total_s: float = 0.0
    phase1_s: float = 0.0
    phase2_s: float = 0.0
    phase3_s: float = 0.0
    ledger: IoLedger = dataclasses.field(default_factory=IoLedger)
    c_checksum: int = 0
    segments: int = 0
    oom: bool = False
    merge_seconds: float = 0.0
    flops: int = 0


@dataclasses.dataclass
class RunResult:
    """scheduler.hpp:39-43; trace = the measured TraceEvents of the run (CUDA-event clocks)."""
    c: CsrMatrix
    report: RunReport
    trace: list


@dataclasses.dataclass
class TraceEvent:
    """tiered_sim.hpp:60-68 with device clocks: timestamp = completion (s after the run's first
    event); kind transfer/compute/alloc/free; phase I/II/III; where = channel or tier name."""
    timestamp: float
    kind: str
    phase: str
    where: str
    buffer: str
    bytes: int
    flops: int
    duration: float = 0.0


_EV_KIND = ("transfer", "compute", "alloc", "free")
_EV_PHASE = ("I", "II", "III")
_EV_CH = ("gds", "s2h", "h2d", "d2h")
_EV_TIER = ("device", "host", "storage")


def _buffer_name(buf: int, index: int) -> str:
    return ("B", f"a_tile_{index}", "C", f"frag_{index}", "A")[buf]


def _trace_events(evs) -> list:
    return [TraceEvent(e.timestamp_ms / 1e3, _EV_KIND[e.kind], _EV_PHASE[e.phase],
                       _EV_CH[e.where] if e.kind == 0 else _EV_TIER[e.where], _buffer_name(e.buffer, e.index),
                       int(e.bytes), int(e.flops), e.duration_ms / 1e3) for e in evs]


def run_maxmemory(a: CsrMatrix, b, budget: MemoryBudget, cfg=None, mode: int = MODE_AUTO, n_buffers: int = 2,
                  with_checksum: bool = True) -> RunResult:
    """scheduler.hpp:174-293 on the B200: the MaxMemory baseline -- the A element stream cut at fixed
    byte boundaries (maxmemory_partition, partition.hpp:140-169), the fragment of every split row
    returned to the host and re-sent with the next tile (merge_partial, :176-197).  Same result as
    run_aires; the ledger shows the extra link traffic (merge_bytes)."""
    res = run_aires(a, b, budget, cfg, mode, c_aware=2, n_buffers=n_buffers, with_checksum=with_checksum)
    res.report.strategy = "maxmemory"
    return res


RUN_STREAM_OUT = 1  # aires_b200_run_config.flags: streamed output (include/aires_b200.h)


def set_option(name: str, value: int) -> None:
    """aires_b200_set_option: a tuning option / test hook for the calling thread (include/aires_b200.h)."""
    _check(lib().aires_b200_set_option(name.encode(), int(value)))


def clear_options() -> None:
    _check(lib().aires_b200_clear_options())


@contextlib.contextmanager
def options(**kw):
    """Temporarily sets tuning options / test hooks on this thread: `with ab.options(wide_at=64): ...`."""
    try:
        for k, v in kw.items():
            set_option(k, v)
        yield
    finally:
        clear_options()


def run_aires(a: CsrMatrix, b, budget: MemoryBudget, cfg=None, mode: int = MODE_AUTO, c_aware: bool = True,
              n_buffers: int = 2, with_checksum: bool = True, stream_out: bool = False) -> RunResult:
    """scheduler.hpp:72-168 as a real three-phase tile pipeline on the B200 (ab2_pipeline.cu).

    A stays in host memory and streams through a ring of device slots sized by A + C bytes;
    C drains tile by tile straight into the result arrays.  ``budget.device_total`` caps the
    device bytes the run may hold (0: free memory).  ``cfg`` (SimConfig) only parameterises
    the reference's simulator and is accepted for signature compatibility.  Raises AiresError
    (insufficient_device_memory / row_too_large) instead of truncating (proj/README.md:58-60).
    ``stream_out`` (uncapped runs): no sizing pass before the product -- the result arrays are
    allocated at an upper bound of nnz(C) and C drains while A is still uploading; same C."""
    del cfg
    L = lib()
    am, keep_a = _matrix_from_np(a.n_rows, a.n_cols, CSR, a.row_ptr, a.col_idx, a.values)
    bm, keep_b = _operand_matrix(b)
    mode = _mode_for(keep_a[2], mode)
    vdt = np.float64 if mode == MODE_FP64_EXACT else np.float32
    if keep_a[2].dtype != vdt:
        keep_a = (keep_a[0], keep_a[1], keep_a[2].astype(vdt))
        am.val = _np_view(keep_a[2])
        am.val_bytes = keep_a[2].dtype.itemsize
    al = _HostAlloc(keep_a[1].dtype, vdt)
    out = al.output()
    events = []

    def _on_trace(_user, evs, n):
        events.extend(_trace_events(evs[i] for i in range(n)))

    trace_fn = _TRACE_FN(_on_trace)
    cfgc = _RunConfig(int(budget.device_total), mode, 2 if c_aware == 2 else int(bool(c_aware)),
                      0 if stream_out and n_buffers == 2 else int(n_buffers), RUN_STREAM_OUT if stream_out else 0,
                      trace_fn, None)
    rep = _RunReport()
    _check(L.aires_b200_run(C.byref(am), C.byref(bm), C.byref(cfgc), C.byref(out), C.byref(rep)))
    c = CsrMatrix(a.n_rows, b.n_cols, al.ptr, al.idx[: out.nnz], al.val[: out.nnz])
    r = RunReport(budget_bytes=int(budget.device_total), total_s=rep.total_ms / 1e3, phase1_s=rep.phase1_ms / 1e3,
                  phase2_s=rep.phase2_ms / 1e3, phase3_s=rep.phase3_ms / 1e3, segments=int(rep.segments),
                  flops=int(rep.flops), merge_seconds=rep.merge_ms / 1e3)
    r.ledger.h2d = ChannelTotals(int(rep.h2d_count), int(rep.h2d_bytes), rep.h2d_ms / 1e3)
    r.ledger.d2h = ChannelTotals(int(rep.d2h_count), int(rep.d2h_bytes), rep.d2h_ms / 1e3)
    r.ledger.peak_device_occupancy = int(rep.peak_device_bytes)
    r.ledger.merge_bytes = int(rep.merge_bytes)
    if with_checksum:
        r.c_checksum = checksum(c)
    return RunResult(c, r, events)


# ---------------------------------------------------------------------------
# GCN layer steps either side of A·X (gcn.hpp:29-132)
# ---------------------------------------------------------------------------

def normalize_adjacency(a: CsrMatrix, val_dtype=None) -> CsrMatrix:
    """gcn.hpp:29-72 on the B200: Ã = D̂^-½(A+I)D̂^-½ (fp64 arithmetic, bit-identical)."""
    L = lib()
    am, keep = _matrix_from_np(a.n_rows, a.n_cols, CSR, a.row_ptr, a.col_idx, a.values)
    al = _HostAlloc(keep[1].dtype, val_dtype or keep[2].dtype)
    out = al.output()
    _check(L.aires_b200_normalize_adjacency(C.byref(am), C.byref(out)))
    return CsrMatrix(a.n_rows, a.n_cols, al.ptr, al.idx[: out.nnz], al.val[: out.nnz])


def combine(x: CsrMatrix, w: np.ndarray) -> CsrMatrix:
    """gcn.hpp:90-116 on the B200: ReLU(X·W) with entries <= 0 dropped.  W dense (in, out), same
    value type as X."""
    L = lib()
    xm, keep = _matrix_from_np(x.n_rows, x.n_cols, CSR, x.row_ptr, x.col_idx, x.values)
    wd = np.ascontiguousarray(w, dtype=keep[2].dtype)
    if wd.ndim != 2:
        raise ValueError("W must be 2-D")
    al = _HostAlloc(keep[1].dtype, keep[2].dtype)
    out = al.output()
    _check(L.aires_b200_combine(C.byref(xm), _np_view(wd), wd.shape[0], wd.shape[1], HOST, C.byref(out)))
    return CsrMatrix(x.n_rows, wd.shape[1], al.ptr, al.idx[: out.nnz], al.val[: out.nnz])


# ---------------------------------------------------------------------------
# containers (serialize.hpp:60-209) and the storage leg
# ---------------------------------------------------------------------------

def _put(arr, width: int) -> bytes:
    a = np.asarray(arr)
    if width == 8:
        return np.ascontiguousarray(a, dtype="<u8").tobytes()
    return np.ascontiguousarray(a, dtype="<u4").tobytes()


def _put_val(arr, width: int) -> bytes:
    a = np.asarray(arr, dtype=np.float64)
    return (np.ascontiguousarray(a, dtype="<f8") if width == 8 else np.ascontiguousarray(a.astype(np.float32),
                                                                                     dtype="<f4")).tobytes()


def write_segments(path: str, segs: list, s: ElementSizes = ElementSizes()) -> None:
    """serialize.hpp:148-174: per segment a length-prefixed little-endian record."""
    with open(path, "wb") as f:
        for seg in segs:
            if s.index_bytes < 8:
                lim = (1 << (8 * s.index_bytes)) - 1
                if (seg.row_ptr_local.size and int(np.max(seg.row_ptr_local)) > lim) or \
                        (seg.col_idx.size and int(np.max(seg.col_idx)) > lim):
                    raise AiresError(1 + errc.capacity_exceeded, "index exceeds index width")
            record = 32 + seg.row_ptr_local.shape[0] * s.index_bytes + seg.nnz() * (s.index_bytes + s.value_bytes)
            f.write(_put([record, seg.seg_index, seg.start_row, seg.end_row, seg.nnz()], 8))
            f.write(_put(seg.row_ptr_local, s.index_bytes))
            f.write(_put(seg.col_idx, s.index_bytes))
            f.write(_put_val(seg.values, s.value_bytes))


def write_matrix(path: str, a: CsrMatrix) -> None:
    """serialize.hpp:102-122: the ARSM container (all 64-bit little-endian)."""
    with open(path, "wb") as f:
        f.write(b"ARSM" + _put([1, a.n_rows, a.n_cols, a.nnz()], 8))
        f.write(_put(a.row_ptr, 8) + _put(a.col_idx, 8) + _put_val(a.values, 8))


def read_matrix(path: str) -> CsrMatrix:
    """serialize.hpp:124-142."""
    raw = np.fromfile(path, dtype=np.uint8)
    if raw[:4].tobytes() != b"ARSM":
        raise AiresError(1 + errc.parse_error, "bad matrix container magic")
    ver, nr, nc, nnz = (int(v) for v in raw[4:36].view("<u8"))
    if ver != 1:
        raise AiresError(1 + errc.unsupported_format, f"matrix container version {ver}")
    o = 36
    rp = raw[o:o + 8 * (nr + 1)].view("<u8").copy(); o += 8 * (nr + 1)
    ci = raw[o:o + 8 * nnz].view("<u8").copy(); o += 8 * nnz
    va = raw[o:o + 8 * nnz].view("<f8").copy()
    return CsrMatrix(nr, nc, rp, ci, va)


def assemble_blocks(blocks: list, n_rows: int, n_cols: int) -> CsrMatrix:
    """spgemm.hpp:155-181: consecutive fragments -> one CSR (throws on gaps / overlaps)."""
    expect = 0
    ptrs, cols, vals = [np.zeros(1, np.uint64)], [], []
    base = 0
    for b in sorted(blocks, key=lambda b: b.start_row):
        if b.start_row != expect:
            raise AiresError(1 + errc.non_adjacent_fragments, f"fragment starts at {b.start_row}, expected {expect}")
        expect = b.end_row
        rp = np.asarray(b.fragment.row_ptr, dtype=np.uint64)
        ptrs.append(rp[1:] - rp[0] + np.uint64(base))
        base += int(rp[-1] - rp[0])
        cols.append(b.fragment.col_idx)
        vals.append(b.fragment.values)
    if expect != n_rows:
        raise AiresError(1 + errc.non_adjacent_fragments, f"fragments cover {expect} of {n_rows} rows")
    return CsrMatrix(n_rows, n_cols, np.concatenate(ptrs),
                     np.concatenate(cols) if cols else np.zeros(0, np.uint64),
                     np.concatenate(vals) if vals else np.zeros(0))


def spgemm_segments_file(path: str, sizes: ElementSizes, a_n_cols: int, b, mode: int = MODE_AUTO) -> tuple:
    """read_segments + spgemm_block per segment on the B200 (the storage leg): the records of a
    segment container go from the file to device memory (cuFile/GDS, or pread + pinned H2D).
    Returns (list of CsrBlockResult, report dict)."""
    L = lib()
    bm, keep = _operand_matrix(b)
    blocks = []
    vdt = np.float64 if (mode == MODE_FP64_EXACT or (mode == MODE_AUTO and sizes.value_bytes == 8)) else np.float32

    def cb(user, seg_index, start_row, end_row, nnz, rp, ci, va, flops):
        rows = end_row - start_row
        ptr = np.ctypeslib.as_array(rp, shape=(rows + 1,)).copy()
        idx = np.ctypeslib.as_array(C.cast(ci, C.POINTER(C.c_uint64)), shape=(max(nnz, 1),))[:nnz].copy()
        vt = C.c_double if vdt == np.float64 else C.c_float
        val = np.ctypeslib.as_array(C.cast(va, C.POINTER(vt)), shape=(max(nnz, 1),))[:nnz].copy()
        blocks.append(CsrBlockResult(start_row, end_row, CsrMatrix(rows, b.n_cols, ptr, idx, val), flops))
        return 0

    fn = _SEG_FN(cb)
    rep = _StorageReport()
    _check(L.aires_b200_spgemm_segments(path.encode(), sizes.index_bytes, sizes.value_bytes, a_n_cols, C.byref(bm),
                                        mode, fn, None, C.byref(rep)))
    return blocks, {"segments": rep.segments, "bytes_read": rep.bytes_read, "flops": rep.flops, "c_nnz": rep.c_nnz,
                    "used_gds": bool(rep.used_gds), "read_ms": rep.read_ms, "total_ms": rep.total_ms}


def layer_fused(a_tilde: CsrMatrix, h: CsrMatrix, w: np.ndarray) -> CsrMatrix:
    """ReLU((Ã·H)·W) in one device pass (fp32, dense-ish H): the aggregate + combine of layer_forward
    without materialising Ã·H; within the fp32 tolerance of the unfused chain."""
    L = lib()
    am, ka = _matrix_from_np(a_tilde.n_rows, a_tilde.n_cols, CSR, a_tilde.row_ptr, a_tilde.col_idx.astype(np.uint32),
                             a_tilde.values.astype(np.float32))
    hm, kh = _matrix_from_np(h.n_rows, h.n_cols, CSR, h.row_ptr, h.col_idx.astype(np.uint32),
                             h.values.astype(np.float32))
    wd = np.ascontiguousarray(w, dtype=np.float32)
    al = _HostAlloc(np.uint32, np.float32)
    out = al.output()
    _check(L.aires_b200_layer_fused(C.byref(am), C.byref(hm), _np_view(wd), wd.shape[0], wd.shape[1], HOST,
                                    C.byref(out)))
    return CsrMatrix(a_tilde.n_rows, wd.shape[1], al.ptr, al.idx[: out.nnz], al.val[: out.nnz])


def gen_weights(in_dim: int, out_dim: int, seed: int) -> np.ndarray:
    """synth.hpp:81-86 (same draws as the reference)."""
    w = np.empty((in_dim, out_dim), dtype=np.float64)
    _check(lib().aires_b200_synth_weights(in_dim, out_dim, seed, w.ctypes.data_as(C.POINTER(C.c_double))), synth=True)
    return w


@dataclasses.dataclass
class LayerResult:
    """gcn.hpp:118-123"""
    h_next: CsrMatrix
    aggregate_report: Optional[RunReport]
    trace: list


def layer_forward(a: CsrMatrix, h, weight: np.ndarray, budget: Optional[MemoryBudget] = None,
                  mode: int = MODE_AUTO) -> LayerResult:
    """gcn.hpp:125-132: normalize, aggregate (A·H; the out-of-core run when a budget is given),
    combine with ReLU -- every step on the B200."""
    at = normalize_adjacency(a)
    if budget is not None:
        res = run_aires(at, h, budget, mode=mode)
        x, rep = res.c, res.report
    else:
        x, rep = spgemm_full(at, h, mode=mode), None
    return LayerResult(combine(x, weight), rep, [])


def last_profile() -> dict:
    L = lib()
    arr = (C.c_double * 7)()
    n = L.aires_b200_last_profile(arr, 7)
    names = ["classify", "symbolic", "scan", "numeric", "x_prep", "h2d", "d2h"]
    d = {names[i]: arr[i] for i in range(n)}
    d["total"] = L.aires_b200_last_kernel_ms()
    return d


def device_count() -> int:
    n = C.c_int()
    _check(lib().aires_b200_device_count(C.byref(n)))
    return n.value


# ---------------------------------------------------------------------------
# synthetic inputs
# ---------------------------------------------------------------------------

def synth_graph(n: int, target_nnz: int, alpha: float = 0.75, degree_cap: int = 20000, seed: int = 1,
                relabel_seed: int = 2, relabel: bool = True, normalize: bool = True, threads: int = 0,
                idx_dtype=np.uint32, val_dtype=np.float64) -> tuple:
    """Chung-Lu power-law graph -> (CsrMatrix Ã (or A), stats dict)."""
    L = lib()
    al = _HostAlloc(idx_dtype, val_dtype)
    out = al.output()
    spec = _GraphSpec(n, target_nnz, alpha, degree_cap, seed, relabel_seed, int(relabel), int(normalize),
                      threads, 0)
    st = (C.c_double * 8)()
    _check(L.aires_b200_synth_graph(C.byref(spec), C.byref(out), st), synth=True)
    m = CsrMatrix(n, n, al.ptr, al.idx[: out.nnz], al.val[: out.nnz])
    stats = dict(nnz_a=int(st[0]), max_degree=int(st[1]), mean_degree=st[2], rounds=int(st[3]),
                 seconds=st[4], i0=st[5])
    return m, stats


def synth_features(n: int, dim: int, sparsity_pct: float = 99.0, seed: int = 3, idx_dtype=np.uint32,
                   val_dtype=np.float64) -> CsrMatrix:
    """gen_features (synth.hpp:73-78), draw-for-draw identical."""
    L = lib()
    al = _HostAlloc(idx_dtype, val_dtype)
    out = al.output()
    _check(L.aires_b200_synth_features(n, dim, sparsity_pct, seed, C.byref(out)), synth=True)
    return CsrMatrix(n, dim, al.ptr, al.idx[: out.nnz], al.val[: out.nnz])
