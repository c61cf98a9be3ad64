/*
 * aires_b200.h -- C ABI of the B200-native AIRES out-of-core A·X SpGEMM path.
 *
 * The reference (arxiv 2507.02006, /root/reference/proj) is a header-only C++20
 * library with no FFI; its "operator API" is the free functions of namespace
 * aires.  This C ABI is the thin layer those functions now forward to (the
 * drop-in C++ headers in include/aires/ call it; see INTEGRATION.md for the
 * ctypes / C++ bindings).  Plain pointers and sizes only; no torch types.
 *
 * Entry point  -> reference interface it replaces
 *   aires_b200_spgemm        -> aires::spgemm_block (raw spans)  spgemm.hpp:60-132
 *                               aires::spgemm_block (segment)    spgemm.hpp:134-139
 *                               aires::spgemm_full (Csr,Csc)     spgemm.hpp:142-146
 *                               aires::spgemm_full (Csr,Csr)     spgemm.hpp:148-151
 *   aires_b200_operand_*     -> the resident B of run_aires Phase I (scheduler.hpp:89-96)
 *   aires_b200_spgemm_op     -> spgemm_block against a resident B (scheduler.hpp:124)
 *   aires_b200_robw_cuts     -> aires::robw_partition cut search partition.hpp:52-74
 *   aires_b200_run           -> aires::run_aires Phases I-III    scheduler.hpp:72-168
 *                               (real multi-stream tile pipeline, C-aware tiles)
 *   aires_b200_checksum      -> aires::checksum (FNV-1a of C)   serialize.hpp:50-59
 *   aires_b200_normalize_adjacency -> aires::normalize_adjacency gcn.hpp:29-72
 *   aires_b200_combine       -> aires::combine (ReLU(X*W))      gcn.hpp:90-116
 *   aires_b200_layer_fused   -> aggregate + combine of layer_forward, fused  gcn.hpp:81-116
 *   aires_b200_spgemm_segments -> read_segments + spgemm_block per segment  serialize.hpp:148-209,
 *                               spgemm.hpp:134-139 (the storage leg: cuFile/GDS or pinned host)
 *   aires_b200_last_error    -> the what() string of aires::error error.hpp:53-62
 *
 * Status codes: 0 = OK, otherwise 1 + (int)aires::errc (error.hpp:9-27), so
 * errc::index_out_of_range (0) is 1.  Codes >= 100 are device/runtime failures
 * with no errc equivalent.  CUDA out-of-memory maps to
 * insufficient_device_memory.  Every entry point is reentrant:
 * each host thread gets its own CUDA stream and workspace on the current device.
 */
#ifndef AIRES_B200_H
#define AIRES_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AIRES_B200_ABI_VERSION 2

/* status codes (1 + errc) */
enum {
  AIRES_B200_OK = 0,
  AIRES_B200_INDEX_OUT_OF_RANGE = 1,
  AIRES_B200_UNSUPPORTED_FORMAT = 3,
  AIRES_B200_INSUFFICIENT_DEVICE_MEMORY = 5,
  AIRES_B200_ROW_TOO_LARGE = 6,
  AIRES_B200_DIMENSION_MISMATCH = 8,
  AIRES_B200_CAPACITY_EXCEEDED = 9,
  AIRES_B200_CONFIG_ERROR = 17,
  AIRES_B200_CUDA_ERROR = 100,
  AIRES_B200_NO_DEVICE = 101,
  AIRES_B200_INVALID_ARGUMENT = 102
};

/* where a buffer lives */
enum { AIRES_B200_HOST = 0, AIRES_B200_DEVICE = 1 };
/* sparse layouts */
enum { AIRES_B200_CSR = 0, AIRES_B200_CSC = 1 };
/* arithmetic modes */
enum {
  AIRES_B200_MODE_AUTO = 0,     /* FP64_EXACT if the values are 8 bytes wide, else FP32 */
  AIRES_B200_MODE_FP32 = 1,     /* fp32 products and sums; order-free accumulation;
                                   values within 1e-5 relative of the reference */
  AIRES_B200_MODE_FP64_EXACT = 2 /* fp64, no FMA, each cell summed in ascending k from
                                   +0.0: bit-identical to the reference (spgemm.hpp:21-42) */
};

/*
 * A borrowed sparse matrix.  CSR: ptr has n_rows+1 entries, idx holds column
 * indices.  CSC: ptr has n_cols+1 entries, idx holds row indices.  ptr is
 * always 64-bit (index_t); it may be absolute, i.e. ptr[0] != 0, indexing into
 * idx/val directly (spgemm.hpp:79-84).  idx_bytes in {4, 8}; val_bytes in {4, 8}.
 * span = number of idx/val entries addressable (>= ptr[last]).
 */
typedef struct aires_b200_matrix {
  uint64_t n_rows;
  uint64_t n_cols;
  uint32_t layout;
  uint32_t location;
  uint32_t idx_bytes;
  uint32_t val_bytes;
  const uint64_t* ptr;
  const void* idx;
  const void* val;
  uint64_t span;
} aires_b200_matrix;

/*
 * Output allocator.  Called once per product, once the exact row and nnz counts are
 * known (the exact allocation of spgemm.hpp:111-112).  Must return buffers in out->location of n_rows+1 u64, nnz idx_bytes-wide and nnz
 * val_bytes-wide entries.  Return 0 on success; any other value is passed back to the
 * caller as the status.
 */
typedef int (*aires_b200_alloc_fn)(void* user, uint64_t n_rows, uint64_t nnz, void** ptr,
                                   void** idx, void** val);

typedef struct aires_b200_output {
  uint32_t location;  /* where alloc() places C */
  uint32_t idx_bytes; /* C col_idx width: 4 or 8 */
  uint32_t val_bytes; /* C value width: 4 or 8 */
  uint32_t reserved;
  aires_b200_alloc_fn alloc;
  void* user;
  /* filled by the call */
  uint64_t n_rows;
  uint64_t n_cols;
  uint64_t nnz;
  uint64_t flops; /* multiply-accumulate count == CsrBlockResult.flops (spgemm.hpp:51) */
} aires_b200_output;

/* ---- library ----------------------------------------------------------- */
int aires_b200_abi_version(void);
const char* aires_b200_last_error(void);
int aires_b200_device_count(int* count);
/* Selects the CUDA device used by the calling thread (default 0). */
int aires_b200_set_device(int device);

/* ---- in-core product: C = A(rows) * B --------------------------------- */
/*
 * A: CSR rows (spgemm_block's row_ptr/col_idx/values spans; a->n_cols is a_n_cols).
 * B: CSR or CSC, host or device.  Result columns are sorted ascending per row and
 * cells with a structural hit are kept even when their sum is zero.
 */
int aires_b200_spgemm(const aires_b200_matrix* a, const aires_b200_matrix* b, uint32_t mode,
                      aires_b200_output* c);

/* ---- resident right operand -------------------------------------------- */
typedef struct aires_b200_operand_s* aires_b200_operand;
/* Uploads / converts B once (B200 row-major feature layout) on the current device. */
int aires_b200_operand_create(const aires_b200_matrix* b, uint32_t mode,
                              aires_b200_operand* out);
int aires_b200_operand_destroy(aires_b200_operand op);
int aires_b200_operand_info(aires_b200_operand op, uint64_t* n_rows, uint64_t* n_cols,
                            uint64_t* nnz, uint32_t* mode, uint64_t* device_bytes);
int aires_b200_spgemm_op(const aires_b200_matrix* a, aires_b200_operand b,
                         aires_b200_output* c);

/* ---- RoBW tiler (Alg. 1) ------------------------------------------------ */
/*
 * Greedy maximal whole-row segments with calc_mem(k,q) = (k+1)*I + q*(I+V) <= m_a,
 * computed on the device (search over F(r) = r*I + row_ptr[r]*(I+V)).  cuts gets
 * n_segs+1 boundaries (cuts[0] = 0, cuts[n_segs] = n_rows); cap = capacity of cuts.
 * Returns AIRES_B200_ROW_TOO_LARGE with *bad_row set exactly as robw_partition
 * throws (partition.hpp:64-69).  row_ptr may be host or device (location).
 */
int aires_b200_robw_cuts(const uint64_t* row_ptr, uint64_t n_rows, uint64_t m_a,
                         uint64_t index_bytes, uint64_t value_bytes, uint32_t location,
                         uint64_t* cuts, uint64_t cap, uint64_t* n_segs, uint64_t* bad_row);

/* ---- out-of-core run (Alg. 2 as a real multi-stream pipeline) ---------- */
/*
 * One measured event of a real run -- the TraceEvent of tiered_sim.hpp:60-68 with device clocks:
 * timestamps are the completion times of CUDA events recorded on the stream that did the work,
 * in ms after the run's first event.  Buffers are named the reference's way by the C++ glue:
 * AIRES_B200_BUF_B -> "B", _A_TILE -> "a_tile_<index>", _C_BLOCK -> "C" (d2h of block <index>),
 * _FRAGMENT -> "frag_<index>" (MaxMemory's returned row fragment), _A -> "A".
 */
enum { AIRES_B200_EV_TRANSFER = 0, AIRES_B200_EV_COMPUTE = 1, AIRES_B200_EV_ALLOC = 2, AIRES_B200_EV_FREE = 3 };
enum { AIRES_B200_CH_GDS = 0, AIRES_B200_CH_S2H = 1, AIRES_B200_CH_H2D = 2, AIRES_B200_CH_D2H = 3 };
enum { AIRES_B200_TIER_DEVICE = 0, AIRES_B200_TIER_HOST = 1, AIRES_B200_TIER_STORAGE = 2 };
enum { AIRES_B200_BUF_B = 0, AIRES_B200_BUF_A_TILE = 1, AIRES_B200_BUF_C_BLOCK = 2, AIRES_B200_BUF_FRAGMENT = 3,
       AIRES_B200_BUF_A = 4 /* A's row pointers / the sizing pass's column chunks -> "A" */ };
typedef struct aires_b200_trace_event {
  double timestamp_ms; /* completion, ms after the run's first event */
  double duration_ms;  /* device time of the span (transfers, compute); 0 for alloc / free */
  uint32_t kind;       /* AIRES_B200_EV_* (EventKind order) */
  uint32_t phase;      /* 0, 1, 2 = Phase I, II, III */
  uint32_t where;      /* transfers: AIRES_B200_CH_* (ChannelId order); otherwise AIRES_B200_TIER_* */
  uint32_t buffer;     /* AIRES_B200_BUF_* */
  uint64_t index;      /* tile / block index of the buffer */
  uint64_t bytes;
  uint64_t flops;
} aires_b200_trace_event;
/* Receives the whole trace once, sorted by timestamp, after the run completed. */
typedef void (*aires_b200_trace_fn)(void* user, const aires_b200_trace_event* events, uint64_t n);

typedef struct aires_b200_run_config {
  uint64_t device_budget; /* bytes the run may hold on the device at once (0 = no cap) */
  uint32_t mode;          /* AIRES_B200_MODE_* */
  uint32_t c_aware;       /* 1: tiles sized by A + C bytes (default); 0: RoBW by A only;
                             2: the MaxMemory baseline (fixed byte tiles, split rows' fragments
                                returned to the host and re-sent, scheduler.hpp:174-293) */
  uint32_t n_buffers;     /* tile ring depth (default 2; 3 for streamed output) */
  uint32_t flags;         /* AIRES_B200_RUN_* bits (0 = the reference's exact-allocation protocol) */
  aires_b200_trace_fn trace; /* optional: the run's measured trace (RunResult::trace) */
  void* trace_user;
} aires_b200_run_config;

/* Streamed output (uncapped runs, device_budget 0): no sizing pass before the product.  c->alloc
 * receives an UPPER BOUND of nnz(C) (min(rows * n_cols, nnz(A) * longest X row)) before the first
 * tile, C is drained tile by tile while A is still crossing the link, and c->nnz reports the exact
 * count (the arrays hold the exact CSR in their first c->nnz entries).  Ignored for capped and
 * MaxMemory runs and for operands wider than the dense accumulator (exact protocol). */
#define AIRES_B200_RUN_STREAM_OUT 1u

typedef struct aires_b200_run_report {
  uint64_t segments;
  uint64_t h2d_bytes; /* bytes actually copied host -> device */
  uint64_t d2h_bytes; /* bytes actually copied device -> host */
  uint64_t flops;
  uint64_t c_nnz;
  uint64_t peak_device_bytes;
  double total_ms;   /* first H2D to last D2H, CUDA events */
  double phase1_ms;  /* operand upload + symbolic sizing + cut */
  double phase2_ms;  /* tile streaming */
  double phase3_ms;  /* final drain / assembly */
  uint64_t merge_bytes; /* MaxMemory: fragment bytes re-sent after the host stitch (IoLedger::merge_bytes) */
  /* ChannelTotals (tiered_sim.hpp:70-76) of the run: one transfer per tile upload / block drain */
  uint64_t h2d_count;
  uint64_t d2h_count;
  double h2d_ms;        /* sum of the transfers' device durations */
  double d2h_ms;
  double merge_ms;      /* MaxMemory: fragment return + the re-sent share of uploads (RunReport::merge_seconds) */
} aires_b200_run_report;

/* A in host memory (CSR); B host or device; C written through c->alloc (host). */
int aires_b200_run(const aires_b200_matrix* a, const aires_b200_matrix* b,
                   const aires_b200_run_config* cfg, aires_b200_output* c,
                   aires_b200_run_report* report);

/* ---- storage leg: RoBW segments from the reference's segment container ------ */
/* Called once per segment with the positioned fragment (CsrBlockResult, spgemm.hpp:47-52): local
   row_ptr (end_row - start_row + 1 u64), col_idx (nnz u64), values (nnz, 4 or 8 bytes per the mode);
   the pointers are valid during the call.  Return 0 to continue. */
typedef int (*aires_b200_segment_fn)(void* user, uint64_t seg_index, uint64_t start_row, uint64_t end_row,
                                     uint64_t nnz, const uint64_t* row_ptr, const void* col_idx,
                                     const void* values, uint64_t flops);
typedef struct aires_b200_storage_report {
  uint64_t segments;
  uint64_t bytes_read; /* file bytes moved to the device */
  uint64_t flops;
  uint64_t c_nnz;
  uint32_t used_gds;   /* 1: cuFileRead into device memory (GPUDirect Storage); 0: pread + pinned H2D */
  uint32_t reserved;
  double read_ms;      /* host time spent reading (overlapped with the products) */
  double total_ms;
} aires_b200_storage_report;
/* Streams the segments of `path` (serialize.hpp:148-209 format, ElementSizes {index_bytes,
   value_bytes}) to the device and multiplies each against B (host or device, CSR or CSC). */
int aires_b200_spgemm_segments(const char* path, uint32_t index_bytes, uint32_t value_bytes, uint64_t a_n_cols,
                               const aires_b200_matrix* b, uint32_t mode, aires_b200_segment_fn cb, void* user,
                               aires_b200_storage_report* report);

/* ---- GCN layer steps either side of A·X ------------------ */
/* Ã = D̂^-½ (A + I) D̂^-½, bit-identical to the reference (fp64 arithmetic; fp32 output is the
   rounded fp64 value).  A square CSR, nonnegative weights; errors: non_square, negative_weight. */
int aires_b200_normalize_adjacency(const aires_b200_matrix* a, aires_b200_output* out);
/* H = ReLU(X * W), entries <= 0 dropped.  X CSR (host or device), W dense row-major w_rows x w_cols
   of X's value type at w_location; fp64 bit-identical to the reference, fp32 within tolerance. */
int aires_b200_combine(const aires_b200_matrix* x, const void* w, uint64_t w_rows, uint64_t w_cols,
                       uint32_t w_location, aires_b200_output* out);

/* H' = ReLU((Ã * H) * W) in one pass without materialising Ã*H (gcn.hpp:81-116 fused): the
   aggregate and combine of layer_forward for a dense-ish H (fp32, u32 columns; H width <= 256,
   W width <= 128).  Terms are re-associated: within the fp32 tolerance, not bit-exact. */
int aires_b200_layer_fused(const aires_b200_matrix* a_tilde, const aires_b200_matrix* h, const void* w,
                           uint64_t w_rows, uint64_t w_cols, uint32_t w_location, aires_b200_output* out);

/* FNV-1a 64 of a CSR in the reference's canonical byte stream (serialize.hpp:50-59); host only.
   row_ptr may be absolute (it is rebased); 4-byte indices / values are widened to u64 / f64. */
uint64_t aires_b200_checksum(uint64_t n_rows, uint64_t n_cols, uint64_t nnz, const uint64_t* row_ptr,
                             const void* col_idx, uint32_t idx_bytes, const void* values, uint32_t val_bytes);

/* ---- tuning options and test hooks (not part of the reference surface) --- */
/*
 * Per calling thread; every option has a measured default, so production callers set none.
 * Unknown names return AIRES_B200_INVALID_ARGUMENT.  The library reads no environment variable
 * for kernel choice or numerics (AB2_TRACE=1 only prints per-run device timelines to stderr).
 *   heavy_deg (1024)        A rows above this degree are computed CTA-cooperatively
 *   sym_heavy_deg (2048)    the same for the out-of-core sizing kernel
 *   num_warps (4)           warps per CTA of the product kernel
 *   short_rows (1)          rows with <= 32 terms take the register-sort path
 *   slot_w (auto)           force the X slot width (2, 4, 8, 16)
 *   numeric_kernel (3)      5: the fp32 step-list kernel instead of the W-slot kernel
 *   n5_warps, w5            step-list kernel: warps per CTA, slot width
 *   wide_at (8192 / 4096)   X column count from which products run in column tiles
 *   wide_tile               column-tile width of those products
 *   run_tiles (16), stream_tiles (16)  tiles of the uncapped exact / streamed runs
 *   run_resident_cols (1)   uncapped exact runs keep A's columns on the device after sizing
 *   run_cslots (1)          out-of-core sizing over 16-wide column slots when X rows average >= 4
 *   combine_one_pass (1), combine_smem (1), combine_v4 (1), fused_reassoc (1)  GCN kernel paths
 *   gds (0) / no_gds (0)    storage leg: force / forbid the cuFile attempt
 *   stage_min_bytes (64 MiB) pageable host arrays at least this large move through pinned bounce
 *                           slots (host copy threads) instead of being registered for the call
 *   narrow_cols (1)         streamed runs move C's column indices as u16 (host threads widen them)
 *   hw_tensor (1)           fused layer: T = H·W on tcgen05 (3xTF32) when W has <= 48 columns
 *   short_dense (1)         rows of <= 32 terms with <= 256 output columns: dense cells instead of a sort
 *   agg_async (1)           fused layer: Ã·T gathers T rows (<= 64 floats) with cp.async into shared memory
 */
int aires_b200_set_option(const char* name, int64_t value);
int aires_b200_clear_options(void);

/* ---- timing helpers for harnesses (not part of the reference surface) --- */
/* The cudaStream_t the calling thread's products run on (current device), so a harness can
   record CUDA events on the stream the kernels are launched on. */
void* aires_b200_stream(void);
/* Number of kernels the last product on this thread launched. */
int aires_b200_last_launches(void);
/* Elapsed ms of the last aires_b200_spgemm/_op on this thread (CUDA events). */
double aires_b200_last_kernel_ms(void);
/* Per-stage ms of the last product on this thread: [classify+mac count, place, scan,
   numeric, x_prep, h2d, d2h]; returns the number of entries written (<= cap). */
int aires_b200_last_profile(double* ms, int cap);

#ifdef __cplusplus
}
#endif
#endif /* AIRES_B200_H */
