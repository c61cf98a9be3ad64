// ab2_internal.h -- host-side internals shared by the library translation units.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "ab2_common.cuh"

namespace ab2 {

// Grow-only device buffer.
struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  void* get(size_t bytes);
  template <class T>
  T* as(size_t n) {
    return static_cast<T*>(get(n * sizeof(T)));
  }
  void release();
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;  // owns its allocation: containers move it, never copy it
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), cap(o.cap) {
    o.p = nullptr;
    o.cap = 0;
  }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p;
      cap = o.cap;
      o.p = nullptr;
      o.cap = 0;
    }
    return *this;
  }
  ~DevBuf() { release(); }
};

// One device allocation carved for a budgeted run: buffers the run keeps come from the bottom, build
// temporaries from the top (dropped together once the build has finished on the device), so every
// byte a run holds at once lies inside `size` and the high-water mark is `peak`.
struct Region {
  char* base = nullptr;
  uint64_t size = 0, lo = 0, hi = 0, peak = 0;
  void init(void* p, uint64_t n) {
    base = static_cast<char*>(p);
    size = n & ~uint64_t(255);  // both ends 256-byte aligned
    lo = 0;
    hi = size;
    peak = 0;
  }
  static uint64_t up(uint64_t b) { return (std::max<uint64_t>(b, 1) + 255) & ~uint64_t(255); }
  void* keep(uint64_t bytes) {
    bytes = up(bytes);
    if (bytes > hi - lo)
      fail(AIRES_B200_INSUFFICIENT_DEVICE_MEMORY, "device budget of " + std::to_string(size) +
                                                      " bytes exhausted (" + std::to_string(bytes) + " more needed)");
    void* p = base + lo;
    lo += bytes;
    peak = std::max(peak, lo + (size - hi));
    return p;
  }
  void* temp(uint64_t bytes) {
    bytes = up(bytes);
    if (bytes > hi - lo)
      fail(AIRES_B200_INSUFFICIENT_DEVICE_MEMORY, "device budget of " + std::to_string(size) +
                                                      " bytes exhausted (" + std::to_string(bytes) + " more needed)");
    hi -= bytes;
    peak = std::max(peak, lo + (size - hi));
    return base + hi;
  }
  void drop_temps() { hi = size; }
};

// Grow-only pinned host buffer.
struct HostBuf {
  void* p = nullptr;
  size_t cap = 0;
  void* get(size_t bytes);
  void release();
  HostBuf() = default;
  HostBuf(const HostBuf&) = delete;
  HostBuf& operator=(const HostBuf&) = delete;
  HostBuf(HostBuf&& o) noexcept : p(o.p), cap(o.cap) {
    o.p = nullptr;
    o.cap = 0;
  }
  HostBuf& operator=(HostBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p;
      cap = o.cap;
      o.p = nullptr;
      o.cap = 0;
    }
    return *this;
  }
  ~HostBuf() { release(); }
};

// kPPlace shares the slot the symbolic pass used before the single-pass design.
enum ProfSlot { kPClassify, kPPlace, kPScan, kPNumeric, kPXPrep, kPH2D, kPD2H, kPCount };
constexpr int kPSymbolic = kPPlace;

// Per-thread, per-device execution context (reentrancy: SURVEY.md §8b Threading).
struct Ctx {
  int device = 0;
  int sms = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev[2 * kPCount + 2] = {};
  DevBuf a_ptr, a_col, a_val, a_col2, a_val2;  // uploaded / converted A
  DevBuf cnt, rflops, cptr, scan_part, sym_heavy, num_heavy, fix_rows, ctl;
  DevBuf c_col, c_val;                          // C staging for host outputs
  DevBuf t_col, t_val;                          // product staging (K_numeric -> K_place)
  DevBuf x_ptr, x_idx, x_val;                   // raw X upload (host operands)
  DevBuf xo_ptr, xo_col, xo_val, xo_slots, xo_cslots, xo_len, xo_desc, xo_ent;  // per-call operand layout
  HostBuf h_ctl;
  double prof[kPCount] = {};
  double last_ms = 0.0;
  int launches = 0;  // kernels launched by the last product
  void* pipe = nullptr;  // out-of-core pipeline cache (ab2_pipeline.cu)
  uint64_t last_fix_rows = 0;
  explicit Ctx(int dev);
  ~Ctx();
};

Ctx& ctx_for_thread();
int current_device();

// A prepared right operand (B200 feature layout), see ab2_operand.cuh.
struct XOperand {
  int device = 0;
  uint32_t mode = 0;  // AIRES_B200_MODE_FP32 or _FP64_EXACT
  int64_t K = 0, n_cols = 0, nnz = 0;
  int W = 0;
  int64_t max_row_len = 0;  // longest X row (bounds C nnz per A entry)
  void* ptr = nullptr;     // int64 K+1
  void* col = nullptr;     // int32 nnz
  void* val = nullptr;     // V nnz
  void* slots = nullptr;   // K*W entries
  void* cslots = nullptr;  // K*kCSlotW u16
  void* xlen = nullptr;    // K+1 u16 row lengths
  void* xdesc = nullptr;   // fp32: K+1 uint2 {slot start, nslot | len << 16} (row K empty)
  void* xent = nullptr;    // fp32: padded W5-entry slots of uint2 {col, value bits}
  int W5 = 0;              // fp32 step-list slot width
  bool wide = false;       // n_cols beyond the dense accumulator: plain CSR only, column-tiled product
  int64_t dummy_slot = 0;  // fp32: index of the all-trash slot
  double xmin = 0.0;       // smallest nonzero |x|
  bool has_zero = false;   // X stores an exact zero
  size_t bytes = 0;        // device bytes of every layout built
  int prep_launches = 0;
  bool owned = true;  // kernels launched to build the operand
  ~XOperand();
};

// Builds an operand from a matrix view (host or device, CSR or CSC).
// temp: storage comes from the context (valid until the next product on this thread).
// Which device layouts of X to build (the plain CSR is always built).
enum OperandPlan : uint32_t {
  kPlanSlots = 1,   // W-slot groups (k_numeric3)
  kPlanCSlots = 2,  // 16-wide column-only slots (symbolic pass over slots)
  kPlanStep = 4,    // padded step-list slots (k_numeric5, fp32 only)
  kPlanLean = 8,    // with kPlanStep (fp32): drop the plain CSR once the step list is built (tight budgets)
  kPlanAuto = 0     // the in-core default for the mode (AB2_NUMERIC selects the fp32 kernel)
};
// Widest X handled by the dense accumulator (wider operands run in column tiles).
int64_t wide_threshold(uint32_t mode);
// rg (budgeted runs): every device buffer of the build comes from the region -- the layouts the run
// reads are kept, the raw upload and the scratch are temporaries dropped (after a stream sync) on return.
struct Region;
std::unique_ptr<XOperand> make_operand(Ctx& ctx, const aires_b200_matrix& b, uint32_t mode, bool temp,
                                       uint32_t plan = kPlanAuto, Region* rg = nullptr);

// C = A * X; A is a CSR rows view (host or device).
void spgemm_rows(Ctx& ctx, const aires_b200_matrix& a, const XOperand& x, aires_b200_output& out);

// ---- tile passes for the out-of-core pipeline (ab2_pipeline.cu), launched on ctx.stream ----
// A tile: rows [0, rows) of a device CSR slice; aptr is absolute (abase = aptr[0] of the slice
// buffer's first entry).  idx_bytes is the width of acol and of the C column output.
struct TileSym {
  const uint64_t* aptr;
  uint64_t abase;
  const void* acol;
  int64_t rows;
  int32_t* cnt;     // rows: C nnz per row (output)
  int64_t* rflops;  // rows: MACs per row (output)
  int64_t* heavy;   // rows scratch
  Ctl* ctl;         // zeroed; ctl->flops accumulates the MACs
};
struct TilePass {
  const uint64_t* aptr;
  uint64_t abase;
  const void* acol;
  const void* aval;
  int64_t rows;
  const int64_t* cpos;  // exact C row offsets for these rows (rows+1), absolute
  int64_t cbase;        // cpos value of the tile's first C entry in ccol/cval
  void* ccol;
  void* cval;
  uint64_t c_cap;
  int64_t* heavy;   // rows scratch
  uint32_t* cnt;    // rows scratch
  uint64_t* toff;   // rows scratch
  Ctl* ctl;         // zeroed; bad_row != 0 afterwards means a count/capacity failure
};
// A tile whose C row counts are not known in advance (streamed-output runs): product into a
// staging area, scan of the row counts -> local C row offsets, placement into a contiguous C block.
struct TileStaged {
  const uint64_t* aptr;
  uint64_t abase;
  const void* acol;
  const void* aval;
  int64_t rows;
  uint64_t a_nnz;    // A entries of the tile (staging bound)
  void* tcol;        // staging, staged_capacity() entries
  void* tval;
  uint64_t t_cap;
  int64_t* cptr;     // rows+1 local C row offsets (out)
  void* ccol;        // C block, >= c_bound() entries
  void* cval;
  int64_t* heavy;    // rows scratch
  uint32_t* cnt;     // rows scratch
  uint64_t* toff;    // rows scratch
  int64_t* part;     // scan partials, (rows + 2047) / 2048
  Ctl* ctl;          // zeroed; afterwards nnz = tile nnz, flops = MACs, bad_row != 0 = staging overflow
};
uint64_t c_bound(const XOperand& x, uint64_t rows, uint64_t a_nnz);  // nnz(C) upper bound of a tile
uint64_t staged_capacity(Ctx& ctx, const XOperand& x, uint64_t rows, uint64_t a_nnz);
// All return the number of kernels launched.
int tile_symbolic(Ctx& ctx, const XOperand& x, uint32_t idx_bytes, const TileSym& t);
int tile_product(Ctx& ctx, const XOperand& x, uint32_t idx_bytes, const TilePass& t);
int tile_product_staged(Ctx& ctx, const XOperand& x, uint32_t idx_bytes, const TileStaged& t);

// GCN layer steps either side of A·X (ab2_gcn.cu, gcn.hpp:29-116).
void normalize_adjacency(Ctx& ctx, const aires_b200_matrix& a, aires_b200_output& out);
void combine(Ctx& ctx, const aires_b200_matrix& x, const void* w, uint64_t w_rows, uint64_t w_cols,
             uint32_t w_location, aires_b200_output& out);
void layer_fused(Ctx& ctx, const aires_b200_matrix& at, const aires_b200_matrix& h, const void* w, uint64_t w_rows,
                 uint64_t w_cols, uint32_t w_location, aires_b200_output& out);

// Storage leg (ab2_storage.cu).
void spgemm_segments(Ctx& ctx, const char* path, uint32_t ib, uint32_t vb, uint64_t a_n_cols,
                     const aires_b200_matrix& b, uint32_t mode, aires_b200_segment_fn cb, void* user,
                     aires_b200_storage_report& rep);

// Out-of-core run (ab2_pipeline.cu).
void destroy_pipe_cache(void* p);
void run_pipeline(Ctx& ctx, const aires_b200_matrix& a, const aires_b200_matrix& b, const aires_b200_run_config& cfg,
                  aires_b200_output& out, aires_b200_run_report& rep);

// RoBW cuts on the device.
int robw_cuts(Ctx& ctx, const uint64_t* row_ptr, uint64_t n_rows, uint64_t m_a, uint64_t I,
              uint64_t V, uint32_t location, uint64_t* cuts, uint64_t cap, uint64_t* n_segs,
              uint64_t* bad_row);

// Tuning option / test hook set through aires_b200_set_option (this thread), else def.
int64_t option(const char* name, int64_t def);
bool option_known(const char* name);
std::vector<std::pair<std::string, int64_t>>& t_options_ref();
// AB2_TRACE=1 in the environment: per-run device timelines on stderr (diagnostics only).
bool trace_enabled();

}  // namespace ab2
