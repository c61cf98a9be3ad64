// ab2_api.cu -- the extern "C" boundary (include/aires_b200.h) and per-thread contexts.
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>

#include "ab2_internal.h"

namespace ab2 {

namespace {
thread_local std::string tl_error;
thread_local int tl_device = 0;
thread_local std::map<int, std::unique_ptr<Ctx>> tl_ctx;
}  // namespace

void fail(int code, const std::string& msg) { throw Error{code, msg}; }

void check_cuda(cudaError_t e, const char* what, const char* file, int line) {
  if (e == cudaSuccess) return;
  cudaGetLastError();
  int code = e == cudaErrorMemoryAllocation ? AIRES_B200_INSUFFICIENT_DEVICE_MEMORY
             : (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) ? AIRES_B200_NO_DEVICE
                                                                             : AIRES_B200_CUDA_ERROR;
  fail(code, std::string(cudaGetErrorString(e)) + " in " + what + " (" + file + ":" + std::to_string(line) + ")");
}

// Tuning options and test hooks (aires_b200_set_option): explicit, per calling thread, validated
// against the list in aires_b200.h; nothing in the library reads the process environment except the
// AB2_TRACE diagnostic timeline (stderr only, never numerics or kernel choice).
namespace {
const char* const kOptionNames[] = {
    "heavy_deg",         "sym_heavy_deg",  "num_warps",         "short_rows", "slot_w",      "numeric_kernel",
    "n5_warps",          "w5",             "wide_at",           "wide_tile",  "run_tiles",   "stream_tiles",
    "run_resident_cols", "run_cslots",     "combine_one_pass",  "combine_smem", "combine_v4", "fused_reassoc",
    "gds",               "no_gds",         "stage_min_bytes",   "narrow_cols",       "hw_tensor",         "agg_async",
    "short_dense"};
thread_local std::vector<std::pair<std::string, int64_t>> t_options;
}  // namespace

std::vector<std::pair<std::string, int64_t>>& t_options_ref() { return t_options; }

bool option_known(const char* name) {
  for (const char* k : kOptionNames)
    if (std::strcmp(k, name) == 0) return true;
  return false;
}

int64_t option(const char* name, int64_t def) {
  for (const auto& kv : t_options)
    if (kv.first == name) return kv.second;
  return def;
}

bool trace_enabled() {
  static const bool on = [] {
    const char* v = std::getenv("AB2_TRACE");
    return v && *v && std::strtoll(v, nullptr, 10) != 0;
  }();
  return on;
}

void* DevBuf::get(size_t bytes) {
  bytes = std::max<size_t>(bytes, 256);
  if (bytes <= cap) return p;
  release();
  size_t want = bytes + bytes / 8;
  cudaError_t e = cudaMalloc(&p, want);
  if (e != cudaSuccess) {
    cudaGetLastError();
    p = nullptr;
    e = cudaMalloc(&p, bytes);
    want = bytes;
  }
  if (e != cudaSuccess) {
    p = nullptr;
    cap = 0;
    check_cuda(e, "cudaMalloc(workspace)", __FILE__, __LINE__);
  }
  cap = want;
  return p;
}

void DevBuf::release() {
  if (p) cudaFree(p);
  p = nullptr;
  cap = 0;
}

void* HostBuf::get(size_t bytes) {
  bytes = std::max<size_t>(bytes, 256);
  if (bytes <= cap) return p;
  release();
  AB2_CUDA(cudaHostAlloc(&p, bytes, cudaHostAllocDefault));
  cap = bytes;
  return p;
}

void HostBuf::release() {
  if (p) cudaFreeHost(p);
  p = nullptr;
  cap = 0;
}

Ctx::Ctx(int dev) : device(dev) {
  AB2_CUDA(cudaSetDevice(dev));
  AB2_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  AB2_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
  for (auto& e : ev) AB2_CUDA(cudaEventCreate(&e));
}

Ctx::~Ctx() {
  // Best effort: the CUDA runtime may already be torn down at thread/process exit.
  if (pipe) destroy_pipe_cache(pipe);
  for (auto& e : ev)
    if (e) cudaEventDestroy(e);
  if (stream) cudaStreamDestroy(stream);
}

int current_device() { return tl_device; }

Ctx& ctx_for_thread() {
  auto it = tl_ctx.find(tl_device);
  if (it != tl_ctx.end()) {
    AB2_CUDA(cudaSetDevice(tl_device));
    return *it->second;
  }
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    cudaGetLastError();
    fail(AIRES_B200_NO_DEVICE, "no CUDA device is visible (the B200 path has no CPU fallback)");
  }
  auto c = std::make_unique<Ctx>(tl_device);
  Ctx& ref = *c;
  tl_ctx[tl_device] = std::move(c);
  return ref;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    tl_error.clear();
    return AIRES_B200_OK;
  } catch (const Error& e) {
    tl_error = e.msg;
    return e.code;
  } catch (const std::exception& e) {
    tl_error = e.what();
    return AIRES_B200_CUDA_ERROR;
  } catch (...) {
    tl_error = "unknown failure";
    return AIRES_B200_CUDA_ERROR;
  }
}

}  // namespace ab2

struct aires_b200_operand_s {
  std::unique_ptr<ab2::XOperand> x;
};

extern "C" {

int aires_b200_abi_version(void) { return AIRES_B200_ABI_VERSION; }

int aires_b200_set_option(const char* name, int64_t value) {
  return ab2::guarded([&] {
    if (!name || !ab2::option_known(name)) ab2::fail(AIRES_B200_INVALID_ARGUMENT, std::string("unknown option ") + (name ? name : "(null)"));
    for (auto& kv : ab2::t_options_ref())
      if (kv.first == name) {
        kv.second = value;
        return;
      }
    ab2::t_options_ref().emplace_back(name, value);
  });
}

int aires_b200_clear_options(void) {
  return ab2::guarded([&] { ab2::t_options_ref().clear(); });
}

const char* aires_b200_last_error(void) { return ab2::tl_error.c_str(); }

int aires_b200_device_count(int* count) {
  return ab2::guarded([&] {
    if (!count) ab2::fail(AIRES_B200_INVALID_ARGUMENT, "count is null");
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess) {
      cudaGetLastError();
      n = 0;
    }
    *count = n;
  });
}

int aires_b200_set_device(int device) {
  return ab2::guarded([&] {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || device < 0 || device >= n) {
      cudaGetLastError();
      ab2::fail(AIRES_B200_NO_DEVICE, "device " + std::to_string(device) + " is not visible");
    }
    ab2::tl_device = device;
  });
}

int aires_b200_spgemm(const aires_b200_matrix* a, const aires_b200_matrix* b, uint32_t mode,
                      aires_b200_output* c) {
  return ab2::guarded([&] {
    if (!a || !b || !c) ab2::fail(AIRES_B200_INVALID_ARGUMENT, "null argument");
    if (a->n_cols != b->n_rows)
      ab2::fail(AIRES_B200_DIMENSION_MISMATCH, "inner dimensions " + std::to_string(a->n_cols) + " and " +
                                                   std::to_string(b->n_rows) + " differ");
    ab2::Ctx& ctx = ab2::ctx_for_thread();
    if (mode == AIRES_B200_MODE_AUTO) mode = c->val_bytes == 8 ? AIRES_B200_MODE_FP64_EXACT : AIRES_B200_MODE_FP32;
    cudaEvent_t t0 = ctx.ev[10], t1 = ctx.ev[11];
    AB2_CUDA(cudaEventRecord(t0, ctx.stream));
    auto x = ab2::make_operand(ctx, *b, mode, /*temp=*/true);
    AB2_CUDA(cudaEventRecord(t1, ctx.stream));
    ctx.launches = x->prep_launches;
    ab2::spgemm_rows(ctx, *a, *x, *c);
    float ms = 0;
    AB2_CUDA(cudaEventElapsedTime(&ms, t0, t1));
    ctx.prof[ab2::kPXPrep] = ms;
  });
}

int aires_b200_operand_create(const aires_b200_matrix* b, uint32_t mode, aires_b200_operand* out) {
  return ab2::guarded([&] {
    if (!b || !out) ab2::fail(AIRES_B200_INVALID_ARGUMENT, "null argument");
    ab2::Ctx& ctx = ab2::ctx_for_thread();
    auto op = std::make_unique<aires_b200_operand_s>();
    op->x = ab2::make_operand(ctx, *b, mode, /*temp=*/false);
    *out = op.release();
  });
}

int aires_b200_operand_destroy(aires_b200_operand op) {
  return ab2::guarded([&] { delete op; });
}

int aires_b200_operand_info(aires_b200_operand op, uint64_t* n_rows, uint64_t* n_cols, uint64_t* nnz,
                            uint32_t* mode, uint64_t* device_bytes) {
  return ab2::guarded([&] {
    if (!op || !op->x) ab2::fail(AIRES_B200_INVALID_ARGUMENT, "null operand");
    if (n_rows) *n_rows = static_cast<uint64_t>(op->x->K);
    if (n_cols) *n_cols = static_cast<uint64_t>(op->x->n_cols);
    if (nnz) *nnz = static_cast<uint64_t>(op->x->nnz);
    if (mode) *mode = op->x->mode;
    if (device_bytes) *device_bytes = op->x->bytes;
  });
}

int aires_b200_spgemm_op(const aires_b200_matrix* a, aires_b200_operand b, aires_b200_output* c) {
  return ab2::guarded([&] {
    if (!a || !b || !b->x || !c) ab2::fail(AIRES_B200_INVALID_ARGUMENT, "null argument");
    ab2::Ctx& ctx = ab2::ctx_for_thread();
    if (b->x->device != ctx.device)
      ab2::fail(AIRES_B200_INVALID_ARGUMENT, "operand lives on another device");
    ctx.launches = 0;
    ab2::spgemm_rows(ctx, *a, *b->x, *c);
    ctx.prof[ab2::kPXPrep] = 0.0;
  });
}

int aires_b200_robw_cuts(const uint64_t* row_ptr, uint64_t n_rows, uint64_t m_a, uint64_t index_bytes,
                         uint64_t value_bytes, uint32_t location, uint64_t* cuts, uint64_t cap,
                         uint64_t* n_segs, uint64_t* bad_row) {
  int rc = AIRES_B200_OK;
  int g = ab2::guarded([&] {
    if (!row_ptr || !cuts || !n_segs) ab2::fail(AIRES_B200_INVALID_ARGUMENT, "null argument");
    ab2::Ctx& ctx = ab2::ctx_for_thread();
    rc = ab2::robw_cuts(ctx, row_ptr, n_rows, m_a, index_bytes, value_bytes, location, cuts, cap, n_segs,
                        bad_row);
  });
  return g != AIRES_B200_OK ? g : rc;
}

int aires_b200_run(const aires_b200_matrix* a, const aires_b200_matrix* b, const aires_b200_run_config* cfg,
                   aires_b200_output* c, aires_b200_run_report* report) {
  return ab2::guarded([&] {
    if (!a || !b || !cfg || !c || !report) ab2::fail(AIRES_B200_INVALID_ARGUMENT, "null argument");
    ab2::Ctx& ctx = ab2::ctx_for_thread();
    ctx.launches = 0;
    ab2::run_pipeline(ctx, *a, *b, *cfg, *c, *report);
  });
}

int aires_b200_normalize_adjacency(const aires_b200_matrix* a, aires_b200_output* out) {
  return ab2::guarded([&] {
    if (!a || !out) ab2::fail(AIRES_B200_INVALID_ARGUMENT, "null argument");
    ab2::Ctx& ctx = ab2::ctx_for_thread();
    ab2::normalize_adjacency(ctx, *a, *out);
  });
}

int aires_b200_combine(const aires_b200_matrix* x, const void* w, uint64_t w_rows, uint64_t w_cols,
                       uint32_t w_location, aires_b200_output* out) {
  return ab2::guarded([&] {
    if (!x || !out || (!w && w_rows * w_cols)) ab2::fail(AIRES_B200_INVALID_ARGUMENT, "null argument");
    ab2::Ctx& ctx = ab2::ctx_for_thread();
    ab2::combine(ctx, *x, w, w_rows, w_cols, w_location, *out);
  });
}

int aires_b200_layer_fused(const aires_b200_matrix* a_tilde, const aires_b200_matrix* h, const void* w,
                           uint64_t w_rows, uint64_t w_cols, uint32_t w_location, aires_b200_output* out) {
  return ab2::guarded([&] {
    if (!a_tilde || !h || !out || (!w && w_rows * w_cols)) ab2::fail(AIRES_B200_INVALID_ARGUMENT, "null argument");
    ab2::Ctx& ctx = ab2::ctx_for_thread();
    ab2::layer_fused(ctx, *a_tilde, *h, w, w_rows, w_cols, w_location, *out);
  });
}

int aires_b200_spgemm_segments(const char* path, uint32_t index_bytes, uint32_t value_bytes, uint64_t a_n_cols,
                               const aires_b200_matrix* b, uint32_t mode, aires_b200_segment_fn cb, void* user,
                               aires_b200_storage_report* report) {
  return ab2::guarded([&] {
    if (!path || !b || !report) ab2::fail(AIRES_B200_INVALID_ARGUMENT, "null argument");
    ab2::Ctx& ctx = ab2::ctx_for_thread();
    ab2::spgemm_segments(ctx, path, index_bytes, value_bytes, a_n_cols, *b, mode, cb, user, *report);
  });
}

void* aires_b200_stream(void) {
  void* s = nullptr;
  ab2::guarded([&] { s = static_cast<void*>(ab2::ctx_for_thread().stream); });
  return s;
}

int aires_b200_last_launches(void) {
  auto it = ab2::tl_ctx.find(ab2::tl_device);
  return it == ab2::tl_ctx.end() ? 0 : it->second->launches;
}

double aires_b200_last_kernel_ms(void) {
  auto it = ab2::tl_ctx.find(ab2::tl_device);
  return it == ab2::tl_ctx.end() ? 0.0 : it->second->last_ms;
}

int aires_b200_last_profile(double* ms, int cap) {
  auto it = ab2::tl_ctx.find(ab2::tl_device);
  int n = 0;
  for (; n < cap && n < ab2::kPCount; n++) ms[n] = it == ab2::tl_ctx.end() ? 0.0 : it->second->prof[n];
  return n;
}

}  // extern "C"
