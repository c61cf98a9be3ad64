// ab2_storage.cu -- the storage leg of the dual-way load (§III-C; scheduler.hpp:89-96 models
// it as the "gds" channel): RoBW segments read from the reference's segment container
// (serialize.hpp:148-209 -- per segment a length-prefixed little-endian record) straight into
// device memory with cuFile (GPUDirect Storage) when the driver opens, otherwise through a pinned
// host buffer and cudaMemcpyAsync (the report says which).  Each segment is multiplied against the
// resident X on arrival (spgemm_block(seg, ...), scheduler.hpp:124) and handed to the caller's
// callback as a positioned fragment (CsrBlockResult, spgemm.hpp:47-52); the next record is read by a
// host thread while the current one is multiplied.
//
// libcufile is loaded with dlopen, so the library has no hard dependency on it.
#include <dlfcn.h>
#include <fcntl.h>
#include <unistd.h>

#include <chrono>
#include <cstring>
#include <future>
#include <mutex>
#include <vector>

#include "ab2_internal.h"

namespace ab2 {

namespace {

// ---- minimal cuFile binding (cufile.h types restated as opaque) ------------
struct CuFileApi {
  void* so = nullptr;
  bool open = false;
  struct Err {
    int err;
    int cu_err;
  };
  struct Descr {
    int type;  // CU_FILE_HANDLE_TYPE_OPAQUE_FD = 1
    union {
      int fd;
      void* handle;
    } handle;
    const void* fs_ops;
  };
  Err (*driver_open)() = nullptr;
  Err (*handle_register)(void**, Descr*) = nullptr;
  void (*handle_deregister)(void*) = nullptr;
  ssize_t (*read)(void*, void*, size_t, off_t, off_t) = nullptr;
  Err (*buf_register)(const void*, size_t, int) = nullptr;
  Err (*buf_deregister)(const void*) = nullptr;

  bool load() {
    if (so) return open;
    if (option("no_gds", 0)) return false;
    // GPUDirect Storage needs the nvidia-fs kernel module; without it cuFileDriverOpen was measured
    // to block for minutes on the B200 boxes, so the driver is only opened when the module is
    // loaded (or AB2_GDS=1 forces the attempt).  Otherwise the pinned-host path is used.
    if (::access("/proc/driver/nvidia-fs", F_OK) != 0 && option("gds", 0) == 0) {
      so = reinterpret_cast<void*>(1);  // probed: unavailable
      return false;
    }
    so = dlopen("libcufile.so.0", RTLD_NOW | RTLD_LOCAL);
    if (!so) so = dlopen("libcufile.so", RTLD_NOW | RTLD_LOCAL);
    if (!so) return false;
    driver_open = reinterpret_cast<Err (*)()>(dlsym(so, "cuFileDriverOpen"));
    handle_register = reinterpret_cast<Err (*)(void**, Descr*)>(dlsym(so, "cuFileHandleRegister"));
    handle_deregister = reinterpret_cast<void (*)(void*)>(dlsym(so, "cuFileHandleDeregister"));
    read = reinterpret_cast<ssize_t (*)(void*, void*, size_t, off_t, off_t)>(dlsym(so, "cuFileRead"));
    buf_register = reinterpret_cast<Err (*)(const void*, size_t, int)>(dlsym(so, "cuFileBufRegister"));
    buf_deregister = reinterpret_cast<Err (*)(const void*)>(dlsym(so, "cuFileBufDeregister"));
    if (!driver_open || !handle_register || !handle_deregister || !read) return false;
    open = driver_open().err == 0;  // CU_FILE_SUCCESS
    return open;
  }
};

CuFileApi& cufile() {
  static CuFileApi api;
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  api.load();
  return api;
}

uint64_t get_le(const unsigned char* p, unsigned w) {
  uint64_t v = 0;
  for (unsigned i = 0; i < w; i++) v |= static_cast<uint64_t>(p[i]) << (8 * i);
  return v;
}

void pread_all(int fd, void* dst, size_t n, off_t off) {
  char* d = static_cast<char*>(dst);
  while (n) {
    const ssize_t r = ::pread(fd, d, n, off);
    if (r <= 0) fail(1 + 15, "short read from the segment file");  // errc::io_error
    d += r;
    n -= static_cast<size_t>(r);
    off += r;
  }
}

struct Record {
  uint64_t seg_index, start_row, end_row, nnz;
  off_t payload_off;
  uint64_t payload_bytes;
};

// Widens the segment's local row pointers (index_bytes wide) to u64 rows+1 entries.
__global__ void k_widen_ptr(const unsigned char* __restrict__ src, unsigned w, uint64_t n, uint64_t* __restrict__ out) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    uint64_t v = 0;
    for (unsigned b = 0; b < w; b++) v |= static_cast<uint64_t>(src[i * w + b]) << (8 * b);
    out[i] = v;
  }
}

struct HostFrag {
  std::vector<uint64_t> ptr;
  HostBuf idx, val;
  static int alloc(void* user, uint64_t n_rows, uint64_t nnz, void** p, void** i, void** v) {
    auto* f = static_cast<HostFrag*>(user);
    try {
      f->ptr.assign(n_rows + 1, 0);
    } catch (...) {
      return 1 + 8;
    }
    *p = f->ptr.data();
    *i = f->idx.get(std::max<uint64_t>(nnz, 1) * 8);
    *v = f->val.get(std::max<uint64_t>(nnz, 1) * 8);
    return 0;
  }
};

}  // namespace

void spgemm_segments(Ctx& ctx, const char* path, uint32_t ib, uint32_t vb, uint64_t a_n_cols,
                     const aires_b200_matrix& b, uint32_t mode, aires_b200_segment_fn cb, void* user,
                     aires_b200_storage_report& rep) {
  if ((ib != 4 && ib != 8) || (vb != 4 && vb != 8)) fail(AIRES_B200_INVALID_ARGUMENT, "element sizes must be 4 or 8");
  if (!cb) fail(AIRES_B200_INVALID_ARGUMENT, "segment callback is null");
  if (a_n_cols != b.n_rows)
    fail(AIRES_B200_DIMENSION_MISMATCH,
         "inner dimensions " + std::to_string(a_n_cols) + " and " + std::to_string(b.n_rows) + " differ");
  if (mode == AIRES_B200_MODE_AUTO) mode = vb == 8 ? AIRES_B200_MODE_FP64_EXACT : AIRES_B200_MODE_FP32;
  const uint32_t ovb = mode == AIRES_B200_MODE_FP32 ? 4 : 8;
  std::memset(&rep, 0, sizeof(rep));
  const auto t0 = std::chrono::steady_clock::now();
  const int fd = ::open(path, O_RDONLY);
  if (fd < 0) fail(1 + 15, std::string("cannot open ") + path);
  struct Closer {
    int fd;
    ~Closer() { ::close(fd); }
  } closer{fd};
  // record index (headers only)
  std::vector<Record> recs;
  {
    const off_t end = ::lseek(fd, 0, SEEK_END);
    off_t off = 0;
    while (off < end) {
      unsigned char h[40];
      pread_all(fd, h, 40, off);
      Record r{get_le(h + 8, 8), get_le(h + 16, 8), get_le(h + 24, 8), get_le(h + 32, 8), off + 40, 0};
      const uint64_t record = get_le(h, 8);
      if (r.end_row < r.start_row) fail(1 + 1, "segment row range inverted");  // parse_error
      const uint64_t rows = r.end_row - r.start_row;
      if (record != 32 + (rows + 1) * ib + r.nnz * (ib + vb)) fail(1 + 1, "segment record length mismatch");
      r.payload_bytes = record - 32;
      recs.push_back(r);
      off += 8 + static_cast<off_t>(record);
    }
  }
  auto x = make_operand(ctx, b, mode, /*temp=*/false);
  CuFileApi& gds = cufile();
  void* gh = nullptr;
  if (gds.open) {
    CuFileApi::Descr d{};
    d.type = 1;
    d.handle.fd = fd;
    if (gds.handle_register(&gh, &d).err != 0) gh = nullptr;
  }
  rep.used_gds = gh != nullptr;
  uint64_t maxp = 0;
  for (const Record& r : recs) maxp = std::max(maxp, r.payload_bytes);
  // two device payload buffers (+ pinned staging when not on the GDS path)
  DevBuf dbuf[2];
  HostBuf hbuf[2];
  for (int i = 0; i < 2; i++) {
    dbuf[i].get(std::max<uint64_t>(maxp, 256));
    if (!gh) hbuf[i].get(std::max<uint64_t>(maxp, 256));
  }
  auto fetch = [&](size_t k) -> double {  // reads record k's payload into dbuf[k & 1] (host thread)
    const auto s = std::chrono::steady_clock::now();
    const Record& r = recs[k];
    void* dst = dbuf[k & 1].p;
    if (gh) {
      AB2_CUDA(cudaSetDevice(ctx.device));
      const ssize_t got = gds.read(gh, dst, r.payload_bytes, r.payload_off, 0);
      if (got < 0 || static_cast<uint64_t>(got) != r.payload_bytes) fail(1 + 15, "cuFileRead failed");
    } else {
      pread_all(fd, hbuf[k & 1].p, r.payload_bytes, r.payload_off);
    }
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - s).count();
  };
  HostFrag frag;
  std::future<double> next;
  if (!recs.empty()) next = std::async(std::launch::async, fetch, 0);
  DevBuf ptr64, vconv;
  for (size_t k = 0; k < recs.size(); k++) {
    rep.read_ms += next.get();
    const Record& r = recs[k];
    const uint64_t rows = r.end_row - r.start_row;
    char* payload = static_cast<char*>(dbuf[k & 1].p);
    if (!gh)
      AB2_CUDA(cudaMemcpyAsync(payload, hbuf[k & 1].p, r.payload_bytes, cudaMemcpyHostToDevice, ctx.stream));
    AB2_CUDA(cudaStreamSynchronize(ctx.stream));  // payload k on the device; buffers of k+1 are free
    if (k + 1 < recs.size()) next = std::async(std::launch::async, fetch, k + 1);
    rep.bytes_read += r.payload_bytes + 40;
    // views into the payload: ptr (rows+1) x ib, col nnz x ib, val nnz x vb
    uint64_t* p64 = ptr64.as<uint64_t>(rows + 1);
    k_widen_ptr<<<static_cast<unsigned>(std::min<uint64_t>((rows + 256) / 256, 4096)), 256, 0, ctx.stream>>>(
        reinterpret_cast<const unsigned char*>(payload), ib, rows + 1, p64);
    AB2_CUDA(cudaGetLastError());
    aires_b200_matrix am{};
    am.n_rows = rows;
    am.n_cols = a_n_cols;
    am.layout = AIRES_B200_CSR;
    am.location = AIRES_B200_DEVICE;
    am.idx_bytes = ib;
    am.val_bytes = vb;
    am.ptr = p64;
    am.idx = payload + (rows + 1) * ib;
    am.val = payload + (rows + 1) * ib + r.nnz * ib;
    am.span = r.nnz;
    aires_b200_output o{};
    o.location = AIRES_B200_HOST;
    o.idx_bytes = 8;
    o.val_bytes = ovb;
    o.alloc = &HostFrag::alloc;
    o.user = &frag;
    spgemm_rows(ctx, am, *x, o);
    rep.flops += o.flops;
    rep.c_nnz += o.nnz;
    const int rc = cb(user, r.seg_index, r.start_row, r.end_row, o.nnz, frag.ptr.data(), frag.idx.p, frag.val.p, o.flops);
    if (rc != 0) fail(rc, "segment callback failed");
    rep.segments++;
  }
  if (gh) gds.handle_deregister(gh);
  rep.total_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  (void)vconv;
}

}  // namespace ab2
