// ab2_pipeline.cu -- the out-of-core run (Alg. 2, run_aires, scheduler.hpp:72-168) as a real
// multi-stream tile pipeline under a device-memory budget.
//
// The reference sizes RoBW segments by A alone (scheduler.hpp:79-82) and admits each segment's C
// block against its Eq. 5 estimate (scheduler.hpp:126-130), which for GCN shapes is ~1e-4 of the
// real C, so every multi-segment budget throws.  Here the tiles are sized by
// A + C bytes, which needs C's row counts before the product -- the reference's own structure
// (symbolic pass, exact allocation, numeric pass, spgemm.hpp:94-130) lifted to the whole run:
//
//   Phase I   (dual-way load + partition, scheduler.hpp:89-100)
//     X -> resident operand; A row_ptr -> device (resident, 8 B/row);
//     symbolic pass streamed over A's column indices in chunks (copy stream || compute stream)
//     -> per-row nnz(C) -> device scan -> C row_ptr (-> host output) and total nnz;
//     C-aware tile cuts (greedy maximal row ranges whose A + C bytes fit a ring slot; with
//     c_aware = 0 the cuts are RoBW's, partition.hpp:52-74, over A alone);
//     the caller's allocator receives the exact (rows, nnz) once (spgemm.hpp:111-112).
//   Phase II  (per segment: H2D -> multiply -> drain C, scheduler.hpp:103-139)
//     ring of n_buffers slots; tile k+1's H2D (copy engine 0) overlaps tile k's product
//     (compute stream, rows written straight to their exact CSR offsets -- no staging) and
//     tile k-1's D2H of C into the final host arrays (copy engine 1).  Events order slot reuse.
//   Phase III (assemble / drain / store, scheduler.hpp:142-166)
//     nothing to assemble: every tile's C already sits at its final offsets; sync and report.
//
// Streamed output (AIRES_B200_RUN_STREAM_OUT, uncapped runs only): run_stream below skips the sizing
// pass -- the allocator gets an upper bound of nnz(C) and C drains tile by tile from the first tile on.
//
// Host memory: A and C host buffers that are not page-locked are registered for the call
// (cudaHostRegister) so every copy is an async DMA; GPUDirect Storage is not used on this path
// (the operands arrive in host memory through the API).
#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <exception>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "ab2_internal.h"
#include "ab2_kernels.cuh"

namespace ab2 {

namespace {

struct Pinned {
  std::vector<void*> regs;
  void ensure(const void* p, size_t bytes) {
    if (!p || bytes == 0) return;
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) == cudaSuccess && at.type != cudaMemoryTypeUnregistered) return;
    cudaGetLastError();
    cudaError_t e = cudaHostRegister(const_cast<void*>(p), bytes, cudaHostRegisterDefault);
    if (e == cudaSuccess) {
      regs.push_back(const_cast<void*>(p));
    } else {
      cudaGetLastError();  // fall back to pageable copies (synchronous staging by the driver)
    }
  }
  ~Pinned() {
    for (void* p : regs) cudaHostUnregister(p);
  }
};

bool is_pinned(const void* p) {
  if (!p) return true;
  cudaPointerAttributes at{};
  const bool ok = cudaPointerGetAttributes(&at, p) == cudaSuccess && at.type != cudaMemoryTypeUnregistered;
  cudaGetLastError();
  return ok;
}

// Host threads that copy between pageable caller arrays and pinned bounce buffers (Stager).
struct CopyPool {
  std::vector<std::thread> th;
  std::mutex m;
  std::condition_variable cv, idle;
  std::vector<std::function<void()>> jobs;
  size_t next = 0, left = 0;
  uint64_t gen = 0;
  bool stop = false;
  explicit CopyPool(unsigned n) {
    for (unsigned i = 0; i < n; i++)
      th.emplace_back([this] {
        uint64_t seen = 0;
        for (;;) {
          std::function<void()> job;
          {
            std::unique_lock<std::mutex> lk(m);
            cv.wait(lk, [&] { return stop || (gen != seen && next < jobs.size()); });
            if (stop) return;
            job = jobs[next++];
            if (next == jobs.size()) seen = gen;
          }
          job();
          std::lock_guard<std::mutex> lk(m);
          if (--left == 0) idle.notify_all();
        }
      });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> lk(m);
      stop = true;
    }
    cv.notify_all();
    for (auto& t : th) t.join();
  }
  // copies every (dst, src, bytes) in ~4 MB pieces across the pool and the calling thread
  void copy(const std::vector<std::tuple<char*, const char*, uint64_t>>& segs) {
    constexpr uint64_t kPiece = 4ull << 20;
    std::vector<std::function<void()>> js;
    for (const auto& sg : segs)
      for (uint64_t o = 0; o < std::get<2>(sg); o += kPiece) {
        const uint64_t n = std::min(kPiece, std::get<2>(sg) - o);
        char* d = std::get<0>(sg) + o;
        const char* s2 = std::get<1>(sg) + o;
        js.emplace_back([d, s2, n] { std::memcpy(d, s2, n); });
      }
    run(std::move(js));
  }
  // widens `count` u16 column indices to u32 / u64 (out_bytes) in ~2M-entry pieces
  void widen(char* dst, const uint16_t* src, uint64_t count, uint32_t out_bytes) {
    constexpr uint64_t kPiece = 512ull << 10;
    std::vector<std::function<void()>> js;
    for (uint64_t o = 0; o < count; o += kPiece) {
      const uint64_t n = std::min(kPiece, count - o);
      if (out_bytes == 4) {
        uint32_t* d = reinterpret_cast<uint32_t*>(dst) + o;
        const uint16_t* q = src + o;
        js.emplace_back([d, q, n] {
          for (uint64_t i = 0; i < n; i++) d[i] = q[i];
        });
      } else {
        uint64_t* d = reinterpret_cast<uint64_t*>(dst) + o;
        const uint16_t* q = src + o;
        js.emplace_back([d, q, n] {
          for (uint64_t i = 0; i < n; i++) d[i] = q[i];
        });
      }
    }
    run(std::move(js));
  }
  std::mutex run_mu;  // one batch at a time (the pipeline thread's uploads, the stager's copy-outs)
  void run(std::vector<std::function<void()>>&& js) {
    if (js.empty()) return;
    std::lock_guard<std::mutex> batch(run_mu);
    if (js.size() == 1 || th.empty()) {
      for (auto& j : js) j();
      return;
    }
    std::unique_lock<std::mutex> lk(m);
    jobs = std::move(js);
    next = 0;
    left = jobs.size();
    gen++;
    cv.notify_all();
    // the caller works too
    while (next < jobs.size()) {
      auto job = jobs[next++];
      lk.unlock();
      job();
      lk.lock();
      if (--left == 0) idle.notify_all();
    }
    idle.wait(lk, [&] { return left == 0; });
    jobs.clear();
  }
};

// Pageable caller arrays (the reference's std::vector storage behind the drop-in headers): instead of
// registering gigabytes with the driver inside every call (cudaHostRegister pins page by page --
// ~0.5 s for cfg2's A and C at the reference's widths), tiles travel through pinned bounce slots:
// host threads copy a tile's A segments into an up-slot and the copy engine moves them to the device;
// C parts come down into a down-slot and host threads copy them out once that DMA has completed
// (before the slot is reused, or at the end of the run).  Page-locked caller buffers skip this.
struct Stager {
  struct Slot {
    char* buf = nullptr;
    cudaEvent_t done = nullptr;
    bool armed = false;
    std::vector<std::tuple<char*, const char*, uint64_t>> out;  // pending copy-outs (down slots)
    std::vector<std::tuple<char*, const uint16_t*, uint64_t, uint32_t>> wide;  // pending u16 -> u32/u64 widenings
  };
  CopyPool& pool;
  std::vector<HostBuf>& ubuf;
  std::vector<HostBuf>& dbuf;
  std::vector<Slot> up, down;
  size_t nu = 0, nd = 0;
  int device = 0;
  // down-slots are retired (DMA landed -> host copies) by a background thread, in arrival order,
  // so the thread that queues the pipeline never stops for them
  std::thread bg;
  std::mutex mu;
  std::condition_variable cv;
  std::vector<uint32_t> fifo;
  size_t head = 0;
  bool stop = false;
  std::exception_ptr err;
  Stager(CopyPool& p, std::vector<HostBuf>& u, std::vector<HostBuf>& d, uint32_t nbuf, std::vector<cudaEvent_t>& ev,
         int dev)
      : pool(p), ubuf(u), dbuf(d), up(nbuf), down(2 * nbuf), device(dev) {
    if (ubuf.size() < nbuf) ubuf.resize(nbuf);
    if (dbuf.size() < 2 * nbuf) dbuf.resize(2 * nbuf);
    while (ev.size() < 3 * nbuf) {
      cudaEvent_t e;
      AB2_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      ev.push_back(e);
    }
    for (uint32_t i = 0; i < nbuf; i++) up[i].done = ev[i];
    for (uint32_t i = 0; i < 2 * nbuf; i++) down[i].done = ev[nbuf + i];
  }
  ~Stager() { halt(); }
  void halt() {
    {
      std::lock_guard<std::mutex> lk(mu);
      stop = true;
    }
    cv.notify_all();
    if (bg.joinable()) bg.join();
  }
  // host -> device: segments (dev, host, bytes) through the next up-slot, queued on stream s
  void h2d(const std::vector<std::tuple<char*, const char*, uint64_t>>& segs, cudaStream_t s) {
    Slot& sl = up[nu % up.size()];
    const uint32_t i = static_cast<uint32_t>(nu++ % up.size());
    uint64_t total = 0;
    for (const auto& g : segs) total += (std::get<2>(g) + 255) & ~uint64_t(255);
    if (sl.armed) AB2_CUDA(cudaEventSynchronize(sl.done));  // its previous upload has left
    sl.buf = static_cast<char*>(ubuf[i].get(total));
    std::vector<std::tuple<char*, const char*, uint64_t>> in;
    uint64_t o = 0;
    for (const auto& g : segs) {
      in.emplace_back(sl.buf + o, std::get<1>(g), std::get<2>(g));
      o += (std::get<2>(g) + 255) & ~uint64_t(255);
    }
    pool.copy(in);
    o = 0;
    for (const auto& g : segs) {
      if (std::get<2>(g)) AB2_CUDA(cudaMemcpyAsync(std::get<0>(g), sl.buf + o, std::get<2>(g), cudaMemcpyHostToDevice, s));
      o += (std::get<2>(g) + 255) & ~uint64_t(255);
    }
    AB2_CUDA(cudaEventRecord(sl.done, s));
    sl.armed = true;
  }
  // device -> host: segments (host, dev, bytes) into the next down-slot, queued on stream s, plus
  // `narrow` u16 column indices (host dst, device u16 src, count, host width 4 or 8) that the host
  // widens; the background thread does the host side once the DMA has landed
  void d2h(const std::vector<std::tuple<char*, const char*, uint64_t>>& segs, cudaStream_t s,
           const std::vector<std::tuple<char*, const uint16_t*, uint64_t, uint32_t>>& narrow = {}) {
    const uint32_t i = static_cast<uint32_t>(nd++ % down.size());
    Slot& sl = down[i];
    {
      std::unique_lock<std::mutex> lk(mu);
      cv.wait(lk, [&] { return !sl.armed || err; });
      if (err) std::rethrow_exception(err);
    }
    uint64_t total = 0;
    for (const auto& g : segs) total += (std::get<2>(g) + 255) & ~uint64_t(255);
    for (const auto& g : narrow) total += (std::get<2>(g) * 2 + 255) & ~uint64_t(255);
    sl.buf = static_cast<char*>(dbuf[i].get(total));
    uint64_t o = 0;
    for (const auto& g : segs) {
      if (std::get<2>(g)) AB2_CUDA(cudaMemcpyAsync(sl.buf + o, std::get<1>(g), std::get<2>(g), cudaMemcpyDeviceToHost, s));
      sl.out.emplace_back(std::get<0>(g), sl.buf + o, std::get<2>(g));
      o += (std::get<2>(g) + 255) & ~uint64_t(255);
    }
    for (const auto& g : narrow) {
      if (std::get<2>(g))
        AB2_CUDA(cudaMemcpyAsync(sl.buf + o, std::get<1>(g), std::get<2>(g) * 2, cudaMemcpyDeviceToHost, s));
      sl.wide.emplace_back(std::get<0>(g), reinterpret_cast<const uint16_t*>(sl.buf + o), std::get<2>(g), std::get<3>(g));
      o += (std::get<2>(g) * 2 + 255) & ~uint64_t(255);
    }
    AB2_CUDA(cudaEventRecord(sl.done, s));
    {
      std::lock_guard<std::mutex> lk(mu);
      sl.armed = true;
      fifo.push_back(i);
    }
    cv.notify_all();
    if (!bg.joinable()) bg = std::thread([this] { loop(); });
  }
  void loop() {
    cudaSetDevice(device);
    for (;;) {
      uint32_t i;
      {
        std::unique_lock<std::mutex> lk(mu);
        cv.wait(lk, [&] { return stop || head < fifo.size(); });
        if (head >= fifo.size()) return;
        i = fifo[head];
      }
      Slot& sl = down[i];
      try {
        AB2_CUDA(cudaEventSynchronize(sl.done));
        pool.copy(sl.out);
        for (const auto& w : sl.wide) pool.widen(std::get<0>(w), std::get<1>(w), std::get<2>(w), std::get<3>(w));
      } catch (...) {
        std::lock_guard<std::mutex> lk(mu);
        if (!err) err = std::current_exception();
      }
      {
        std::lock_guard<std::mutex> lk(mu);
        sl.out.clear();
        sl.wide.clear();
        sl.armed = false;
        head++;
      }
      cv.notify_all();
    }
  }
  // every queued copy-out done (call after the run's last synchronisation)
  void finish() {
    {
      std::unique_lock<std::mutex> lk(mu);
      cv.wait(lk, [&] { return head >= fifo.size() || err; });
    }
    halt();
    if (err) std::rethrow_exception(err);
  }
};

// Routes the kernels a helper launches on ctx.stream to another stream for a scope.
struct StreamSwap {
  Ctx& ctx;
  cudaStream_t saved;
  StreamSwap(Ctx& c, cudaStream_t s) : ctx(c), saved(c.stream) { c.stream = s; }
  ~StreamSwap() { ctx.stream = saved; }
};

// Waits for every stream of a run before its host buffers can go away: a run that throws midway
// (an allocation failure, an overflow found at a drain) still has copies into / out of the caller's
// arrays and registered memory queued, and the Pinned registrations are dropped right after.
struct SyncGuard {
  cudaStream_t s[4];
  ~SyncGuard() {
    for (cudaStream_t q : s)
      if (q) cudaStreamSynchronize(q);
    cudaGetLastError();
  }
};

// Streams, events and device buffers of the pipeline, cached per (thread, device) context so
// repeated runs pay no cudaMalloc / stream creation on the host path.
struct PipeCacheImpl {
  cudaStream_t h2d = nullptr, d2h = nullptr, aux = nullptr;  // aux: sizing (capped streamed run), fragments (MaxMemory)
  std::vector<cudaEvent_t> ev, tev;  // disable-timing / timing
  std::vector<DevBuf> bufs;
  DevBuf region;  // the capped streamed run's budget, carved by a Region
  // pageable caller arrays: pinned bounce slots and the host copy threads (Stager)
  std::vector<HostBuf> bounce_up, bounce_down;
  std::vector<cudaEvent_t> stage_ev;
  std::unique_ptr<CopyPool> pool;
  CopyPool& copy_pool() {
    if (!pool) pool = std::make_unique<CopyPool>(std::max(1u, std::min(15u, std::thread::hardware_concurrency() - 1)));
    return *pool;
  }
  PipeCacheImpl() {
    AB2_CUDA(cudaStreamCreateWithFlags(&h2d, cudaStreamNonBlocking));
    AB2_CUDA(cudaStreamCreateWithFlags(&d2h, cudaStreamNonBlocking));
    AB2_CUDA(cudaStreamCreateWithFlags(&aux, cudaStreamNonBlocking));
    bufs.resize(32);
  }
  ~PipeCacheImpl() {
    pool.reset();
    for (auto e : stage_ev) cudaEventDestroy(e);
    for (auto e : ev) cudaEventDestroy(e);
    for (auto e : tev) cudaEventDestroy(e);
    if (h2d) cudaStreamDestroy(h2d);
    if (d2h) cudaStreamDestroy(d2h);
    if (aux) cudaStreamDestroy(aux);
  }
};

struct Streams {
  PipeCacheImpl& c;
  cudaStream_t h2d, d2h, aux;
  size_t ne = 0, nt = 0;
  explicit Streams(PipeCacheImpl& pc) : c(pc), h2d(pc.h2d), d2h(pc.d2h), aux(pc.aux) {}
  cudaEvent_t make() {
    if (ne == c.ev.size()) {
      cudaEvent_t e;
      AB2_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      c.ev.push_back(e);
    }
    return c.ev[ne++];
  }
  cudaEvent_t make_timed() {
    if (nt == c.tev.size()) {
      cudaEvent_t e;
      AB2_CUDA(cudaEventCreate(&e));
      c.tev.push_back(e);
    }
    return c.tev[nt++];
  }
};

// The measured trace of a run (RunResult::trace, tiered_sim.hpp:60-98): every transfer, compute span
// and device allocation is bracketed by timed CUDA events on the stream that does the work, the
// NVTX range of the enclosing phase marks the host side, and finish() turns the events into the
// ChannelTotals of the report (count, bytes, seconds) and the time-sorted event list.
struct Tracer {
  struct Rec {
    cudaEvent_t a, b;  // a == b for alloc / free
    aires_b200_trace_event e;
  };
  Streams& st;
  std::vector<Rec> recs;
  uint32_t phase = 0;
  explicit Tracer(Streams& s) : st(s) {}
  void set_phase(uint32_t p, const char* name) {
    if (phase_open) nvtxRangePop();
    phase = p;
    nvtxRangePushA(name);
    phase_open = true;
  }
  ~Tracer() {
    if (phase_open) nvtxRangePop();
  }
  // brackets the work fn() enqueues on stream s; returns the record (flops may be filled in later)
  template <class F>
  size_t span(cudaStream_t s, uint32_t kind, uint32_t where, uint32_t buf, uint64_t index, uint64_t bytes,
              uint64_t flops, F&& fn) {
    Rec r{st.make_timed(), st.make_timed(), {}};
    r.e.kind = kind;
    r.e.phase = phase;
    r.e.where = where;
    r.e.buffer = buf;
    r.e.index = index;
    r.e.bytes = bytes;
    r.e.flops = flops;
    AB2_CUDA(cudaEventRecord(r.a, s));
    fn();
    AB2_CUDA(cudaEventRecord(r.b, s));
    recs.push_back(r);
    return recs.size() - 1;
  }
  void point(cudaStream_t s, uint32_t kind, uint32_t buf, uint64_t index, uint64_t bytes) {
    Rec r{st.make_timed(), nullptr, {}};
    r.b = r.a;
    r.e.kind = kind;
    r.e.phase = phase;
    r.e.where = AIRES_B200_TIER_DEVICE;
    r.e.buffer = buf;
    r.e.index = index;
    r.e.bytes = bytes;
    AB2_CUDA(cudaEventRecord(r.a, s));
    recs.push_back(r);
  }
  // after the run's last synchronisation
  // MaxMemory: records whose duration (times the share) is merge time -- fragment returns, re-sends
  std::vector<std::pair<size_t, double>> merge_share;
  void finish(cudaEvent_t t0, aires_b200_run_report& rep, const aires_b200_run_config& cfg) {
    std::vector<aires_b200_trace_event> ev;
    ev.reserve(recs.size());
    rep.h2d_count = rep.d2h_count = 0;
    rep.h2d_ms = rep.d2h_ms = 0.0;
    for (Rec& r : recs) {
      float t = 0.f, d = 0.f;
      AB2_CUDA(cudaEventElapsedTime(&t, t0, r.b));
      if (r.b != r.a) AB2_CUDA(cudaEventElapsedTime(&d, r.a, r.b));
      r.e.timestamp_ms = std::max(0.0, static_cast<double>(t));
      r.e.duration_ms = d;
      if (r.e.kind == AIRES_B200_EV_TRANSFER && r.e.where == AIRES_B200_CH_H2D) {
        rep.h2d_count++;
        rep.h2d_ms += d;
      } else if (r.e.kind == AIRES_B200_EV_TRANSFER && r.e.where == AIRES_B200_CH_D2H) {
        rep.d2h_count++;
        rep.d2h_ms += d;
      }
      ev.push_back(r.e);
    }
    rep.merge_ms = 0.0;
    for (const auto& m : merge_share) rep.merge_ms += recs[m.first].e.duration_ms * m.second;
    if (!cfg.trace) return;
    std::stable_sort(ev.begin(), ev.end(), [](const aires_b200_trace_event& x, const aires_b200_trace_event& y) {
      return x.timestamp_ms < y.timestamp_ms || (x.timestamp_ms == y.timestamp_ms && x.phase < y.phase);
    });
    cfg.trace(cfg.trace_user, ev.data(), ev.size());
  }

 private:
  bool phase_open = false;
};

// Device allocations of the run (charged against the budget), from the cached grow-only buffers.
struct Arena {
  PipeCacheImpl& c;
  size_t next = 0;
  uint64_t used = 0;
  explicit Arena(PipeCacheImpl& pc) : c(pc) {}
  void* get(size_t bytes) {
    bytes = std::max<size_t>(bytes, 256);
    if (next == c.bufs.size()) c.bufs.resize(c.bufs.size() * 2);
    DevBuf& d = c.bufs[next++];
    if (d.cap < bytes) {
      d.release();
      cudaError_t e = cudaMalloc(&d.p, bytes);
      if (e != cudaSuccess) {
        cudaGetLastError();
        d.p = nullptr;
        fail(AIRES_B200_INSUFFICIENT_DEVICE_MEMORY, "cudaMalloc of " + std::to_string(bytes) + " bytes failed");
      }
      d.cap = bytes;
    }
    used += bytes;
    return d.p;
  }
};

// Greedy maximal cuts over rows [0, n): tile [s, e) costs
//   (e - s + 1) * row_bytes + (pa[e] - pa[s]) * a_bytes + (pc[e] - pc[s]) * c_bytes,
// the calc_mem form of memory_model.hpp:84-86 extended by C.  Returns false (and the row) if a
// single row does not fit.
bool greedy_cuts(const uint64_t* pa, const uint64_t* pc, uint64_t n, uint64_t row_bytes, uint64_t a_bytes,
                 uint64_t c_bytes, uint64_t budget, std::vector<uint64_t>& cuts, uint64_t* bad) {
  auto cost = [&](uint64_t s, uint64_t e) -> unsigned __int128 {
    unsigned __int128 v = static_cast<unsigned __int128>(e - s + 1) * row_bytes +
                          static_cast<unsigned __int128>(pa[e] - pa[s]) * a_bytes;
    if (pc) v += static_cast<unsigned __int128>(pc[e] - pc[s]) * c_bytes;
    return v;
  };
  cuts.assign(1, 0);
  uint64_t s = 0;
  while (s < n) {
    if (cost(s, s + 1) > budget) {
      *bad = s;
      return false;
    }
    uint64_t lo = s + 1, hi = n;  // largest e with cost(s, e) <= budget
    while (lo < hi) {
      const uint64_t mid = lo + (hi - lo + 1) / 2;
      if (cost(s, mid) <= budget)
        lo = mid;
      else
        hi = mid - 1;
    }
    cuts.push_back(lo);
    s = lo;
  }
  return true;
}

double ms_between(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0;
  AB2_CUDA(cudaEventElapsedTime(&ms, a, b));
  return ms;
}

// Global C row offsets of a streamed tile: local offsets + the nnz of every earlier tile (a device
// running total, so the compute stream needs nothing from the host); the last block carries the
// total on to the next tile.
// The tile's {nnz, MACs, bad_row} also go straight to pinned host memory (UVA-mapped), so the host
// learns them without a copy queued behind the D2H of C on the copy engine.
__global__ void k_tile_ptr(const int64_t* __restrict__ in, int64_t n, const Ctl* __restrict__ ctl,
                           unsigned long long* __restrict__ base, uint64_t* __restrict__ out,
                           volatile unsigned long long* host) {
  const unsigned long long b = base[0];
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = static_cast<uint64_t>(in[i]) + b;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    base[1] = b + ctl->nnz;
    host[0] = ctl->nnz;
    host[1] = ctl->flops;
    host[2] = ctl->bad_row;
    __threadfence_system();
  }
}

// C's column indices on the wire: every feature column fits 16 bits (the dense accumulator is at most
// 8192 wide), so a tile's columns cross the link as u16 and host threads widen them into the
// caller's u32 / u64 array (CopyPool::widen) -- 2 bytes per C entry instead of 4 or 8 on the binding
// D2H direction.  The count comes from the tile's Ctl (the device knows it before the host does).
__global__ void k_narrow_cols(const void* __restrict__ in, uint32_t in_bytes, uint16_t* __restrict__ out,
                              const Ctl* __restrict__ ctl) {
  const uint64_t n = ctl->nnz;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  if (in_bytes == 4) {
    const uint32_t* q = static_cast<const uint32_t*>(in);
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n; i += stride)
      out[i] = static_cast<uint16_t>(q[i]);
  } else {
    const uint64_t* q = static_cast<const uint64_t*>(in);
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n; i += stride)
      out[i] = static_cast<uint16_t>(q[i]);
  }
}

// Streamed-output run (AIRES_B200_RUN_STREAM_OUT, uncapped): no sizing pass before the product.
// The caller's allocator receives an upper bound of nnz(C) up front (min(rows * n_cols, nnz(A) *
// longest X row)); A is cut into ~AB2_STREAM_TILES row blocks of equal nnz and every tile goes
// H2D (copy engine 0) -> product into staging + scan + placement (compute stream) -> D2H of its
// exact C block to the running offset (copy engine 1).  The host learns tile j's nnz (one pinned
// Ctl readback) while tile j+1 is already queued, so the D2H of C overlaps the H2D of A from the
// first tile on -- with exact sizing first, D2H cannot start before every column of A has crossed
// the link (the run's Phase I).  Same results as the exact run; out.nnz is the exact count.
void run_stream(Ctx& ctx, const aires_b200_matrix& a, const aires_b200_matrix& b, uint32_t mode, uint32_t nbuf,
                aires_b200_output& out, aires_b200_run_report& rep, Streams& st, Arena& arena, Pinned& pin, Tracer& tr,
                const aires_b200_run_config& cfg, Stager& sg, bool stage_a) {
  const uint32_t ib = a.idx_bytes, vb = mode == AIRES_B200_MODE_FP32 ? 4 : 8;
  const uint64_t n = a.n_rows;
  const uint64_t p0 = a.ptr[0], pend = a.ptr[n];
  cudaStream_t cs = ctx.stream;
  cudaEvent_t t_begin = st.make_timed(), t_p1 = st.make_timed(), t_p2 = st.make_timed(), t_end = st.make_timed();
  AB2_CUDA(cudaEventRecord(t_begin, cs));
  AB2_CUDA(cudaStreamWaitEvent(st.h2d, t_begin, 0));
  tr.set_phase(0, "aires phase I (X operand, A row_ptr)");
  std::unique_ptr<XOperand> x;
  const uint64_t x_h2d = b.location == AIRES_B200_HOST
                             ? (b.layout == AIRES_B200_CSR ? b.n_rows : b.n_cols) * 8 + 8 +
                                   (b.ptr[b.layout == AIRES_B200_CSR ? b.n_rows : b.n_cols] - b.ptr[0]) *
                                       (b.idx_bytes + b.val_bytes)
                             : 0;
  tr.span(cs, AIRES_B200_EV_TRANSFER, AIRES_B200_CH_H2D, AIRES_B200_BUF_B, 0, x_h2d, 0,
          [&] { x = make_operand(ctx, b, mode, /*temp=*/true, kPlanSlots); });
  tr.point(cs, AIRES_B200_EV_ALLOC, AIRES_B200_BUF_B, 0, x->bytes);
  rep.h2d_bytes += x_h2d;
  uint64_t* d_aptr = static_cast<uint64_t*>(arena.get((n + 1) * 8));
  tr.span(st.h2d, AIRES_B200_EV_TRANSFER, AIRES_B200_CH_H2D, AIRES_B200_BUF_A, 0, (n + 1) * 8, 0, [&] {
    AB2_CUDA(cudaMemcpyAsync(d_aptr, a.ptr, (n + 1) * 8, cudaMemcpyHostToDevice, st.h2d));
  });
  rep.h2d_bytes += (n + 1) * 8;
  // row blocks of ~equal A nnz, the first one a quarter of the others (the D2H of C starts sooner)
  const uint64_t T = static_cast<uint64_t>(std::max<int64_t>(1, option("stream_tiles", 16)));
  std::vector<uint64_t> cuts{0};
  const double unit = static_cast<double>(pend - p0) / (static_cast<double>(T) - 0.75);
  for (uint64_t i = 1; i < T; i++) {
    const uint64_t target = p0 + static_cast<uint64_t>(unit * (static_cast<double>(i) - 0.75));
    const uint64_t r = static_cast<uint64_t>(std::lower_bound(a.ptr, a.ptr + n + 1, target) - a.ptr);
    if (r > cuts.back() && r < n) cuts.push_back(r);
  }
  if (n > 0) cuts.push_back(n);
  const uint64_t n_tiles = cuts.size() - 1;
  uint64_t max_rows = 1, max_annz = 1, max_cb = 1, max_stage = 1;
  for (uint64_t j = 0; j < n_tiles; j++) {
    const uint64_t rows = cuts[j + 1] - cuts[j], an = a.ptr[cuts[j + 1]] - a.ptr[cuts[j]];
    max_rows = std::max(max_rows, rows);
    max_annz = std::max(max_annz, an);
    max_cb = std::max(max_cb, c_bound(*x, rows, an));
    max_stage = std::max(max_stage, staged_capacity(ctx, *x, rows, an));
  }
  // the caller's allocator: an upper bound of nnz(C); the exact count is reported in out.nnz
  const uint64_t bound = c_bound(*x, n, pend - p0);
  void *optr = nullptr, *oidx = nullptr, *oval = nullptr;
  int rc = out.alloc(out.user, n, bound, &optr, &oidx, &oval);
  if (rc != 0) fail(rc, "output allocator failed for a bound of " + std::to_string(bound) + " nonzeros");
  // pageable output arrays come down through the stager's pinned bounce slots
  const bool stage_c = bound * (ib + vb) >= static_cast<uint64_t>(option("stage_min_bytes", 64ll << 20)) && (!is_pinned(oidx) || !is_pinned(oval) || !is_pinned(optr));
  if (!stage_c) {
    pin.ensure(optr, (n + 1) * 8);
    pin.ensure(oidx, bound * ib);
    pin.ensure(oval, bound * vb);
  }
  // C's columns cross the link as u16 (k_narrow_cols) unless the option turns it off
  const bool narrow = x->n_cols <= 65536 && option("narrow_cols", 1) != 0;
  struct Slot {
    void *acol, *aval, *tcol, *tval, *ccol, *cval;
    uint16_t* c16;
    int64_t *cptr, *heavy, *part;
    uint64_t* optr;
    uint32_t* cnt;
    uint64_t* toff;
    cudaEvent_t loaded, computed, drained;
  };
  // AB2_TRACE=1: per-tile device timeline (loaded / computed / drained, ms from the start) on stderr
  const bool trace = trace_enabled();
  std::vector<cudaEvent_t> tl;
  if (trace)
    for (uint64_t j = 0; j < 3 * n_tiles; j++) tl.push_back(st.make_timed());
  std::vector<Slot> slot(nbuf);
  for (auto& s : slot) {
    s.acol = arena.get(max_annz * ib);
    s.aval = arena.get(max_annz * vb);
    s.tcol = arena.get(max_stage * ib);
    s.tval = arena.get(max_stage * vb);
    s.ccol = arena.get(max_cb * ib);
    s.cval = arena.get(max_cb * vb);
    s.c16 = narrow ? static_cast<uint16_t*>(arena.get(max_cb * 2)) : nullptr;
    s.cptr = static_cast<int64_t*>(arena.get((max_rows + 1) * 8));
    s.optr = static_cast<uint64_t*>(arena.get((max_rows + 1) * 8));
    s.heavy = static_cast<int64_t*>(arena.get(max_rows * 8));
    s.part = static_cast<int64_t*>(arena.get(((max_rows + kScanTile - 1) / kScanTile + 1) * 8));
    s.cnt = static_cast<uint32_t*>(arena.get(max_rows * 4));
    s.toff = static_cast<uint64_t*>(arena.get(max_rows * 8));
    s.loaded = st.make();
    s.computed = st.make();
    s.drained = st.make();
  }
  Ctl* d_ctl = static_cast<Ctl*>(arena.get(sizeof(Ctl) * std::max<uint64_t>(n_tiles, 1)));
  auto* h_rep = static_cast<unsigned long long*>(ctx.h_ctl.get(24 * std::max<uint64_t>(n_tiles, 1)));
  AB2_CUDA(cudaMemsetAsync(d_ctl, 0, sizeof(Ctl) * std::max<uint64_t>(n_tiles, 1), cs));
  auto* d_base = static_cast<unsigned long long*>(arena.get(8 * (n_tiles + 1)));
  AB2_CUDA(cudaMemsetAsync(d_base, 0, 8 * (n_tiles + 1), cs));
  cudaEvent_t e_ptr = st.make();
  AB2_CUDA(cudaEventRecord(e_ptr, st.h2d));
  AB2_CUDA(cudaStreamWaitEvent(cs, e_ptr, 0));
  AB2_CUDA(cudaEventRecord(t_p1, cs));
  cudaEvent_t e_zero = st.make();
  AB2_CUDA(cudaEventRecord(e_zero, cs));
  AB2_CUDA(cudaStreamWaitEvent(st.h2d, e_zero, 0));
  AB2_CUDA(cudaStreamWaitEvent(st.d2h, e_zero, 0));
  tr.set_phase(1, "aires phase II (tiles)");

  uint64_t running = 0, flops = 0;
  std::vector<size_t> compute_rec(n_tiles, 0);
  std::vector<uint64_t> up_bytes(n_tiles, 0);
  auto drain = [&](uint64_t j) {
    Slot& s = slot[j % nbuf];
    AB2_CUDA(cudaEventSynchronize(s.computed));
    const volatile unsigned long long* c = h_rep + 3 * j;
    if (c[2]) fail(AIRES_B200_CAPACITY_EXCEEDED, "tile staging overflow");
    const uint64_t r0 = cuts[j], rows = cuts[j + 1] - r0, nz = c[0];
    if (running + nz > bound) fail(AIRES_B200_CAPACITY_EXCEEDED, "C exceeds its bound");
    flops += c[1];
    tr.recs[compute_rec[j]].e.flops = c[1];
    AB2_CUDA(cudaStreamWaitEvent(st.d2h, s.computed, 0));  // (already complete: the host waited on it)
    const uint64_t dn_bytes = (rows + 1) * 8 + nz * ((narrow ? 2 : ib) + vb);
    tr.span(st.d2h, AIRES_B200_EV_TRANSFER, AIRES_B200_CH_D2H, AIRES_B200_BUF_C_BLOCK, j, dn_bytes, 0, [&] {
      if (narrow) {
        std::vector<std::tuple<char*, const char*, uint64_t>> direct{
            {reinterpret_cast<char*>(static_cast<uint64_t*>(optr) + r0), reinterpret_cast<const char*>(s.optr),
             (rows + 1) * 8},
            {static_cast<char*>(oval) + running * vb, static_cast<const char*>(s.cval), nz * vb}};
        if (!stage_c) {
          for (const auto& g : direct)
            if (std::get<2>(g))
              AB2_CUDA(cudaMemcpyAsync(std::get<0>(g), std::get<1>(g), std::get<2>(g), cudaMemcpyDeviceToHost, st.d2h));
          direct.clear();
        }
        sg.d2h(direct, st.d2h, {{static_cast<char*>(oidx) + running * ib, s.c16, nz, ib}});
        return;
      }
      if (stage_c) {
        sg.d2h({{reinterpret_cast<char*>(static_cast<uint64_t*>(optr) + r0), reinterpret_cast<const char*>(s.optr),
                 (rows + 1) * 8},
                {static_cast<char*>(oidx) + running * ib, static_cast<const char*>(s.ccol), nz * ib},
                {static_cast<char*>(oval) + running * vb, static_cast<const char*>(s.cval), nz * vb}},
               st.d2h);
        return;
      }
      AB2_CUDA(cudaMemcpyAsync(static_cast<uint64_t*>(optr) + r0, s.optr, (rows + 1) * 8, cudaMemcpyDeviceToHost, st.d2h));
      if (nz) {
        AB2_CUDA(cudaMemcpyAsync(static_cast<char*>(oidx) + running * ib, s.ccol, nz * ib, cudaMemcpyDeviceToHost, st.d2h));
        AB2_CUDA(cudaMemcpyAsync(static_cast<char*>(oval) + running * vb, s.cval, nz * vb, cudaMemcpyDeviceToHost, st.d2h));
      }
    });
    rep.d2h_bytes += dn_bytes;
    tr.point(st.d2h, AIRES_B200_EV_FREE, AIRES_B200_BUF_A_TILE, j, up_bytes[j]);
    AB2_CUDA(cudaEventRecord(s.drained, st.d2h));
    if (trace) AB2_CUDA(cudaEventRecord(tl[3 * j + 2], st.d2h));
    running += nz;
  };
  for (uint64_t j = 0; j < n_tiles; j++) {
    Slot& s = slot[j % nbuf];
    const uint64_t r0 = cuts[j], r1 = cuts[j + 1];
    const uint64_t q0 = a.ptr[r0], q1 = a.ptr[r1];
    if (j >= nbuf) AB2_CUDA(cudaStreamWaitEvent(st.h2d, s.drained, 0));
    up_bytes[j] = (q1 - q0) * (ib + vb);
    tr.point(st.h2d, AIRES_B200_EV_ALLOC, AIRES_B200_BUF_A_TILE, j, up_bytes[j]);
    tr.span(st.h2d, AIRES_B200_EV_TRANSFER, AIRES_B200_CH_H2D, AIRES_B200_BUF_A_TILE, j, up_bytes[j], 0, [&] {
      if (q1 > q0 && stage_a) {
        sg.h2d({{static_cast<char*>(s.acol), static_cast<const char*>(a.idx) + q0 * ib, (q1 - q0) * ib},
                {static_cast<char*>(s.aval), static_cast<const char*>(a.val) + q0 * vb, (q1 - q0) * vb}},
               st.h2d);
      } else if (q1 > q0) {
        AB2_CUDA(cudaMemcpyAsync(s.acol, static_cast<const char*>(a.idx) + q0 * ib, (q1 - q0) * ib,
                                 cudaMemcpyHostToDevice, st.h2d));
        AB2_CUDA(cudaMemcpyAsync(s.aval, static_cast<const char*>(a.val) + q0 * vb, (q1 - q0) * vb,
                                 cudaMemcpyHostToDevice, st.h2d));
      }
    });
    rep.h2d_bytes += up_bytes[j];
    AB2_CUDA(cudaEventRecord(s.loaded, st.h2d));
    if (trace) AB2_CUDA(cudaEventRecord(tl[3 * j], st.h2d));
    AB2_CUDA(cudaStreamWaitEvent(cs, s.loaded, 0));
    if (j >= nbuf) AB2_CUDA(cudaStreamWaitEvent(cs, s.drained, 0));  // staging / C block of tile j-nbuf
    TileStaged t{};
    t.aptr = d_aptr + r0;
    t.abase = q0;
    t.acol = s.acol;
    t.aval = s.aval;
    t.rows = static_cast<int64_t>(r1 - r0);
    t.a_nnz = q1 - q0;
    t.tcol = s.tcol;
    t.tval = s.tval;
    t.t_cap = staged_capacity(ctx, *x, r1 - r0, q1 - q0);
    t.cptr = s.cptr;
    t.ccol = s.ccol;
    t.cval = s.cval;
    t.heavy = s.heavy;
    t.cnt = s.cnt;
    t.toff = s.toff;
    t.part = s.part;
    t.ctl = d_ctl + j;
    compute_rec[j] = tr.span(cs, AIRES_B200_EV_COMPUTE, AIRES_B200_TIER_DEVICE, AIRES_B200_BUF_A_TILE, j, 0, 0, [&] {
      ctx.launches += tile_product_staged(ctx, *x, ib, t);
      const int g = static_cast<int>(std::min<uint64_t>((r1 - r0 + 256) / 256, static_cast<uint64_t>(ctx.sms) * 4));
      k_tile_ptr<<<g, 256, 0, cs>>>(s.cptr, static_cast<int64_t>(r1 - r0 + 1), d_ctl + j, d_base + j, s.optr,
                                    h_rep + 3 * j);
      AB2_CUDA(cudaGetLastError());
      ctx.launches++;
      if (narrow) {
        k_narrow_cols<<<ctx.sms * 4, 256, 0, cs>>>(s.ccol, ib, s.c16, d_ctl + j);
        AB2_CUDA(cudaGetLastError());
        ctx.launches++;
      }
    });
    AB2_CUDA(cudaEventRecord(s.computed, cs));
    if (trace) AB2_CUDA(cudaEventRecord(tl[3 * j + 1], cs));
    if (j >= 1) drain(j - 1);
  }
  AB2_CUDA(cudaEventRecord(t_p2, cs));
  if (n_tiles) drain(n_tiles - 1);
  if (n == 0) static_cast<uint64_t*>(optr)[0] = 0;
  cudaEvent_t e_d2h = st.make();
  AB2_CUDA(cudaEventRecord(e_d2h, st.d2h));
  AB2_CUDA(cudaStreamWaitEvent(cs, e_d2h, 0));
  tr.set_phase(2, "aires phase III (drain)");
  tr.point(cs, AIRES_B200_EV_FREE, AIRES_B200_BUF_B, 0, x->bytes);
  AB2_CUDA(cudaEventRecord(t_end, cs));
  AB2_CUDA(cudaStreamSynchronize(cs));
  sg.finish();  // pageable outputs: the last parts' host copies
  if (trace) {
    std::fprintf(stderr, "[ab2 stream] phase1 (X, A row_ptr) %.3f ms\n", ms_between(t_begin, t_p1));
    for (uint64_t j = 0; j < n_tiles; j++)
      std::fprintf(stderr, "[ab2 stream] tile %3llu  loaded %8.3f  computed %8.3f  drained %8.3f ms\n",
                   static_cast<unsigned long long>(j), ms_between(t_begin, tl[3 * j]),
                   ms_between(t_begin, tl[3 * j + 1]), ms_between(t_begin, tl[3 * j + 2]));
  }
  rep.segments = n_tiles;
  rep.flops = flops;
  rep.c_nnz = running;
  rep.peak_device_bytes = arena.used + x->bytes;
  tr.finish(t_begin, rep, cfg);
  rep.phase1_ms = ms_between(t_begin, t_p1);
  rep.phase2_ms = ms_between(t_p1, t_p2);
  rep.phase3_ms = ms_between(t_p2, t_end);
  rep.total_ms = ms_between(t_begin, t_end);
  ctx.last_ms = rep.total_ms;
  out.n_rows = n;
  out.n_cols = static_cast<uint64_t>(x->n_cols);
  out.nnz = running;
  out.flops = flops;
}

// C row pointers of a part of a tile: local offsets (cptr_local[i] - sub) + the running total; the
// part's product status (ctl->bad_row) is folded into the run's flag.
__global__ void k_part_ptr(const int64_t* __restrict__ in, int64_t n, int64_t sub, uint64_t add,
                           uint64_t* __restrict__ out, const Ctl* __restrict__ ctl, unsigned long long* bad) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = static_cast<uint64_t>(in[i] - sub) + add;
  if (blockIdx.x == 0 && threadIdx.x == 0 && ctl->bad_row) atomicMax(bad, ctl->bad_row);
}

// Capped streamed run: the report of a sized tile, written by the device into pinned host memory.
constexpr int kMaxParts = 30;
struct TileReport {
  unsigned long long nnz, flops, n_parts, bad;
  long long split[kMaxParts + 1];  // part boundaries (local rows), split[0] = 0
  long long base[kMaxParts + 1];   // cptr_local at each boundary
};

// One thread: the tile's nnz / MACs and its parts -- greedy maximal row ranges whose C entries fit
// the slot's C region (cap entries).  A row that does not fit on its own, or more than kMaxParts
// parts, sets bad.
__global__ void k_tile_report(const Ctl* __restrict__ ctl, const int64_t* __restrict__ cptr, int64_t rows,
                              uint64_t cap, volatile TileReport* rep) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  rep->nnz = ctl->nnz;
  rep->flops = ctl->flops;
  unsigned long long bad = ctl->bad_row ? 1ull : 0ull;
  int parts = 0;
  int64_t p = 0;
  rep->split[0] = 0;
  rep->base[0] = 0;
  while (p < rows && !bad) {
    int64_t lo = p, hi = rows;  // largest q with cptr[q] - cptr[p] <= cap
    while (lo < hi) {
      const int64_t mid = lo + (hi - lo + 1) / 2;
      if (static_cast<uint64_t>(cptr[mid] - cptr[p]) <= cap)
        lo = mid;
      else
        hi = mid - 1;
    }
    if (lo == p || parts == kMaxParts) {
      bad = 2;
      break;
    }
    parts++;
    rep->split[parts] = lo;
    rep->base[parts] = cptr[lo];
    p = lo;
  }
  rep->n_parts = static_cast<unsigned long long>(parts);
  rep->bad = bad;
  __threadfence_system();
}

// Capped streamed run (AIRES_B200_RUN_STREAM_OUT with a device budget): A crosses the link once.
// The exact protocol sizes C before the first byte of it is placed -- a sizing pass over A's
// column indices, then the tiles, so A's columns cross the link twice whenever the budget cannot
// hold them (cfg3 at 25%: 1.45x the algorithmic H2D bytes).  Here each tile is sized on the device
// right after its upload, from the columns already in its slot: classify + symbolic -> row counts
// -> scan -> exact local offsets -> k_tile_report (parts that fit the slot's C region, straight
// into pinned host memory).  The host reads the report of tile j while tile j+1 uploads and sizes,
// then queues tile j's product in direct mode (rows written at their exact offsets, no staging)
// part by part, each part's row_ptr rebased to the running total and drained to its final host
// position.  Tiles are cut by A bytes with C bytes estimated from the ratio observed so far (the
// first tile a quarter slot); an estimate that is off only costs an extra part (a D2H round trip
// inside the tile), never a re-upload.  Slot layout: [A cols | A vals | per-row scratch | C region].
void run_stream_capped(Ctx& ctx, const aires_b200_matrix& a, const aires_b200_matrix& b, uint32_t mode,
                       uint32_t nbuf, uint64_t budget, aires_b200_output& out, aires_b200_run_report& rep,
                       Streams& st, Arena& arena, Pinned& pin, Tracer& tr, const aires_b200_run_config& cfg, Stager& sg,
                       bool stage_a) {
  const uint32_t ib = a.idx_bytes, vb = mode == AIRES_B200_MODE_FP32 ? 4 : 8;
  const uint64_t n = a.n_rows;
  const uint64_t p0 = a.ptr[0], pend = a.ptr[n];
  cudaStream_t cs = ctx.stream;
  cudaEvent_t t_begin = st.make_timed(), t_p1 = st.make_timed(), t_p2 = st.make_timed(), t_end = st.make_timed();
  AB2_CUDA(cudaEventRecord(t_begin, cs));
  AB2_CUDA(cudaStreamWaitEvent(st.h2d, t_begin, 0));
  // X: W-slots (k_numeric3) when a 16-wide slot array takes <= 1/8 of the budget, else the lean
  // step list (fp32); 16-wide column slots for the sizing kernel when rows average >= 4 entries
  const uint64_t xk = b.layout == AIRES_B200_CSR ? b.n_rows : b.n_cols;
  const uint64_t xnnz = b.location == AIRES_B200_HOST ? b.ptr[xk] - b.ptr[0] : b.span;
  // (the step list alone: the sizing kernel walks it too, so the plain CSR is released after the build)
  uint32_t plan = mode == AIRES_B200_MODE_FP32 && (xk + 1) * 16 * 8 * 8 > budget ? kPlanStep | kPlanLean : kPlanSlots;
  if (!(plan & kPlanLean) && xk > 0 && xnnz >= 4 * xk && xk * kCSlotW * 2 * 16 <= budget) plan |= kPlanCSlots;
  // Everything the run holds on the device -- X's layouts, the build's temporaries (raw upload,
  // scratch, the plain CSR of a lean build), the tile ring -- is carved from one budget-sized region
  // (cached across calls, so no cudaMalloc / cudaFree on the run's path).
  (void)arena;
  Region rg;
  rg.init(st.c.region.get(budget), budget);
  tr.set_phase(0, "aires phase I (X operand)");
  std::unique_ptr<XOperand> x;
  const uint64_t x_h2d = b.location == AIRES_B200_HOST ? xk * 8 + 8 + xnnz * (b.idx_bytes + b.val_bytes) : 0;
  tr.span(cs, AIRES_B200_EV_TRANSFER, AIRES_B200_CH_H2D, AIRES_B200_BUF_B, 0, x_h2d, 0,
          [&] { x = make_operand(ctx, b, mode, /*temp=*/true, plan, &rg); });
  tr.point(cs, AIRES_B200_EV_ALLOC, AIRES_B200_BUF_B, 0, rg.lo);
  const uint64_t x_keep = rg.lo;
  rep.h2d_bytes += x_h2d;
  Ctl* d_ctl = static_cast<Ctl*>(rg.keep(sizeof(Ctl) * nbuf * (kMaxParts + 1)));
  auto* d_bad = static_cast<unsigned long long*>(rg.keep(8));  // max of every part's ctl->bad_row
  AB2_CUDA(cudaMemsetAsync(d_bad, 0, 8, cs));
  const uint64_t fixed = rg.lo + (64 << 10);
  if (budget <= fixed)
    fail(AIRES_B200_INSUFFICIENT_DEVICE_MEMORY, "device budget " + std::to_string(budget) +
                                                    " does not cover the resident operand and row arrays (" +
                                                    std::to_string(fixed) + " bytes)");
  const uint64_t slot_bytes = ((budget - fixed) / nbuf) & ~uint64_t(255);
  std::vector<char*> slot_mem(nbuf);
  for (uint32_t s = 0; s < nbuf; s++) slot_mem[s] = static_cast<char*>(rg.keep(slot_bytes));
  auto* h_rep = static_cast<TileReport*>(ctx.h_ctl.get(sizeof(TileReport) * nbuf));
  // the caller's allocator: an upper bound of nnz(C); the exact count is reported in out.nnz
  const uint64_t bound = c_bound(*x, n, pend - p0);
  void *optr = nullptr, *oidx = nullptr, *oval = nullptr;
  int rc = out.alloc(out.user, n, bound, &optr, &oidx, &oval);
  if (rc != 0) fail(rc, "output allocator failed for a bound of " + std::to_string(bound) + " nonzeros");
  const bool stage_c = bound * (ib + vb) >= static_cast<uint64_t>(option("stage_min_bytes", 64ll << 20)) && (!is_pinned(oidx) || !is_pinned(oval) || !is_pinned(optr));
  if (!stage_c) {
    pin.ensure(optr, (n + 1) * 8);
    pin.ensure(oidx, bound * ib);
    pin.ensure(oval, bound * vb);
  }
  AB2_CUDA(cudaEventRecord(t_p1, cs));
  tr.set_phase(1, "aires phase II (tiles)");

  auto r256 = [](uint64_t v) { return (v + 255) & ~uint64_t(255); };
  struct Tile {
    uint64_t r0, r1, q0, q1;
    uint32_t slot;
    uint64_t* aptr;  // the tile's A row pointers (absolute), uploaded with its columns and values
    char *acol, *aval, *ccol, *cval;
    int64_t *heavy, *cptr, *rflops;
    uint64_t* toff;
    uint64_t* optr;
    int32_t* cnt;
    uint64_t c_cap;
    cudaEvent_t sized;
    cudaEvent_t tl_loaded = nullptr, tl_computed = nullptr, tl_drained = nullptr;  // AB2_TRACE
    uint64_t parts = 0;
    uint64_t up_bytes = 0;
  };
  // AB2_TRACE=1: per-tile device timeline (loaded / sized / last part computed / drained) on stderr
  const bool trace = trace_enabled();
  std::vector<cudaEvent_t> slot_free(nbuf, nullptr);
  // C entries per A entry, observed; the first tile assumes the mean X row length
  double rho = std::max(0.05, std::min(static_cast<double>(x->n_cols),
                                       static_cast<double>(x->nnz) / static_cast<double>(std::max<int64_t>(x->K, 1))));
  uint64_t seen_a = 0, seen_c = 0, cursor = 0, running = 0, flops = 0, parts_total = 0;
  auto bytes_of = [&](uint64_t r0, uint64_t r1, double ratio) {
    const uint64_t an = a.ptr[r1] - a.ptr[r0];
    return static_cast<double>(r256(an * ib) + r256(an * vb)) + static_cast<double>(r256((r1 - r0 + 1) * 8)) * 6 +
           static_cast<double>(r256((r1 - r0 + 1) * 4)) + ratio * 1.1 * static_cast<double>(an) * (ib + vb) + 1024.0;
  };
  std::vector<Tile> tiles;
  auto launch_tile = [&]() {
    Tile t{};
    t.slot = static_cast<uint32_t>(tiles.size() % nbuf);
    t.r0 = cursor;
    const double cap_bytes = tiles.empty() ? static_cast<double>(slot_bytes) / 4 : static_cast<double>(slot_bytes);
    uint64_t lo = cursor + 1, hi = n;  // largest r1 whose estimated bytes fit
    if (bytes_of(cursor, cursor + 1, 0.0) + static_cast<double>(x->n_cols) * (ib + vb) > static_cast<double>(slot_bytes))
      fail(AIRES_B200_ROW_TOO_LARGE, "row " + std::to_string(cursor) + " does not fit a ring slot of " +
                                         std::to_string(slot_bytes) + " bytes");
    while (lo < hi) {
      const uint64_t mid = lo + (hi - lo + 1) / 2;
      if (bytes_of(cursor, mid, rho) <= cap_bytes)
        lo = mid;
      else
        hi = mid - 1;
    }
    t.r1 = lo;
    t.q0 = a.ptr[t.r0];
    t.q1 = a.ptr[t.r1];
    const uint64_t rows = t.r1 - t.r0, an = t.q1 - t.q0;
    char* m = slot_mem[t.slot];
    auto take = [&](uint64_t bytes) {
      char* q = m;
      m += r256(bytes);
      return q;
    };
    t.aptr = reinterpret_cast<uint64_t*>(take((rows + 1) * 8));
    t.acol = take(std::max<uint64_t>(an, 1) * ib);
    t.aval = take(std::max<uint64_t>(an, 1) * vb);
    t.heavy = reinterpret_cast<int64_t*>(take((rows + 1) * 8));
    t.toff = reinterpret_cast<uint64_t*>(take((rows + 1) * 8));
    t.cptr = reinterpret_cast<int64_t*>(take((rows + 1) * 8));
    t.optr = reinterpret_cast<uint64_t*>(take((rows + 1) * 8));
    t.rflops = reinterpret_cast<int64_t*>(take((rows + 1) * 8));
    t.cnt = reinterpret_cast<int32_t*>(take((rows + 1) * 4));
    const uint64_t used = static_cast<uint64_t>(m - slot_mem[t.slot]);
    if (used > slot_bytes) fail(AIRES_B200_INSUFFICIENT_DEVICE_MEMORY, "ring slot overflow");
    // C region: c_cap column indices, then (256-byte aligned) c_cap values
    t.c_cap = slot_bytes - used > 256 ? (slot_bytes - used - 256) / (ib + vb) : 0;
    t.ccol = m;
    t.cval = m + r256(t.c_cap * ib);
    // upload (copy engine 0) once the slot's previous tile has drained
    if (slot_free[t.slot]) AB2_CUDA(cudaStreamWaitEvent(st.h2d, slot_free[t.slot], 0));
    const uint64_t up_bytes = (rows + 1) * 8 + an * (ib + vb);
    const uint64_t j = tiles.size();
    tr.point(st.h2d, AIRES_B200_EV_ALLOC, AIRES_B200_BUF_A_TILE, j, up_bytes);
    tr.span(st.h2d, AIRES_B200_EV_TRANSFER, AIRES_B200_CH_H2D, AIRES_B200_BUF_A_TILE, j, up_bytes, 0, [&] {
      if (stage_a) {
        sg.h2d({{reinterpret_cast<char*>(t.aptr), reinterpret_cast<const char*>(a.ptr + t.r0), (rows + 1) * 8},
                {t.acol, static_cast<const char*>(a.idx) + t.q0 * ib, an * ib},
                {t.aval, static_cast<const char*>(a.val) + t.q0 * vb, an * vb}},
               st.h2d);
        return;
      }
      AB2_CUDA(cudaMemcpyAsync(t.aptr, a.ptr + t.r0, (rows + 1) * 8, cudaMemcpyHostToDevice, st.h2d));
      if (an) {
        AB2_CUDA(cudaMemcpyAsync(t.acol, static_cast<const char*>(a.idx) + t.q0 * ib, an * ib, cudaMemcpyHostToDevice, st.h2d));
        AB2_CUDA(cudaMemcpyAsync(t.aval, static_cast<const char*>(a.val) + t.q0 * vb, an * vb, cudaMemcpyHostToDevice, st.h2d));
      }
    });
    t.up_bytes = up_bytes;
    rep.h2d_bytes += up_bytes;
    cudaEvent_t loaded = st.make();
    AB2_CUDA(cudaEventRecord(loaded, st.h2d));
    if (trace) {
      t.tl_loaded = st.make_timed();
      AB2_CUDA(cudaEventRecord(t.tl_loaded, st.h2d));
    }
    // size it on the device (sizing stream, so tile j's product never queues behind tile j+1's
    // upload): row counts -> local exact offsets -> parts that fit the C region
    cudaStream_t zs = st.aux;
    AB2_CUDA(cudaStreamWaitEvent(zs, loaded, 0));
    Ctl* c = d_ctl + t.slot * (kMaxParts + 1);
    AB2_CUDA(cudaMemsetAsync(c, 0, sizeof(Ctl) * (kMaxParts + 1), zs));
    StreamSwap swap(ctx, zs);
    tr.span(zs, AIRES_B200_EV_COMPUTE, AIRES_B200_TIER_DEVICE, AIRES_B200_BUF_A_TILE, j, 0, 0, [&] {
      TileSym sy{};
      sy.aptr = t.aptr;
      sy.abase = t.q0;
      sy.acol = t.acol;
      sy.rows = static_cast<int64_t>(rows);
      sy.cnt = t.cnt;
      sy.rflops = t.rflops;
      sy.heavy = t.heavy;
      sy.ctl = c;
      ctx.launches += tile_symbolic(ctx, *x, ib, sy);
      const int64_t nb = (static_cast<int64_t>(rows) + kScanTile - 1) / kScanTile;
      int64_t* part = reinterpret_cast<int64_t*>(t.optr);  // scan partials: optr is written later
      if (rows > 0) {
        k_scan_reduce<<<static_cast<unsigned>(nb), kScanThreads, 0, zs>>>(t.cnt, static_cast<int64_t>(rows), part);
        k_scan_part<<<1, 1024, 0, zs>>>(part, nb, c);
        k_scan_down<<<static_cast<unsigned>(nb), kScanThreads, 0, zs>>>(t.cnt, static_cast<int64_t>(rows), part, t.cptr);
        ctx.launches += 3;
      } else {
        AB2_CUDA(cudaMemsetAsync(t.cptr, 0, 8, zs));
      }
      k_tile_report<<<1, 32, 0, zs>>>(c, t.cptr, static_cast<int64_t>(rows), t.c_cap, h_rep + t.slot);
      AB2_CUDA(cudaGetLastError());
      ctx.launches++;
    });
    t.sized = trace ? st.make_timed() : st.make();
    AB2_CUDA(cudaEventRecord(t.sized, zs));
    cursor = t.r1;
    tiles.push_back(t);
  };

  size_t j = 0;
  if (cursor < n) launch_tile();
  while (j < tiles.size()) {
    while (cursor < n && tiles.size() - j < nbuf) launch_tile();  // later tiles upload and size meanwhile
    Tile& t = tiles[j];
    AB2_CUDA(cudaEventSynchronize(t.sized));
    const TileReport& r = h_rep[t.slot];
    if (r.bad) fail(AIRES_B200_CAPACITY_EXCEEDED, r.bad == 2 ? "tile C row does not fit the slot's C region"
                                                             : "tile sizing overflow");
    const uint64_t rows = t.r1 - t.r0, tnnz = r.nnz;
    flops += r.flops;
    seen_a += t.q1 - t.q0;
    seen_c += tnnz;
    if (seen_a) rho = std::max(0.01, static_cast<double>(seen_c) / static_cast<double>(seen_a));
    if (running + tnnz > bound) fail(AIRES_B200_CAPACITY_EXCEEDED, "C exceeds its bound");
    const int n_parts = static_cast<int>(r.n_parts);
    std::vector<long long> split(r.split, r.split + n_parts + 1), base(r.base, r.base + n_parts + 1);
    cudaEvent_t prev_drain = nullptr;
    Ctl* c = d_ctl + t.slot * (kMaxParts + 1);
    for (int q = 0; q < n_parts; q++) {
      const uint64_t pa = static_cast<uint64_t>(split[q]), pb = static_cast<uint64_t>(split[q + 1]);
      const uint64_t pn = static_cast<uint64_t>(base[q + 1] - base[q]);
      if (prev_drain) AB2_CUDA(cudaStreamWaitEvent(cs, prev_drain, 0));  // the C region is reused
      TilePass tp{};
      tp.aptr = t.aptr + pa;
      tp.abase = t.q0;
      tp.acol = t.acol;
      tp.aval = t.aval;
      tp.rows = static_cast<int64_t>(pb - pa);
      tp.cpos = t.cptr + pa;
      tp.cbase = base[q];
      tp.ccol = t.ccol;
      tp.cval = t.cval;
      tp.c_cap = t.c_cap;
      tp.heavy = t.heavy;
      tp.cnt = reinterpret_cast<uint32_t*>(t.cnt) + pa;  // scratch (the counts are in cptr now)
      tp.toff = t.toff;
      tp.ctl = c + 1 + q;
      tr.span(cs, AIRES_B200_EV_COMPUTE, AIRES_B200_TIER_DEVICE, AIRES_B200_BUF_A_TILE, j, 0, q == 0 ? r.flops : 0, [&] {
        ctx.launches += tile_product(ctx, *x, ib, tp);
        const int g = static_cast<int>(std::min<uint64_t>((pb - pa + 256) / 256, static_cast<uint64_t>(ctx.sms) * 4));
        k_part_ptr<<<g, 256, 0, cs>>>(t.cptr + pa, static_cast<int64_t>(pb - pa + 1), base[q], running, t.optr + pa,
                                      c + 1 + q, d_bad);
        AB2_CUDA(cudaGetLastError());
        ctx.launches++;
      });
      cudaEvent_t computed = trace ? st.make_timed() : st.make();
      AB2_CUDA(cudaEventRecord(computed, cs));
      AB2_CUDA(cudaStreamWaitEvent(st.d2h, computed, 0));
      const uint64_t dn_bytes = (pb - pa + 1) * 8 + pn * (ib + vb);
      tr.span(st.d2h, AIRES_B200_EV_TRANSFER, AIRES_B200_CH_D2H, AIRES_B200_BUF_C_BLOCK, j, dn_bytes, 0, [&] {
        if (stage_c) {
          sg.d2h({{reinterpret_cast<char*>(static_cast<uint64_t*>(optr) + t.r0 + pa),
                   reinterpret_cast<const char*>(t.optr + pa), (pb - pa + 1) * 8},
                  {static_cast<char*>(oidx) + running * ib, t.ccol, pn * ib},
                  {static_cast<char*>(oval) + running * vb, t.cval, pn * vb}},
                 st.d2h);
          return;
        }
        AB2_CUDA(cudaMemcpyAsync(static_cast<uint64_t*>(optr) + t.r0 + pa, t.optr + pa, (pb - pa + 1) * 8,
                                 cudaMemcpyDeviceToHost, st.d2h));
        if (pn) {
          AB2_CUDA(cudaMemcpyAsync(static_cast<char*>(oidx) + running * ib, t.ccol, pn * ib, cudaMemcpyDeviceToHost, st.d2h));
          AB2_CUDA(cudaMemcpyAsync(static_cast<char*>(oval) + running * vb, t.cval, pn * vb, cudaMemcpyDeviceToHost, st.d2h));
        }
      });
      rep.d2h_bytes += dn_bytes;
      if (q + 1 == n_parts) tr.point(st.d2h, AIRES_B200_EV_FREE, AIRES_B200_BUF_A_TILE, j, t.up_bytes);
      prev_drain = trace ? st.make_timed() : st.make();
      AB2_CUDA(cudaEventRecord(prev_drain, st.d2h));
      if (trace) t.tl_computed = computed;
      running += pn;
      parts_total++;
    }
    t.parts = static_cast<uint64_t>(n_parts);
    if (trace) t.tl_drained = prev_drain;
    if (n_parts == 0) {  // rows without entries still get their row pointers
      tr.point(st.d2h, AIRES_B200_EV_FREE, AIRES_B200_BUF_A_TILE, j, t.up_bytes);
      prev_drain = st.make();
      AB2_CUDA(cudaEventRecord(prev_drain, st.d2h));
    }
    (void)rows;
    slot_free[t.slot] = prev_drain;
    j++;
  }
  AB2_CUDA(cudaEventRecord(t_p2, cs));
  if (n == 0) static_cast<uint64_t*>(optr)[0] = 0;
  cudaEvent_t e_d2h = st.make();
  AB2_CUDA(cudaEventRecord(e_d2h, st.d2h));
  AB2_CUDA(cudaStreamWaitEvent(cs, e_d2h, 0));
  tr.set_phase(2, "aires phase III (drain)");
  tr.point(cs, AIRES_B200_EV_FREE, AIRES_B200_BUF_B, 0, x_keep);
  AB2_CUDA(cudaEventRecord(t_end, cs));
  AB2_CUDA(cudaStreamSynchronize(cs));
  sg.finish();  // pageable outputs: the last parts' host copies
  {
    unsigned long long hb = 0;
    AB2_CUDA(cudaMemcpy(&hb, d_bad, 8, cudaMemcpyDeviceToHost));
    if (hb == 2) fail(AIRES_B200_CUDA_ERROR, "numeric row counts disagree with the sizing pass");
    if (hb) fail(AIRES_B200_CAPACITY_EXCEEDED, "tile output overflow");
  }
  if (trace) {
    std::fprintf(stderr, "[ab2 capped] phase1 (X operand) %.3f ms, slot %llu bytes, %zu tiles\n",
                 ms_between(t_begin, t_p1), static_cast<unsigned long long>(slot_bytes), tiles.size());
    for (size_t q = 0; q < tiles.size(); q++) {
      const Tile& t = tiles[q];
      std::fprintf(stderr, "[ab2 capped] tile %3zu rows %8llu A %10llu  loaded %8.3f sized %8.3f computed %8.3f drained %8.3f  parts %llu\n",
                   q, static_cast<unsigned long long>(t.r1 - t.r0), static_cast<unsigned long long>(t.q1 - t.q0),
                   ms_between(t_begin, t.tl_loaded), ms_between(t_begin, t.sized),
                   t.tl_computed ? ms_between(t_begin, t.tl_computed) : 0.0,
                   t.tl_drained ? ms_between(t_begin, t.tl_drained) : 0.0, static_cast<unsigned long long>(t.parts));
    }
  }
  rep.segments = parts_total;
  rep.flops = flops;
  rep.c_nnz = running;
  rep.peak_device_bytes = rg.peak;
  tr.finish(t_begin, rep, cfg);
  rep.phase1_ms = ms_between(t_begin, t_p1);
  rep.phase2_ms = ms_between(t_p1, t_p2);
  rep.phase3_ms = ms_between(t_p2, t_end);
  rep.total_ms = ms_between(t_begin, t_end);
  ctx.last_ms = rep.total_ms;
  out.n_rows = n;
  out.n_cols = static_cast<uint64_t>(x->n_cols);
  out.nnz = running;
  out.flops = flops;
}

}  // namespace

void destroy_pipe_cache(void* p) { delete static_cast<PipeCacheImpl*>(p); }

void run_pipeline(Ctx& ctx, const aires_b200_matrix& a, const aires_b200_matrix& b, const aires_b200_run_config& cfg,
                  aires_b200_output& out, aires_b200_run_report& rep) {
  if (a.layout != AIRES_B200_CSR || a.location != AIRES_B200_HOST)
    fail(AIRES_B200_INVALID_ARGUMENT, "run: A must be a host CSR matrix");
  if ((a.idx_bytes != 4 && a.idx_bytes != 8) || (a.val_bytes != 4 && a.val_bytes != 8))
    fail(AIRES_B200_INVALID_ARGUMENT, "run: A idx_bytes/val_bytes must be 4 or 8");
  if (!out.alloc) fail(AIRES_B200_INVALID_ARGUMENT, "output allocator is null");
  if (out.location != AIRES_B200_HOST) fail(AIRES_B200_INVALID_ARGUMENT, "run: C is drained to host memory");
  if (a.n_cols != b.n_rows)
    fail(AIRES_B200_DIMENSION_MISMATCH,
         "inner dimensions " + std::to_string(a.n_cols) + " and " + std::to_string(b.n_rows) + " differ");
  uint32_t mode = cfg.mode;
  if (mode == AIRES_B200_MODE_AUTO) mode = out.val_bytes == 8 ? AIRES_B200_MODE_FP64_EXACT : AIRES_B200_MODE_FP32;
  const uint32_t vb = mode == AIRES_B200_MODE_FP32 ? 4 : 8;
  if (out.val_bytes != vb) fail(AIRES_B200_INVALID_ARGUMENT, "output value width must match the arithmetic mode");
  if (a.val_bytes != vb) fail(AIRES_B200_INVALID_ARGUMENT, "run: A value width must match the arithmetic mode");
  if (out.idx_bytes != a.idx_bytes) fail(AIRES_B200_INVALID_ARGUMENT, "run: C index width must equal A's");
  const uint32_t ib = a.idx_bytes;
  const uint64_t n = a.n_rows;
  const uint64_t p0 = a.ptr[0], pend = a.ptr[n];
  if (pend < p0 || pend > a.span) fail(AIRES_B200_INDEX_OUT_OF_RANGE, "A row pointers exceed the index span");
  const uint32_t nbuf = std::max<uint32_t>(2, std::min<uint32_t>(cfg.n_buffers ? cfg.n_buffers : 2, 8));
  std::memset(&rep, 0, sizeof(rep));
  // AB2_TRACE=1: host-side milestones on stderr (where the wall time of a run goes)
  const bool trace = trace_enabled();
  const auto t_host0 = std::chrono::steady_clock::now();
  auto mark = [&](const char* what) {
    if (!trace) return;
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_host0).count();
    std::fprintf(stderr, "[ab2 run] %8.3f ms  %s\n", ms, what);
  };

  if (!ctx.pipe) ctx.pipe = new PipeCacheImpl();
  Streams st(*static_cast<PipeCacheImpl*>(ctx.pipe));
  cudaStream_t cs = ctx.stream;
  Arena arena(*static_cast<PipeCacheImpl*>(ctx.pipe));
  Pinned pin;
  SyncGuard sync{{cs, st.h2d, st.d2h, st.aux}};  // destroyed before pin (no copy outlives its buffers)
  Tracer tr(st);
  cudaEvent_t t_begin = st.make_timed(), t_p1 = st.make_timed(), t_p2 = st.make_timed(), t_end = st.make_timed();
  // tiles hold whole C rows in the dense accumulator: wider features are the in-core product's
  // column tiles (aires_b200_spgemm) -- the drop-in's run_aires falls back to the reference scheduler
  if (static_cast<int64_t>(b.n_cols) > wide_threshold(mode))
    fail(AIRES_B200_UNSUPPORTED_FORMAT, "run: feature matrix has " + std::to_string(b.n_cols) +
                                            " columns; the out-of-core pipeline supports " +
                                            std::to_string(wide_threshold(mode)));
  const bool streamed = (cfg.flags & AIRES_B200_RUN_STREAM_OUT) && cfg.c_aware != 2 &&
                        (cfg.device_budget == 0 || cfg.c_aware == 1) &&
                        static_cast<int64_t>(b.n_cols) <= wide_threshold(mode);
  // streamed runs move pageable A arrays through pinned bounce slots instead of registering them
  const bool stage_a = streamed && (pend - p0) * (ib + vb) >= static_cast<uint64_t>(option("stage_min_bytes", 64ll << 20)) &&
                       (!is_pinned(static_cast<const char*>(a.idx) + p0 * ib) ||
                        !is_pinned(static_cast<const char*>(a.val) + p0 * vb));
  pin.ensure(a.ptr, (n + 1) * 8);
  if (!stage_a) {
    pin.ensure(static_cast<const char*>(a.idx) + p0 * ib, (pend - p0) * ib);
    pin.ensure(static_cast<const char*>(a.val) + p0 * vb, (pend - p0) * vb);
  }
  if (streamed) {
    PipeCacheImpl& pc = *static_cast<PipeCacheImpl*>(ctx.pipe);
    const uint32_t nb = cfg.n_buffers ? nbuf : 3;
    Stager sg(pc.copy_pool(), pc.bounce_up, pc.bounce_down, nb, pc.stage_ev, ctx.device);
    if (cfg.device_budget == 0)
      run_stream(ctx, a, b, mode, nb, out, rep, st, arena, pin, tr, cfg, sg, stage_a);
    else
      run_stream_capped(ctx, a, b, mode, nb, cfg.device_budget, out, rep, st, arena, pin, tr, cfg, sg, stage_a);
    return;
  }

  // ---------------- Phase I ----------------
  mark("pinned checks done");
  AB2_CUDA(cudaEventRecord(t_begin, cs));
  AB2_CUDA(cudaStreamWaitEvent(st.h2d, t_begin, 0));
  tr.set_phase(0, "aires phase I (X operand, sizing pass)");
  // lean operand: the step-list layout (fp32) or W-slots (fp64-exact) plus the plain CSR, which
  // the sizing pass reads directly (the device staging of a host X's raw arrays is transient and
  // not charged to the budget)
  // (+ 16-wide column slots for the sizing pass when X rows average >= 4 entries and the slots take
  // <= 1/16 of a capped budget: the lane-per-entry walk over the plain CSR serialises long rows)
  uint32_t plan = mode == AIRES_B200_MODE_FP32 ? kPlanStep : kPlanSlots;
  {
    const uint64_t xk = b.layout == AIRES_B200_CSR ? b.n_rows : b.n_cols;
    const uint64_t xnnz = b.location == AIRES_B200_HOST ? b.ptr[(b.layout == AIRES_B200_CSR ? b.n_rows : b.n_cols)] - b.ptr[0]
                                                        : b.span;
    const uint64_t cs_bytes = xk * kCSlotW * 2;
    if (xk > 0 && xnnz >= 4 * xk && (cfg.device_budget == 0 || cs_bytes * 16 <= cfg.device_budget) &&
        option("run_cslots", 1) != 0)
      plan |= kPlanCSlots;
  }
  std::unique_ptr<XOperand> x;
  const uint64_t xk_ = b.layout == AIRES_B200_CSR ? b.n_rows : b.n_cols;
  const uint64_t x_h2d =
      b.location == AIRES_B200_HOST ? xk_ * 8 + 8 + (b.ptr[xk_] - b.ptr[0]) * (b.idx_bytes + b.val_bytes) : 0;
  tr.span(cs, AIRES_B200_EV_TRANSFER, AIRES_B200_CH_H2D, AIRES_B200_BUF_B, 0, x_h2d, 0,
          [&] { x = make_operand(ctx, b, mode, /*temp=*/true, plan); });
  mark("operand built (host synced)");
  // Uncapped runs keep A's column indices resident and stream them right after X (X first: its
  // build synchronises the host once and must not queue behind A on the link).
  const uint64_t a_col_bytes = (pend - p0) * ib;
  const bool maxmem = cfg.c_aware == 2;  // the MaxMemory baseline (scheduler.hpp:174-293)
  const bool early_cols = !maxmem && cfg.device_budget == 0 && option("run_resident_cols", 1) != 0 && n > 0;
  char* d_acol_full = nullptr;
  std::vector<uint64_t> early_cuts;
  std::vector<cudaEvent_t> early_ev;
  uint64_t bad = 0;
  if (early_cols) {
    d_acol_full = static_cast<char*>(arena.get(a_col_bytes));
    if (!greedy_cuts(a.ptr, nullptr, n, 0, ib, 0, std::max<uint64_t>(a_col_bytes / 8, 16ull << 20), early_cuts, &bad))
      early_cuts = {0, n};  // a row longer than the chunk target: one chunk
    for (size_t c = 0; c + 1 < early_cuts.size(); c++) {
      const uint64_t q0 = a.ptr[early_cuts[c]], q1 = a.ptr[early_cuts[c + 1]];
      tr.span(st.h2d, AIRES_B200_EV_TRANSFER, AIRES_B200_CH_H2D, AIRES_B200_BUF_A, c + 1, (q1 - q0) * ib, 0, [&] {
        if (q1 > q0)
          AB2_CUDA(cudaMemcpyAsync(d_acol_full + (q0 - p0) * ib, static_cast<const char*>(a.idx) + q0 * ib,
                                   (q1 - q0) * ib, cudaMemcpyHostToDevice, st.h2d));
      });
      early_ev.push_back(st.make());
      AB2_CUDA(cudaEventRecord(early_ev.back(), st.h2d));
    }
  }
  uint64_t x_dev = x->bytes;
  if (b.location == AIRES_B200_HOST) {
    const uint64_t raw = ctx.x_ptr.cap + ctx.x_idx.cap + ctx.x_val.cap;
    x_dev = x_dev > raw ? x_dev - raw : 0;
  }
  tr.point(cs, AIRES_B200_EV_ALLOC, AIRES_B200_BUF_B, 0, x_dev);
  rep.h2d_bytes += x_h2d;
  // resident per-row arrays: A row_ptr, C row_ptr, counts
  mark("A columns enqueued");
  uint64_t* d_aptr = static_cast<uint64_t*>(arena.get((n + 1) * 8));
  int64_t* d_cptr = static_cast<int64_t*>(arena.get((n + 1) * 8));
  int32_t* d_cnt = static_cast<int32_t*>(arena.get(std::max<uint64_t>(n, 1) * 4));
  tr.span(st.h2d, AIRES_B200_EV_TRANSFER, AIRES_B200_CH_H2D, AIRES_B200_BUF_A, 0, (n + 1) * 8, 0, [&] {
    AB2_CUDA(cudaMemcpyAsync(d_aptr, a.ptr, (n + 1) * 8, cudaMemcpyHostToDevice, st.h2d));
  });
  rep.h2d_bytes += (n + 1) * 8;
  cudaEvent_t e_ptr = st.make();
  AB2_CUDA(cudaEventRecord(e_ptr, st.h2d));

  // budget left for the ring: per slot A col/val + C col/val + per-row scratch
  const uint64_t fixed = x_dev + arena.used + (64 << 10) + 8 * sizeof(Ctl);
  uint64_t budget = cfg.device_budget;
  // Uncapped (device_budget 0): no cap to divide -- every buffer is sized to what the run needs and
  // an allocation failure surfaces as insufficient_device_memory (cudaMemGetInfo would wait for
  // the copies already in flight).
  if (budget == 0) budget = fixed + (uint64_t(1) << 60);
  mark("budget sized");
  if (budget <= fixed)
    fail(AIRES_B200_INSUFFICIENT_DEVICE_MEMORY, "device budget " + std::to_string(budget) +
                                                    " does not cover the resident operand and row arrays (" +
                                                    std::to_string(fixed) + " bytes)");
  // A's column indices stay resident after the sizing pass when they take at most half of the
  // budget left (then Phase II streams only A's values): one column pass over the link instead of two
  const bool cols_resident =
      early_cols || (!maxmem && option("run_resident_cols", 1) != 0 && budget - fixed >= 2 * a_col_bytes + 4096);
  if (cols_resident && !d_acol_full) d_acol_full = static_cast<char*>(arena.get(a_col_bytes));
  const uint64_t fixed2 = fixed + (cols_resident && !early_cols ? std::max<uint64_t>(a_col_bytes, 256) : 0);
  const uint64_t slot_budget = (budget - fixed2) / nbuf;
  // per-row scratch per slot: heavy (8) + cnt (4) + toff (8) + rflops (8)
  const uint64_t row_bytes = 28;
  const uint64_t a_tile_bytes = cols_resident ? vb : ib + vb;  // A bytes per entry streamed in Phase II

  // Symbolic chunks: A columns only, sized like a slot's A + C space.
  std::vector<uint64_t> sym_cuts;
  // (uncapped runs: chunks of ~1/8 of A's columns so the copies overlap the sizing kernels)
  const uint64_t sym_budget = cfg.device_budget == 0
                                  ? std::min<uint64_t>(slot_budget, std::max<uint64_t>(a_col_bytes / 8, 16ull << 20))
                                  : slot_budget;
  if (early_cols)
    sym_cuts = early_cuts;
  else if (!greedy_cuts(a.ptr, nullptr, n, row_bytes, ib, 0, sym_budget, sym_cuts, &bad))
    fail(AIRES_B200_ROW_TOO_LARGE, "row " + std::to_string(bad) + " does not fit a ring slot of " +
                                       std::to_string(slot_budget) + " bytes");
  // shift to relative offsets: greedy_cuts used absolute pointers; differences are what count
  struct Slot {
    void* acol = nullptr;
    void* aval = nullptr;
    void* ccol = nullptr;
    void* cval = nullptr;
    int64_t* heavy = nullptr;
    uint32_t* cnt = nullptr;
    uint64_t* toff = nullptr;
    int64_t* rflops = nullptr;
    Ctl* ctl = nullptr;
    cudaEvent_t loaded = nullptr, computed = nullptr, drained = nullptr;
    uint64_t a_cap = 0, c_cap = 0, rows_cap = 0;
  };
  // Slot memory is carved from one allocation per slot (reused by both phases).
  std::vector<Slot> slot(nbuf);
  // Capped runs give every slot the whole per-slot budget once; uncapped runs size the slots to
  // the largest chunk (Phase I) and again to the largest tile (Phase II).
  auto carve_bytes = [&](uint64_t rows, uint64_t a_nnz, bool with_val, uint64_t c_nnz) {
    auto r = [](uint64_t b) { return (b + 255) & ~uint64_t(255); };
    return (cols_resident ? 0 : r(a_nnz * ib)) + (with_val ? r(a_nnz * vb) : 0) + (c_nnz ? r(c_nnz * ib) + r(c_nnz * vb) : 0) +
           r(std::max<uint64_t>(rows, 1) * 8) * 3 + r(std::max<uint64_t>(rows, 1) * 4);
  };
  uint64_t slot_cap = slot_budget;
  if (cfg.device_budget == 0) {
    slot_cap = 0;
    for (size_t c = 0; c + 1 < sym_cuts.size(); c++)
      slot_cap = std::max(slot_cap, carve_bytes(sym_cuts[c + 1] - sym_cuts[c], a.ptr[sym_cuts[c + 1]] - a.ptr[sym_cuts[c]],
                                                false, 0));
  }
  std::vector<char*> slot_mem(nbuf);
  for (uint32_t s = 0; s < nbuf; s++) {
    slot_mem[s] = static_cast<char*>(arena.get(slot_cap + 4096));
    slot[s].loaded = st.make();
    slot[s].computed = st.make();
    slot[s].drained = st.make();
  }
  Ctl* d_ctl = static_cast<Ctl*>(arena.get(sizeof(Ctl) * 2));
  AB2_CUDA(cudaMemsetAsync(d_ctl, 0, sizeof(Ctl) * 2, cs));
  AB2_CUDA(cudaStreamWaitEvent(cs, e_ptr, 0));
  auto carve = [&](uint32_t s, uint64_t rows, uint64_t a_nnz, bool with_val, uint64_t c_nnz) {
    char* m = slot_mem[s];
    auto take = [&](uint64_t bytes) {
      char* p = m;
      m += (bytes + 255) & ~uint64_t(255);
      return static_cast<void*>(p);
    };
    Slot& sl = slot[s];
    sl.acol = cols_resident ? nullptr : take(a_nnz * ib);
    sl.aval = with_val ? take(a_nnz * vb) : nullptr;
    sl.ccol = c_nnz ? take(c_nnz * ib) : nullptr;
    sl.cval = c_nnz ? take(c_nnz * vb) : nullptr;
    sl.heavy = static_cast<int64_t*>(take(std::max<uint64_t>(rows, 1) * 8));
    sl.cnt = static_cast<uint32_t*>(take(std::max<uint64_t>(rows, 1) * 4));
    sl.toff = static_cast<uint64_t*>(take(std::max<uint64_t>(rows, 1) * 8));
    sl.rflops = static_cast<int64_t*>(take(std::max<uint64_t>(rows, 1) * 8));
    if (static_cast<uint64_t>(m - slot_mem[s]) > slot_cap + 4096)
      fail(AIRES_B200_INSUFFICIENT_DEVICE_MEMORY, "ring slot overflow");
  };

  const uint64_t n_sym = sym_cuts.size() - 1;
  std::vector<Ctl*> sym_ctl(nbuf);
  Ctl* d_ctls = static_cast<Ctl*>(arena.get(sizeof(Ctl) * std::max<uint64_t>(n_sym, 1)));
  AB2_CUDA(cudaMemsetAsync(d_ctls, 0, sizeof(Ctl) * std::max<uint64_t>(n_sym, 1), cs));
  cudaEvent_t e_zero = st.make();
  AB2_CUDA(cudaEventRecord(e_zero, cs));
  AB2_CUDA(cudaStreamWaitEvent(st.h2d, e_zero, 0));
  for (uint64_t c = 0; c < n_sym; c++) {
    const uint32_t s = static_cast<uint32_t>(c % nbuf);
    const uint64_t r0 = sym_cuts[c], r1 = sym_cuts[c + 1];
    const uint64_t q0 = a.ptr[r0], q1 = a.ptr[r1];
    if (c >= nbuf) AB2_CUDA(cudaStreamWaitEvent(st.h2d, slot[s].computed, 0));
    carve(s, r1 - r0, q1 - q0, false, 0);
    if (cols_resident) slot[s].acol = d_acol_full + (q0 - p0) * ib;
    rep.h2d_bytes += (q1 - q0) * ib;
    if (early_cols) {
      AB2_CUDA(cudaStreamWaitEvent(cs, early_ev[c], 0));
    } else {
      tr.span(st.h2d, AIRES_B200_EV_TRANSFER, AIRES_B200_CH_H2D, AIRES_B200_BUF_A, c + 1, (q1 - q0) * ib, 0, [&] {
        if (q1 > q0)
          AB2_CUDA(cudaMemcpyAsync(slot[s].acol, static_cast<const char*>(a.idx) + q0 * ib, (q1 - q0) * ib,
                                   cudaMemcpyHostToDevice, st.h2d));
      });
      AB2_CUDA(cudaEventRecord(slot[s].loaded, st.h2d));
      AB2_CUDA(cudaStreamWaitEvent(cs, slot[s].loaded, 0));
    }
    TileSym t{};
    t.aptr = d_aptr + r0;
    t.abase = q0;
    t.acol = slot[s].acol;
    t.rows = static_cast<int64_t>(r1 - r0);
    t.cnt = d_cnt + r0;
    t.rflops = slot[s].rflops;
    t.heavy = slot[s].heavy;
    t.ctl = d_ctls + c;
    tr.span(cs, AIRES_B200_EV_COMPUTE, AIRES_B200_TIER_DEVICE, AIRES_B200_BUF_A, c + 1, 0, 0,
            [&] { ctx.launches += tile_symbolic(ctx, *x, ib, t); });
    AB2_CUDA(cudaEventRecord(slot[s].computed, cs));
  }
  // scan -> C row_ptr, total nnz and MACs
  mark("sizing pass enqueued");
  {
    const int64_t nb = (static_cast<int64_t>(n) + kScanTile - 1) / kScanTile;
    int64_t* part = static_cast<int64_t*>(arena.get(std::max<int64_t>(nb, 1) * 8));
    if (n > 0) {
      k_scan_reduce<<<static_cast<unsigned>(nb), kScanThreads, 0, cs>>>(d_cnt, n, part);
      k_scan_part<<<1, 1024, 0, cs>>>(part, nb, d_ctl);
      k_scan_down<<<static_cast<unsigned>(nb), kScanThreads, 0, cs>>>(d_cnt, n, part, d_cptr);
      ctx.launches += 3;
    } else {
      AB2_CUDA(cudaMemsetAsync(d_cptr, 0, 8, cs));
    }
    AB2_CUDA(cudaGetLastError());
  }
  std::vector<Ctl> h_ctls(std::max<uint64_t>(n_sym, 1));
  Ctl* h = static_cast<Ctl*>(ctx.h_ctl.get(sizeof(Ctl)));
  AB2_CUDA(cudaMemcpyAsync(h, d_ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, cs));
  AB2_CUDA(cudaMemcpyAsync(h_ctls.data(), d_ctls, sizeof(Ctl) * std::max<uint64_t>(n_sym, 1), cudaMemcpyDeviceToHost, cs));
  AB2_CUDA(cudaStreamSynchronize(cs));
  const uint64_t nnz = n > 0 ? h->nnz : 0;
  uint64_t flops = 0;
  for (uint64_t c = 0; c < n_sym; c++) flops += h_ctls[c].flops;

  // exact allocation by the caller (spgemm.hpp:111-112), C row_ptr straight into it
  mark("sizing pass done (synced)");
  void *optr = nullptr, *oidx = nullptr, *oval = nullptr;
  int rc = out.alloc(out.user, n, nnz, &optr, &oidx, &oval);
  if (rc != 0) fail(rc, "output allocator failed for " + std::to_string(nnz) + " nonzeros");
  pin.ensure(optr, (n + 1) * 8);
  pin.ensure(oidx, nnz * ib);
  pin.ensure(oval, nnz * vb);
  tr.span(cs, AIRES_B200_EV_TRANSFER, AIRES_B200_CH_D2H, AIRES_B200_BUF_C_BLOCK, 0, (n + 1) * 8, 0, [&] {
    AB2_CUDA(cudaMemcpyAsync(optr, d_cptr, (n + 1) * 8, cudaMemcpyDeviceToHost, cs));
  });
  AB2_CUDA(cudaStreamSynchronize(cs));
  rep.d2h_bytes += (n + 1) * 8;
  const uint64_t* cp = static_cast<const uint64_t*>(optr);

  // tile cuts: C-aware (A + C + scratch per slot), or RoBW over A alone
  mark("allocated + C row_ptr copied");
  // (c_aware = 0: RoBW-style cuts that fill a slot with A alone, then the C block of each
  // segment must fit the rest -- the reference's admission, which fails on GCN shapes)
  // Uncapped runs (device_budget 0) still cut ~AB2_RUN_TILES (16) tiles so that tile k+1's H2D, tile k's
  // product and tile k-1's D2H overlap; capped runs use maximal tiles.
  uint64_t tile_budget = slot_budget;
  if (cfg.device_budget == 0) {
    const uint64_t p2_bytes = (pend - p0) * a_tile_bytes + nnz * (ib + vb) + n * row_bytes;
    const uint64_t want = std::max<uint64_t>(option("run_tiles", 16), 1);
    tile_budget = std::min<uint64_t>(slot_budget, std::max<uint64_t>(p2_bytes / want, 64ull << 20));
  }
  // MaxMemory (partition.hpp:140-169): the element stream is cut at fixed byte boundaries, rows split
  // mid-way; tile j ships its raw bytes plus the fragment of the row cut by the previous tile, which
  // came back to the host (D2H) and is stitched on in front (merge_partial, partition.hpp:176-197).
  struct MmTile {
    uint64_t q_frag, q0, q1;  // entries [q_frag, q0) re-sent fragment, [q0, q1) raw bytes
    uint64_t r0, r1;          // complete rows multiplied in this tile
  };
  std::vector<MmTile> mm;
  // The reference reserves C statically from its Eq. 5 estimate (~1e-4 of the real C on GCN
  // shapes, so it cannot run them); here the baseline gets the generous version: the slot is split
  // between A bytes and output bytes in the proportion of the whole product (known from the sizing
  // pass), and the tile is halved until every tile's fragment + raw bytes + output block fits.
  auto mm_build = [&](uint64_t te) {
    mm.clear();
    uint64_t cursor = 0, frag = p0;
    for (uint64_t e0 = p0; e0 < pend; e0 += te) {
      const uint64_t e1 = std::min(e0 + te, pend);
      MmTile t{frag, e0, e1, cursor, cursor};
      while (t.r1 < n && a.ptr[t.r1 + 1] <= e1) t.r1++;
      cursor = t.r1;
      frag = cursor < n ? a.ptr[cursor] : pend;  // start of the row cut at e1 (a row longer than a
                                                  // tile is re-sent from its start, partition.hpp:110-114)
      mm.push_back(t);
    }
    while (cursor < n) {  // trailing empty rows
      mm.push_back(MmTile{pend, pend, pend, cursor, n});
      cursor = n;
    }
  };
  if (maxmem) {
    const double a_share = static_cast<double>((pend - p0) * (ib + vb)) /
                           std::max<double>(1.0, static_cast<double>((pend - p0) * (ib + vb) + nnz * (ib + vb)));
    uint64_t te = std::max<uint64_t>(static_cast<uint64_t>(slot_budget * a_share * 0.9) / (ib + vb), 1);
    for (;;) {
      mm_build(te);
      bool fits = true;
      for (const MmTile& t : mm)
        fits = fits && carve_bytes(t.r1 - t.r0, t.q1 - t.q_frag, true, cp[t.r1] - cp[t.r0]) <= slot_budget + 4096;
      if (fits || te == 1) break;
      te = std::max<uint64_t>(te / 2, 1);
    }
  }
  std::vector<uint64_t> cuts;
  if (maxmem) {
    cuts.assign(1, 0);
    for (const MmTile& t : mm) cuts.push_back(t.r1);
  } else if (!greedy_cuts(a.ptr, cfg.c_aware ? cp : nullptr, n, row_bytes, a_tile_bytes, ib + vb,
                          cfg.c_aware ? tile_budget : slot_budget - slot_budget / 16, cuts, &bad))
    fail(AIRES_B200_ROW_TOO_LARGE, "row " + std::to_string(bad) + " does not fit a ring slot of " +
                                       std::to_string(slot_budget) + " bytes");
  if (maxmem) {
    for (size_t j = 0; j < mm.size(); j++) {
      const MmTile& t = mm[j];
      if (carve_bytes(t.r1 - t.r0, t.q1 - t.q_frag, true, cp[t.r1] - cp[t.r0]) > slot_budget + 4096)
        fail(AIRES_B200_INSUFFICIENT_DEVICE_MEMORY,
             "MaxMemory tile " + std::to_string(j) + " (fragment + raw bytes + output block) does not fit a slot");
    }
  }
  if (!cfg.c_aware) {
    for (size_t j = 0; j + 1 < cuts.size(); j++) {
      const uint64_t r0 = cuts[j], r1 = cuts[j + 1];
      const uint64_t need =
          (r1 - r0) * row_bytes + (a.ptr[r1] - a.ptr[r0]) * a_tile_bytes + (cp[r1] - cp[r0]) * (ib + vb);
      if (need > slot_budget)
        fail(AIRES_B200_INSUFFICIENT_DEVICE_MEMORY,
             "segment " + std::to_string(j) + "'s C block does not fit the remaining device memory (A-only tiling)");
    }
  }
  const uint64_t n_tiles = cuts.size() - 1;
  if (cfg.device_budget == 0) {  // resize the ring to the largest tile
    uint64_t need = 0;
    for (uint64_t j = 0; j < n_tiles; j++)
      need = std::max(need, carve_bytes(cuts[j + 1] - cuts[j],
                                        maxmem ? mm[j].q1 - mm[j].q_frag : a.ptr[cuts[j + 1]] - a.ptr[cuts[j]], true,
                                        cp[cuts[j + 1]] - cp[cuts[j]]));
    if (need > slot_cap) {
      slot_cap = need;
      for (uint32_t s = 0; s < nbuf; s++) slot_mem[s] = static_cast<char*>(arena.get(slot_cap + 4096));
    }
  }
  Ctl* d_tctl = static_cast<Ctl*>(arena.get(sizeof(Ctl) * std::max<uint64_t>(n_tiles, 1)));
  AB2_CUDA(cudaMemsetAsync(d_tctl, 0, sizeof(Ctl) * std::max<uint64_t>(n_tiles, 1), cs));
  AB2_CUDA(cudaEventRecord(t_p1, cs));

  // MaxMemory's host merge buffer (pinned): the trailing fragment of tile j, re-sent with tile j+1
  void* merge_col = nullptr;
  void* merge_val = nullptr;
  cudaEvent_t frag_back = st.make();
  HostBuf merge_buf;
  if (maxmem) {
    uint64_t maxfrag = 1;
    for (const MmTile& m : mm) maxfrag = std::max(maxfrag, m.q0 - m.q_frag);
    char* mb = static_cast<char*>(merge_buf.get(maxfrag * (ib + vb) + 256));
    merge_col = mb;
    merge_val = mb + ((maxfrag * ib + 127) & ~uint64_t(127));
  }

  // ---------------- Phase II ----------------
  mark("tiles cut");
  AB2_CUDA(cudaEventRecord(e_zero, cs));
  AB2_CUDA(cudaStreamWaitEvent(st.h2d, e_zero, 0));
  tr.set_phase(1, "aires phase II (tiles)");
  std::vector<size_t> compute_rec(n_tiles, 0);
  for (uint64_t j = 0; j < n_tiles; j++) {
    const uint32_t s = static_cast<uint32_t>(j % nbuf);
    const uint64_t r0 = cuts[j], r1 = cuts[j + 1];
    const uint64_t q0 = a.ptr[r0], q1 = a.ptr[r1];
    const uint64_t c0 = cp[r0], c1 = cp[r1];
    // slot s is free for A once tile j-nbuf was computed (Phase I chunks were awaited above)
    if (j >= nbuf) AB2_CUDA(cudaStreamWaitEvent(st.h2d, slot[s].computed, 0));
    // its C space is free once tile j-nbuf was drained
    if (j >= nbuf) AB2_CUDA(cudaStreamWaitEvent(st.h2d, slot[s].drained, 0));
    if (maxmem) {
      // fragment (from the host merge buffer, filled by tile j-1's D2H) + raw tile (from A)
      const MmTile& m = mm[j];
      carve(s, r1 - r0, m.q1 - m.q_frag, true, c1 - c0);
      if (j > 0) AB2_CUDA(cudaStreamWaitEvent(st.h2d, frag_back, 0));
      const uint64_t nf = m.q0 - m.q_frag, nr = m.q1 - m.q0;
      tr.point(st.h2d, AIRES_B200_EV_ALLOC, AIRES_B200_BUF_A_TILE, j, (nf + nr) * (ib + vb));
      const size_t up = tr.span(st.h2d, AIRES_B200_EV_TRANSFER, AIRES_B200_CH_H2D, AIRES_B200_BUF_A_TILE, j,
                                (nf + nr) * (ib + vb), 0, [&] {
        if (nf) {
          AB2_CUDA(cudaMemcpyAsync(slot[s].acol, merge_col, nf * ib, cudaMemcpyHostToDevice, st.h2d));
          AB2_CUDA(cudaMemcpyAsync(slot[s].aval, merge_val, nf * vb, cudaMemcpyHostToDevice, st.h2d));
        }
        if (nr) {
          AB2_CUDA(cudaMemcpyAsync(static_cast<char*>(slot[s].acol) + nf * ib, static_cast<const char*>(a.idx) + m.q0 * ib,
                                   nr * ib, cudaMemcpyHostToDevice, st.h2d));
          AB2_CUDA(cudaMemcpyAsync(static_cast<char*>(slot[s].aval) + nf * vb, static_cast<const char*>(a.val) + m.q0 * vb,
                                   nr * vb, cudaMemcpyHostToDevice, st.h2d));
        }
      });
      if (nf) tr.merge_share.emplace_back(up, static_cast<double>(nf) / static_cast<double>(nf + nr));
      rep.h2d_bytes += (nf + nr) * (ib + vb);
      rep.merge_bytes += nf * (ib + vb);
      AB2_CUDA(cudaEventRecord(slot[s].loaded, st.h2d));
      AB2_CUDA(cudaStreamWaitEvent(cs, slot[s].loaded, 0));
      // the trailing fragment goes back to the host once this tile is on the device -- on its own
      // stream, so the next upload waits for this fragment only (not behind earlier C drains)
      const uint64_t fb = j + 1 < mm.size() ? mm[j + 1].q_frag : pend;
      const uint64_t tail = m.q1 > fb ? m.q1 - fb : 0;
      AB2_CUDA(cudaStreamWaitEvent(st.aux, slot[s].loaded, 0));
      if (tail) {
        const size_t fr = tr.span(st.aux, AIRES_B200_EV_TRANSFER, AIRES_B200_CH_D2H, AIRES_B200_BUF_FRAGMENT, j,
                                  tail * (ib + vb), 0, [&] {
          AB2_CUDA(cudaMemcpyAsync(merge_col, static_cast<char*>(slot[s].acol) + (fb - m.q_frag) * ib, tail * ib,
                                   cudaMemcpyDeviceToHost, st.aux));
          AB2_CUDA(cudaMemcpyAsync(merge_val, static_cast<char*>(slot[s].aval) + (fb - m.q_frag) * vb, tail * vb,
                                   cudaMemcpyDeviceToHost, st.aux));
        });
        tr.merge_share.emplace_back(fr, 1.0);
        rep.d2h_bytes += tail * (ib + vb);
      }
      AB2_CUDA(cudaEventRecord(frag_back, st.aux));
      TilePass t{};
      t.aptr = d_aptr + r0;
      t.abase = m.q_frag;
      t.acol = slot[s].acol;
      t.aval = slot[s].aval;
      t.rows = static_cast<int64_t>(r1 - r0);
      t.cpos = d_cptr + r0;
      t.cbase = static_cast<int64_t>(c0);
      t.ccol = slot[s].ccol;
      t.cval = slot[s].cval;
      t.c_cap = c1 - c0;
      t.heavy = slot[s].heavy;
      t.cnt = slot[s].cnt;
      t.toff = slot[s].toff;
      t.ctl = d_tctl + j;
      compute_rec[j] = tr.span(cs, AIRES_B200_EV_COMPUTE, AIRES_B200_TIER_DEVICE, AIRES_B200_BUF_A_TILE, j, 0, 0,
                               [&] { ctx.launches += tile_product(ctx, *x, ib, t); });
      AB2_CUDA(cudaEventRecord(slot[s].computed, cs));
      AB2_CUDA(cudaStreamWaitEvent(st.d2h, slot[s].computed, 0));
      tr.span(st.d2h, AIRES_B200_EV_TRANSFER, AIRES_B200_CH_D2H, AIRES_B200_BUF_C_BLOCK, j, (c1 - c0) * (ib + vb), 0, [&] {
        if (c1 > c0) {
          AB2_CUDA(cudaMemcpyAsync(static_cast<char*>(oidx) + c0 * ib, slot[s].ccol, (c1 - c0) * ib,
                                   cudaMemcpyDeviceToHost, st.d2h));
          AB2_CUDA(cudaMemcpyAsync(static_cast<char*>(oval) + c0 * vb, slot[s].cval, (c1 - c0) * vb,
                                   cudaMemcpyDeviceToHost, st.d2h));
        }
      });
      rep.d2h_bytes += (c1 - c0) * (ib + vb);
      tr.point(st.d2h, AIRES_B200_EV_FREE, AIRES_B200_BUF_A_TILE, j, (nf + nr) * (ib + vb));
      AB2_CUDA(cudaEventRecord(slot[s].drained, st.d2h));
      continue;
    }
    carve(s, r1 - r0, q1 - q0, true, c1 - c0);
    if (cols_resident) slot[s].acol = d_acol_full + (q0 - p0) * ib;
    tr.point(st.h2d, AIRES_B200_EV_ALLOC, AIRES_B200_BUF_A_TILE, j, (q1 - q0) * a_tile_bytes);
    tr.span(st.h2d, AIRES_B200_EV_TRANSFER, AIRES_B200_CH_H2D, AIRES_B200_BUF_A_TILE, j, (q1 - q0) * a_tile_bytes, 0, [&] {
      if (q1 > q0) {
        if (!cols_resident)
          AB2_CUDA(cudaMemcpyAsync(slot[s].acol, static_cast<const char*>(a.idx) + q0 * ib, (q1 - q0) * ib,
                                   cudaMemcpyHostToDevice, st.h2d));
        AB2_CUDA(cudaMemcpyAsync(slot[s].aval, static_cast<const char*>(a.val) + q0 * vb, (q1 - q0) * vb,
                                 cudaMemcpyHostToDevice, st.h2d));
      }
    });
    rep.h2d_bytes += (q1 - q0) * a_tile_bytes;
    AB2_CUDA(cudaEventRecord(slot[s].loaded, st.h2d));
    AB2_CUDA(cudaStreamWaitEvent(cs, slot[s].loaded, 0));
    TilePass t{};
    t.aptr = d_aptr + r0;
    t.abase = q0;
    t.acol = slot[s].acol;
    t.aval = slot[s].aval;
    t.rows = static_cast<int64_t>(r1 - r0);
    t.cpos = d_cptr + r0;
    t.cbase = static_cast<int64_t>(c0);
    t.ccol = slot[s].ccol;
    t.cval = slot[s].cval;
    t.c_cap = c1 - c0;
    t.heavy = slot[s].heavy;
    t.cnt = slot[s].cnt;
    t.toff = slot[s].toff;
    t.ctl = d_tctl + j;
    compute_rec[j] = tr.span(cs, AIRES_B200_EV_COMPUTE, AIRES_B200_TIER_DEVICE, AIRES_B200_BUF_A_TILE, j, 0, 0,
                             [&] { ctx.launches += tile_product(ctx, *x, ib, t); });
    AB2_CUDA(cudaEventRecord(slot[s].computed, cs));
    AB2_CUDA(cudaStreamWaitEvent(st.d2h, slot[s].computed, 0));
    tr.span(st.d2h, AIRES_B200_EV_TRANSFER, AIRES_B200_CH_D2H, AIRES_B200_BUF_C_BLOCK, j, (c1 - c0) * (ib + vb), 0, [&] {
      if (c1 > c0) {
        AB2_CUDA(cudaMemcpyAsync(static_cast<char*>(oidx) + c0 * ib, slot[s].ccol, (c1 - c0) * ib,
                                 cudaMemcpyDeviceToHost, st.d2h));
        AB2_CUDA(cudaMemcpyAsync(static_cast<char*>(oval) + c0 * vb, slot[s].cval, (c1 - c0) * vb,
                                 cudaMemcpyDeviceToHost, st.d2h));
      }
    });
    rep.d2h_bytes += (c1 - c0) * (ib + vb);
    tr.point(st.d2h, AIRES_B200_EV_FREE, AIRES_B200_BUF_A_TILE, j, (q1 - q0) * a_tile_bytes);
    AB2_CUDA(cudaEventRecord(slot[s].drained, st.d2h));
  }
  AB2_CUDA(cudaEventRecord(t_p2, cs));

  // ---------------- Phase III ----------------
  mark("phase II enqueued");
  AB2_CUDA(cudaStreamWaitEvent(cs, slot[0].drained, 0));
  for (uint32_t s = 0; s < nbuf; s++) AB2_CUDA(cudaStreamWaitEvent(cs, slot[s].drained, 0));
  if (maxmem) {  // the fragment stream too
    AB2_CUDA(cudaEventRecord(frag_back, st.aux));
    AB2_CUDA(cudaStreamWaitEvent(cs, frag_back, 0));
  }
  tr.set_phase(2, "aires phase III (drain)");
  tr.point(cs, AIRES_B200_EV_FREE, AIRES_B200_BUF_B, 0, x_dev);
  AB2_CUDA(cudaEventRecord(t_end, cs));
  std::vector<Ctl> h_t(std::max<uint64_t>(n_tiles, 1));
  AB2_CUDA(cudaMemcpyAsync(h_t.data(), d_tctl, sizeof(Ctl) * std::max<uint64_t>(n_tiles, 1), cudaMemcpyDeviceToHost, cs));
  AB2_CUDA(cudaStreamSynchronize(cs));
  AB2_CUDA(cudaStreamSynchronize(st.d2h));
  for (uint64_t j = 0; j < n_tiles; j++) {
    if (h_t[j].bad_row == 2) fail(AIRES_B200_CUDA_ERROR, "numeric row counts disagree with the symbolic pass");
    if (h_t[j].bad_row) fail(AIRES_B200_CAPACITY_EXCEEDED, "tile output overflow");
  }
  mark("phase III synced");
  rep.segments = n_tiles;
  rep.flops = flops;
  rep.c_nnz = nnz;
  rep.peak_device_bytes = arena.used + x_dev;
  for (uint64_t j = 0; j < n_tiles; j++) tr.recs[compute_rec[j]].e.flops = h_t[j].flops;
  tr.finish(t_begin, rep, cfg);
  rep.phase1_ms = ms_between(t_begin, t_p1);
  rep.phase2_ms = ms_between(t_p1, t_p2);
  rep.phase3_ms = ms_between(t_p2, t_end);
  rep.total_ms = ms_between(t_begin, t_end);
  ctx.last_ms = rep.total_ms;
  out.n_rows = n;
  out.n_cols = static_cast<uint64_t>(x->n_cols);
  out.nnz = nnz;
  out.flops = flops;
}

}  // namespace ab2
