// ab2_spgemm.cu -- host orchestration of one A·X product (spgemm_block, spgemm.hpp:60-132).
//
//   upload (host A only) -> K_classify -> K_numeric (staging) -> K_scan -> [nnz readback, exact
//   allocation through the caller's allocator, spgemm.hpp:111-112] -> K_place -> row_ptr copy
//   -> (host C) D2H.  Operands wider than the dense accumulator run in column tiles (wide_product).
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstring>
#include <mutex>
#include <type_traits>
#include <unordered_map>

#include "ab2_internal.h"
#include "ab2_numeric.cuh"
#include "ab2_numeric5.cuh"

namespace ab2 {

namespace {

template <class K>
int occupancy_grid(K kernel, int threads, size_t smem, int sms) {
  static std::mutex mu;
  static std::unordered_map<const void*, size_t> attr_set;
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = attr_set.find(reinterpret_cast<const void*>(kernel));
    if (it == attr_set.end() || it->second < smem) {
      AB2_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
      attr_set[reinterpret_cast<const void*>(kernel)] = smem;
    }
  }
  int nb = 0;
  AB2_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kernel, threads, smem));
  if (nb < 1) fail(AIRES_B200_INSUFFICIENT_DEVICE_MEMORY, "kernel does not fit on an SM (shared memory)");
  return nb * sms;
}

template <class V, class IdxT, int W>
void launch_numeric_w(Ctx& ctx, const Num3Args<V, IdxT>& p, int threads, size_t smem, bool xz) {
  auto k = xz ? k_numeric3<V, IdxT, W, true> : k_numeric3<V, IdxT, W, false>;
  int grid = occupancy_grid(k, threads, smem, ctx.sms);
  k<<<grid, threads, smem, ctx.stream>>>(p);
}

template <class V, class IdxT>
int numeric_warps(const Num3Args<V, IdxT>& p) {
  // fp32 over 16-entry slots (walk_pair; cfg2): one-warp CTAs -- more resident warps, heavy rows one
  // warp each -- measured 2.10 ms vs 2.13 (2 warps) and 2.20 (4 warps); fp64 is neutral and narrow
  // slots (cfg3) prefer 4 (1.92 vs 1.94 ms at 2)
  const int def = sizeof(V) == 4 && p.copies == 2 ? 1 : 4;
  int nw = std::min<int>(static_cast<int>(option("num_warps", def)), AB2_NUM_MAXT / 32);
  return std::max(1, std::min<int>(nw, static_cast<int>((200 * 1024) / p.warp_bytes)));
}

template <class V, class IdxT>
void launch_numeric(Ctx& ctx, const Num3Args<V, IdxT>& p, int W, bool xz) {
  const int nw = numeric_warps(p);
  const int threads = nw * 32;
  const size_t smem = static_cast<size_t>(nw) * p.warp_bytes;
  switch (W) {
    case 2: launch_numeric_w<V, IdxT, 2>(ctx, p, threads, smem, xz); break;
    case 4: launch_numeric_w<V, IdxT, 4>(ctx, p, threads, smem, xz); break;
    case 8: launch_numeric_w<V, IdxT, 8>(ctx, p, threads, smem, xz); break;
    case 16: launch_numeric_w<V, IdxT, 16>(ctx, p, threads, smem, xz); break;
    default: fail(AIRES_B200_INVALID_ARGUMENT, "bad slot width");
  }
  AB2_CUDA(cudaGetLastError());
}

// fp32 step-list pass (ab2_numeric5.cuh); shares the staging / direct-offset set-up of the
// k_numeric3 args.
template <class IdxT, int W>
void launch_numeric5_w(Ctx& ctx, const Num5Args<IdxT>& p, bool xz) {
  int nw = static_cast<int>(option("n5_warps", AB2_N5_MAXT / 32));
  nw = std::max(1, std::min<int>({nw, AB2_N5_MAXT / 32, static_cast<int>((200 * 1024) / p.warp_bytes)}));
  const int threads = nw * 32;
  const size_t smem = static_cast<size_t>(nw) * p.warp_bytes;
  auto k = xz ? k_numeric5<IdxT, W, true> : k_numeric5<IdxT, W, false>;
  const int grid = occupancy_grid(k, threads, smem, ctx.sms);
  k<<<grid, threads, smem, ctx.stream>>>(p);
  AB2_CUDA(cudaGetLastError());
}

template <class IdxT>
void launch_numeric5(Ctx& ctx, const Num3Args<float, IdxT>& q, const XOperand& x) {
  Num5Args<IdxT> p{};
  p.aptr = q.aptr;
  p.abase = q.abase;
  p.acol = q.acol;
  p.aval = q.aval;
  p.rows = q.rows;
  p.K = x.K;
  p.n_cols = static_cast<int32_t>(x.n_cols);
  p.stride = q.stride;
  p.warp_bytes = static_cast<int32_t>(static_cast<size_t>(32 / x.W5) * p.stride * 4 + p.stride + kN5List * 8);
  p.xdesc = static_cast<const uint2*>(x.xdesc);
  p.xent = static_cast<const uint2*>(x.xent);
  p.dummy_slot = static_cast<uint32_t>(x.dummy_slot);
  p.heavy = q.heavy;
  p.heavy_deg = q.heavy_deg;
  p.cnt = q.cnt;
  p.toff = q.toff;
  p.tcol = q.tcol;
  p.tval = q.tval;
  p.t_cap = q.t_cap;
  p.tiny = q.tiny;
  p.stage_block = q.stage_block;
  p.ctl = q.ctl;
  p.cpos = q.cpos;
  p.cbase = q.cbase;
  switch (x.W5) {
    case 2: launch_numeric5_w<IdxT, 2>(ctx, p, x.has_zero); break;
    case 4: launch_numeric5_w<IdxT, 4>(ctx, p, x.has_zero); break;
    case 8: launch_numeric5_w<IdxT, 8>(ctx, p, x.has_zero); break;
    case 16: launch_numeric5_w<IdxT, 16>(ctx, p, x.has_zero); break;
    case 32: launch_numeric5_w<IdxT, 32>(ctx, p, x.has_zero); break;
    default: fail(AIRES_B200_INVALID_ARGUMENT, "bad step-list slot width");
  }
}

template <class Src, class Dst>
__global__ void k_convert(const Src* __restrict__ in, Dst* __restrict__ out, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = static_cast<Dst>(in[i]);
}

template <class Src, class Dst>
void convert(Ctx& ctx, const void* in, void* out, int64_t n) {
  if (n <= 0) return;
  int grid = static_cast<int>(std::min<int64_t>((n + 255) / 256, static_cast<int64_t>(ctx.sms) * 32));
  k_convert<Src, Dst><<<grid, 256, 0, ctx.stream>>>(static_cast<const Src*>(in), static_cast<Dst*>(out), n);
  ctx.launches++;
  AB2_CUDA(cudaGetLastError());
}


template <class V, class IdxT>
Num3Args<V, IdxT> make_num3(const XOperand& x, const uint64_t* aptr, uint64_t abase, const IdxT* acol, const V* aval,
                            int64_t rows, int64_t* heavy, int64_t heavy_deg, uint32_t* cnt, uint64_t* toff, Ctl* ctl) {
  Num3Args<V, IdxT> np{};
  np.aptr = aptr;
  np.abase = abase;
  np.acol = acol;
  np.aval = aval;
  np.rows = rows;
  np.x.K = x.K;
  np.x.n_cols = static_cast<int32_t>(x.n_cols);
  np.x.W = x.W;
  np.x.ptr = static_cast<const int64_t*>(x.ptr);
  np.x.col = static_cast<const int32_t*>(x.col);
  np.x.val = static_cast<const V*>(x.val);
  np.x.slots = static_cast<const typename SlotOf<V>::type*>(x.slots);
  np.x.cslots = static_cast<const uint16_t*>(x.cslots);
  np.stride = static_cast<int32_t>((x.n_cols + 1 + 31) & ~int64_t(31));
  // fp32: one accumulator copy per lane group (two 16-lane groups over 16-entry slots)
  np.copies = sizeof(V) == 8 ? 1 : 32 / x.W;
  np.warp_bytes = static_cast<int32_t>(
      ((static_cast<size_t>(np.copies) * np.stride * sizeof(V) + np.stride + 15) & ~size_t(15)) +
      36 * sizeof(ChunkPair));  // chunk tables (walk_pair: two 288-byte buffers)
  np.heavy = heavy;
  np.heavy_deg = heavy_deg;
  np.cnt = cnt;
  np.toff = toff;
  np.ctl = ctl;
  np.xlen = static_cast<const uint16_t*>(x.xlen);
  // |a| below `tiny` may round a*x to zero (fp32: |a*x| < 2^-149 incl. the FFMA path;
  // fp64: < 2^-1074); such weights send the row to the explicit-mark path.
  np.tiny = x.xmin > 0 ? static_cast<V>((sizeof(V) == 4 ? std::ldexp(1.0, -147) : std::ldexp(1.0, -1072)) / x.xmin)
                       : V(0);
  np.stage_block = static_cast<uint32_t>(std::max<int64_t>(4096, 8 * static_cast<int64_t>(np.stride)));
  np.pad0 = option("short_rows", 1) == 0 ? 0 : (x.n_cols <= 256 && option("short_dense", 1) != 0 ? 2 : 1);
  return np;
}

// The product kernel: k_numeric3 (W-lane slot groups; fp32 and fp64-exact) by default, the fp32
// step-list k_numeric5 with AB2_NUMERIC=5 (measured 3.5 ms vs 3.0 ms at cfg2: both are bound by
// L1/shared-memory wavefronts, profiles/r01*).
template <class V, class IdxT>
void launch_product(Ctx& ctx, const Num3Args<V, IdxT>& np, const XOperand& x) {
  if constexpr (std::is_same<V, float>::value) {
    if (x.xdesc != nullptr && (x.slots == nullptr || option("numeric_kernel", 3) == 5)) {
      launch_numeric5<IdxT>(ctx, np, x);
      return;
    }
  }
  launch_numeric<V, IdxT>(ctx, np, x.W, x.has_zero);
}

// One product: classify -> MAC count -> K_numeric (staging) -> scan -> [nnz readback,
// exact allocation through the caller's allocator, spgemm.hpp:111-112] -> K_place.
template <class V, class IdxT>
void run_product(Ctx& ctx, const aires_b200_matrix& a, const XOperand& x, aires_b200_output& out,
                 const uint64_t* aptr, uint64_t abase, const IdxT* acol, const V* aval, uint64_t span_hint) {
  const int64_t rows = static_cast<int64_t>(a.n_rows);
  if (x.K >= (int64_t(1) << 31) / 16) fail(AIRES_B200_CAPACITY_EXCEEDED, "inner dimension too large for slot indexing");
  Ctl* ctl = ctx.ctl.as<Ctl>(1);
  Ctl* h = static_cast<Ctl*>(ctx.h_ctl.get(sizeof(Ctl)));
  const int64_t heavy_deg = option("heavy_deg", 1024);
  int64_t* heavy = ctx.sym_heavy.as<int64_t>(std::max<int64_t>(rows, 1));
  uint32_t* cnt = reinterpret_cast<uint32_t*>(ctx.cnt.as<int32_t>(std::max<int64_t>(rows, 1)));
  uint64_t* toff = reinterpret_cast<uint64_t*>(ctx.rflops.as<int64_t>(std::max<int64_t>(rows, 1)));
  int64_t* cptr = ctx.cptr.as<int64_t>(rows + 1);
  const uint64_t n_cols = static_cast<uint64_t>(x.n_cols);

  Num3Args<V, IdxT> np = make_num3<V, IdxT>(x, aptr, abase, acol, aval, rows, heavy, heavy_deg, cnt, toff, ctl);
  // staging: nnz bound (dense rows, or A entries x longest X row) * 8/7 + one block per warp
  const uint64_t maxlen = std::max<int64_t>(x.max_row_len, 1);
  const uint64_t bound = std::min<uint64_t>(static_cast<uint64_t>(rows) * n_cols, span_hint * maxlen);
  np.stage_block = static_cast<uint32_t>(std::max<int64_t>(4096, 8 * static_cast<int64_t>(np.stride)));
  const int nw = numeric_warps(np);
  const uint64_t warps_total = static_cast<uint64_t>(ctx.sms) * 64;  // upper bound of resident warps
  np.t_cap = bound + bound / 7 + (warps_total + 1) * np.stage_block;
  (void)nw;
  np.tcol = ctx.t_col.as<IdxT>(np.t_cap);
  np.tval = ctx.t_val.as<V>(np.t_cap);

  AB2_CUDA(cudaMemsetAsync(ctl, 0, sizeof(Ctl), ctx.stream));
  AB2_CUDA(cudaEventRecord(ctx.ev[0], ctx.stream));
  if (rows > 0) {
    int g = static_cast<int>(std::min<int64_t>((rows + 255) / 256, static_cast<int64_t>(ctx.sms) * 16));
    k_classify<<<g, 256, 0, ctx.stream>>>(aptr, rows, heavy_deg, heavy, ctl);
    AB2_CUDA(cudaGetLastError());
  }
  AB2_CUDA(cudaEventRecord(ctx.ev[1], ctx.stream));
  if (rows > 0) launch_product<V, IdxT>(ctx, np, x);
  AB2_CUDA(cudaEventRecord(ctx.ev[2], ctx.stream));
  const int64_t nb = (rows + kScanTile - 1) / kScanTile;
  int64_t* part = ctx.scan_part.as<int64_t>(std::max<int64_t>(nb, 1));
  if (rows > 0) {
    const int32_t* cin = reinterpret_cast<const int32_t*>(cnt);
    k_scan_reduce<<<static_cast<unsigned>(nb), kScanThreads, 0, ctx.stream>>>(cin, rows, part);
    k_scan_part<<<1, 1024, 0, ctx.stream>>>(part, nb, ctl);
    k_scan_down<<<static_cast<unsigned>(nb), kScanThreads, 0, ctx.stream>>>(cin, rows, part, cptr);
    AB2_CUDA(cudaGetLastError());
  } else {
    AB2_CUDA(cudaMemsetAsync(cptr, 0, sizeof(int64_t), ctx.stream));
  }
  AB2_CUDA(cudaEventRecord(ctx.ev[3], ctx.stream));
  AB2_CUDA(cudaMemcpyAsync(h, ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, ctx.stream));
  AB2_CUDA(cudaStreamSynchronize(ctx.stream));
  if (h->bad_row) fail(AIRES_B200_CAPACITY_EXCEEDED, "staging area overflow");
  const uint64_t nnz = h->nnz;
  const uint64_t flops = h->flops;

  // exact allocation by the caller (spgemm.hpp:111-112)
  void *optr = nullptr, *oidx = nullptr, *oval = nullptr;
  int rc = out.alloc(out.user, static_cast<uint64_t>(rows), nnz, &optr, &oidx, &oval);
  if (rc != 0) fail(rc, "output allocator failed for " + std::to_string(nnz) + " nonzeros");
  IdxT* ccol;
  V* cval;
  if (out.location == AIRES_B200_DEVICE) {
    ccol = static_cast<IdxT*>(oidx);
    cval = static_cast<V*>(oval);
  } else {
    ccol = ctx.c_col.as<IdxT>(std::max<uint64_t>(nnz, 1));
    cval = ctx.c_val.as<V>(std::max<uint64_t>(nnz, 1));
  }
  AB2_CUDA(cudaEventRecord(ctx.ev[4], ctx.stream));
  if (rows > 0 && nnz > 0) {
    k_place<V, IdxT><<<ctx.sms * 8, 256, 0, ctx.stream>>>(cnt, toff, cptr, np.tcol, np.tval, rows, ccol, cval);
    AB2_CUDA(cudaGetLastError());
  }
  AB2_CUDA(cudaEventRecord(ctx.ev[5], ctx.stream));
  // row_ptr (int64 == u64 bits; all values are >= 0)
  if (out.location == AIRES_B200_DEVICE) {
    AB2_CUDA(cudaMemcpyAsync(optr, cptr, (rows + 1) * 8, cudaMemcpyDeviceToDevice, ctx.stream));
    AB2_CUDA(cudaEventRecord(ctx.ev[6], ctx.stream));
  } else {
    AB2_CUDA(cudaEventRecord(ctx.ev[6], ctx.stream));
    AB2_CUDA(cudaMemcpyAsync(optr, cptr, (rows + 1) * 8, cudaMemcpyDeviceToHost, ctx.stream));
    if (nnz) {
      AB2_CUDA(cudaMemcpyAsync(oidx, ccol, nnz * sizeof(IdxT), cudaMemcpyDeviceToHost, ctx.stream));
      AB2_CUDA(cudaMemcpyAsync(oval, cval, nnz * sizeof(V), cudaMemcpyDeviceToHost, ctx.stream));
    }
  }
  AB2_CUDA(cudaEventRecord(ctx.ev[7], ctx.stream));
  AB2_CUDA(cudaStreamSynchronize(ctx.stream));
  float ms = 0;
  auto el = [&](int a0, int b0) {
    AB2_CUDA(cudaEventElapsedTime(&ms, ctx.ev[a0], ctx.ev[b0]));
    return static_cast<double>(ms);
  };
  ctx.prof[kPClassify] = el(0, 1);
  ctx.prof[kPSymbolic] = el(4, 5);  // slot reused: K_place
  ctx.prof[kPScan] = el(2, 3);
  ctx.prof[kPNumeric] = el(1, 2);
  ctx.prof[kPD2H] = el(6, 7);
  ctx.last_ms = el(0, 7);
  ctx.launches += rows > 0 ? 5 + (nnz > 0 ? 1 : 0) : 0;
  out.n_rows = static_cast<uint64_t>(rows);
  out.n_cols = n_cols;
  out.nnz = nnz;
  out.flops = flops;
}

}  // namespace

namespace {
template <class V, class IdxT>
int tile_product_t(Ctx& ctx, const XOperand& x, const TilePass& t) {
  if (t.rows <= 0) return 0;
  const int64_t heavy_deg = option("heavy_deg", 1024);
  const int g = static_cast<int>(std::min<int64_t>((t.rows + 255) / 256, static_cast<int64_t>(ctx.sms) * 16));
  k_classify<<<g, 256, 0, ctx.stream>>>(t.aptr, t.rows, heavy_deg, t.heavy, t.ctl);
  AB2_CUDA(cudaGetLastError());
  Num3Args<V, IdxT> np = make_num3<V, IdxT>(x, t.aptr, t.abase, static_cast<const IdxT*>(t.acol),
                                            static_cast<const V*>(t.aval), t.rows, t.heavy, heavy_deg, t.cnt,
                                            t.toff, t.ctl);
  np.cpos = t.cpos;
  np.cbase = t.cbase;
  np.tcol = static_cast<IdxT*>(t.ccol);
  np.tval = static_cast<V*>(t.cval);
  np.t_cap = t.c_cap;
  launch_product<V, IdxT>(ctx, np, x);
  return 2;
}

template <class IdxT>
int tile_symbolic_t(Ctx& ctx, const XOperand& x, const TileSym& t) {
  if (t.rows <= 0) return 0;
  const int64_t heavy_deg = option("sym_heavy_deg", 2048);
  const int g = static_cast<int>(std::min<int64_t>((t.rows + 255) / 256, static_cast<int64_t>(ctx.sms) * 16));
  k_classify<<<g, 256, 0, ctx.stream>>>(t.aptr, t.rows, heavy_deg, t.heavy, t.ctl);
  AB2_CUDA(cudaGetLastError());
  SymArgs sp{};
  sp.aptr = t.aptr;
  sp.abase = t.abase;
  sp.rows = t.rows;
  sp.K = x.K;
  sp.n_cols = static_cast<int32_t>(x.n_cols);
  sp.region_bytes = static_cast<int32_t>((x.n_cols + 15) & ~int64_t(15));
  sp.xptr = static_cast<const int64_t*>(x.ptr);
  sp.xcol = static_cast<const int32_t*>(x.col);
  sp.cslots = static_cast<const uint16_t*>(x.cslots);
  sp.cnt = t.cnt;
  sp.rflops = t.rflops;
  sp.sym_heavy = t.heavy;
  sp.heavy_deg = heavy_deg;
  sp.num_heavy = t.heavy;  // unused: heavy_flops is never exceeded
  sp.heavy_flops = INT64_MAX;
  sp.ctl = t.ctl;
  sp.xdesc = static_cast<const uint2*>(x.xdesc);
  sp.xent = static_cast<const uint2*>(x.xent);
  sp.w5 = x.W5;
  auto k = x.cslots ? k_symbolic<IdxT, kCSlotW> : (x.ptr ? k_symbolic<IdxT, 0> : k_symbolic<IdxT, -1>);
  const size_t smem = 8 * static_cast<size_t>(sp.region_bytes);
  const int grid = occupancy_grid(k, 256, smem, ctx.sms);
  k<<<grid, 256, smem, ctx.stream>>>(sp, static_cast<const IdxT*>(t.acol));
  AB2_CUDA(cudaGetLastError());
  return 2;
}
// ---------------------------------------------------------------------------
// Wide operands (n_cols(X) beyond the dense shared-memory accumulator): C is computed in column
// tiles of X -- the reference's own B column tiling (spgemm.hpp:94-130, tile_cols), which never
// changes a cell's terms or their ascending-k order -- each tile through the regular product
// pass into its own staging area; the tiles' row counts are summed, scanned, and every tile is
// placed at row offset cptr[r] + (entries of earlier tiles in row r), so each row comes out in
// ascending column order.
// ---------------------------------------------------------------------------
template <class V>
__global__ void k_tile_count(const int64_t* __restrict__ xptr, const int32_t* __restrict__ xcol, int64_t K,
                             int32_t c0, int32_t c1, int32_t* __restrict__ cnt) {
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < K;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t n = 0;
    for (int64_t t = xptr[k]; t < xptr[k + 1]; t++) n += xcol[t] >= c0 && xcol[t] < c1;
    cnt[k] = static_cast<int32_t>(n);
  }
}

template <class V>
__global__ void k_tile_fill(const int64_t* __restrict__ xptr, const int32_t* __restrict__ xcol,
                            const V* __restrict__ xval, int64_t K, int32_t c0, int32_t c1,
                            const int64_t* __restrict__ tptr, uint32_t* __restrict__ tcol, V* __restrict__ tval) {
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < K;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t o = tptr[k];
    for (int64_t t = xptr[k]; t < xptr[k + 1]; t++)
      if (xcol[t] >= c0 && xcol[t] < c1) {
        tcol[o] = static_cast<uint32_t>(xcol[t] - c0);
        tval[o] = xval[t];
        o++;
      }
  }
}

__global__ void k_add_counts(uint32_t* __restrict__ acc, const uint32_t* __restrict__ add, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    acc[i] += add[i];
}

template <class V, class IdxT>
__global__ void __launch_bounds__(256) k_place_tile(const uint32_t* __restrict__ cnt, const uint64_t* __restrict__ toff,
                                                    const int64_t* __restrict__ cptr, uint32_t* __restrict__ roff,
                                                    const IdxT* __restrict__ tcol, const V* __restrict__ tval,
                                                    int64_t rows, IdxT col0, IdxT* __restrict__ ccol,
                                                    V* __restrict__ cval) {
  const int lane = lane_id();
  const int64_t wid = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r = wid; r < rows; r += nwarps) {
    const uint32_t n = cnt[r];
    const uint64_t src = toff[r];
    const int64_t dst = cptr[r] + roff[r];
    for (uint32_t i = lane; i < n; i += 32) {
      ccol[dst + i] = tcol[src + i] + col0;
      cval[dst + i] = tval[src + i];
    }
    __syncwarp();
    if (lane == 0) roff[r] += n;
  }
}

template <class V, class IdxT>
void wide_product(Ctx& ctx, const aires_b200_matrix& a, const XOperand& x, aires_b200_output& out,
                  const uint64_t* aptr, uint64_t abase, const IdxT* acol, const V* aval, uint64_t span_hint) {
  const int64_t rows = static_cast<int64_t>(a.n_rows);
  const int64_t n_cols = x.n_cols;
  const int64_t tw = std::min<int64_t>(wide_threshold(x.mode), std::max<int64_t>(32, option("wide_tile", 2048)));
  const int64_t T = (n_cols + tw - 1) / tw;
  const int64_t K = x.K;
  const uint32_t mode = x.mode;
  const int64_t heavy_deg = option("heavy_deg", 1024);
  int64_t* heavy = ctx.sym_heavy.as<int64_t>(std::max<int64_t>(rows, 1));
  struct Tile {
    DevBuf ptr, col, val, cnt, toff, tcol, tval;
    int64_t c0 = 0;
  };
  std::vector<Tile> tiles(T);
  DevBuf ctl_buf, cnt_sum, roff;
  Ctl* ctls = static_cast<Ctl*>(ctl_buf.get(sizeof(Ctl) * (T + 1)));
  AB2_CUDA(cudaMemsetAsync(ctls, 0, sizeof(Ctl) * (T + 1), ctx.stream));
  const auto* xp = static_cast<const int64_t*>(x.ptr);
  const auto* xc = static_cast<const int32_t*>(x.col);
  const auto* xv = static_cast<const V*>(x.val);
  const int gK = static_cast<int>(std::min<int64_t>((K + 255) / 256 + 1, static_cast<int64_t>(ctx.sms) * 32));
  const int64_t nbK = (K + kScanTile - 1) / kScanTile;
  int64_t* partK = ctx.scan_part.as<int64_t>(std::max<int64_t>(nbK, 1) + 1);
  for (int64_t t = 0; t < T; t++) {
    Tile& tl = tiles[t];
    tl.c0 = t * tw;
    const int32_t c0 = static_cast<int32_t>(tl.c0), c1 = static_cast<int32_t>(std::min(n_cols, tl.c0 + tw));
    // one buffer: X-row counts of the tile first, then the product's C row counts
    int32_t* kc = static_cast<int32_t*>(tl.cnt.get(std::max<int64_t>(std::max<int64_t>(rows, K), 1) * 4));
    int64_t* tp = static_cast<int64_t*>(tl.ptr.get((K + 1) * 8));
    k_tile_count<V><<<gK, 256, 0, ctx.stream>>>(xp, xc, K, c0, c1, kc);
    if (K > 0) {
      k_scan_reduce<<<static_cast<unsigned>(nbK), kScanThreads, 0, ctx.stream>>>(kc, K, partK);
      k_scan_part<<<1, 1024, 0, ctx.stream>>>(partK, nbK, ctls + T);
      k_scan_down<<<static_cast<unsigned>(nbK), kScanThreads, 0, ctx.stream>>>(kc, K, partK, tp);
    } else {
      AB2_CUDA(cudaMemsetAsync(tp, 0, 8, ctx.stream));
    }
    auto* tc = static_cast<uint32_t*>(tl.col.get(std::max<int64_t>(x.nnz, 1) * 4));
    auto* tv = static_cast<V*>(tl.val.get(std::max<int64_t>(x.nnz, 1) * sizeof(V)));
    k_tile_fill<V><<<gK, 256, 0, ctx.stream>>>(xp, xc, xv, K, c0, c1, tp, tc, tv);
    AB2_CUDA(cudaGetLastError());
    aires_b200_matrix tv_m{};
    tv_m.n_rows = static_cast<uint64_t>(K);
    tv_m.n_cols = static_cast<uint64_t>(c1 - c0);
    tv_m.layout = AIRES_B200_CSR;
    tv_m.location = AIRES_B200_DEVICE;
    tv_m.idx_bytes = 4;
    tv_m.val_bytes = sizeof(V);
    tv_m.ptr = reinterpret_cast<const uint64_t*>(tp);
    tv_m.idx = tc;
    tv_m.val = tv;
    tv_m.span = static_cast<uint64_t>(std::max<int64_t>(x.nnz, 1));
    auto xt = make_operand(ctx, tv_m, mode, /*temp=*/false, kPlanSlots);
    ctx.launches += xt->prep_launches + 6;
    uint32_t* cnt = reinterpret_cast<uint32_t*>(kc);
    uint64_t* toff = static_cast<uint64_t*>(tl.toff.get(std::max<int64_t>(rows, 1) * 8));
    Num3Args<V, IdxT> np =
        make_num3<V, IdxT>(*xt, aptr, abase, acol, aval, rows, heavy, heavy_deg, cnt, toff, ctls + t);
    const uint64_t maxlen = std::max<int64_t>(xt->max_row_len, 1);
    const uint64_t bound = std::min<uint64_t>(static_cast<uint64_t>(rows) * (c1 - c0), span_hint * maxlen);
    np.t_cap = bound + bound / 7 + (static_cast<uint64_t>(ctx.sms) * 64 + 1) * np.stage_block;
    np.tcol = static_cast<IdxT*>(tl.tcol.get(np.t_cap * sizeof(IdxT)));
    np.tval = static_cast<V*>(tl.tval.get(np.t_cap * sizeof(V)));
    if (rows > 0) {
      const int g = static_cast<int>(std::min<int64_t>((rows + 255) / 256, static_cast<int64_t>(ctx.sms) * 16));
      k_classify<<<g, 256, 0, ctx.stream>>>(aptr, rows, heavy_deg, heavy, ctls + t);
      launch_product<V, IdxT>(ctx, np, *xt);
    }
    AB2_CUDA(cudaStreamSynchronize(ctx.stream));  // xt is freed at scope exit
  }
  // row counts -> row_ptr
  uint32_t* csum = static_cast<uint32_t*>(cnt_sum.get(std::max<int64_t>(rows, 1) * 4));
  uint32_t* ro = static_cast<uint32_t*>(roff.get(std::max<int64_t>(rows, 1) * 4));
  AB2_CUDA(cudaMemsetAsync(csum, 0, std::max<int64_t>(rows, 1) * 4, ctx.stream));
  AB2_CUDA(cudaMemsetAsync(ro, 0, std::max<int64_t>(rows, 1) * 4, ctx.stream));
  const int gR = static_cast<int>(std::min<int64_t>((rows + 255) / 256 + 1, static_cast<int64_t>(ctx.sms) * 32));
  for (int64_t t = 0; t < T && rows > 0; t++)
    k_add_counts<<<gR, 256, 0, ctx.stream>>>(csum, static_cast<uint32_t*>(tiles[t].cnt.p), rows);
  int64_t* cptr = ctx.cptr.as<int64_t>(rows + 1);
  const int64_t nb = (rows + kScanTile - 1) / kScanTile;
  int64_t* part = ctx.scan_part.as<int64_t>(std::max<int64_t>(nb, 1));
  if (rows > 0) {
    const int32_t* cin = reinterpret_cast<const int32_t*>(csum);
    k_scan_reduce<<<static_cast<unsigned>(nb), kScanThreads, 0, ctx.stream>>>(cin, rows, part);
    k_scan_part<<<1, 1024, 0, ctx.stream>>>(part, nb, ctls + T);
    k_scan_down<<<static_cast<unsigned>(nb), kScanThreads, 0, ctx.stream>>>(cin, rows, part, cptr);
  } else {
    AB2_CUDA(cudaMemsetAsync(cptr, 0, 8, ctx.stream));
  }
  AB2_CUDA(cudaGetLastError());
  std::vector<Ctl> h(T + 1);
  AB2_CUDA(cudaMemcpyAsync(h.data(), ctls, sizeof(Ctl) * (T + 1), cudaMemcpyDeviceToHost, ctx.stream));
  AB2_CUDA(cudaStreamSynchronize(ctx.stream));
  uint64_t flops = 0;
  for (int64_t t = 0; t < T; t++) {
    if (h[t].bad_row) fail(AIRES_B200_CAPACITY_EXCEEDED, "staging area overflow");
    flops += h[t].flops;
  }
  const uint64_t nnz = rows > 0 ? h[T].nnz : 0;
  void *optr = nullptr, *oidx = nullptr, *oval = nullptr;
  int rc = out.alloc(out.user, static_cast<uint64_t>(rows), nnz, &optr, &oidx, &oval);
  if (rc != 0) fail(rc, "output allocator failed for " + std::to_string(nnz) + " nonzeros");
  IdxT* ccol;
  V* cval;
  if (out.location == AIRES_B200_DEVICE) {
    ccol = static_cast<IdxT*>(oidx);
    cval = static_cast<V*>(oval);
  } else {
    ccol = ctx.c_col.as<IdxT>(std::max<uint64_t>(nnz, 1));
    cval = ctx.c_val.as<V>(std::max<uint64_t>(nnz, 1));
  }
  for (int64_t t = 0; t < T && rows > 0 && nnz > 0; t++)
    k_place_tile<V, IdxT><<<ctx.sms * 8, 256, 0, ctx.stream>>>(
        static_cast<const uint32_t*>(tiles[t].cnt.p), static_cast<const uint64_t*>(tiles[t].toff.p), cptr, ro,
        static_cast<const IdxT*>(tiles[t].tcol.p), static_cast<const V*>(tiles[t].tval.p), rows,
        static_cast<IdxT>(tiles[t].c0), ccol, cval);
  AB2_CUDA(cudaGetLastError());
  if (out.location == AIRES_B200_DEVICE) {
    AB2_CUDA(cudaMemcpyAsync(optr, cptr, (rows + 1) * 8, cudaMemcpyDeviceToDevice, ctx.stream));
  } else {
    AB2_CUDA(cudaMemcpyAsync(optr, cptr, (rows + 1) * 8, cudaMemcpyDeviceToHost, ctx.stream));
    if (nnz) {
      AB2_CUDA(cudaMemcpyAsync(oidx, ccol, nnz * sizeof(IdxT), cudaMemcpyDeviceToHost, ctx.stream));
      AB2_CUDA(cudaMemcpyAsync(oval, cval, nnz * sizeof(V), cudaMemcpyDeviceToHost, ctx.stream));
    }
  }
  AB2_CUDA(cudaStreamSynchronize(ctx.stream));
  ctx.launches += static_cast<int>(2 * T + 3);
  out.n_rows = static_cast<uint64_t>(rows);
  out.n_cols = static_cast<uint64_t>(n_cols);
  out.nnz = nnz;
  out.flops = flops;
}

}  // namespace

namespace {
template <class V, class IdxT>
int tile_product_staged_t(Ctx& ctx, const XOperand& x, const TileStaged& t) {
  if (t.rows <= 0) return 0;
  const int64_t heavy_deg = option("heavy_deg", 1024);
  const int g = static_cast<int>(std::min<int64_t>((t.rows + 255) / 256, static_cast<int64_t>(ctx.sms) * 16));
  k_classify<<<g, 256, 0, ctx.stream>>>(t.aptr, t.rows, heavy_deg, t.heavy, t.ctl);
  AB2_CUDA(cudaGetLastError());
  Num3Args<V, IdxT> np = make_num3<V, IdxT>(x, t.aptr, t.abase, static_cast<const IdxT*>(t.acol),
                                            static_cast<const V*>(t.aval), t.rows, t.heavy, heavy_deg, t.cnt,
                                            t.toff, t.ctl);
  np.tcol = static_cast<IdxT*>(t.tcol);
  np.tval = static_cast<V*>(t.tval);
  np.t_cap = t.t_cap;
  launch_product<V, IdxT>(ctx, np, x);
  const int64_t nb = (t.rows + kScanTile - 1) / kScanTile;
  const int32_t* cin = reinterpret_cast<const int32_t*>(t.cnt);
  k_scan_reduce<<<static_cast<unsigned>(nb), kScanThreads, 0, ctx.stream>>>(cin, t.rows, t.part);
  k_scan_part<<<1, 1024, 0, ctx.stream>>>(t.part, nb, t.ctl);
  k_scan_down<<<static_cast<unsigned>(nb), kScanThreads, 0, ctx.stream>>>(cin, t.rows, t.part, t.cptr);
  k_place<V, IdxT><<<ctx.sms * 8, 256, 0, ctx.stream>>>(t.cnt, t.toff, t.cptr, np.tcol, np.tval, t.rows,
                                                        static_cast<IdxT*>(t.ccol), static_cast<V*>(t.cval));
  AB2_CUDA(cudaGetLastError());
  return 6;
}
}  // namespace

uint64_t c_bound(const XOperand& x, uint64_t rows, uint64_t a_nnz) {
  const uint64_t maxlen = static_cast<uint64_t>(std::max<int64_t>(x.max_row_len, 1));
  return std::min<uint64_t>(rows * static_cast<uint64_t>(x.n_cols), a_nnz * maxlen);
}

// Staging entries of one product pass over `rows` rows: the nnz bound + 1/7 (each warp's bump
// reservation wastes less than one row out of >= 8 rows' worth) + one reservation block per
// resident warp (the same sizing as run_product).
uint64_t staged_capacity(Ctx& ctx, const XOperand& x, uint64_t rows, uint64_t a_nnz) {
  const uint64_t bound = c_bound(x, rows, a_nnz);
  const uint64_t stride = static_cast<uint64_t>((x.n_cols + 1 + 31) & ~int64_t(31));
  const uint64_t block = std::max<uint64_t>(4096, 8 * stride);
  return bound + bound / 7 + (static_cast<uint64_t>(ctx.sms) * 64 + 1) * block;
}

int tile_product_staged(Ctx& ctx, const XOperand& x, uint32_t idx_bytes, const TileStaged& t) {
  const bool f32 = x.mode == AIRES_B200_MODE_FP32;
  if (idx_bytes == 4)
    return f32 ? tile_product_staged_t<float, uint32_t>(ctx, x, t) : tile_product_staged_t<double, uint32_t>(ctx, x, t);
  return f32 ? tile_product_staged_t<float, uint64_t>(ctx, x, t) : tile_product_staged_t<double, uint64_t>(ctx, x, t);
}

int tile_product(Ctx& ctx, const XOperand& x, uint32_t idx_bytes, const TilePass& t) {
  const bool f32 = x.mode == AIRES_B200_MODE_FP32;
  if (idx_bytes == 4) return f32 ? tile_product_t<float, uint32_t>(ctx, x, t) : tile_product_t<double, uint32_t>(ctx, x, t);
  return f32 ? tile_product_t<float, uint64_t>(ctx, x, t) : tile_product_t<double, uint64_t>(ctx, x, t);
}

int tile_symbolic(Ctx& ctx, const XOperand& x, uint32_t idx_bytes, const TileSym& t) {
  return idx_bytes == 4 ? tile_symbolic_t<uint32_t>(ctx, x, t) : tile_symbolic_t<uint64_t>(ctx, x, t);
}

void spgemm_rows(Ctx& ctx, const aires_b200_matrix& a, const XOperand& x, aires_b200_output& out) {
  if (a.layout != AIRES_B200_CSR) fail(AIRES_B200_INVALID_ARGUMENT, "A must be CSR");
  if ((a.idx_bytes != 4 && a.idx_bytes != 8) || (a.val_bytes != 4 && a.val_bytes != 8))
    fail(AIRES_B200_INVALID_ARGUMENT, "A idx_bytes/val_bytes must be 4 or 8");
  if ((out.idx_bytes != 4 && out.idx_bytes != 8) || (out.val_bytes != 4 && out.val_bytes != 8))
    fail(AIRES_B200_INVALID_ARGUMENT, "output idx_bytes/val_bytes must be 4 or 8");
  if (!out.alloc) fail(AIRES_B200_INVALID_ARGUMENT, "output allocator is null");
  if (a.n_cols != static_cast<uint64_t>(x.K))
    fail(AIRES_B200_DIMENSION_MISMATCH, "inner dimensions " + std::to_string(a.n_cols) + " and " +
                                            std::to_string(x.K) + " differ");
  if (a.ptr == nullptr) fail(AIRES_B200_INVALID_ARGUMENT, "A ptr is null");
  const size_t vsize = x.mode == AIRES_B200_MODE_FP32 ? 4 : 8;
  if (out.val_bytes != vsize)
    fail(AIRES_B200_INVALID_ARGUMENT, "output value width must match the operand's arithmetic mode");
  const int64_t rows = static_cast<int64_t>(a.n_rows);

  // Stage A on the device.
  const uint64_t* aptr = a.ptr;
  uint64_t abase = 0;
  const void* acol = a.idx;
  const void* aval = a.val;
  uint64_t p0 = 0, p1 = 0;
  AB2_CUDA(cudaEventRecord(ctx.ev[8], ctx.stream));
  if (a.location == AIRES_B200_HOST) {
    p0 = a.ptr[0];
    p1 = a.ptr[rows];
    if (p1 < p0 || p1 > a.span) fail(AIRES_B200_INDEX_OUT_OF_RANGE, "A row pointers exceed the index span");
    uint64_t* dptr = ctx.a_ptr.as<uint64_t>(rows + 1);
    void* dcol = ctx.a_col.get(std::max<uint64_t>(p1 - p0, 1) * a.idx_bytes);
    void* dval = ctx.a_val.get(std::max<uint64_t>(p1 - p0, 1) * a.val_bytes);
    AB2_CUDA(cudaMemcpyAsync(dptr, a.ptr, (rows + 1) * 8, cudaMemcpyHostToDevice, ctx.stream));
    if (p1 > p0) {
      AB2_CUDA(cudaMemcpyAsync(dcol, static_cast<const char*>(a.idx) + p0 * a.idx_bytes, (p1 - p0) * a.idx_bytes,
                               cudaMemcpyHostToDevice, ctx.stream));
      AB2_CUDA(cudaMemcpyAsync(dval, static_cast<const char*>(a.val) + p0 * a.val_bytes, (p1 - p0) * a.val_bytes,
                               cudaMemcpyHostToDevice, ctx.stream));
    }
    aptr = dptr;
    abase = p0;
    acol = dcol;
    aval = dval;
  } else if (a.idx_bytes != out.idx_bytes || a.val_bytes != vsize) {
    // conversions need the span ends
    AB2_CUDA(cudaMemcpyAsync(&p0, a.ptr, 8, cudaMemcpyDeviceToHost, ctx.stream));
    AB2_CUDA(cudaMemcpyAsync(&p1, a.ptr + rows, 8, cudaMemcpyDeviceToHost, ctx.stream));
    AB2_CUDA(cudaStreamSynchronize(ctx.stream));
    if (p1 < p0 || p1 > a.span) fail(AIRES_B200_INDEX_OUT_OF_RANGE, "A row pointers exceed the index span");
    abase = p0;
    acol = static_cast<const char*>(a.idx) + p0 * a.idx_bytes;
    aval = static_cast<const char*>(a.val) + p0 * a.val_bytes;
  }
  AB2_CUDA(cudaEventRecord(ctx.ev[9], ctx.stream));
  // Width conversions: kernels read A's columns at the output index width and A's
  // values at the arithmetic width.
  const int64_t span = static_cast<int64_t>(p1 - p0);
  if (a.idx_bytes != out.idx_bytes) {
    void* c2 = ctx.a_col2.get(std::max<int64_t>(span, 1) * out.idx_bytes);
    if (a.idx_bytes == 8)
      convert<uint64_t, uint32_t>(ctx, acol, c2, span);
    else
      convert<uint32_t, uint64_t>(ctx, acol, c2, span);
    acol = c2;
  }
  if (a.val_bytes != vsize) {
    void* v2 = ctx.a_val2.get(std::max<int64_t>(span, 1) * vsize);
    if (a.val_bytes == 8)
      convert<double, float>(ctx, aval, v2, span);
    else
      convert<float, double>(ctx, aval, v2, span);
    aval = v2;
  }
  const uint64_t span_hint = a.location == AIRES_B200_HOST || p1 > p0 ? p1 - p0 : a.span;
  if (x.wide) {
    if (out.idx_bytes == 4 && vsize == 4)
      wide_product<float, uint32_t>(ctx, a, x, out, aptr, abase, static_cast<const uint32_t*>(acol),
                                    static_cast<const float*>(aval), span_hint);
    else if (out.idx_bytes == 4)
      wide_product<double, uint32_t>(ctx, a, x, out, aptr, abase, static_cast<const uint32_t*>(acol),
                                     static_cast<const double*>(aval), span_hint);
    else if (vsize == 4)
      wide_product<float, uint64_t>(ctx, a, x, out, aptr, abase, static_cast<const uint64_t*>(acol),
                                    static_cast<const float*>(aval), span_hint);
    else
      wide_product<double, uint64_t>(ctx, a, x, out, aptr, abase, static_cast<const uint64_t*>(acol),
                                     static_cast<const double*>(aval), span_hint);
  } else if (out.idx_bytes == 4 && vsize == 4)
    run_product<float, uint32_t>(ctx, a, x, out, aptr, abase, static_cast<const uint32_t*>(acol),
                             static_cast<const float*>(aval), span_hint);
  else if (out.idx_bytes == 4)
    run_product<double, uint32_t>(ctx, a, x, out, aptr, abase, static_cast<const uint32_t*>(acol),
                              static_cast<const double*>(aval), span_hint);
  else if (vsize == 4)
    run_product<float, uint64_t>(ctx, a, x, out, aptr, abase, static_cast<const uint64_t*>(acol),
                             static_cast<const float*>(aval), span_hint);
  else
    run_product<double, uint64_t>(ctx, a, x, out, aptr, abase, static_cast<const uint64_t*>(acol),
                              static_cast<const double*>(aval), span_hint);
  float ms = 0;
  AB2_CUDA(cudaEventElapsedTime(&ms, ctx.ev[8], ctx.ev[9]));
  ctx.prof[kPH2D] = ms;
}

}  // namespace ab2
