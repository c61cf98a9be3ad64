// ab2_gcn.cu -- the steps either side of A·X in a GCN layer, on the device.
//
//   K9 normalize_adjacency (gcn.hpp:29-72): Ã = D̂^-½ (A + I) D̂^-½.  Self loops are inserted at
//      their sorted position (a diagonal entry present in A becomes a_rr + 1), the weighted degree
//      of each row is summed left to right in fp64 exactly as the reference does, and every entry
//      becomes v / sqrt(d_i * d_j) with one IEEE multiply, sqrt and divide (the division form keeps
//      1/sqrt(4) = 0.5 exact) -- bit-identical to the reference.
//   K8 combine (gcn.hpp:90-116): H' = ReLU(X · W), X sparse CSR, W dense row-major; entries <= 0
//      after the activation are dropped (re-sparsified CSR).  One warp per row, lanes over output
//      columns (tiles of 256), terms added in ascending k with separate multiply and add: fp64 is
//      bit-identical to the reference; fp32 is within tolerance.  One-tile widths (<= 256 output
//      columns) run one pass: positives go to a bump-allocated staging area with per-row counts,
//      then scan + K_place give the exact CSR (the product is computed once; the extra bytes are
//      one streaming copy of the output).  Wider W: two passes (count, fill) around a scan.
#include <algorithm>
#include <cmath>

#include "ab2_internal.h"
#include "ab2_kernels.cuh"
#include "ab2_numeric.cuh"

namespace ab2 {

namespace {

template <class IdxT>
__global__ void k_norm_count(const uint64_t* __restrict__ ptr, uint64_t base, const IdxT* __restrict__ col,
                             int64_t n, int32_t* __restrict__ cnt, Ctl* __restrict__ ctl) {
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < n;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t lo = static_cast<int64_t>(ptr[r] - base), hi = static_cast<int64_t>(ptr[r + 1] - base);
    const int64_t len = hi - lo;
    while (lo < hi) {  // lower_bound(r)
      const int64_t mid = (lo + hi) >> 1;
      if (static_cast<int64_t>(col[mid]) < r)
        lo = mid + 1;
      else
        hi = mid;
    }
    const bool diag = lo < static_cast<int64_t>(ptr[r + 1] - base) && static_cast<int64_t>(col[lo]) == r;
    cnt[r] = static_cast<int32_t>(len + (diag ? 0 : 1));
  }
  (void)ctl;
}

template <class IdxT, class VIn>
__global__ void k_norm_check(const IdxT* __restrict__ col, const VIn* __restrict__ val, uint64_t nnz, int64_t n,
                             Ctl* __restrict__ ctl) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < nnz;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    if (val[i] < VIn(0)) ctl->bad_row = 1;                                // negative_weight
    if (static_cast<uint64_t>(col[i]) >= static_cast<uint64_t>(n)) ctl->n_fix = 1;  // index_out_of_range
  }
}

// Â = A + I at its sorted positions (values before normalisation, fp64).
template <class IdxT, class VIn, class IdxO>
__global__ void k_norm_fill(const uint64_t* __restrict__ ptr, uint64_t base, const IdxT* __restrict__ col,
                            const VIn* __restrict__ val, int64_t n, const int64_t* __restrict__ optr,
                            IdxO* __restrict__ ocol, double* __restrict__ oval, int32_t* __restrict__ orow) {
  const int lane = lane_id();
  const int64_t wid = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r = wid; r < n; r += nw) {
    const int64_t s = static_cast<int64_t>(ptr[r] - base), e = static_cast<int64_t>(ptr[r + 1] - base);
    int64_t lo = s, hi = e;
    if (e - s <= 32) {  // short row: one coalesced load and a ballot instead of a dependent search
      const bool below = s + lane < e && static_cast<int64_t>(col[s + lane]) < r;
      lo = s + __popc(__ballot_sync(kFull, below));
      hi = lo;
    }
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (static_cast<int64_t>(col[mid]) < r)
        lo = mid + 1;
      else
        hi = mid;
    }
    const int64_t p = lo;  // first entry with col >= r
    const bool diag = p < e && static_cast<int64_t>(col[p]) == r;
    const int64_t o = optr[r];
    for (int64_t i = s + lane; i < e; i += 32) {
      if (diag && i == p) continue;
      const int64_t dst = o + (i - s) + (i >= p && !diag ? 1 : 0);
      ocol[dst] = static_cast<IdxO>(col[i]);
      oval[dst] = static_cast<double>(val[i]);
      if (orow) orow[dst] = static_cast<int32_t>(r);
    }
    if (lane == 0) {
      ocol[o + (p - s)] = static_cast<IdxO>(r);
      oval[o + (p - s)] = diag ? static_cast<double>(val[p]) + 1.0 : 1.0;
      if (orow) orow[o + (p - s)] = static_cast<int32_t>(r);
    }
  }
}

// Rows of Â are short on GCN graphs (~26 entries on the products shape) with a power-law tail. A warp
// takes 32 consecutive rows (one per lane) and streams their contiguous entries through shared memory
// in coalesced windows; each lane adds its own row's values left to right as the windows pass, so
// the sum keeps the reference's order (gcn.hpp:61-64).  Rows longer than kNormHeavy are summed by the
// whole warp instead (coalesced 32-entry loads, the next chunk in flight).  Earlier forms: a thread
// per row reading its row from global (0.73 ms for the products-shaped Â: 32 rows' strided loads per
// instruction), a warp per row (1.2 ms, lanes idle).
constexpr int64_t kNormHeavy = 256;
constexpr int kNormWin = 512, kNormWarps = 8;

// weighted degrees, summed left to right, exact for any weights.
__global__ void __launch_bounds__(kNormWarps * 32) k_norm_degree(const int64_t* __restrict__ optr,
                                                                  const double* __restrict__ oval, int64_t n,
                                                                  double* __restrict__ deg) {
  __shared__ double win[kNormWarps][kNormWin];
  double* buf = win[threadIdx.x >> 5];
  const int lane = lane_id();
  const int64_t wid = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t rb = wid * 32; rb < n; rb += nw * 32) {
    const int64_t r = rb + lane;
    int64_t s = 0, e = 0;
    if (r < n) s = optr[r], e = optr[r + 1];
    const bool heavy = e - s > kNormHeavy;
    const int64_t S = optr[rb], E = optr[rb + 32 < n ? rb + 32 : n];
    double d = 0.0;
    int64_t pos = heavy ? e : s;
    for (int64_t w0 = S; w0 < E; w0 += kNormWin) {
      const int64_t w1 = w0 + kNormWin < E ? w0 + kNormWin : E;
      if (__any_sync(kFull, pos < e && pos < w1)) {  // some light row has entries in this window
#pragma unroll 4
        for (int64_t i = w0 + lane; i < w1; i += 32) buf[i - w0] = oval[i];
        __syncwarp();
        const int64_t lim = e < w1 ? e : w1;
        for (; pos + 4 <= lim; pos += 4) {  // loads ahead of the (ordered) adds
          const double v0 = buf[pos - w0], v1 = buf[pos - w0 + 1], v2 = buf[pos - w0 + 2], v3 = buf[pos - w0 + 3];
          d = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(d, v0), v1), v2), v3);
        }
        for (; pos < lim; pos++) d = __dadd_rn(d, buf[pos - w0]);
        __syncwarp();
      }
    }
    if (r < n && !heavy) deg[r] = d;
    for (unsigned hm = __ballot_sync(kFull, heavy); hm; hm &= hm - 1) {
      const int h = __ffs(hm) - 1;
      const int64_t hs = __shfl_sync(kFull, s, h), he = __shfl_sync(kFull, e, h);
      double hd = 0.0;
      double v = hs + lane < he ? oval[hs + lane] : 0.0;
      for (int64_t b = hs; b < he; b += 32) {
        const double nv = b + 32 + lane < he ? oval[b + 32 + lane] : 0.0;  // next chunk in flight
        const int m = static_cast<int>(he - b < 32 ? he - b : 32);
        for (int i = 0; i < m; i++) hd = __dadd_rn(hd, __shfl_sync(kFull, v, i));
        v = nv;
      }
      if (lane == h) deg[rb + h] = hd;
    }
  }
}

// v / sqrt(d_i * d_j): one IEEE multiply, sqrt and divide, one thread per entry (the fill pass
// records each entry's row): every lane busy and every stream coalesced; only deg[] is gathered
// (L2-resident).  A warp per row measured 1.21 ms at cfg5 (lanes idle on ~26-entry rows, the
// per-row load chain exposed), a thread per row 1.40 ms; this form 0.37 ms.  (Summing the degree
// inside the fill's warp-per-row pass measured slower: 2.57 ms vs 0.90 + 0.73.)
template <class IdxO, class VO>
__global__ void k_norm_scale_flat(const int32_t* __restrict__ orow, const IdxO* __restrict__ ocol,
                                  const double* __restrict__ oval, const double* __restrict__ deg, int64_t nnz,
                                  VO* __restrict__ out) {
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < nnz;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[k] = static_cast<VO>(
        __ddiv_rn(oval[k], __dsqrt_rn(__dmul_rn(deg[orow[k]], deg[static_cast<int64_t>(ocol[k])]))));
}

// (row form, used when the row ids do not fit int32)
template <class IdxO, class VO>
__global__ void k_norm_scale(const int64_t* __restrict__ optr, const IdxO* __restrict__ ocol,
                             const double* __restrict__ oval, const double* __restrict__ deg, int64_t n,
                             VO* __restrict__ out) {
  const int lane = lane_id();
  const int64_t wid = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r = wid; r < n; r += nw) {
    const double dr = deg[r];
    for (int64_t k = optr[r] + lane; k < optr[r + 1]; k += 32)
      out[k] = static_cast<VO>(__ddiv_rn(oval[k], __dsqrt_rn(__dmul_rn(dr, deg[static_cast<int64_t>(ocol[k])]))));
  }
}

// ---- combine ---------------------------------------------------------------
template <class V>
__device__ __forceinline__ V mul_add(V acc, V a, V b) {
  if constexpr (sizeof(V) == 8)
    return __dadd_rn(acc, __dmul_rn(a, b));
  else
    return __fadd_rn(acc, __fmul_rn(a, b));
}

// FILL = false: per-row positive counts; FILL = true: writes the positives at optr[r].
// SMEM: W is staged once per CTA in shared memory (every X entry reads a whole W row, so from
// global memory the L1 datapath bound the kernel: 36 ms for the products-shaped layer 2).
// STAGE (w_cols <= 32 * J): one pass; the row's positives go to a warp's bump reservation in the
// staging area (ocol/oval, capacity t_cap), cnt[r] / toff[r] record where (K_place finishes).
template <class V, class IdxT, class IdxO, int J, bool FILL, bool SMEM, bool STAGE = false>
__global__ void __launch_bounds__(256) k_combine(const uint64_t* __restrict__ xptr, uint64_t xbase,
                                                 const IdxT* __restrict__ xcol, const V* __restrict__ xval,
                                                 int64_t rows, const V* __restrict__ wg, int64_t w_rows, int64_t w_cols,
                                                 int32_t* __restrict__ cnt, const int64_t* __restrict__ optr,
                                                 IdxO* __restrict__ ocol, V* __restrict__ oval, Ctl* __restrict__ ctl,
                                                 uint64_t* __restrict__ toff = nullptr, uint64_t t_cap = 0) {
  StageCursor stage;
  constexpr int TW = 32 * J;  // output columns per tile
  extern __shared__ __align__(16) unsigned char smem_w[];
  const V* __restrict__ w = wg;
  if constexpr (SMEM) {
    V* ws = reinterpret_cast<V*>(smem_w);
    for (int64_t i = threadIdx.x; i < w_rows * w_cols; i += blockDim.x) ws[i] = wg[i];
    __syncthreads();
    w = ws;
  }
  const int lane = lane_id();
  const int64_t wid = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r = wid; r < rows; r += nw) {
    const int64_t s = static_cast<int64_t>(xptr[r] - xbase), e = static_cast<int64_t>(xptr[r + 1] - xbase);
    uint32_t written = 0;
    for (int64_t t0 = 0; t0 < w_cols; t0 += TW) {
      V acc[J];
#pragma unroll
      for (int j = 0; j < J; j++) acc[j] = V(0);
      // the row's entries are read 32 at a time (coalesced) and broadcast with SHFL, in order
      for (int64_t k0 = s; k0 < e; k0 += 32) {
        uint64_t lin = 0;
        V lv = V(0);
        if (k0 + lane < e) {
          lin = static_cast<uint64_t>(xcol[k0 + lane]);
          lv = xval[k0 + lane];
          if (lin >= static_cast<uint64_t>(w_rows)) {
            ctl->bad_row = 1;
            lin = 0;
            lv = V(0);
          }
        }
        const int cnt_k = static_cast<int>(e - k0 < 32 ? e - k0 : 32);
        for (int kk = 0; kk < cnt_k; kk++) {
          const uint64_t in = __shfl_sync(kFull, lin, kk);
          const V v = __shfl_sync(kFull, lv, kk);
          const V* wr = w + in * w_cols + t0;
#pragma unroll
          for (int j = 0; j < J; j++) {
            const int64_t c = lane + 32 * j;
            if (t0 + c < w_cols) acc[j] = mul_add<V>(acc[j], v, wr[c]);
          }
        }
      }
      if constexpr (STAGE) {
        unsigned m[J];
        uint32_t total = 0;
#pragma unroll
        for (int j = 0; j < J; j++) {
          m[j] = __ballot_sync(kFull, t0 + lane + 32 * j < w_cols && acc[j] > V(0));
          total += __popc(m[j]);
        }
        const unsigned long long off = stage.take(total, ctl, 4096);
        if (off + total <= t_cap) {
#pragma unroll
          for (int j = 0; j < J; j++) {
            if (m[j] >> lane & 1u) {
              const unsigned long long dst = off + written + __popc(m[j] & ((1u << lane) - 1));
              ocol[dst] = static_cast<IdxO>(t0 + lane + 32 * j);
              oval[dst] = acc[j];
            }
            written += __popc(m[j]);
          }
        } else if (lane == 0) {
          ctl->bad_row = 2;  // staging overflow (the host sized it for the dense bound)
        }
        if (lane == 0) {
          cnt[r] = static_cast<int32_t>(total);
          toff[r] = off;
        }
        continue;
      }
#pragma unroll
      for (int j = 0; j < J; j++) {
        const int64_t c = t0 + lane + 32 * j;
        const bool pos = c < w_cols && acc[j] > V(0);
        const unsigned m = __ballot_sync(kFull, pos);
        if constexpr (FILL) {
          if (pos) {
            const int64_t dst = optr[r] + written + __popc(m & ((1u << lane) - 1));
            ocol[dst] = static_cast<IdxO>(c);
            oval[dst] = acc[j];
          }
        }
        written += __popc(m);
      }
    }
    if constexpr (!FILL && !STAGE) {
      if (lane == 0) cnt[r] = static_cast<int32_t>(written);
    }
  }
}

void scan_counts(Ctx& ctx, const int32_t* cnt, int64_t n, int64_t* out, Ctl* ctl, int* launches) {
  if (n <= 0) {
    AB2_CUDA(cudaMemsetAsync(out, 0, 8, ctx.stream));
    AB2_CUDA(cudaMemsetAsync(&ctl->nnz, 0, 8, ctx.stream));
    return;
  }
  const int64_t nb = (n + kScanTile - 1) / kScanTile;
  int64_t* part = ctx.scan_part.as<int64_t>(std::max<int64_t>(nb, 1));
  k_scan_reduce<<<static_cast<unsigned>(nb), kScanThreads, 0, ctx.stream>>>(cnt, n, part);
  k_scan_part<<<1, 1024, 0, ctx.stream>>>(part, nb, ctl);
  k_scan_down<<<static_cast<unsigned>(nb), kScanThreads, 0, ctx.stream>>>(cnt, n, part, out);
  AB2_CUDA(cudaGetLastError());
  *launches += 3;
}

int grid_of(int64_t n, int threads, int sms) {
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((n + threads - 1) / threads, int64_t(sms) * 32)));
}

// Stages a host CSR (ptr, idx, val) on the device through the context's A buffers.
struct Staged {
  const uint64_t* ptr;
  uint64_t base;   // ptr value of idx[0] / val[0]
  const void* idx;
  const void* val;
  uint64_t nnz;
  uint64_t first;  // index of the first used entry in idx / val
};

Staged stage_csr(Ctx& ctx, const aires_b200_matrix& m) {
  Staged s{m.ptr, 0, m.idx, m.val, 0, 0};
  const uint64_t n = m.n_rows;
  if (m.location == AIRES_B200_HOST) {
    const uint64_t p0 = m.ptr[0], p1 = m.ptr[n];
    if (p1 < p0 || p1 > m.span) fail(AIRES_B200_INDEX_OUT_OF_RANGE, "row pointers exceed the index span");
    uint64_t* dp = ctx.a_ptr.as<uint64_t>(n + 1);
    void* di = ctx.a_col.get(std::max<uint64_t>(p1 - p0, 1) * m.idx_bytes);
    void* dv = ctx.a_val.get(std::max<uint64_t>(p1 - p0, 1) * m.val_bytes);
    AB2_CUDA(cudaMemcpyAsync(dp, m.ptr, (n + 1) * 8, cudaMemcpyHostToDevice, ctx.stream));
    if (p1 > p0) {
      AB2_CUDA(cudaMemcpyAsync(di, static_cast<const char*>(m.idx) + p0 * m.idx_bytes, (p1 - p0) * m.idx_bytes,
                               cudaMemcpyHostToDevice, ctx.stream));
      AB2_CUDA(cudaMemcpyAsync(dv, static_cast<const char*>(m.val) + p0 * m.val_bytes, (p1 - p0) * m.val_bytes,
                               cudaMemcpyHostToDevice, ctx.stream));
    }
    s = Staged{dp, p0, di, dv, p1 - p0, 0};
  } else {
    uint64_t p[2] = {0, 0};
    AB2_CUDA(cudaMemcpyAsync(&p[0], m.ptr, 8, cudaMemcpyDeviceToHost, ctx.stream));
    AB2_CUDA(cudaMemcpyAsync(&p[1], m.ptr + n, 8, cudaMemcpyDeviceToHost, ctx.stream));
    AB2_CUDA(cudaStreamSynchronize(ctx.stream));
    if (p[1] < p[0] || p[1] > m.span) fail(AIRES_B200_INDEX_OUT_OF_RANGE, "row pointers exceed the index span");
    s.nnz = p[1] - p[0];
    s.first = p[0];  // kernels index idx/val by ptr[r] - base with base 0 (absolute pointers)
  }
  return s;
}

// The result's arrays, allocated through the caller's allocator as soon as nnz is known: a device
// result is written in place by the kernels (no staging copy of idx/val), a host result is built in
// the context's buffers and copied down by deliver().
template <class IdxO, class VO>
struct OutBufs {
  void *optr = nullptr, *oidx = nullptr, *oval = nullptr;
  IdxO* col = nullptr;  // where the kernels write
  VO* val = nullptr;
  bool device = false;
};
template <class IdxO, class VO>
OutBufs<IdxO, VO> out_alloc(Ctx& ctx, aires_b200_output& out, uint64_t rows, uint64_t nnz) {
  OutBufs<IdxO, VO> o;
  const int rc = out.alloc(out.user, rows, nnz, &o.optr, &o.oidx, &o.oval);
  if (rc != 0) fail(rc, "output allocator failed for " + std::to_string(nnz) + " nonzeros");
  o.device = out.location == AIRES_B200_DEVICE;
  o.col = o.device ? static_cast<IdxO*>(o.oidx) : static_cast<IdxO*>(ctx.c_col.get(std::max<uint64_t>(nnz, 1) * sizeof(IdxO)));
  o.val = o.device ? static_cast<VO*>(o.oval) : static_cast<VO*>(ctx.c_val.get(std::max<uint64_t>(nnz, 1) * sizeof(VO)));
  return o;
}
// row_ptr (and, for a host result, idx/val) to the caller's arrays; waits for the stream.
template <class IdxO, class VO>
void deliver(Ctx& ctx, aires_b200_output& out, uint64_t rows, uint64_t cols, uint64_t nnz, const int64_t* dptr,
             const OutBufs<IdxO, VO>& o) {
  const cudaMemcpyKind kind = o.device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
  AB2_CUDA(cudaMemcpyAsync(o.optr, dptr, (rows + 1) * 8, kind, ctx.stream));
  if (nnz && !o.device) {
    AB2_CUDA(cudaMemcpyAsync(o.oidx, o.col, nnz * sizeof(IdxO), kind, ctx.stream));
    AB2_CUDA(cudaMemcpyAsync(o.oval, o.val, nnz * sizeof(VO), kind, ctx.stream));
  }
  AB2_CUDA(cudaStreamSynchronize(ctx.stream));
  out.n_rows = rows;
  out.n_cols = cols;
  out.nnz = nnz;
  out.flops = 0;
}

template <class IdxT, class VIn, class IdxO, class VO>
void normalize_t(Ctx& ctx, const aires_b200_matrix& a, aires_b200_output& out) {
  const int64_t n = static_cast<int64_t>(a.n_rows);
  Staged s = stage_csr(ctx, a);
  Ctl* ctl = ctx.ctl.as<Ctl>(1);
  AB2_CUDA(cudaMemsetAsync(ctl, 0, sizeof(Ctl), ctx.stream));
  int32_t* cnt = ctx.cnt.as<int32_t>(std::max<int64_t>(n, 1));
  int64_t* optr = ctx.cptr.as<int64_t>(n + 1);
  const IdxT* col = static_cast<const IdxT*>(s.idx);
  const VIn* val = static_cast<const VIn*>(s.val);
  int launches = 0;
  if (s.nnz) {
    k_norm_check<IdxT, VIn><<<grid_of(static_cast<int64_t>(s.nnz), 256, ctx.sms), 256, 0, ctx.stream>>>(
        col + s.first, val + s.first, s.nnz, n, ctl);
    launches++;
  }
  if (n > 0) {
    k_norm_count<IdxT><<<grid_of(n, 256, ctx.sms), 256, 0, ctx.stream>>>(s.ptr, s.base, col, n, cnt, ctl);
    launches++;
  }
  scan_counts(ctx, cnt, n, optr, ctl, &launches);
  Ctl* h = static_cast<Ctl*>(ctx.h_ctl.get(sizeof(Ctl)));
  AB2_CUDA(cudaMemcpyAsync(h, ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, ctx.stream));
  AB2_CUDA(cudaStreamSynchronize(ctx.stream));
  if (h->bad_row) fail(1 + 14, "adjacency weights must be nonnegative");  // errc::negative_weight
  if (h->n_fix) fail(AIRES_B200_INDEX_OUT_OF_RANGE, "column index outside the square adjacency");
  const uint64_t nnz = n > 0 ? h->nnz : 0;
  const OutBufs<IdxO, VO> ob = out_alloc<IdxO, VO>(ctx, out, static_cast<uint64_t>(n), nnz);
  IdxO* ocol = ob.col;
  double* oval = static_cast<double*>(ctx.t_val.get(std::max<uint64_t>(nnz, 1) * 8));
  const bool flat = n < (int64_t(1) << 31);  // per-entry row ids for the flat scale pass
  int32_t* orow = flat ? static_cast<int32_t*>(ctx.t_col.get(std::max<uint64_t>(nnz, 1) * 4)) : nullptr;
  double* deg = static_cast<double*>(ctx.rflops.get(std::max<int64_t>(n, 1) * 8));
  VO* outv = ob.val;
  if (n > 0) {
    k_norm_fill<IdxT, VIn, IdxO><<<grid_of(n * 32, 256, ctx.sms), 256, 0, ctx.stream>>>(s.ptr, s.base, col, val, n,
                                                                                       optr, ocol, oval, orow);
    k_norm_degree<<<static_cast<unsigned>(std::min<int64_t>((n + 32 * kNormWarps - 1) / (32 * kNormWarps),
                                                            static_cast<int64_t>(ctx.sms) * 8)),
                    kNormWarps * 32, 0, ctx.stream>>>(optr, oval, n, deg);
    if (flat)
      k_norm_scale_flat<IdxO, VO><<<grid_of(static_cast<int64_t>(nnz), 256, ctx.sms), 256, 0, ctx.stream>>>(
          orow, ocol, oval, deg, static_cast<int64_t>(nnz), outv);
    else
      k_norm_scale<IdxO, VO><<<grid_of(n * 32, 256, ctx.sms), 256, 0, ctx.stream>>>(optr, ocol, oval, deg, n, outv);
    AB2_CUDA(cudaGetLastError());
    launches += 3;
  }
  deliver<IdxO, VO>(ctx, out, static_cast<uint64_t>(n), static_cast<uint64_t>(n), nnz, optr, ob);
  ctx.launches = launches;
}

template <class V, class IdxT, class IdxO, int J, bool FILL, bool SMEM, bool STAGE = false>
void combine_launch2(Ctx& ctx, const Staged& s, int64_t rows, const V* w, int64_t w_rows, int64_t w_cols, int32_t* cnt,
                     int64_t* optr, IdxO* ocol, V* oval, Ctl* ctl, uint64_t* toff = nullptr, uint64_t t_cap = 0) {
  auto k = k_combine<V, IdxT, IdxO, J, FILL, SMEM, STAGE>;
  size_t smem = 0;
  int grid = grid_of(rows * 32, 256, ctx.sms);
  if constexpr (SMEM) {
    smem = static_cast<size_t>(w_rows * w_cols) * sizeof(V);
    AB2_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    int nb = 0;
    AB2_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k, 256, smem));
    grid = std::max(1, std::min(grid, std::max(nb, 1) * ctx.sms));  // persistent: W staged once per CTA
  }
  k<<<grid, 256, smem, ctx.stream>>>(s.ptr, s.base, static_cast<const IdxT*>(s.idx), static_cast<const V*>(s.val),
                                     rows, w, w_rows, w_cols, cnt, optr, ocol, oval, ctl, toff, t_cap);
  AB2_CUDA(cudaGetLastError());
}

// fp32, 96 <= w_cols <= 256, W in shared memory: each lane owns 4 consecutive output columns per
// 128-column group (one LDS.128 of the zero-padded W row per group and X entry, FFMA -- fp32 mode
// is within tolerance, not bit-exact), so an X entry costs 2 SHFL + H LDS.128 + 4H FFMA instead of
// 8 LDS + 8 FMUL + 8 FADD + 8 bounds checks.  Padded columns hold W = 0, so they are never
// positive and drop out with the ReLU.  Output in ascending columns: group-major, then lane
// (warp scan of the per-lane positive counts), then the lane's 4 columns.  One pass into staging.
template <class IdxT, class IdxO, int H>
__global__ void __launch_bounds__(512) k_combine_v4(const uint64_t* __restrict__ xptr, uint64_t xbase,
                                                    const IdxT* __restrict__ xcol, const float* __restrict__ xval,
                                                    int64_t rows, const float* __restrict__ wg, int64_t w_rows,
                                                    int64_t w_cols, int32_t* __restrict__ cnt,
                                                    IdxO* __restrict__ ocol, float* __restrict__ oval,
                                                    Ctl* __restrict__ ctl, uint64_t* __restrict__ toff, uint64_t t_cap) {
  constexpr int P = 128 * H;  // padded row length
  extern __shared__ __align__(16) unsigned char smem_w[];
  float* ws = reinterpret_cast<float*>(smem_w);
  for (int64_t i = threadIdx.x; i < w_rows * P; i += blockDim.x) {
    const int64_t rr = i / P, c = i % P;
    ws[i] = c < w_cols ? wg[rr * w_cols + c] : 0.f;
  }
  __syncthreads();
  const float4* __restrict__ w4 = reinterpret_cast<const float4*>(ws);
  StageCursor stage;
  const int lane = lane_id();
  const int64_t wid = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r = wid; r < rows; r += nw) {
    const int64_t s = static_cast<int64_t>(xptr[r] - xbase), e = static_cast<int64_t>(xptr[r + 1] - xbase);
    float4 acc[H];
#pragma unroll
    for (int h = 0; h < H; h++) acc[h] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int64_t k0 = s; k0 < e; k0 += 32) {
      uint32_t lin = 0;
      float lv = 0.f;
      if (k0 + lane < e) {
        const uint64_t c = static_cast<uint64_t>(xcol[k0 + lane]);
        lv = xval[k0 + lane];
        if (c >= static_cast<uint64_t>(w_rows)) {
          ctl->bad_row = 1;
          lv = 0.f;
        } else {
          lin = static_cast<uint32_t>(c);
        }
      }
      const int n = static_cast<int>(e - k0 < 32 ? e - k0 : 32);
      for (int kk = 0; kk < n; kk++) {
        const uint32_t in = __shfl_sync(kFull, lin, kk);
        const float v = __shfl_sync(kFull, lv, kk);
        const float4* wr = w4 + in * (P / 4) + lane;
#pragma unroll
        for (int h = 0; h < H; h++) {
          const float4 q = wr[32 * h];
          acc[h].x = fmaf(v, q.x, acc[h].x);
          acc[h].y = fmaf(v, q.y, acc[h].y);
          acc[h].z = fmaf(v, q.z, acc[h].z);
          acc[h].w = fmaf(v, q.w, acc[h].w);
        }
      }
    }
    uint32_t c_h[H], ex_h[H], total = 0;
#pragma unroll
    for (int h = 0; h < H; h++) {
      c_h[h] = (acc[h].x > 0.f) + (acc[h].y > 0.f) + (acc[h].z > 0.f) + (acc[h].w > 0.f);
      const uint32_t incl = warp_incl_scan(c_h[h]);
      ex_h[h] = total + incl - c_h[h];
      total += __shfl_sync(kFull, incl, 31);
    }
    const unsigned long long off = stage.take(total, ctl, 4096);
    if (off + total <= t_cap) {
#pragma unroll
      for (int h = 0; h < H; h++) {
        unsigned long long pos = off + ex_h[h];
        const uint32_t c0 = static_cast<uint32_t>(128 * h + 4 * lane);
        const float vv[4] = {acc[h].x, acc[h].y, acc[h].z, acc[h].w};
#pragma unroll
        for (int q = 0; q < 4; q++)
          if (vv[q] > 0.f) {
            ocol[pos] = static_cast<IdxO>(c0 + q);
            oval[pos] = vv[q];
            pos++;
          }
      }
    } else if (lane == 0) {
      ctl->bad_row = 2;
    }
    if (lane == 0) {
      cnt[r] = static_cast<int32_t>(total);
      toff[r] = off;
    }
  }
}

// Staging entries of the one-pass combine: the dense bound + 1/15 (a 4096-entry reservation wastes
// less than one <= 256-entry row) + one reservation per warp of the largest grid.
uint64_t combine_stage_cap(Ctx& ctx, int64_t rows, int64_t w_cols) {
  const uint64_t dense = static_cast<uint64_t>(rows) * static_cast<uint64_t>(w_cols);
  return dense + dense / 15 + (static_cast<uint64_t>(ctx.sms) * 32 * 8 + 1) * 4096;
}

template <class V, class IdxT, class IdxO, int J>
void combine_stage(Ctx& ctx, const Staged& s, int64_t rows, const V* w, int64_t w_rows, int64_t w_cols, int32_t* cnt,
                   IdxO* tcol, V* tval, uint64_t* toff, uint64_t t_cap, Ctl* ctl) {
  if constexpr (sizeof(V) == 4) {
    const int H = w_cols > 128 ? 2 : 1;
    const size_t smem4 = static_cast<size_t>(w_rows) * 128 * H * 4;
    if (w_cols >= 96 && w_cols <= 256 && smem4 <= 200 * 1024 && option("combine_v4", 1)) {
      auto k = H == 2 ? k_combine_v4<IdxT, IdxO, 2> : k_combine_v4<IdxT, IdxO, 1>;
      AB2_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem4)));
      int nb = 0;
      AB2_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k, 512, smem4));
      const int grid = std::max(1, std::min(grid_of(rows * 32, 512, ctx.sms), std::max(nb, 1) * ctx.sms));
      k<<<grid, 512, smem4, ctx.stream>>>(s.ptr, s.base, static_cast<const IdxT*>(s.idx),
                                          static_cast<const float*>(s.val), rows, w, w_rows, w_cols, cnt, tcol, tval,
                                          ctl, toff, t_cap);
      AB2_CUDA(cudaGetLastError());
      return;
    }
  }
  const bool smem = static_cast<size_t>(w_rows * w_cols) * sizeof(V) <= 200 * 1024 && option("combine_smem", 1);
  if (smem)
    combine_launch2<V, IdxT, IdxO, J, false, true, true>(ctx, s, rows, w, w_rows, w_cols, cnt, nullptr, tcol, tval, ctl,
                                                          toff, t_cap);
  else
    combine_launch2<V, IdxT, IdxO, J, false, false, true>(ctx, s, rows, w, w_rows, w_cols, cnt, nullptr, tcol, tval,
                                                           ctl, toff, t_cap);
}

template <class V, class IdxT, class IdxO, int J>
void combine_launch(Ctx& ctx, const Staged& s, int64_t rows, const V* w, int64_t w_rows, int64_t w_cols, int32_t* cnt,
                    int64_t* optr, IdxO* ocol, V* oval, Ctl* ctl, bool fill) {
  const bool smem = static_cast<size_t>(w_rows * w_cols) * sizeof(V) <= 200 * 1024 && option("combine_smem", 1);
  if (fill && smem)
    combine_launch2<V, IdxT, IdxO, J, true, true>(ctx, s, rows, w, w_rows, w_cols, cnt, optr, ocol, oval, ctl);
  else if (fill)
    combine_launch2<V, IdxT, IdxO, J, true, false>(ctx, s, rows, w, w_rows, w_cols, cnt, optr, ocol, oval, ctl);
  else if (smem)
    combine_launch2<V, IdxT, IdxO, J, false, true>(ctx, s, rows, w, w_rows, w_cols, cnt, optr, ocol, oval, ctl);
  else
    combine_launch2<V, IdxT, IdxO, J, false, false>(ctx, s, rows, w, w_rows, w_cols, cnt, optr, ocol, oval, ctl);
}

template <class V, class IdxT, class IdxO>
void combine_t(Ctx& ctx, const aires_b200_matrix& x, const void* w_in, uint64_t w_rows, uint64_t w_cols,
               uint32_t w_location, aires_b200_output& out) {
  const int64_t rows = static_cast<int64_t>(x.n_rows);
  Staged s = stage_csr(ctx, x);
  const V* w = static_cast<const V*>(w_in);
  if (w_location == AIRES_B200_HOST) {
    V* dw = static_cast<V*>(ctx.x_val.get(std::max<uint64_t>(w_rows * w_cols, 1) * sizeof(V)));
    AB2_CUDA(cudaMemcpyAsync(dw, w_in, w_rows * w_cols * sizeof(V), cudaMemcpyHostToDevice, ctx.stream));
    w = dw;
  }
  Ctl* ctl = ctx.ctl.as<Ctl>(1);
  AB2_CUDA(cudaMemsetAsync(ctl, 0, sizeof(Ctl), ctx.stream));
  int32_t* cnt = ctx.cnt.as<int32_t>(std::max<int64_t>(rows, 1));
  int64_t* optr = ctx.cptr.as<int64_t>(rows + 1);
  const int J = w_cols >= 256 ? 8 : static_cast<int>((w_cols + 31) / 32);
  auto run = [&](bool fill, IdxO* ocol, V* oval) {
    if (rows <= 0 || w_cols == 0) return;
    switch (std::max(J, 1)) {
      case 1: combine_launch<V, IdxT, IdxO, 1>(ctx, s, rows, w, w_rows, w_cols, cnt, optr, ocol, oval, ctl, fill); break;
      case 2: combine_launch<V, IdxT, IdxO, 2>(ctx, s, rows, w, w_rows, w_cols, cnt, optr, ocol, oval, ctl, fill); break;
      case 3:
      case 4: combine_launch<V, IdxT, IdxO, 4>(ctx, s, rows, w, w_rows, w_cols, cnt, optr, ocol, oval, ctl, fill); break;
      default: combine_launch<V, IdxT, IdxO, 8>(ctx, s, rows, w, w_rows, w_cols, cnt, optr, ocol, oval, ctl, fill); break;
    }
  };
  int launches = 0;
  // one pass when the output fits one column tile and its dense-bound staging fits in memory
  const uint64_t t_cap = combine_stage_cap(ctx, rows, static_cast<int64_t>(w_cols));
  const bool one_pass = rows > 0 && w_cols > 0 && static_cast<int64_t>(w_cols) <= 32 * std::max(J, 1) &&
                        t_cap * (sizeof(IdxO) + sizeof(V)) <= (uint64_t(48) << 30) && option("combine_one_pass", 1);
  if (one_pass) {
    IdxO* tcol = static_cast<IdxO*>(ctx.t_col.get(t_cap * sizeof(IdxO)));
    V* tval = static_cast<V*>(ctx.t_val.get(t_cap * sizeof(V)));
    uint64_t* toff = static_cast<uint64_t*>(ctx.rflops.get(static_cast<size_t>(rows) * 8));
    switch (std::max(J, 1)) {
      case 1: combine_stage<V, IdxT, IdxO, 1>(ctx, s, rows, w, w_rows, w_cols, cnt, tcol, tval, toff, t_cap, ctl); break;
      case 2: combine_stage<V, IdxT, IdxO, 2>(ctx, s, rows, w, w_rows, w_cols, cnt, tcol, tval, toff, t_cap, ctl); break;
      case 3:
      case 4: combine_stage<V, IdxT, IdxO, 4>(ctx, s, rows, w, w_rows, w_cols, cnt, tcol, tval, toff, t_cap, ctl); break;
      default: combine_stage<V, IdxT, IdxO, 8>(ctx, s, rows, w, w_rows, w_cols, cnt, tcol, tval, toff, t_cap, ctl); break;
    }
    launches++;
    scan_counts(ctx, cnt, rows, optr, ctl, &launches);
    Ctl* h = static_cast<Ctl*>(ctx.h_ctl.get(sizeof(Ctl)));
    AB2_CUDA(cudaMemcpyAsync(h, ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, ctx.stream));
    AB2_CUDA(cudaStreamSynchronize(ctx.stream));
    if (h->bad_row == 1) fail(AIRES_B200_INDEX_OUT_OF_RANGE, "feature column outside the weight rows");
    if (h->bad_row) fail(AIRES_B200_CAPACITY_EXCEEDED, "combine staging overflow");
    const uint64_t nnz = h->nnz;
    const OutBufs<IdxO, V> ob = out_alloc<IdxO, V>(ctx, out, static_cast<uint64_t>(rows), nnz);
    if (nnz) {
      k_place<V, IdxO><<<ctx.sms * 8, 256, 0, ctx.stream>>>(reinterpret_cast<const uint32_t*>(cnt), toff, optr, tcol,
                                                           tval, rows, ob.col, ob.val);
      AB2_CUDA(cudaGetLastError());
      launches++;
    }
    deliver<IdxO, V>(ctx, out, static_cast<uint64_t>(rows), w_cols, nnz, optr, ob);
    ctx.launches = launches;
    return;
  }
  if (rows > 0 && w_cols > 0) {
    run(false, nullptr, nullptr);
    launches++;
    scan_counts(ctx, cnt, rows, optr, ctl, &launches);
  } else {
    AB2_CUDA(cudaMemsetAsync(optr, 0, (rows + 1) * 8, ctx.stream));
  }
  Ctl* h = static_cast<Ctl*>(ctx.h_ctl.get(sizeof(Ctl)));
  AB2_CUDA(cudaMemcpyAsync(h, ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, ctx.stream));
  AB2_CUDA(cudaStreamSynchronize(ctx.stream));
  if (h->bad_row) fail(AIRES_B200_INDEX_OUT_OF_RANGE, "feature column outside the weight rows");
  const uint64_t nnz = rows > 0 && w_cols > 0 ? h->nnz : 0;
  const OutBufs<IdxO, V> ob = out_alloc<IdxO, V>(ctx, out, static_cast<uint64_t>(rows), nnz);
  if (nnz) {
    run(true, ob.col, ob.val);
    launches++;
  }
  deliver<IdxO, V>(ctx, out, static_cast<uint64_t>(rows), w_cols, nnz, optr, ob);
  ctx.launches = launches;
}

// ---- fused aggregate + combine for a dense-ish H (fp32) ---------------------
// H' = ReLU((Ã·H)·W) without materialising Ã·H.  When H is dense enough (post-ReLU GCN features
// are ~50% dense) its rows are gathered as dense fp32 rows: lane l accumulates the H columns
// l + 32m in registers (no shared-memory scatter, no bank conflicts), then the row is multiplied
// by W from shared memory (stored lane-major, Wt[m][j][l], conflict-free) and the 32 partial sums
// per output chunk are reduce-scattered across the warp (31 SHFLs per 32 outputs).  fp32 only:
// the terms are re-associated (within the stated tolerance); fp64 layers run unfused (exact).
template <int M>
__global__ void k_densify(const uint64_t* __restrict__ ptr, uint64_t base, const uint32_t* __restrict__ col,
                          const float* __restrict__ val, int64_t K, int64_t hc, float* __restrict__ hd) {
  const int lane = lane_id();
  const int64_t wid = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t k = wid; k < K; k += nw) {
    float* row = hd + k * (32 * M);
#pragma unroll
    for (int m = 0; m < M; m++) row[lane + 32 * m] = 0.f;
    __syncwarp();
    for (int64_t t = static_cast<int64_t>(ptr[k] - base) + lane; t < static_cast<int64_t>(ptr[k + 1] - base); t += 32)
      if (col[t] < hc) row[col[t]] = val[t];
  }
}

// Wt[(m * w_cols + j) * 32 + l] = W[(l + 32 m) * w_cols + j]  (zero past the rows of W)
__global__ void k_w_lane_major(const float* __restrict__ w, int64_t w_rows, int64_t w_cols, int M,
                               float* __restrict__ wt) {
  const int64_t total = static_cast<int64_t>(M) * w_cols * 32;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t l = i % 32, j = (i / 32) % w_cols, m = i / (32 * w_cols);
    const int64_t c = l + 32 * m;
    wt[i] = c < w_rows ? w[c * w_cols + j] : 0.f;
  }
}

// Reduce-scatter of 32 per-lane partials p[0..31]: afterwards lane l holds sum over lanes of p[l].
__device__ __forceinline__ float reduce_scatter32(float (&p)[32]) {
  const int lane = lane_id();
#pragma unroll
  for (int h = 16; h >= 1; h >>= 1) {
    const bool upper = (lane & h) != 0;
#pragma unroll
    for (int i = 0; i < h; i++) {
      // keep the half of the values this lane will own; send the other half to the partner
      const float send = upper ? p[i] : p[i + h];
      const float keep = upper ? p[i + h] : p[i];
      p[i] = keep + __shfl_xor_sync(kFull, send, h);
    }
  }
  return p[0];
}

template <int M, int JC>
__global__ void __launch_bounds__(256) k_agg_comb(const uint64_t* __restrict__ aptr, uint64_t abase,
                                                  const uint32_t* __restrict__ acol, const float* __restrict__ aval,
                                                  int64_t rows, int64_t K, const float* __restrict__ hd,
                                                  const float* __restrict__ wt_g, int64_t w_cols,
                                                  float* __restrict__ dense_out, int32_t* __restrict__ cnt) {
  extern __shared__ __align__(16) float wt[];
  for (int64_t i = threadIdx.x; i < static_cast<int64_t>(M) * w_cols * 32; i += blockDim.x) wt[i] = wt_g[i];
  __syncthreads();
  const int lane = lane_id();
  const int64_t wid = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r = wid; r < rows; r += nw) {
    float acc[M];
#pragma unroll
    for (int m = 0; m < M; m++) acc[m] = 0.f;
    const int64_t s = static_cast<int64_t>(aptr[r] - abase), e = static_cast<int64_t>(aptr[r + 1] - abase);
    for (int64_t b = s; b < e; b += 32) {
      uint32_t k = 0;
      float a = 0.f;
      if (b + lane < e) {
        k = acol[b + lane];
        a = aval[b + lane];
        if (k >= K) a = 0.f, k = 0;
      }
      const int n = static_cast<int>(e - b < 32 ? e - b : 32);
      int kk = 0;
      for (; kk + 4 <= n; kk += 4) {  // four dense rows in flight
        float x[4][M];
        float av[4];
#pragma unroll
        for (int q = 0; q < 4; q++) {
          const uint32_t kq = __shfl_sync(kFull, k, kk + q);
          av[q] = __shfl_sync(kFull, a, kk + q);
          const float* row = hd + static_cast<int64_t>(kq) * (32 * M) + lane;
#pragma unroll
          for (int m = 0; m < M; m++) x[q][m] = __ldg(row + 32 * m);
        }
#pragma unroll
        for (int q = 0; q < 4; q++)
#pragma unroll
          for (int m = 0; m < M; m++) acc[m] = fmaf(av[q], x[q][m], acc[m]);
      }
      for (; kk < n; kk++) {
        const uint32_t kq = __shfl_sync(kFull, k, kk);
        const float aq = __shfl_sync(kFull, a, kk);
        const float* row = hd + static_cast<int64_t>(kq) * (32 * M) + lane;
#pragma unroll
        for (int m = 0; m < M; m++) acc[m] = fmaf(aq, __ldg(row + 32 * m), acc[m]);
      }
    }
    int32_t count = 0;
#pragma unroll
    for (int jc = 0; jc < JC; jc++) {
      float p[32];
#pragma unroll
      for (int jj = 0; jj < 32; jj++) {
        const int64_t j = jc * 32 + jj;
        float v = 0.f;
        if (j < w_cols) {
#pragma unroll
          for (int m = 0; m < M; m++) v = fmaf(acc[m], wt[(m * w_cols + j) * 32 + lane], v);
        }
        p[jj] = v;
      }
      const float o = reduce_scatter32(p);
      const int64_t j = jc * 32 + lane;
      const bool pos = j < w_cols && o > 0.f;
      if (j < w_cols) dense_out[r * w_cols + j] = pos ? o : 0.f;
      count += __popc(__ballot_sync(kFull, pos));
    }
    if (lane == 0) cnt[r] = count;
  }
}

template <class IdxO>
__global__ void k_compact_rows(const float* __restrict__ dense, int64_t rows, int64_t w_cols,
                               const int64_t* __restrict__ optr, IdxO* __restrict__ ocol, float* __restrict__ oval) {
  const int lane = lane_id();
  const int64_t wid = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r = wid; r < rows; r += nw) {
    int64_t o = optr[r];
    for (int64_t j0 = 0; j0 < w_cols; j0 += 128) {  // four 32-column chunks loaded before any is used
      float v[4];
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const int64_t j = j0 + 32 * u + lane;
        v[u] = j < w_cols ? dense[r * w_cols + j] : 0.f;
      }
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const unsigned m = __ballot_sync(kFull, v[u] > 0.f);
        if (v[u] > 0.f) {
          const int64_t d = o + __popc(m & ((1u << lane) - 1));
          ocol[d] = static_cast<IdxO>(j0 + 32 * u + lane);
          oval[d] = v[u];
        }
        o += __popc(m);
      }
    }
  }
}

template <int M, int JC>
void agg_comb_launch(Ctx& ctx, const uint64_t* aptr, uint64_t abase, const uint32_t* acol, const float* aval,
                     int64_t rows, int64_t K, const float* hd, const float* wt, int64_t w_cols, float* dense,
                     int32_t* cnt) {
  auto k = k_agg_comb<M, JC>;
  const size_t smem = static_cast<size_t>(M) * w_cols * 32 * sizeof(float);
  AB2_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  int nb = 0;
  AB2_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k, 256, smem));
  if (nb < 1) fail(AIRES_B200_UNSUPPORTED_FORMAT, "weights too large for the fused layer");
  const int grid = std::max(1, std::min(grid_of(rows * 32, 256, ctx.sms), nb * ctx.sms));
  k<<<grid, 256, smem, ctx.stream>>>(aptr, abase, acol, aval, rows, K, hd, wt, w_cols, dense, cnt);
  AB2_CUDA(cudaGetLastError());
}

template <int M>
void agg_comb_m(Ctx& ctx, int jc, const uint64_t* aptr, uint64_t abase, const uint32_t* acol, const float* aval,
                int64_t rows, int64_t K, const float* hd, const float* wt, int64_t w_cols, float* dense, int32_t* cnt) {
  switch (jc) {
    case 1: agg_comb_launch<M, 1>(ctx, aptr, abase, acol, aval, rows, K, hd, wt, w_cols, dense, cnt); break;
    case 2: agg_comb_launch<M, 2>(ctx, aptr, abase, acol, aval, rows, K, hd, wt, w_cols, dense, cnt); break;
    case 3: agg_comb_launch<M, 3>(ctx, aptr, abase, acol, aval, rows, K, hd, wt, w_cols, dense, cnt); break;
    default: agg_comb_launch<M, 4>(ctx, aptr, abase, acol, aval, rows, K, hd, wt, w_cols, dense, cnt); break;
  }
}

// ---- reassociated layer: ReLU(Ã·(H·W)) when W narrows the features -----------------------------
// (Ã·H)·W = Ã·(H·W) exactly in real arithmetic; in fp32 the terms are summed in another order,
// within the stated tolerance (the cell's scale sum |Ã||H||W| bounds both orders' rounding).  The
// point is the gather: the aggregation reads one row of its right operand per Ã entry, 4·h_cols
// bytes for H (1 KB at the products shape: 64 GB of gathers for layer 2, the bound of k_agg_comb)
// but only 4·w_cols for T = H·W (188 B).  T costs one pass over H's rows with W in shared memory.

// W packed for LDS.128: wt4[(j * M4 + m4) * 32 + l] = {W[l + 32 (4 m4 + q)][j], q = 0..3} (zero past W).
__global__ void k_w_lane_major4(const float* __restrict__ w, int64_t w_rows, int64_t w_cols, int M4,
                                float4* __restrict__ wt4) {
  const int64_t total = static_cast<int64_t>(M4) * w_cols * 32;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t l = i % 32, m4 = (i / 32) % M4, j = i / (32 * M4);
    float q[4];
    for (int k = 0; k < 4; k++) {
      const int64_t c = l + 32 * (4 * m4 + k);
      q[k] = c < w_rows ? w[c * w_cols + j] : 0.f;
    }
    wt4[i] = make_float4(q[0], q[1], q[2], q[3]);
  }
}

// T[r, :w_cols] = H[r, :] · W, one warp per H row: the sparse row is scattered into a per-warp
// shared row (lane l then holds columns l + 32 m), multiplied by W from shared memory (LDS.128 of
// four W rows per output column), and the 32-lane partials are reduce-scattered (lane l gets
// output column 32 jc + l).  T rows are tp floats apart (w_cols rounded to 8: whole sectors).
template <int M4, int JC>
__global__ void __launch_bounds__(256) k_hw(const uint64_t* __restrict__ hptr, uint64_t hbase,
                                            const uint32_t* __restrict__ hcol, const float* __restrict__ hval,
                                            int64_t K, int64_t h_cols, const float4* __restrict__ wt4_g,
                                            int64_t w_cols, int64_t tp, float* __restrict__ t, Ctl* __restrict__ ctl) {
  // Bound by the shared-memory reads of W (L1 95% at cfg5, 4.5 ms).  Measured slower: two H rows per
  // warp step sharing the W loads (113 registers, 5.8 ms); a register-tiled GEMM over dense 56/64-row
  // tiles of H scattered into shared memory (5.3-6.7 ms: the scatter's global-load latency, with one
  // or two CTAs per SM, stalls the FFMAs)
  extern __shared__ __align__(16) float4 sm4[];
  const int64_t nwt = static_cast<int64_t>(M4) * w_cols * 32;
  for (int64_t i = threadIdx.x; i < nwt; i += blockDim.x) sm4[i] = wt4_g[i];
  __syncthreads();
  const int lane = lane_id(), warp = warp_id();
  float* row = reinterpret_cast<float*>(sm4 + nwt) + warp * (128 * M4);
  const int64_t wid = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r = wid; r < K; r += nw) {
#pragma unroll
    for (int m = 0; m < 4 * M4; m++) row[lane + 32 * m] = 0.f;
    __syncwarp();
    const int64_t s = static_cast<int64_t>(hptr[r] - hbase), e = static_cast<int64_t>(hptr[r + 1] - hbase);
    for (int64_t k = s + lane; k < e; k += 32) {
      const uint32_t c = hcol[k];
      if (c < static_cast<uint64_t>(h_cols))
        row[c] = hval[k];
      else
        ctl->bad_row = 1;
    }
    __syncwarp();
    float4 a4[M4];
#pragma unroll
    for (int m4 = 0; m4 < M4; m4++)
      a4[m4] = make_float4(row[lane + 32 * (4 * m4)], row[lane + 32 * (4 * m4 + 1)], row[lane + 32 * (4 * m4 + 2)],
                           row[lane + 32 * (4 * m4 + 3)]);
    __syncwarp();
#pragma unroll
    for (int jc = 0; jc < JC; jc++) {
      float p[32];
#pragma unroll
      for (int jj = 0; jj < 32; jj++) {
        const int64_t j = jc * 32 + jj;
        float v = 0.f;
        if (j < w_cols) {
#pragma unroll
          for (int m4 = 0; m4 < M4; m4++) {
            const float4 q = sm4[(j * M4 + m4) * 32 + lane];
            v = fmaf(a4[m4].x, q.x, v);
            v = fmaf(a4[m4].y, q.y, v);
            v = fmaf(a4[m4].z, q.z, v);
            v = fmaf(a4[m4].w, q.w, v);
          }
        }
        p[jj] = v;
      }
      const float o = reduce_scatter32(p);
      const int64_t j = jc * 32 + lane;
      if (j < w_cols) t[r * tp + j] = o;
    }
  }
}

// out[r, j] = ReLU(sum_k Ã[r, k] T[k, j]) as a dense row + the row's positive count (then scan +
// k_compact_rows, as for k_agg_comb).  One warp per Ã row, lane l owns columns l + 32 jc; eight T
// rows in flight per step.
#ifndef AB2_AGG_INFLIGHT
#define AB2_AGG_INFLIGHT 8  // T rows in flight per warp (16 measured slower: 102 registers, layer 2 9.3 -> 12.0 ms)
#endif
template <int JC>
__global__ void __launch_bounds__(256) k_agg_t(const uint64_t* __restrict__ aptr, uint64_t abase,
                                               const uint32_t* __restrict__ acol, const float* __restrict__ aval,
                                               int64_t rows, int64_t K, const float* __restrict__ t, int64_t tp,
                                               int64_t w_cols, float* __restrict__ dense_out,
                                               int32_t* __restrict__ cnt) {
  const int lane = lane_id();
  const int64_t wid = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  bool mine[JC];
#pragma unroll
  for (int jc = 0; jc < JC; jc++) mine[jc] = jc * 32 + lane < w_cols;
  for (int64_t r = wid; r < rows; r += nw) {
    float acc[JC];
#pragma unroll
    for (int jc = 0; jc < JC; jc++) acc[jc] = 0.f;
    const int64_t s = static_cast<int64_t>(aptr[r] - abase), e = static_cast<int64_t>(aptr[r + 1] - abase);
    for (int64_t b = s; b < e; b += 32) {
      uint32_t k = 0;
      float a = 0.f;
      if (b + lane < e) {
        k = acol[b + lane];
        a = aval[b + lane];
        if (k >= K) a = 0.f, k = 0;
      }
      const int n = static_cast<int>(e - b < 32 ? e - b : 32);
      int kk = 0;
      for (; kk + AB2_AGG_INFLIGHT <= n; kk += AB2_AGG_INFLIGHT) {
        float x[AB2_AGG_INFLIGHT][JC], av[AB2_AGG_INFLIGHT];
#pragma unroll
        for (int q = 0; q < AB2_AGG_INFLIGHT; q++) {
          const uint32_t kq = __shfl_sync(kFull, k, kk + q);
          av[q] = __shfl_sync(kFull, a, kk + q);
          const float* tr = t + static_cast<int64_t>(kq) * tp + lane;
#pragma unroll
          for (int jc = 0; jc < JC; jc++) x[q][jc] = mine[jc] ? __ldg(tr + 32 * jc) : 0.f;
        }
#pragma unroll
        for (int q = 0; q < AB2_AGG_INFLIGHT; q++)
#pragma unroll
          for (int jc = 0; jc < JC; jc++) acc[jc] = fmaf(av[q], x[q][jc], acc[jc]);
      }
      for (; kk < n; kk++) {
        const uint32_t kq = __shfl_sync(kFull, k, kk);
        const float aq = __shfl_sync(kFull, a, kk);
        const float* tr = t + static_cast<int64_t>(kq) * tp + lane;
#pragma unroll
        for (int jc = 0; jc < JC; jc++)
          if (mine[jc]) acc[jc] = fmaf(aq, __ldg(tr + 32 * jc), acc[jc]);
      }
    }
    int32_t count = 0;
#pragma unroll
    for (int jc = 0; jc < JC; jc++) {
      const bool pos = mine[jc] && acc[jc] > 0.f;
      if (mine[jc]) dense_out[r * w_cols + jc * 32 + lane] = pos ? acc[jc] : 0.f;
      count += __popc(__ballot_sync(kFull, pos));
    }
    if (lane == 0) cnt[r] = count;
  }
}

// k_agg_t for T rows of <= 64 floats, with the gathers made asynchronous: k_agg_t holds its eight
// in-flight T rows in registers, so the kernel is latency-bound (ncu: DRAM 21%, long-scoreboard
// stalls, occupancy capped by registers).  Here a warp owns blocks of 32 consecutive Ã rows (wid,
// wid + nw, ...) and streams each block's entries as full 32-entry chunks across row boundaries (rows
// average ~26 entries on GCN graphs); chunk i+1's T rows are copied global -> shared with cp.async (no
// registers held) while chunk i is summed from shared memory.  A row's terms are added in ascending
// entry order with fmaf, as in k_agg_t.  TP is T's row pitch (floats), K * TP < 2^32.
#ifndef AB2_AGG_WARPS
#define AB2_AGG_WARPS 4
#endif
#ifndef AB2_AGG_CH
#define AB2_AGG_CH 32
#endif
constexpr int kAggWarps = AB2_AGG_WARPS, kAggStages = 2;  // (3 / 4 buffers: fewer warps, slower)
constexpr int kAggCh = AB2_AGG_CH;  // entries per chunk (<= 32; cfg5 layer 2: 16 -> 6.54, 24 -> 6.18, 32 -> 6.20 ms)
template <int TP>
__global__ void __launch_bounds__(kAggWarps * 32) k_agg_t_cp(const uint64_t* __restrict__ aptr, uint64_t abase,
                                                          const uint32_t* __restrict__ acol,
                                                          const float* __restrict__ aval, int64_t rows, int64_t K,
                                                          const float* __restrict__ t, int64_t w_cols,
                                                          float* __restrict__ dense_out, int32_t* __restrict__ cnt) {
  constexpr int JC = (TP + 31) / 32, TP4 = TP / 4;
  extern __shared__ __align__(16) float agg_smem[];
  const int lane = lane_id();
  const int64_t wid = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  float* const sb = agg_smem + (threadIdx.x >> 5) * (kAggStages * kAggCh * TP);
  const int piece = lane & 15, half = lane >> 4;
  bool mine[JC];
#pragma unroll
  for (int jc = 0; jc < JC; jc++) mine[jc] = jc * 32 + lane < w_cols;
  auto blk_end = [&](int64_t rb) { return rb + 32 < rows ? rb + 32 : rows; };

  // producer: chunks [b, min(b + 32, e)) of block rb's entry range [., e)
  int64_t p_rb = wid * 32, p_b = 0, p_e = 0;
  if (p_rb < rows) p_b = static_cast<int64_t>(aptr[p_rb] - abase), p_e = static_cast<int64_t>(aptr[blk_end(p_rb)] - abase);
  // advance the producer to its next non-empty chunk; false when the warp's entries are exhausted
  auto p_next = [&]() -> bool {
    while (p_rb < rows && p_b >= p_e) {
      p_rb += 32 * nw;
      if (p_rb < rows) p_b = static_cast<int64_t>(aptr[p_rb] - abase), p_e = static_cast<int64_t>(aptr[blk_end(p_rb)] - abase);
    }
    return p_rb < rows;
  };
  // issue the producer's chunk into buffer buf (returns this lane's Ã value; entries [cb, ce))
  auto issue = [&](int buf, int64_t& cb, int64_t& ce) -> float {
    float a = 0.f;
    cb = ce = -1;
    if (p_next()) {
      cb = p_b;
      const int n = static_cast<int>(p_e - p_b < kAggCh ? p_e - p_b : kAggCh);
      uint32_t k = 0;
      if (lane < n) {
        k = acol[p_b + lane];
        a = aval[p_b + lane];
        if (k >= K) a = 0.f, k = 0;
      }
      const uint32_t off = k * TP;
      float* dst = sb + buf * (kAggCh * TP) + piece * 4;
#pragma unroll 4
      for (int q = 0; q < n; q += 2) {
        const int qq = q + half;
        const uint32_t o = __shfl_sync(kFull, off, qq & 31);
        if (qq < n && piece < TP4) {
          const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst + qq * TP));
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(t + o + piece * 4) : "memory");
        }
      }
      p_b += n;
      ce = p_b;
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    return a;
  };

  int64_t cb0, ce0, cb1, ce1;
  float a0 = issue(0, cb0, ce0), a1 = issue(1, cb1, ce1);
  int buf = 0;
  asm volatile("cp.async.wait_group 1;" ::: "memory");
  __syncwarp();
  // consumer: rows in order; entries [s, e) of row r come from the chunk at cb0 (buffer buf)
  for (int64_t rb = wid * 32; rb < rows; rb += 32 * nw) {
    const int nr = static_cast<int>(blk_end(rb) - rb);
    uint64_t ps = 0, pe = 0;
    if (lane < nr) ps = aptr[rb + lane], pe = aptr[rb + lane + 1];
    for (int i = 0; i < nr; i++) {
      int64_t s = static_cast<int64_t>(__shfl_sync(kFull, ps, i) - abase);
      const int64_t e = static_cast<int64_t>(__shfl_sync(kFull, pe, i) - abase);
      float acc[JC];
#pragma unroll
      for (int jc = 0; jc < JC; jc++) acc[jc] = 0.f;
      while (s < e) {
        if (s >= ce0) {  // chunk exhausted: refill its buffer, move to the next chunk
          __syncwarp();
          int64_t cb2, ce2;
          const float a2 = issue(buf, cb2, ce2);
          asm volatile("cp.async.wait_group 1;" ::: "memory");
          __syncwarp();
          cb0 = cb1, ce0 = ce1, a0 = a1, cb1 = cb2, ce1 = ce2, a1 = a2, buf ^= 1;
        }
        const int q0 = static_cast<int>(s - cb0);
        const int q1 = static_cast<int>((e < ce0 ? e : ce0) - cb0);
        const float* src = sb + buf * (kAggCh * TP) + lane;
        int q = q0;
        for (; q + 8 <= q1; q += 8) {
          float x[8][JC], av[8];
#pragma unroll
          for (int u = 0; u < 8; u++) {
            av[u] = __shfl_sync(kFull, a0, q + u);
#pragma unroll
            for (int jc = 0; jc < JC; jc++) x[u][jc] = mine[jc] ? src[(q + u) * TP + 32 * jc] : 0.f;
          }
#pragma unroll
          for (int u = 0; u < 8; u++)
#pragma unroll
            for (int jc = 0; jc < JC; jc++) acc[jc] = fmaf(av[u], x[u][jc], acc[jc]);
        }
        for (; q < q1; q++) {
          const float aq = __shfl_sync(kFull, a0, q);
#pragma unroll
          for (int jc = 0; jc < JC; jc++)
            if (mine[jc]) acc[jc] = fmaf(aq, src[q * TP + 32 * jc], acc[jc]);
        }
        s = cb0 + q1;
      }
      const int64_t r = rb + i;
      int32_t pos_count = 0;
#pragma unroll
      for (int jc = 0; jc < JC; jc++) {
        const bool pos = mine[jc] && acc[jc] > 0.f;
        if (mine[jc]) dense_out[r * w_cols + jc * 32 + lane] = pos ? acc[jc] : 0.f;
        pos_count += __popc(__ballot_sync(kFull, pos));
      }
      if (lane == 0) cnt[r] = pos_count;
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}

// ---------------------------------------------------------------------------------------------
// T = H·W on the 5th-generation tensor cores (tcgen05.mma kind::tf32), for the reassociated layer's
// narrow W (w_cols <= 48, h_cols <= 256).  fp32 accuracy from a 3xTF32 split: a = a_hi + a_lo with
// a_hi the tf32 truncation, and T = A_hi·W_hi + A_hi·W_lo + A_lo·W_hi accumulated in fp32 (error
// ~2^-21 of the cell's scale; the layer's tolerance is 1e-5).
//
// One persistent CTA per SM (512 threads), one 128-row tile of H at a time:
//   shared: W^T hi / lo for all of K (N rows x K, K-major, 128-byte swizzle: 2 x 48 KB at N = 48),
//           the tile's A hi / lo for one K half of 128 (2 x 64 KB), an mbarrier;
//   TMEM:   the 128 x N fp32 accumulator (64 columns).
// Per K half: zero A, densify the tile's CSR rows into the swizzled layout (warp w owns rows w + 16i;
// the rows' offsets are read once per tile, then every row's next 32 entries are loaded together:
// 16 loads per lane in flight), then one thread issues 16 K-steps x 3 MMAs and commits them to the
// mbarrier; the epilogue reads the accumulator with tcgen05.ld (warp w: lane quarter w % 4, column
// group w / 4) into T.
// ---------------------------------------------------------------------------------------------
namespace tc {
constexpr int kRows = 128, kHalf = 128, kThreads = 512, kWarps = kThreads / 32, kRowsPerWarp = kRows / kWarps;
#ifndef AB2_HW_CHUNKS
#define AB2_HW_CHUNKS 4
#endif
constexpr int kChunks = AB2_HW_CHUNKS;  // 32-entry chunks of every row loaded per densify round
__device__ __forceinline__ uint32_t swz(int m, int k) {  // byte offset of (row m, k < 32) in a K atom
  return static_cast<uint32_t>((m >> 3) * 1024 + (m & 7) * 128 + ((((k >> 2) ^ (m & 7)) & 7) << 4) + (k & 3) * 4);
}
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return static_cast<uint64_t>((saddr & 0x3FFFFu) >> 4) | (static_cast<uint64_t>(1) << 16) |
         (static_cast<uint64_t>(1024 >> 4) << 32) | (static_cast<uint64_t>(1) << 46) | (static_cast<uint64_t>(2) << 61);
}
__device__ __forceinline__ void split(float a, float& hi, float& lo) {
  hi = __uint_as_float(__float_as_uint(a) & 0xFFFFE000u);
  lo = a - hi;
}
__device__ __forceinline__ void mma_tf32(uint32_t tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
               "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t phase) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
                 : "=r"(done)
                 : "r"(mbar), "r"(phase)
                 : "memory");
}
}  // namespace tc

template <int N>
__global__ void __launch_bounds__(tc::kThreads, 1)
    k_hw_tc(const uint64_t* __restrict__ hptr, uint64_t hbase, const uint32_t* __restrict__ hcol,
            const float* __restrict__ hval, int64_t K, int64_t h_cols, const float* __restrict__ w, int64_t w_cols,
            int64_t tp, float* __restrict__ t, Ctl* __restrict__ ctl) {
  using namespace tc;
  extern __shared__ __align__(1024) unsigned char sm_raw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  const int katoms = static_cast<int>((h_cols + 31) / 32);  // K atoms of 32 (<= 8)
  const uint32_t w_atom = N * 128;                           // bytes of one K atom of W^T
  unsigned char* wt_hi = sm;
  unsigned char* wt_lo = sm + 8 * w_atom;
  unsigned char* a_hi = sm + 16 * w_atom;
  unsigned char* a_lo = a_hi + 65536;
  uint64_t* mbar = reinterpret_cast<uint64_t*>(a_lo + 65536);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(mbar + 1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  // W^T, split, swizzled (zero beyond h_cols / w_cols)
  for (int i = tid; i < N * katoms * 32; i += kThreads) {
    const int n = i / (katoms * 32), k = i % (katoms * 32);
    const float v = (n < w_cols && k < h_cols) ? w[static_cast<int64_t>(k) * w_cols + n] : 0.f;
    float hi, lo;
    split(v, hi, lo);
    const uint32_t off = (k >> 5) * w_atom + swz(n, k & 31);
    *reinterpret_cast<float*>(wt_hi + off) = hi;
    *reinterpret_cast<float*>(wt_lo + off) = lo;
  }
  const uint32_t mbar_s = static_cast<uint32_t>(__cvta_generic_to_shared(mbar));
  if (tid == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbar_s));
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(
        static_cast<uint32_t>(__cvta_generic_to_shared(tslot))));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tslot;
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
                         (static_cast<uint32_t>(kRows >> 4) << 24);
  const uint32_t ah_s = static_cast<uint32_t>(__cvta_generic_to_shared(a_hi));
  const uint32_t al_s = static_cast<uint32_t>(__cvta_generic_to_shared(a_lo));
  const uint32_t wh_s = static_cast<uint32_t>(__cvta_generic_to_shared(wt_hi));
  const uint32_t wl_s = static_cast<uint32_t>(__cvta_generic_to_shared(wt_lo));
  const int halves = (katoms + 3) / 4;
  uint32_t phase = 0;
  const int64_t ntiles = (K + kRows - 1) / kRows;
  // The tile loop is lock-step across the CTA (densify -> MMA -> epilogue), so the entries' load
  // latency is exposed once per tile: one thread pulls the NEXT tile's row offsets and CSR entries
  // into L2 with bulk prefetches (its offsets were read one tile earlier, so nothing waits).
  const bool pf = tid == 32;
  int64_t pf_b = 0, pf_e = 0;
  auto pf_range = [&](int64_t tl) {
    if (tl < ntiles) {
      const int64_t q0 = tl * kRows, q1 = q0 + kRows < K ? q0 + kRows : K;
      pf_b = static_cast<int64_t>(hptr[q0] - hbase), pf_e = static_cast<int64_t>(hptr[q1] - hbase);
    } else {
      pf_b = pf_e = 0;
    }
  };
  auto bulk_pf = [](const void* p, int64_t bytes) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(p) & ~uintptr_t(15);
    const uintptr_t e = (reinterpret_cast<uintptr_t>(p) + bytes + 15) & ~uintptr_t(15);
    for (uintptr_t x = a; x < e; x += 65536) {
      const uint32_t n = static_cast<uint32_t>(e - x < 65536 ? e - x : 65536);
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(x), "r"(n) : "memory");
    }
  };
  if (pf) pf_range(blockIdx.x + static_cast<int64_t>(gridDim.x));
  // densification state of the tile being loaded: this warp's rows (offsets relative to the tile's
  // first entry; a tile holds <= 128 x 256 entries) and one round of entries in registers
  int32_t cur[kRowsPerWarp], end[kRowsPerWarp];
  const uint32_t* tcol = hcol;
  const float* tval = hval;
  uint32_t c[kChunks][kRowsPerWarp];
  float v[kChunks][kRowsPerWarp];
  auto setup_tile = [&](int64_t tl) {
    const int64_t q0 = tl * kRows;
    const int nrows = static_cast<int>(K - q0 < kRows ? K - q0 : kRows);
    const int64_t tile_base = static_cast<int64_t>(hptr[q0] - hbase);
#pragma unroll
    for (int j = 0; j < kRowsPerWarp; j++) {
      const int m = warp + kWarps * j;
      cur[j] = end[j] = 0;
      if (m < nrows) {
        cur[j] = static_cast<int32_t>(static_cast<int64_t>(hptr[q0 + m] - hbase) - tile_base);
        end[j] = static_cast<int32_t>(static_cast<int64_t>(hptr[q0 + m + 1] - hbase) - tile_base);
      }
    }
    tcol = hcol + tile_base;
    tval = hval + tile_base;
  };
  // the next 32 * kChunks entries of each of the warp's rows: kChunks x 8 x 2 loads per lane in flight
  auto load_round = [&]() {
#pragma unroll
    for (int h2 = 0; h2 < kChunks; h2++)
#pragma unroll
      for (int j = 0; j < kRowsPerWarp; j++) {
        const int32_t i = cur[j] + 32 * h2 + lane;
        c[h2][j] = 0xffffffffu;
        v[h2][j] = 0.f;
        if (i < end[j]) {
          c[h2][j] = __ldg(tcol + i);
          v[h2][j] = __ldg(tval + i);
        }
      }
  };
  // scatter the round's entries of columns [klo, khi) into A; true if a row may have more of them
  auto scatter = [&](uint32_t klo, uint32_t khi) -> bool {
    bool more = false;
#pragma unroll
    for (int j = 0; j < kRowsPerWarp; j++) {
      const int m = warp + kWarps * j;
      int took = 0;
#pragma unroll
      for (int h2 = 0; h2 < kChunks; h2++) {
        const uint32_t cc = c[h2][j];
        const bool in = cc >= klo && cc < khi;  // (columns are sorted: the half's entries come first)
        if (in) {
          if (cc < static_cast<uint32_t>(h_cols)) {
            float hi, lo;
            split(v[h2][j], hi, lo);
            const uint32_t k = cc - klo;
            const uint32_t off = (k >> 5) * 16384 + swz(m, static_cast<int>(k & 31));
            asm volatile("st.shared.f32 [%0], %1;" ::"r"(ah_s + off), "f"(hi) : "memory");
            asm volatile("st.shared.f32 [%0], %1;" ::"r"(al_s + off), "f"(lo) : "memory");
          } else {
            ctl->bad_row = 1;
          }
        }
        took += __popc(__ballot_sync(0xffffffffu, in));
      }
      cur[j] += took;
      more |= took == 32 * kChunks;
    }
    return more;
  };
  if (static_cast<int64_t>(blockIdx.x) < ntiles) {
    setup_tile(blockIdx.x);
    load_round();
  }
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t r0 = tile * kRows;
    const int rows = static_cast<int>(K - r0 < kRows ? K - r0 : kRows);
    if (pf) {
      const int64_t nt = tile + gridDim.x;
      if (nt < ntiles && pf_e > pf_b) {
        const int64_t q0 = nt * kRows, q1 = q0 + kRows < K ? q0 + kRows : K;
        bulk_pf(hptr + q0, (q1 - q0 + 1) * 8);
        bulk_pf(hcol + pf_b, (pf_e - pf_b) * 4);
        bulk_pf(hval + pf_b, (pf_e - pf_b) * 4);
      }
      pf_range(nt + gridDim.x);
    }
    for (int hf = 0; hf < halves; hf++) {
      // zero this warp's rows of the half (the MMAs that read A have completed: mbarrier waited
      // below) -- warp-local, so no CTA barrier between zeroing and the scatter
#pragma unroll
      for (int z = 0; z < (kRowsPerWarp * 4 * 2 * 128) / (32 * 16); z++) {
        const int idx = z * 32 + lane;                       // 16-byte piece of (row j, atom, hi/lo)
        const int j = idx >> 6, atom = (idx >> 3) & 3, lohi = (idx >> 5) & 1, pc = idx & 7;
        const int m = warp + kWarps * j;
        const uint32_t base = lohi ? al_s : ah_s;
        asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(base + atom * 16384 + (m >> 3) * 1024 +
                                                                       (m & 7) * 128 + pc * 16),
                     "r"(0u)
                     : "memory");
      }
      __syncwarp();
      const uint32_t klo = static_cast<uint32_t>(hf * kHalf), khi = klo + kHalf;
      bool more = scatter(klo, khi);
      while (__any_sync(0xffffffffu, more)) {
        load_round();
        more = scatter(klo, khi);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (tid == 0) {
        const int ksteps = min(16, (katoms - 4 * hf) * 4);
        for (int kk = 0; kk < ksteps; kk++) {
          const uint32_t ao = (kk >> 2) * 16384 + (kk & 3) * 32;
          const uint32_t wo = (4 * hf + (kk >> 2)) * w_atom + (kk & 3) * 32;
          const uint64_t dah = sw128_desc(ah_s + ao), dal = sw128_desc(al_s + ao);
          const uint64_t dwh = sw128_desc(wh_s + wo), dwl = sw128_desc(wl_s + wo);
          const uint32_t acc0 = (hf == 0 && kk == 0) ? 0u : 1u;
          mma_tf32(tmem, dah, dwh, idesc, acc0);
          mma_tf32(tmem, dah, dwl, idesc, 1u);
          mma_tf32(tmem, dal, dwh, idesc, 1u);
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(mbar_s)
                     : "memory");
      }
      // while the MMAs run: the first entries of the next half, or of the next tile
      if (hf + 1 < halves) {
        load_round();
      } else if (tile + gridDim.x < ntiles) {
        setup_tile(tile + gridDim.x);
        load_round();
      }
      mbar_wait(mbar_s, phase);
      phase ^= 1u;
    }
    // epilogue: accumulator rows 32 (w % 4) + lane; warp group w / 4 takes N / 4 columns (x4 loads)
    asm volatile("tcgen05.fence::after_thread_sync;");
    {
      const int q = warp & 3, cg = warp >> 2;
      const int m = 32 * q + lane;
      constexpr int NQ = N / (kWarps / 4);  // 12 at N = 48
      static_assert(NQ % 4 == 0, "column group must be whole x4 loads");
#pragma unroll
      for (int c0 = 0; c0 < NQ; c0 += 4) {
        uint32_t r[4];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                     : "r"(tmem + (static_cast<uint32_t>(32 * q) << 16) + static_cast<uint32_t>(cg * NQ + c0)));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        const int col = cg * NQ + c0;
        if (m < rows && col < tp)  // tp is a multiple of 8: a group of 4 is wholly inside the pitch or not
          *reinterpret_cast<float4*>(t + (r0 + m) * tp + col) =
              make_float4(__uint_as_float(r[0]), __uint_as_float(r[1]), __uint_as_float(r[2]), __uint_as_float(r[3]));
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();  // the accumulator is free for the next tile's MMAs
  }
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem));
}

void hw_tc_launch(Ctx& ctx, const Staged& hs, int64_t K, int64_t h_cols, const float* w, int64_t w_cols, int64_t tp,
                  float* t, Ctl* ctl) {
  constexpr int N = 48;
  const size_t smem = 1024 + 16 * N * 128 + 2 * 65536 + 64;
  AB2_CUDA(cudaFuncSetAttribute(k_hw_tc<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  const int64_t ntiles = (K + tc::kRows - 1) / tc::kRows;
  if (ntiles > 0)
    k_hw_tc<N><<<static_cast<int>(std::min<int64_t>(ntiles, ctx.sms)), tc::kThreads, smem, ctx.stream>>>(
        hs.ptr, hs.base, static_cast<const uint32_t*>(hs.idx), static_cast<const float*>(hs.val), K, h_cols, w,
        w_cols, tp, t, ctl);
  AB2_CUDA(cudaGetLastError());
}

template <int M4, int JC>
void hw_launch(Ctx& ctx, const Staged& hs, int64_t K, int64_t h_cols, const float4* wt4, int64_t w_cols, int64_t tp,
               float* t, Ctl* ctl) {
  const size_t smem = static_cast<size_t>(M4) * w_cols * 32 * 16 + 8 * 128 * M4 * 4;
  auto k1 = k_hw<M4, JC>;
  AB2_CUDA(cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  int nb = 0;
  AB2_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k1, 256, smem));
  if (K > 0)
    k1<<<std::max(1, std::min(grid_of(K * 32, 256, ctx.sms), std::max(nb, 1) * ctx.sms)), 256, smem, ctx.stream>>>(
        hs.ptr, hs.base, static_cast<const uint32_t*>(hs.idx), static_cast<const float*>(hs.val), K, h_cols, wt4,
        w_cols, tp, t, ctl);
  AB2_CUDA(cudaGetLastError());
}

template <int JC>
void agg_t_launch(Ctx& ctx, const Staged& as, int64_t rows, int64_t K, const float* t, int64_t tp, int64_t w_cols,
                  float* dense, int32_t* cnt) {
  if (rows > 0)
    k_agg_t<JC><<<grid_of(rows * 32, 256, ctx.sms), 256, 0, ctx.stream>>>(
        as.ptr, as.base, static_cast<const uint32_t*>(as.idx), static_cast<const float*>(as.val), rows, K, t, tp,
        w_cols, dense, cnt);
  AB2_CUDA(cudaGetLastError());
}

template <int TP>
void agg_t_cp_launch(Ctx& ctx, const Staged& as, int64_t rows, int64_t K, const float* t, int64_t w_cols,
                     float* dense, int32_t* cnt) {
  const int smem = kAggWarps * kAggStages * kAggCh * TP * static_cast<int>(sizeof(float));
  auto k1 = k_agg_t_cp<TP>;
  AB2_CUDA(cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int nb = 0;
  AB2_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k1, kAggWarps * 32, smem));
  const int64_t want = (rows + 32 * kAggWarps - 1) / (32 * kAggWarps);  // warps own 32-row blocks
  const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, static_cast<int64_t>(std::max(nb, 1)) * ctx.sms)));
  if (rows > 0)
    k1<<<grid, kAggWarps * 32, smem, ctx.stream>>>(as.ptr, as.base, static_cast<const uint32_t*>(as.idx),
                                                   static_cast<const float*>(as.val), rows, K, t, w_cols, dense, cnt);
  AB2_CUDA(cudaGetLastError());
}

}  // namespace

void normalize_adjacency(Ctx& ctx, const aires_b200_matrix& a, aires_b200_output& out) {
  if (a.layout != AIRES_B200_CSR) fail(AIRES_B200_INVALID_ARGUMENT, "adjacency must be CSR");
  if (a.n_rows != a.n_cols)
    fail(1 + 13, std::to_string(a.n_rows) + "x" + std::to_string(a.n_cols) + " adjacency is not square");  // non_square
  if ((a.idx_bytes != 4 && a.idx_bytes != 8) || (a.val_bytes != 4 && a.val_bytes != 8) ||
      (out.idx_bytes != 4 && out.idx_bytes != 8) || (out.val_bytes != 4 && out.val_bytes != 8))
    fail(AIRES_B200_INVALID_ARGUMENT, "index / value widths must be 4 or 8");
  if (!out.alloc) fail(AIRES_B200_INVALID_ARGUMENT, "output allocator is null");
#define AB2_NORM(IT, VI, IO, VO_)                                                      \
  if (a.idx_bytes == sizeof(IT) && a.val_bytes == sizeof(VI) && out.idx_bytes == sizeof(IO) && \
      out.val_bytes == sizeof(VO_))                                                    \
    return normalize_t<IT, VI, IO, VO_>(ctx, a, out);
  AB2_NORM(uint32_t, float, uint32_t, float)
  AB2_NORM(uint32_t, double, uint32_t, float)
  AB2_NORM(uint32_t, float, uint32_t, double)
  AB2_NORM(uint32_t, double, uint32_t, double)
  AB2_NORM(uint64_t, double, uint64_t, double)
  AB2_NORM(uint64_t, float, uint64_t, float)
  AB2_NORM(uint64_t, double, uint64_t, float)
  AB2_NORM(uint64_t, float, uint64_t, double)
#undef AB2_NORM
  fail(AIRES_B200_INVALID_ARGUMENT, "output index width must equal the adjacency's");
}

void combine(Ctx& ctx, const aires_b200_matrix& x, const void* w, uint64_t w_rows, uint64_t w_cols,
             uint32_t w_location, aires_b200_output& out) {
  if (x.layout != AIRES_B200_CSR) fail(AIRES_B200_INVALID_ARGUMENT, "features must be CSR");
  if (x.n_cols != w_rows)
    fail(AIRES_B200_DIMENSION_MISMATCH, "feature width " + std::to_string(x.n_cols) + " does not match weight rows " +
                                            std::to_string(w_rows));
  if (x.val_bytes != out.val_bytes) fail(AIRES_B200_INVALID_ARGUMENT, "value widths of X, W and H must agree");
  if (!out.alloc) fail(AIRES_B200_INVALID_ARGUMENT, "output allocator is null");
#define AB2_COMB(V, IT, IO)                                                                     \
  if (x.val_bytes == sizeof(V) && x.idx_bytes == sizeof(IT) && out.idx_bytes == sizeof(IO)) \
    return combine_t<V, IT, IO>(ctx, x, w, w_rows, w_cols, w_location, out);
  AB2_COMB(float, uint32_t, uint32_t)
  AB2_COMB(double, uint32_t, uint32_t)
  AB2_COMB(float, uint64_t, uint64_t)
  AB2_COMB(double, uint64_t, uint64_t)
  AB2_COMB(float, uint32_t, uint64_t)
  AB2_COMB(double, uint64_t, uint32_t)
  AB2_COMB(double, uint32_t, uint64_t)
  AB2_COMB(float, uint64_t, uint32_t)
#undef AB2_COMB
  fail(AIRES_B200_INVALID_ARGUMENT, "index widths must be 4 or 8");
}

}  // namespace ab2

namespace ab2 {

// H' = ReLU((Ã·H)·W), fp32, fused (dense-H path); Ã and H device or host CSR (u32 columns, f32).
// Scan of the positive counts, the caller's allocation, compaction of the dense ReLU rows and the
// copies out (both fused-layer forms).
static void finish_fused(Ctx& ctx, aires_b200_output& out, int64_t rows, uint64_t w_cols, const float* dense, int32_t* cnt,
                  Ctl* ctl, int launches) {
  int64_t* optr = ctx.cptr.as<int64_t>(rows + 1);
  scan_counts(ctx, cnt, rows, optr, ctl, &launches);
  Ctl* hc = static_cast<Ctl*>(ctx.h_ctl.get(sizeof(Ctl)));
  AB2_CUDA(cudaMemcpyAsync(hc, ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, ctx.stream));
  AB2_CUDA(cudaStreamSynchronize(ctx.stream));
  const uint64_t nnz = rows > 0 ? hc->nnz : 0;
  void *optr_o = nullptr, *oidx = nullptr, *oval = nullptr;
  const int rc = out.alloc(out.user, static_cast<uint64_t>(rows), nnz, &optr_o, &oidx, &oval);
  if (rc != 0) fail(rc, "output allocator failed for " + std::to_string(nnz) + " nonzeros");
  void* dcol = out.location == AIRES_B200_DEVICE ? oidx : ctx.c_col.get(std::max<uint64_t>(nnz, 1) * out.idx_bytes);
  float* dval = out.location == AIRES_B200_DEVICE ? static_cast<float*>(oval)
                                                  : static_cast<float*>(ctx.c_val.get(std::max<uint64_t>(nnz, 1) * 4));
  if (rows > 0 && nnz > 0) {
    if (out.idx_bytes == 4)
      k_compact_rows<uint32_t><<<grid_of(rows * 32, 256, ctx.sms), 256, 0, ctx.stream>>>(
          dense, rows, static_cast<int64_t>(w_cols), optr, static_cast<uint32_t*>(dcol), dval);
    else
      k_compact_rows<uint64_t><<<grid_of(rows * 32, 256, ctx.sms), 256, 0, ctx.stream>>>(
          dense, rows, static_cast<int64_t>(w_cols), optr, static_cast<uint64_t*>(dcol), dval);
    AB2_CUDA(cudaGetLastError());
    launches++;
  }
  const cudaMemcpyKind kind = out.location == AIRES_B200_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
  AB2_CUDA(cudaMemcpyAsync(optr_o, optr, (rows + 1) * 8, kind, ctx.stream));
  if (out.location != AIRES_B200_DEVICE && nnz) {
    AB2_CUDA(cudaMemcpyAsync(oidx, dcol, nnz * out.idx_bytes, kind, ctx.stream));
    AB2_CUDA(cudaMemcpyAsync(oval, dval, nnz * 4, kind, ctx.stream));
  }
  AB2_CUDA(cudaStreamSynchronize(ctx.stream));
  float ms = 0;
  AB2_CUDA(cudaEventElapsedTime(&ms, ctx.ev[0], ctx.ev[1]));
  ctx.last_ms = ms;
  ctx.launches = launches;
  out.n_rows = static_cast<uint64_t>(rows);
  out.n_cols = w_cols;
  out.nnz = nnz;
  out.flops = 0;
}

void layer_fused(Ctx& ctx, const aires_b200_matrix& at, const aires_b200_matrix& h, const void* w, uint64_t w_rows,
                 uint64_t w_cols, uint32_t w_location, aires_b200_output& out) {
  if (at.layout != AIRES_B200_CSR || h.layout != AIRES_B200_CSR)
    fail(AIRES_B200_INVALID_ARGUMENT, "Ã and H must be CSR");
  if (at.idx_bytes != 4 || at.val_bytes != 4 || h.idx_bytes != 4 || h.val_bytes != 4 || out.val_bytes != 4)
    fail(AIRES_B200_INVALID_ARGUMENT, "the fused layer is fp32 with 4-byte column indices");
  if (at.n_cols != h.n_rows || h.n_cols != w_rows)
    fail(AIRES_B200_DIMENSION_MISMATCH, "Ã, H and W dimensions do not chain");
  const int M = static_cast<int>((h.n_cols + 31) / 32);
  const int JC = static_cast<int>((w_cols + 31) / 32);
  if (M < 1 || M > 8 || JC < 1 || JC > 4)
    fail(AIRES_B200_UNSUPPORTED_FORMAT, "fused layer supports H widths <= 256 and W widths <= 128");
  if (!out.alloc) fail(AIRES_B200_INVALID_ARGUMENT, "output allocator is null");
  const int64_t rows = static_cast<int64_t>(at.n_rows), K = static_cast<int64_t>(h.n_rows);
  int launches = 0;
  // W narrower than H: aggregate T = H·W instead of H (see k_hw / k_agg_t)
  if (w_cols < h.n_cols && option("fused_reassoc", 1) != 0) {
    const int M4 = (M + 3) / 4;
    const size_t smem = static_cast<size_t>(M4) * w_cols * 32 * 16 + 8 * 128 * M4 * 4;
    if (smem <= 200 * 1024) {
      const Staged hs = stage_csr(ctx, h);
      const float* wsrc = static_cast<const float*>(w);
      if (w_location == AIRES_B200_HOST) {
        float* dw = static_cast<float*>(ctx.x_idx.get(std::max<uint64_t>(w_rows * w_cols, 1) * sizeof(float)));
        AB2_CUDA(cudaMemcpyAsync(dw, w, w_rows * w_cols * sizeof(float), cudaMemcpyHostToDevice, ctx.stream));
        wsrc = dw;
      }
      // T = H·W on tcgen05 (3xTF32) when W fits the tensor-core kernel's 48 output columns
      const bool tensor = w_cols <= 48 && h.n_cols <= 256 && option("hw_tensor", 1) != 0;
      float4* wt4 = nullptr;
      if (!tensor) {
        wt4 = static_cast<float4*>(ctx.xo_desc.get(static_cast<size_t>(M4) * w_cols * 32 * sizeof(float4)));
        k_w_lane_major4<<<grid_of(static_cast<int64_t>(M4) * w_cols * 32, 256, ctx.sms), 256, 0, ctx.stream>>>(
            wsrc, static_cast<int64_t>(w_rows), static_cast<int64_t>(w_cols), M4, wt4);
      }
      const int64_t tp = (static_cast<int64_t>(w_cols) + 7) & ~int64_t(7);
      float* t = static_cast<float*>(ctx.xo_val.get(std::max<int64_t>(K, 1) * tp * sizeof(float)));
      float* dense = static_cast<float*>(ctx.t_val.get(std::max<int64_t>(rows, 1) * w_cols * sizeof(float)));
      int32_t* cnt = ctx.cnt.as<int32_t>(std::max<int64_t>(rows, 1));
      Ctl* ctl = ctx.ctl.as<Ctl>(1);
      AB2_CUDA(cudaMemsetAsync(ctl, 0, sizeof(Ctl), ctx.stream));
      AB2_CUDA(cudaEventRecord(ctx.ev[0], ctx.stream));
      const int64_t hc = static_cast<int64_t>(h.n_cols), wc = static_cast<int64_t>(w_cols);
      // T = H·W is enqueued before Ã is staged: both stagings use the context's A buffers
      if (tensor) {
        hw_tc_launch(ctx, hs, K, hc, wsrc, wc, tp, t, ctl);
      } else {
        switch (M4 * 8 + JC) {
#define AB2_RA(A, B) case A * 8 + B: hw_launch<A, B>(ctx, hs, K, hc, wt4, wc, tp, t, ctl); break;
          AB2_RA(1, 1) AB2_RA(1, 2) AB2_RA(1, 3) AB2_RA(1, 4) AB2_RA(2, 1) AB2_RA(2, 2) AB2_RA(2, 3) AB2_RA(2, 4)
#undef AB2_RA
          default: fail(AIRES_B200_UNSUPPORTED_FORMAT, "fused layer shape");
        }
      }
      const Staged as = stage_csr(ctx, at);
      if (tp <= 64 && K * tp < (int64_t(1) << 32) && option("agg_async", 1) != 0) {
        switch (tp) {
#define AB2_CP(TP) case TP: agg_t_cp_launch<TP>(ctx, as, rows, K, t, wc, dense, cnt); break;
          AB2_CP(8) AB2_CP(16) AB2_CP(24) AB2_CP(32) AB2_CP(40) AB2_CP(48) AB2_CP(56) AB2_CP(64)
#undef AB2_CP
        }
      } else switch (JC) {
        case 1: agg_t_launch<1>(ctx, as, rows, K, t, tp, wc, dense, cnt); break;
        case 2: agg_t_launch<2>(ctx, as, rows, K, t, tp, wc, dense, cnt); break;
        case 3: agg_t_launch<3>(ctx, as, rows, K, t, tp, wc, dense, cnt); break;
        default: agg_t_launch<4>(ctx, as, rows, K, t, tp, wc, dense, cnt); break;
      }
      launches += 3;
      AB2_CUDA(cudaEventRecord(ctx.ev[1], ctx.stream));
      finish_fused(ctx, out, rows, w_cols, dense, cnt, ctl, launches);
      return;
    }
  }
  // H -> dense rows (32*M floats each)
  const Staged hs = stage_csr(ctx, h);
  float* hd = static_cast<float*>(ctx.xo_val.get(std::max<int64_t>(K, 1) * 32 * M * sizeof(float)));
  switch (M) {
#define AB2_DENS(MM) case MM: k_densify<MM><<<grid_of(K * 32, 256, ctx.sms), 256, 0, ctx.stream>>>(hs.ptr, hs.base, static_cast<const uint32_t*>(hs.idx), static_cast<const float*>(hs.val), K, static_cast<int64_t>(h.n_cols), hd); break;
    AB2_DENS(1) AB2_DENS(2) AB2_DENS(3) AB2_DENS(4) AB2_DENS(5) AB2_DENS(6) AB2_DENS(7) AB2_DENS(8)
#undef AB2_DENS
  }
  launches++;
  // W -> lane-major
  const float* wsrc = static_cast<const float*>(w);
  if (w_location == AIRES_B200_HOST) {
    float* dw = static_cast<float*>(ctx.x_idx.get(std::max<uint64_t>(w_rows * w_cols, 1) * sizeof(float)));
    AB2_CUDA(cudaMemcpyAsync(dw, w, w_rows * w_cols * sizeof(float), cudaMemcpyHostToDevice, ctx.stream));
    wsrc = dw;
  }
  float* wt = static_cast<float*>(ctx.xo_desc.get(static_cast<size_t>(M) * w_cols * 32 * sizeof(float)));
  k_w_lane_major<<<grid_of(static_cast<int64_t>(M) * w_cols * 32, 256, ctx.sms), 256, 0, ctx.stream>>>(
      wsrc, static_cast<int64_t>(w_rows), static_cast<int64_t>(w_cols), M, wt);
  launches++;
  // Ã rows (staged after H: the A buffers of the context)
  const Staged as = stage_csr(ctx, at);
  float* dense = static_cast<float*>(ctx.t_val.get(std::max<int64_t>(rows, 1) * w_cols * sizeof(float)));
  int32_t* cnt = ctx.cnt.as<int32_t>(std::max<int64_t>(rows, 1));
  int64_t* optr = ctx.cptr.as<int64_t>(rows + 1);
  Ctl* ctl = ctx.ctl.as<Ctl>(1);
  AB2_CUDA(cudaMemsetAsync(ctl, 0, sizeof(Ctl), ctx.stream));
  AB2_CUDA(cudaEventRecord(ctx.ev[0], ctx.stream));
  if (rows > 0) {
    const auto* ac = static_cast<const uint32_t*>(as.idx);
    const auto* av = static_cast<const float*>(as.val);
    switch (M) {
#define AB2_AC(MM) case MM: agg_comb_m<MM>(ctx, JC, as.ptr, as.base, ac, av, rows, K, hd, wt, static_cast<int64_t>(w_cols), dense, cnt); break;
      AB2_AC(1) AB2_AC(2) AB2_AC(3) AB2_AC(4) AB2_AC(5) AB2_AC(6) AB2_AC(7) AB2_AC(8)
#undef AB2_AC
    }
    launches++;
  }
  AB2_CUDA(cudaEventRecord(ctx.ev[1], ctx.stream));
  finish_fused(ctx, out, rows, w_cols, dense, cnt, ctl, launches);
}

}  // namespace ab2
