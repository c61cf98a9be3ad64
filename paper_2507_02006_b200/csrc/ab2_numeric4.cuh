// ab2_numeric4.cuh -- fp32 A·X product pass with flattened multiply-accumulates (sm_100a).
//
// Same contract as k_numeric3 (ab2_numeric.cuh): one pass over A, each row accumulated once in
// a dense shared-memory accumulator, emitted in ascending column order into the bump-allocated
// staging area, then K_place moves rows to their exact CSR offsets (spgemm.hpp:60-132).
//
// What changes is how the terms a_ik * x_kj are spread over the lanes.  k_numeric3 gives each
// A entry a fixed W-lane group, so with Reddit-shaped X (mean 6 entries per row, W = 16) ~60%
// of the lanes idle in every step.  Here the terms of a 32-entry chunk of an A row are laid
// end to end (an exclusive scan of the X row lengths) and lane t of a window takes term
// p0 + t, so every lane carries a term in every window:
//   * chunk: lanes load (k, a) coalesced, gather the 8-byte X row descriptor {start, len},
//     compact the non-empty entries (ballot rank, one STS/LDS), scan the lengths;
//   * window: the entries starting inside [p0, p0+32) form a 32-bit mask (REDUX.OR); the
//     owner of lane t is (# entries starting at or before p0+t) - 1, fetched with SHFL; lane t
//     gathers its {col, value} pair with one 8-byte load from the flat X layout.
// Collisions: two lanes of a window may hit the same column only if they belong to different
// X rows.  Entry ranks r map to accumulator copy r mod NC; the window's entries are applied
// in ceil(#entries / NC) phases of at most NC consecutive ranks, so within a phase every lane
// owning a copy belongs to the same X row and its columns are distinct.  Copies are summed at
// fold time (fp32 mode: order-free within the stated tolerance).
//
// Marker and structural zeros exactly as ab2_numeric.cuh (cells start at -0.0; any possibly
// zero product sends the row through the explicit-mark path).
#pragma once
#include "ab2_numeric.cuh"

#ifndef AB2_N4_BATCH
#define AB2_N4_BATCH 8
#endif

namespace ab2 {

template <class IdxT>
struct Num4Args {
  const uint64_t* aptr;
  uint64_t abase;
  const IdxT* acol;
  const float* aval;
  int64_t rows;
  int64_t K;
  int32_t n_cols;
  int32_t stride;      // accumulator floats per copy (>= n_cols + 1, multiple of 32)
  int32_t copies;      // NC, power of two
  int32_t log2c;
  int32_t warp_bytes;  // copies*stride*4 + stride marks + 32 * 16 compaction slots
  int32_t pad0;
  const uint2* xdesc;  // K+1 {start, len}
  const uint2* xent;   // {col, value bits}
  const int64_t* heavy;
  int64_t heavy_deg;
  uint32_t* cnt;
  uint64_t* toff;
  IdxT* tcol;
  float* tval;
  uint64_t t_cap;
  float tiny;
  uint32_t stage_block;
  Ctl* ctl;
  const int64_t* cpos;
  int64_t cbase;
};

__device__ __forceinline__ void smem_fma_rmw(uint32_t addr, float a, float x) {
  asm volatile(
      "{\n\t.reg .f32 t;\n\tld.shared.f32 t, [%0];\n\tfma.rn.f32 t, %1, %2, t;\n\tst.shared.f32 [%0], t;\n\t}" ::"r"(addr),
      "f"(a), "f"(x)
      : "memory");
}

// Walks A entries [0, n) in 32-entry chunks c == chunk0 (mod chunk_stride); returns the MACs.
template <class IdxT, bool XZ>
__device__ __forceinline__ uint32_t walk4(const Num4Args<IdxT>& p, const IdxT* __restrict__ ac,
                                          const float* __restrict__ av, uint32_t n, uint32_t chunk0,
                                          uint32_t chunk_stride, float* acc, uint4* cbuf, bool& zero) {
  constexpr int U = AB2_N4_BATCH;
  const int lane = lane_id();
  const uint32_t lt_mask = (1u << lane) - 1u;
  const uint32_t le_mask = 0xffffffffu >> (31 - lane);
  const uint64_t K = static_cast<uint64_t>(p.K);
  const uint32_t acc_s = static_cast<uint32_t>(__cvta_generic_to_shared(acc));
  const uint32_t cbuf_s = static_cast<uint32_t>(__cvta_generic_to_shared(cbuf));
  const uint32_t stride4 = static_cast<uint32_t>(p.stride) * 4u;
  const uint32_t cmask = static_cast<uint32_t>(p.copies) - 1u;
  const int log2c = p.log2c;
  const uint2* __restrict__ xent = p.xent;
  const float tiny = p.tiny;
  uint32_t macs = 0;
  // Two-deep prefetch: the descriptor gather of chunk c+1 and the (k, a) loads of chunk c+2 are
  // in flight while chunk c's terms are gathered and accumulated.
  const uint32_t step = chunk_stride * 32;
  auto load_ka = [&](uint32_t b, uint64_t& k, float& a) {
    const uint32_t i = b + lane;
    k = K;
    a = 0.f;
    if (i < n) {
      k = static_cast<uint64_t>(ac[i]);
      a = av[i];
    }
  };
  auto load_d = [&](uint64_t k) { return k < K ? __ldg(p.xdesc + k) : make_uint2(0u, 0u); };
  uint64_t k1 = K, k2 = K;
  float a1 = 0.f, a2 = 0.f;
  uint32_t b = chunk0 * 32;
  load_ka(b, k1, a1);
  uint2 d1 = load_d(k1);
  load_ka(b + step, k2, a2);
  for (; b < n; b += step) {
    const uint2 d = d1;
    const float a = a1;
    zero |= (b + lane < n) && !(fabsf(a) >= tiny);  // zero, tiny or NaN weight: explicit path
    d1 = load_d(k2);
    a1 = a2;
    load_ka(b + 2 * step, k2, a2);
    macs += d.y;
    const uint32_t nem = __ballot_sync(kFull, d.y != 0);
    if (nem == 0) continue;
    const uint32_t n_ne = __popc(nem);
    __syncwarp();
    if (d.y != 0) {
      const uint32_t dst = cbuf_s + __popc(nem & lt_mask) * 16u;
      asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(dst), "r"(d.x), "r"(d.y),
                   "r"(__float_as_uint(a)), "r"(0u)
                   : "memory");
    }
    __syncwarp();
    uint32_t start = 0, len = 0;
    float aa = 0.f;
    if (static_cast<uint32_t>(lane) < n_ne) {
      uint4 t;
      asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(t.x), "=r"(t.y), "=r"(t.z), "=r"(t.w)
                   : "r"(cbuf_s + lane * 16u)
                   : "memory");
      start = t.x;
      len = t.y;
      aa = __uint_as_float(t.z);
    }
    const uint32_t incl = warp_incl_scan(len);
    const uint32_t T = __shfl_sync(kFull, incl, 31);
    const uint32_t excl = incl - len;
    const uint32_t base = start - excl;  // term p of this entry sits at xent[base + p]
    uint32_t before = 0;                 // entries starting before the current window
#pragma unroll 1
    for (uint32_t p0 = 0; p0 < T; p0 += 32u * U) {
      uint2 xe[U];
      float ax[U];
      uint32_t own[U], lo[U], cnt[U];
#pragma unroll
      for (int u = 0; u < U; u++) {
        const uint32_t q0 = p0 + 32u * u;
        const uint32_t d0 = excl - q0;
        const uint32_t bit = (len != 0 && d0 < 32u) ? (1u << d0) : 0u;
        const uint32_t M = __reduce_or_sync(kFull, bit);
        const uint32_t J = before + __popc(M & le_mask) - 1u;
        lo[u] = before + (M & 1u) - 1u;  // owner of the window's first term
        before += __popc(M);
        cnt[u] = q0 < T ? before - lo[u] : 0u;
        own[u] = J;
        const uint32_t src = J & 31u;
        const uint32_t bJ = __shfl_sync(kFull, base, src);
        ax[u] = __shfl_sync(kFull, aa, src);
        xe[u] = make_uint2(0xffffffffu, 0u);
        if (q0 + lane < T) xe[u] = __ldg(xent + (bJ + q0 + lane));
      }
#pragma unroll
      for (int u = 0; u < U; u++) {
        if (cnt[u] == 0) break;
        const bool act = xe[u].x != 0xffffffffu;
        const float xv = __uint_as_float(xe[u].y);
        if constexpr (XZ) zero |= act && ax[u] * xv == 0.f;
        const uint32_t addr = acc_s + (own[u] & cmask) * stride4 + xe[u].x * 4u;
        if (cnt[u] <= cmask + 1u) {
          if (act) smem_fma_rmw(addr, ax[u], xv);
        } else {
          const uint32_t nph = (cnt[u] + cmask) >> log2c;
          const uint32_t myph = (own[u] - lo[u]) >> log2c;
          for (uint32_t ph = 0; ph < nph; ph++) {
            if (act && myph == ph) smem_fma_rmw(addr, ax[u], xv);
            __syncwarp();
          }
        }
        __syncwarp();
      }
    }
  }
  return macs;
}

// Explicit-mark slow path over the flat layout (one k at a time in ascending order, +0.0 start,
// byte marks); leaves copy 0 with the values of marked cells and the marker elsewhere.
template <class IdxT>
__device__ void slow_row4(const Num4Args<IdxT>& p, const IdxT* __restrict__ ac, const float* __restrict__ av,
                          uint32_t n, float* acc, unsigned char* mark) {
  const int lane = lane_id();
  const int n_cols = p.n_cols;
  for (int c = lane; c < p.stride * p.copies; c += 32) acc[c] = c < n_cols ? 0.f : Sentinel<float>::value();
  for (int c = lane; c < p.stride; c += 32) mark[c] = 0;
  __syncwarp();
  for (uint32_t i = 0; i < n; i++) {
    const uint64_t k = static_cast<uint64_t>(ac[i]);
    if (k >= static_cast<uint64_t>(p.K)) continue;
    const float a = av[i];
    const uint2 d = p.xdesc[k];
    for (uint32_t t = lane; t < d.y; t += 32) {
      const uint2 e = p.xent[d.x + t];
      acc[e.x] = __fadd_rn(acc[e.x], __fmul_rn(a, __uint_as_float(e.y)));
      mark[e.x] = 1;
    }
    __syncwarp();
  }
  for (int c = lane; c < n_cols; c += 32)
    if (!mark[c]) acc[c] = Sentinel<float>::value();
  __syncwarp();
}

template <class IdxT, bool XZ>
__global__ void __launch_bounds__(256, 2) k_numeric4(Num4Args<IdxT> p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ unsigned long long s_ticket;
  __shared__ int s_zero;
  const int lane = lane_id(), warp = warp_id(), nw = blockDim.x >> 5;
  const int n_cols = p.n_cols;
  const int acc_elems = p.stride * p.copies;
  auto warp_acc = [&](int w) { return reinterpret_cast<float*>(smem_raw + static_cast<size_t>(w) * p.warp_bytes); };
  auto warp_mark = [&](int w) {
    return smem_raw + static_cast<size_t>(w) * p.warp_bytes + static_cast<size_t>(acc_elems) * 4;
  };
  auto warp_cbuf = [&](int w) {
    return reinterpret_cast<uint4*>(smem_raw + static_cast<size_t>(w) * p.warp_bytes +
                                    static_cast<size_t>(acc_elems) * 4 + p.stride);
  };
  for (int w = 0; w < nw; w++)
    for (int i = threadIdx.x; i < acc_elems; i += blockDim.x) warp_acc(w)[i] = Sentinel<float>::value();
  __syncthreads();
  StageCursor stage;
  unsigned long long my_nnz = 0, my_macs = 0;
  const unsigned long long n_heavy = p.ctl->n_sym_heavy;

  // ---- Phase 1: heavy rows, one CTA per row (warps interleave over the row's chunks) ----
  for (;;) {
    if (threadIdx.x == 0) {
      s_ticket = atomicAdd(&p.ctl->heavy_next, 1ull);
      s_zero = 0;
    }
    __syncthreads();
    const unsigned long long h = s_ticket;
    if (h >= n_heavy) break;
    const int64_t r = p.heavy[h];
    const uint64_t s = p.aptr[r] - p.abase, e = p.aptr[r + 1] - p.abase;
    const uint32_t n = static_cast<uint32_t>(e - s);
    const IdxT* ac = p.acol + s;
    const float* av = p.aval + s;
    bool zero = false;
    my_macs += walk4<IdxT, XZ>(p, ac, av, n, warp, nw, warp_acc(warp), warp_cbuf(warp), zero);
    if (__any_sync(kFull, zero) && lane == 0) s_zero = 1;
    __syncthreads();
    if (s_zero) {
      if (warp == 0) slow_row4<IdxT>(p, ac, av, n, warp_acc(0), warp_mark(0));
      if (warp != 0)
        for (int i = lane; i < acc_elems; i += 32) warp_acc(warp)[i] = Sentinel<float>::value();
    } else {
      for (int c = threadIdx.x; c < p.stride; c += blockDim.x) {
        float v = Sentinel<float>::value();
        for (int w = 0; w < nw; w++)
          for (int g = 0; g < p.copies; g++) {
            float* q = warp_acc(w) + g * p.stride + c;
            v += *q;
            *q = Sentinel<float>::value();
          }
        warp_acc(0)[c] = v;
      }
    }
    __syncthreads();
    if (warp == 0) {
      const uint32_t cnt = fold_count<float>(warp_acc(0), p.stride, 1, n_cols);
      const unsigned long long off = out_offset(p, r, cnt, stage);
      if (off <= p.t_cap && off + cnt <= p.t_cap) {
        emit_copy0<float, IdxT>(warp_acc(0), n_cols, p.tcol + off, p.tval + off);
      } else {
        fold_count<float>(warp_acc(0), p.stride, 1, 0);
        if (lane == 0) atomicMax(&p.ctl->bad_row, 1ull);
      }
      if (lane == 0) {
        p.cnt[r] = cnt;
        p.toff[r] = off;
        my_nnz += cnt;
      }
    }
    __syncthreads();
  }

  // ---- Phase 2: light rows, one warp per row ----
  float* acc = warp_acc(warp);
  for (;;) {
    unsigned long long r0 = 0;
    if (lane == 0) r0 = atomicAdd(&p.ctl->light_next, static_cast<unsigned long long>(kLightBatch));
    r0 = __shfl_sync(kFull, r0, 0);
    if (r0 >= static_cast<unsigned long long>(p.rows)) break;
    const int64_t r1 = min(static_cast<int64_t>(r0) + kLightBatch, p.rows);
    for (int64_t r = static_cast<int64_t>(r0); r < r1; r++) {
      const uint64_t s = p.aptr[r] - p.abase, e = p.aptr[r + 1] - p.abase;
      if (static_cast<int64_t>(e - s) > p.heavy_deg) continue;
      const uint32_t n = static_cast<uint32_t>(e - s);
      const IdxT* ac = p.acol + s;
      const float* av = p.aval + s;
      bool zero = false;
      my_macs += walk4<IdxT, XZ>(p, ac, av, n, 0, 1, acc, warp_cbuf(warp), zero);
      if (__any_sync(kFull, zero)) slow_row4<IdxT>(p, ac, av, n, acc, warp_mark(warp));
      const uint32_t cnt = fold_count<float>(acc, p.stride, p.copies, n_cols);
      const unsigned long long off = out_offset(p, r, cnt, stage);
      if (off <= p.t_cap && off + cnt <= p.t_cap) {
        emit_copy0<float, IdxT>(acc, n_cols, p.tcol + off, p.tval + off);
      } else {
        fold_count<float>(acc, p.stride, 1, 0);
        if (lane == 0) atomicMax(&p.ctl->bad_row, 1ull);
      }
      if (lane == 0) {
        p.cnt[r] = cnt;
        p.toff[r] = off;
        my_nnz += cnt;
      }
    }
  }
  my_macs = warp_sum(my_macs);
  if (lane == 0 && my_nnz) atomicAdd(&p.ctl->nnz, my_nnz);
  if (lane == 0 && my_macs) atomicAdd(&p.ctl->flops, my_macs);
}

}  // namespace ab2
