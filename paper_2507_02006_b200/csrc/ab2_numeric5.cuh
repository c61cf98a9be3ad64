// ab2_numeric5.cuh -- fp32 A·X product pass over a per-chunk step list (sm_100a).
//
// Same contract as k_numeric3 (ab2_numeric.cuh): one pass over A, each row accumulated once in a
// dense shared-memory accumulator, emitted in ascending column order (canonical, sparse.hpp:26-28)
// either into the bump-allocated staging area (then K_place) or, when the row offsets are known
// (out-of-core tiles), straight to the exact CSR offsets (spgemm.hpp:60-132).
//
// Work mapping.  The warp is G = 32 / W groups of W lanes; group g owns accumulator copy g.
// X is stored in padded W-entry slots (ab2_operand.cu, k_x_pfill): row k = nslot_k consecutive
// slots, entries past the row's length aim at the trash column.  For a 32-entry chunk of an A row
// every lane expands its entry (k, a) into nslot_k step descriptors {slot, a} in a per-warp list
// (positions from a warp scan of nslot); warp step t then hands descriptor t*G + g to group g.
// So the steps of all entries are spread evenly over the groups (no per-group imbalance, no
// overflow tails), each step is one 8-byte LDS of the descriptor, one 8-byte gather of a slot
// entry per lane and one shared-memory FMA read-modify-write.  Two lanes of one step never touch
// the same cell: within a group the slot's columns are distinct; across groups the copies differ.
// Copies are summed at fold time (fp32 mode: order-free within the stated 1e-5 tolerance).
//
// Memory-level parallelism: the (k, a) loads of chunk c+2 and the descriptor gather of chunk c+1
// are in flight while chunk c runs; within a chunk B warp steps issue their gathers before any of
// their accumulations.
//
// Marker and structural zeros as in ab2_numeric.cuh: cells start at -0.0; a weight that can round
// a product to zero (or an exact zero stored in X, flag XZ) sends the row to the explicit path.
#pragma once
#include "ab2_numeric.cuh"

#ifndef AB2_N5_BATCH
#define AB2_N5_BATCH 8
#endif
#ifndef AB2_N5_MAXT
#define AB2_N5_MAXT 256
#endif
#ifndef AB2_N5_MINB
#define AB2_N5_MINB 3
#endif

namespace ab2 {

constexpr int kN5List = 64;  // step descriptors per warp per round

template <class IdxT>
struct Num5Args {
  const uint64_t* aptr;
  uint64_t abase;
  const IdxT* acol;
  const float* aval;
  int64_t rows;
  int64_t K;
  int32_t n_cols;
  int32_t stride;      // accumulator floats per copy (>= n_cols + 1, multiple of 32)
  int32_t warp_bytes;  // (32/W)*stride*4 + stride marks + kN5List * 8
  int32_t pad0;
  const uint2* xdesc;  // K+1 {slot start, nslot | len << 16}
  const uint2* xent;   // padded slots {col * 4, value bits}
  uint32_t dummy_slot; // an all-trash slot
  uint32_t pad1;
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

__device__ __forceinline__ void smem_fma5(uint32_t addr, float a, float x) {
  asm volatile(
      "{\n\t.reg .f32 t;\n\tld.shared.f32 t, [%0];\n\tfma.rn.f32 t, %1, %2, t;\n\tst.shared.f32 [%0], t;\n\t}" ::"r"(addr),
      "f"(a), "f"(x)
      : "memory");
}

// Walks A entries [0, n) in 32-entry chunks c == chunk0 (mod chunk_stride); returns the MACs.
template <class IdxT, int W, bool XZ>
__device__ __forceinline__ uint32_t walk5(const Num5Args<IdxT>& p, const IdxT* __restrict__ ac,
                                          const float* __restrict__ av, uint32_t n, uint32_t chunk0,
                                          uint32_t chunk_stride, float* acc, uint2* list, bool& zero) {
  constexpr int G = 32 / W;
  constexpr int B = AB2_N5_BATCH;
  const int lane = lane_id();
  const uint32_t g = lane / W, e = lane % W;
  const uint64_t K = static_cast<uint64_t>(p.K);
  const uint32_t copy_s = static_cast<uint32_t>(__cvta_generic_to_shared(acc)) + g * static_cast<uint32_t>(p.stride) * 4u;
  const uint32_t list_s = static_cast<uint32_t>(__cvta_generic_to_shared(list));
  const uint32_t trash4 = static_cast<uint32_t>(p.n_cols) * 4u;
  const uint2* __restrict__ xbase = p.xent + e;  // slot entries hold the accumulator byte offset col * 4
  const float tiny = p.tiny;
  uint32_t macs = 0;
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
  uint64_t k1, k2;
  float a1, a2;
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
    const uint32_t ns = d.y & 0xffffu;
    macs += d.y >> 16;
    const uint32_t incl = warp_incl_scan(ns);
    const uint32_t TS = __shfl_sync(kFull, incl, 31);
    const uint32_t pos = incl - ns;
    for (uint32_t r0 = 0; r0 < TS; r0 += kN5List) {
      // my steps [pos, pos + ns) that fall in [r0, r0 + kN5List); the list is padded to a whole
      // warp step with descriptors of the all-trash dummy slot
      __syncwarp();
      const uint32_t lo = max(pos, r0), hi = min(pos + ns, r0 + kN5List);
      for (uint32_t q = lo; q < hi; q++) {
        const uint32_t dst = list_s + (q - r0) * 8u;
        asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(dst), "r"(d.x + (q - pos)), "r"(__float_as_uint(a))
                     : "memory");
      }
      const uint32_t nsteps = min(TS - r0, static_cast<uint32_t>(kN5List));
      const uint32_t nb = (nsteps + G - 1) / G;  // warp steps this round
      if (lane < nb * G - nsteps) {
        asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(list_s + (nsteps + lane) * 8u), "r"(p.dummy_slot),
                     "r"(0u)
                     : "memory");
      }
      __syncwarp();
#pragma unroll 1
      for (uint32_t t0 = 0; t0 < nb; t0 += B) {
        const uint32_t cu = min(static_cast<uint32_t>(B), nb - t0);
        uint2 xe[B];
        float ax[B];
#pragma unroll
        for (int u = 0; u < B; u++) {
          if (u < cu) {
            uint2 ds;
            asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];"
                         : "=r"(ds.x), "=r"(ds.y)
                         : "r"(list_s + ((t0 + u) * G + g) * 8u)
                         : "memory");
            xe[u] = __ldg(xbase + static_cast<uint64_t>(ds.x) * W);
            ax[u] = __uint_as_float(ds.y);
          }
        }
#pragma unroll
        for (int u = 0; u < B; u++) {
          // padding lanes (trash column) skip the access: the groups' trash cells share a bank,
          // which made every step a >= 4-way bank conflict (3.9 wavefronts per RMW measured)
          if (u < cu && xe[u].x != trash4) {
            const float xv = __uint_as_float(xe[u].y);
            if constexpr (XZ) zero |= ax[u] * xv == 0.f;
            smem_fma5(copy_s + xe[u].x, ax[u], xv);
          }
          __syncwarp();  // consecutive steps of one group may hit the same cell
        }
        __syncwarp();
      }
    }
  }
  return macs;
}

// Explicit-mark slow path (one k at a time in ascending order, +0.0 start, byte marks); leaves
// copy 0 with the values of marked cells and the marker elsewhere, other copies reset.
template <class IdxT, int W>
__device__ void slow_row5(const Num5Args<IdxT>& p, const IdxT* __restrict__ ac, const float* __restrict__ av,
                          uint32_t n, float* acc, unsigned char* mark) {
  const int lane = lane_id();
  const int n_cols = p.n_cols;
  for (int c = lane; c < p.stride * (32 / W); c += 32) acc[c] = c < n_cols ? 0.f : Sentinel<float>::value();
  for (int c = lane; c < p.stride; c += 32) mark[c] = 0;
  __syncwarp();
  for (uint32_t i = 0; i < n; i++) {
    const uint64_t k = static_cast<uint64_t>(ac[i]);
    if (k >= static_cast<uint64_t>(p.K)) continue;
    const float a = av[i];
    const uint2 d = p.xdesc[k];
    const uint32_t len = d.y >> 16;
    for (uint32_t t = lane; t < len; t += 32) {
      const uint2 en = p.xent[static_cast<uint64_t>(d.x) * W + t];
      const uint32_t c = en.x >> 2;
      acc[c] = __fadd_rn(acc[c], __fmul_rn(a, __uint_as_float(en.y)));
      mark[c] = 1;
    }
    __syncwarp();
  }
  for (int c = lane; c < n_cols; c += 32)
    if (!mark[c]) acc[c] = Sentinel<float>::value();
  __syncwarp();
}

template <class IdxT, int W, bool XZ>
__global__ void __launch_bounds__(AB2_N5_MAXT, AB2_N5_MINB) k_numeric5(Num5Args<IdxT> p) {
  constexpr int G = 32 / W;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ unsigned long long s_ticket;
  __shared__ int s_zero;
  const int lane = lane_id(), warp = warp_id(), nw = blockDim.x >> 5;
  const int n_cols = p.n_cols;
  const int acc_elems = p.stride * G;
  auto warp_acc = [&](int w) { return reinterpret_cast<float*>(smem_raw + static_cast<size_t>(w) * p.warp_bytes); };
  auto warp_mark = [&](int w) {
    return smem_raw + static_cast<size_t>(w) * p.warp_bytes + static_cast<size_t>(acc_elems) * 4;
  };
  auto warp_list = [&](int w) {
    return reinterpret_cast<uint2*>(smem_raw + static_cast<size_t>(w) * p.warp_bytes +
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
    my_macs += walk5<IdxT, W, XZ>(p, ac, av, n, warp, nw, warp_acc(warp), warp_list(warp), zero);
    if (__any_sync(kFull, zero) && lane == 0) s_zero = 1;
    __syncthreads();
    if (s_zero) {
      if (warp == 0) slow_row5<IdxT, W>(p, ac, av, n, warp_acc(0), warp_mark(0));
      if (warp != 0)
        for (int i = lane; i < acc_elems; i += 32) warp_acc(warp)[i] = Sentinel<float>::value();
    } else {
      for (int c = threadIdx.x; c < p.stride; c += blockDim.x) {
        float v = Sentinel<float>::value();
        for (int w = 0; w < nw; w++)
          for (int g = 0; g < G; g++) {
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
      my_macs += walk5<IdxT, W, XZ>(p, ac, av, n, 0, 1, acc, warp_list(warp), zero);
      if (__any_sync(kFull, zero)) slow_row5<IdxT, W>(p, ac, av, n, acc, warp_mark(warp));
      const uint32_t cnt = fold_count<float>(acc, p.stride, G, n_cols);
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
