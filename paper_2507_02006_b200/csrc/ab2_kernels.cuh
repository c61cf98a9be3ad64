// ab2_kernels.cuh -- sm_100a kernels of the B200 AIRES A·X SpGEMM shared by the in-core product and
// the out-of-core pipeline.
//
// Replaces the reference's inner-product spgemm_block (spgemm.hpp:60-132):
//   K_classify  : rows whose A-degree exceeds the warp budget -> CTA-wide (heavy) list
//   K_numeric   : (ab2_numeric.cuh) one pass per row into a dense shared-memory accumulator,
//                 counted and emitted in ascending column order (spgemm.hpp:114-130; canonical,
//                 sparse.hpp:26-28) into a bump-allocated staging area
//   K_scan      : exclusive scan of the row counts -> int64 C row_ptr (spgemm.hpp:107, :111)
//   K_place     : staging -> exact CSR offsets (after the caller's exact allocation, :111-112)
//   K_symbolic  : per-row nnz(C) = |U_k cols(X_k)| (byte flags in shared memory) and per-row MACs
//                 -- only where C's sizes are needed before any product: the out-of-core tiles
//                 (scheduler.hpp:103-139), each sized on the device before it is multiplied
//
// Work distribution: heavy rows are claimed first, one CTA per row; light rows then go one warp per
// row from a ticket counter in batches.  No shared-memory fp atomics (smem CAS add measured 11.7
// SM-cycles per warp op on B200) and no MATCH.ANY.
//
// Accumulator marker: cells start at -0.0.  -0.0 + p == p for every p except p == -0.0, so a cell
// still reads -0.0 only if it got no contribution or only -0.0 ones; rows where a product can be
// exactly zero (zero / tiny weights, zeros stored in X) are re-run on the explicit-mark path with a
// +0.0 start (dot_row_col's `sum = 0.0; if (hit)`, spgemm.hpp:27-41) -- see ab2_numeric.cuh.
#pragma once
#include "ab2_common.cuh"
#include "ab2_operand.cuh"

namespace ab2 {

#ifndef AB2_LIGHT_BATCH
#define AB2_LIGHT_BATCH 4
#endif
constexpr int kLightBatch = AB2_LIGHT_BATCH;  // light rows per ticket

template <class V>
struct Sentinel;
template <>
struct Sentinel<float> {
  using Bits = uint32_t;
  static __device__ __forceinline__ float value() { return __uint_as_float(0x80000000u); }
  static __device__ __forceinline__ bool is(float v) { return __float_as_uint(v) == 0x80000000u; }
};
template <>
struct Sentinel<double> {
  using Bits = unsigned long long;
  static __device__ __forceinline__ double value() {
    return __longlong_as_double(static_cast<long long>(0x8000000000000000ull));
  }
  static __device__ __forceinline__ bool is(double v) {
    return static_cast<unsigned long long>(__double_as_longlong(v)) == 0x8000000000000000ull;
  }
};

// Warp-aggregated append of `r` (when pred) to list[] with counter *n.
__device__ __forceinline__ void warp_append(bool pred, int64_t r, int64_t* list,
                                            unsigned long long* n) {
  unsigned m = __ballot_sync(__activemask(), pred);
  if (!m) return;
  int lane = lane_id();
  int leader = __ffs(m) - 1;
  unsigned long long base = 0;
  if (lane == leader) base = atomicAdd(n, static_cast<unsigned long long>(__popc(m)));
  base = __shfl_sync(__activemask(), base, leader);
  if (pred) list[base + __popc(m & ((1u << lane) - 1))] = r;
}

// ---------------------------------------------------------------------------
// K_classify: heavy rows for the symbolic pass (A-degree > heavy_deg).
// ---------------------------------------------------------------------------
static __global__ void k_classify(const uint64_t* __restrict__ aptr, int64_t rows, int64_t heavy_deg,
                           int64_t* __restrict__ sym_heavy, Ctl* __restrict__ ctl) {
  int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t r0 = static_cast<int64_t>(blockIdx.x) * blockDim.x; r0 < rows; r0 += stride) {
    int64_t r = r0 + threadIdx.x;
    bool heavy = false;
    if (r < rows) heavy = static_cast<int64_t>(aptr[r + 1] - aptr[r]) > heavy_deg;
    warp_append(heavy, r, sym_heavy, &ctl->n_sym_heavy);
  }
}

// ---------------------------------------------------------------------------
// Column-only slot loads (W u16 per row).
// ---------------------------------------------------------------------------
template <int W>
struct CSlot {
  uint32_t w[W / 2];
  __device__ __forceinline__ uint32_t at(int e) const { return (w[e >> 1] >> (16 * (e & 1))) & 0xffffu; }
};

template <int W>
__device__ __forceinline__ CSlot<W> load_cslot(const uint16_t* __restrict__ cs, uint64_t k) {
  CSlot<W> s;
  const uint16_t* p = cs + k * W;
  if constexpr (W == 2) {
    s.w[0] = __ldg(reinterpret_cast<const uint32_t*>(p));
  } else if constexpr (W == 4) {
    uint2 v = __ldg(reinterpret_cast<const uint2*>(p));
    s.w[0] = v.x;
    s.w[1] = v.y;
  } else if constexpr (W == 8) {
    uint4 v = __ldg(reinterpret_cast<const uint4*>(p));
    s.w[0] = v.x;
    s.w[1] = v.y;
    s.w[2] = v.z;
    s.w[3] = v.w;
  } else {
    static_assert(W == 16, "slot width");
    uint4 v = __ldg(reinterpret_cast<const uint4*>(p));
    uint4 u = __ldg(reinterpret_cast<const uint4*>(p) + 1);
    s.w[0] = v.x;
    s.w[1] = v.y;
    s.w[2] = v.z;
    s.w[3] = v.w;
    s.w[4] = u.x;
    s.w[5] = u.y;
    s.w[6] = u.z;
    s.w[7] = u.w;
  }
  return s;
}

template <int W>
__device__ __forceinline__ CSlot<W> empty_cslot() {
  CSlot<W> s;
#pragma unroll
  for (int i = 0; i < W / 2; i++) s.w[i] = 0xffffffffu;
  return s;
}

// Marks the inline columns of X row k in `flags` (predicated byte stores; concurrent
// writers only ever store 1) and returns their count; *ovf reports an overflow marker.
template <int W>
__device__ __forceinline__ uint32_t mark_cslot(const CSlot<W>& s, unsigned char* flags, bool& ovf) {
  uint32_t f = 0;
#pragma unroll
  for (int e = 0; e < W; e++) {
    const uint32_t c = s.at(e);
    if (c < kCOvf) flags[c] = 1;
    f += c < kCOvf;
    ovf |= c == kCOvf;
  }
  return f;
}

// Overflow tail of X row k (rows longer than the slot; rare on the GCN shapes).
template <int W>
__device__ __noinline__ uint32_t mark_tail(uint64_t k, const int64_t* __restrict__ xptr,
                                           const int32_t* __restrict__ xcol, unsigned char* flags) {
  const int64_t t0 = xptr[k] + (W - 1), t1 = xptr[k + 1];
  for (int64_t t = t0; t < t1; t++) flags[xcol[t]] = 1;
  return static_cast<uint32_t>(t1 - t0);
}

// ---------------------------------------------------------------------------
// K_symbolic
// ---------------------------------------------------------------------------
struct SymArgs {
  const uint64_t* aptr;
  uint64_t abase;
  int64_t rows;
  int64_t K;
  int32_t n_cols;
  int32_t region_bytes;  // per-warp flag region (multiple of 16)
  const int64_t* xptr;
  const int32_t* xcol;
  const uint16_t* cslots;
  int32_t* cnt;
  int64_t* rflops;
  const int64_t* sym_heavy;
  int64_t heavy_deg;
  int64_t* num_heavy;
  int64_t heavy_flops;
  Ctl* ctl;
  const uint2* xdesc;  // W == -1: the fp32 step list (ab2_numeric5.cuh) instead of the plain CSR
  const uint2* xent;
  int32_t w5;
};

__device__ __forceinline__ int count_flags(uint32_t* f, int words, int start, int stride) {
  int c = 0;
  for (int i = start; i < words; i += stride) {
    uint32_t v = f[i];
    c += __popc(v);
    f[i] = 0;
  }
  return c;
}

// Lane-per-A-entry: each lane loads one whole column-only slot (2W bytes, one vector load)
// and sets its flags; 32 entries per warp step, two steps in flight.
template <class IdxT, int W>
__device__ __forceinline__ uint32_t sym_walk(const SymArgs& p, const IdxT* __restrict__ ac, uint32_t n, uint32_t first,
                                             uint32_t stride, unsigned char* flags) {
  const uint32_t K = static_cast<uint32_t>(p.K);
  uint32_t f = 0;
  for (uint32_t b = first; b < n; b += 2 * stride) {
    const uint32_t i0 = b, i1 = b + stride;
    uint32_t k0 = 0xffffffffu, k1 = 0xffffffffu;
    if (i0 < n) {
      const uint64_t k = static_cast<uint64_t>(ac[i0]);
      k0 = k < K ? static_cast<uint32_t>(k) : 0xffffffffu;
    }
    if (i1 < n) {
      const uint64_t k = static_cast<uint64_t>(ac[i1]);
      k1 = k < K ? static_cast<uint32_t>(k) : 0xffffffffu;
    }
    const CSlot<W> c0 = k0 != 0xffffffffu ? load_cslot<W>(p.cslots, k0) : empty_cslot<W>();
    const CSlot<W> c1 = k1 != 0xffffffffu ? load_cslot<W>(p.cslots, k1) : empty_cslot<W>();
    bool o0 = false, o1 = false;
    f += mark_cslot<W>(c0, flags, o0);
    f += mark_cslot<W>(c1, flags, o1);
    if (o0) f += mark_tail<W>(k0, p.xptr, p.xcol, flags);
    if (o1) f += mark_tail<W>(k1, p.xptr, p.xcol, flags);
  }
  return f;
}

// Lane-per-A-entry over the plain CSR of X (W == 0): each lane marks its X row's columns.  Used
// by the out-of-core sizing pass, whose operand carries no column slots (short X rows, e.g. the
// ogbn-products shape with ~1 entry per row, make 32-byte slots mostly padding).
template <class IdxT>
__device__ __forceinline__ uint32_t sym_walk_plain(const SymArgs& p, const IdxT* __restrict__ ac, uint32_t n,
                                                   uint32_t first, uint32_t stride, unsigned char* flags) {
  const uint64_t K = static_cast<uint64_t>(p.K);
  uint32_t f = 0;
  for (uint32_t i = first; i < n; i += stride) {
    const uint64_t k = static_cast<uint64_t>(ac[i]);
    if (k >= K) continue;
    const int64_t s = p.xptr[k], e = p.xptr[k + 1];
    f += static_cast<uint32_t>(e - s);
    for (int64_t t = s; t < e; t++) flags[p.xcol[t]] = 1;
  }
  return f;
}

// Lane-per-A-entry over the fp32 step list (W == -1; tight budgets keep no plain CSR): the X row's
// descriptor {slot start, nslot | len << 16}, then its len entries {col * 4, value bits}.
template <class IdxT>
__device__ __forceinline__ uint32_t sym_walk_steps(const SymArgs& p, const IdxT* __restrict__ ac, uint32_t n,
                                                   uint32_t first, uint32_t stride, unsigned char* flags) {
  const uint64_t K = static_cast<uint64_t>(p.K);
  uint32_t f = 0;
  for (uint32_t i = first; i < n; i += stride) {
    const uint64_t k = static_cast<uint64_t>(ac[i]);
    if (k >= K) continue;
    const uint2 d = __ldg(p.xdesc + k);
    const uint32_t len = d.y >> 16;
    const uint2* e = p.xent + static_cast<uint64_t>(d.x) * p.w5;
    f += len;
    for (uint32_t t = 0; t < len; t++) flags[__ldg(e + t).x >> 2] = 1;
  }
  return f;
}

template <class IdxT, int W>
__device__ __forceinline__ uint32_t sym_any(const SymArgs& p, const IdxT* __restrict__ ac, uint32_t n, uint32_t first,
                                            uint32_t stride, unsigned char* flags) {
  if constexpr (W == -1)
    return sym_walk_steps<IdxT>(p, ac, n, first, stride, flags);
  else if constexpr (W == 0)
    return sym_walk_plain<IdxT>(p, ac, n, first, stride, flags);
  else
    return sym_walk<IdxT, W>(p, ac, n, first, stride, flags);
}

template <class IdxT, int W>
__global__ void __launch_bounds__(256) k_symbolic(SymArgs p, const IdxT* __restrict__ acol) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int64_t s_red[32];
  __shared__ unsigned long long s_ticket;
  const int lane = lane_id(), warp = warp_id(), nw = blockDim.x >> 5;
  const int words = p.region_bytes / 4;
  for (int i = threadIdx.x; i < nw * words; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  __syncthreads();
  unsigned long long my_flops = 0;
  const unsigned long long n_heavy = p.ctl->n_sym_heavy;

  // Phase 1: heavy rows (A-degree > heavy_deg), one CTA per row, flags in warp 0's region.
  for (;;) {
    if (threadIdx.x == 0) s_ticket = atomicAdd(&p.ctl->heavy_next, 1ull);
    __syncthreads();
    const unsigned long long h = s_ticket;
    __syncthreads();
    if (h >= n_heavy) break;
    const int64_t r = p.sym_heavy[h];
    const uint64_t s = p.aptr[r] - p.abase, e = p.aptr[r + 1] - p.abase;
    int64_t f = sym_any<IdxT, W>(p, acol + s, static_cast<uint32_t>(e - s), threadIdx.x, blockDim.x, smem);
    __syncthreads();
    int64_t c = count_flags(reinterpret_cast<uint32_t*>(smem), words, threadIdx.x, blockDim.x);
    c = block_sum<int64_t>(c, s_red);
    f = block_sum<int64_t>(f, s_red);
    if (threadIdx.x == 0) {
      p.cnt[r] = static_cast<int32_t>(c);
      p.rflops[r] = f;
      my_flops += f;
      if (f > p.heavy_flops) p.num_heavy[atomicAdd(&p.ctl->n_num_heavy, 1ull)] = r;
    }
    __syncthreads();
  }

  // Phase 2: light rows, one warp per row.
  unsigned char* flags = smem + warp * p.region_bytes;
  for (;;) {
    unsigned long long r0 = 0;
    if (lane == 0) r0 = atomicAdd(&p.ctl->light_next, static_cast<unsigned long long>(kLightBatch));
    r0 = __shfl_sync(kFull, r0, 0);
    if (r0 >= static_cast<unsigned long long>(p.rows)) break;
    const int64_t r1 = min(static_cast<int64_t>(r0) + kLightBatch, p.rows);
    for (int64_t r = static_cast<int64_t>(r0); r < r1; r++) {
      const uint64_t s = p.aptr[r] - p.abase, e = p.aptr[r + 1] - p.abase;
      if (static_cast<int64_t>(e - s) > p.heavy_deg) continue;
      uint32_t f = sym_any<IdxT, W>(p, acol + s, static_cast<uint32_t>(e - s), lane, 32, flags);
      __syncwarp();
      int c = count_flags(reinterpret_cast<uint32_t*>(flags), words, lane, 32);
      c = warp_sum(c);
      f = warp_sum(f);
      if (lane == 0) {
        p.cnt[r] = c;
        p.rflops[r] = f;
        my_flops += f;
      }
      warp_append(lane == 0 && f > p.heavy_flops, r, p.num_heavy, &p.ctl->n_num_heavy);
      __syncwarp();
    }
  }
  if (lane == 0 && my_flops) atomicAdd(&p.ctl->flops, my_flops);
}

// ---------------------------------------------------------------------------
// Exclusive scan int32 counts -> int64 row_ptr (n+1 entries), total in ctl->nnz.
// ---------------------------------------------------------------------------
constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

static __global__ void __launch_bounds__(kScanThreads) k_scan_reduce(const int32_t* __restrict__ in,
                                                              int64_t n, int64_t* __restrict__ part) {
  __shared__ int64_t tmp[32];
  int64_t base = static_cast<int64_t>(blockIdx.x) * kScanTile;
  int64_t s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; i++) {
    int64_t j = base + static_cast<int64_t>(i) * kScanThreads + threadIdx.x;
    if (j < n) s += in[j];
  }
  s = block_sum<int64_t>(s, tmp);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

static __global__ void __launch_bounds__(1024) k_scan_part(int64_t* __restrict__ part, int64_t nb,
                                                    Ctl* __restrict__ ctl) {
  __shared__ int64_t tmp[32];
  int64_t carry = 0;
  for (int64_t b0 = 0; b0 < nb; b0 += blockDim.x) {
    int64_t j = b0 + threadIdx.x;
    int64_t v = j < nb ? part[j] : 0;
    int64_t tot;
    int64_t incl = block_incl_scan<int64_t>(v, tmp, &tot);
    if (j < nb) part[j] = carry + incl - v;
    carry += tot;
  }
  if (threadIdx.x == 0) ctl->nnz = static_cast<unsigned long long>(carry);
}

template <class OutT = int64_t>
static __global__ void __launch_bounds__(kScanThreads) k_scan_down(const int32_t* __restrict__ in, int64_t n,
                                                            const int64_t* __restrict__ part,
                                                            OutT* __restrict__ out) {
  __shared__ int64_t tmp[32];
  int64_t base = static_cast<int64_t>(blockIdx.x) * kScanTile;
  // each thread owns kScanItems consecutive items
  int64_t v[kScanItems];
  int64_t s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; i++) {
    int64_t j = base + static_cast<int64_t>(threadIdx.x) * kScanItems + i;
    v[i] = j < n ? in[j] : 0;
    s += v[i];
  }
  int64_t tot;
  int64_t incl = block_incl_scan<int64_t>(s, tmp, &tot);
  int64_t run = part[blockIdx.x] + incl - s;
#pragma unroll
  for (int i = 0; i < kScanItems; i++) {
    int64_t j = base + static_cast<int64_t>(threadIdx.x) * kScanItems + i;
    run += v[i];
    if (j < n) out[j + 1] = static_cast<OutT>(run);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = 0;
}

}  // namespace ab2
