// ab2_kernels.cuh -- sm_100a kernels of the B200 AIRES A·X SpGEMM.
//
// Replaces the reference's inner-product spgemm_block (spgemm.hpp:60-132):
//   K_classify  : rows whose A-degree exceeds the warp budget -> CTA-wide symbolic list
//   K_symbolic  : per-row nnz(C) = |U_k cols(X_k)| (byte flags in shared memory) and
//                 per-row MACs (spgemm.hpp:94-109 counts; :51 flops)
//   K_scan      : exclusive scan of the counts -> int64 C row_ptr (spgemm.hpp:107, :111)
//   K_numeric   : per-row dense shared-memory accumulator, emitted in ascending column
//                 order (spgemm.hpp:114-130; canonical, sparse.hpp:26-28)
//   K_fix       : rows whose fast-path marker disagreed with the symbolic count
//                 (all contributions were -0.0) are recomputed with explicit marks.
//
// Work distribution: heavy rows (by A-degree for symbolic, by MACs for numeric) are
// claimed first, one CTA per row; light rows then go one warp per row from a ticket
// counter in batches.  No shared-memory fp atomics other than the fp32 CAS add (ATOMS
// .CAST.SPIN, measured 11.7 SM-cycles per warp op on B200) and no MATCH.ANY (63).
//
// Accumulator marker: cells start at -0.0.  -0.0 + p == p for every p except p == -0.0,
// so a cell reads -0.0 afterwards only if every contribution was -0.0; such rows are
// detected by comparing the emitted count with the symbolic count and re-run by K_fix
// with explicit marks and a +0.0 start (dot_row_col's `sum = 0.0`, spgemm.hpp:27).
#pragma once
#include "ab2_common.cuh"
#include "ab2_operand.cuh"

namespace ab2 {

constexpr int kLightBatch = 4;   // light rows per ticket
constexpr int kUnrollSym = 4;    // A entries in flight per lane (symbolic)
constexpr int kUnrollNum = 4;    // group steps in flight (numeric)

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

// Marks the columns of X row k in `flags`; returns the row's MAC count.
template <int W>
__device__ __forceinline__ int64_t mark_cslot(const CSlot<W>& s, uint64_t k,
                                              const int64_t* __restrict__ xptr,
                                              const int32_t* __restrict__ xcol,
                                              unsigned char* flags) {
  int64_t f = 0;
#pragma unroll
  for (int e = 0; e < W; e++) {
    uint32_t c = s.at(e);
    if (c < kCOvf) {
      flags[c] = 1;
      f++;
    } else if (c == kCOvf) {  // only ever in entry W-1
      int64_t t0 = xptr[k] + (W - 1), t1 = xptr[k + 1];
      for (int64_t t = t0; t < t1; t++) flags[xcol[t]] = 1;
      f += t1 - t0;
    }
  }
  return f;
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

  // Phase 1: heavy rows, one CTA per row (flags in warp 0's region).
  for (;;) {
    if (threadIdx.x == 0) s_ticket = atomicAdd(&p.ctl->heavy_next, 1ull);
    __syncthreads();
    const unsigned long long h = s_ticket;
    __syncthreads();
    if (h >= n_heavy) break;
    const int64_t r = p.sym_heavy[h];
    const uint64_t s = p.aptr[r] - p.abase, e = p.aptr[r + 1] - p.abase;
    int64_t f = 0;
    for (uint64_t i = s + threadIdx.x; i < e; i += blockDim.x) {
      uint64_t k = static_cast<uint64_t>(acol[i]);
      if (k < static_cast<uint64_t>(p.K))
        f += mark_cslot<W>(load_cslot<W>(p.cslots, k), k, p.xptr, p.xcol, smem);
    }
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
      int64_t f = 0;
      for (uint64_t b = s; b < e; b += 32 * kUnrollSym) {
        uint64_t kk[kUnrollSym];
#pragma unroll
        for (int u = 0; u < kUnrollSym; u++) {
          uint64_t i = b + u * 32 + lane;
          kk[u] = i < e ? static_cast<uint64_t>(acol[i]) : ~0ull;
        }
        CSlot<W> cs[kUnrollSym];
#pragma unroll
        for (int u = 0; u < kUnrollSym; u++)
          cs[u] = kk[u] < static_cast<uint64_t>(p.K) ? load_cslot<W>(p.cslots, kk[u]) : empty_cslot<W>();
#pragma unroll
        for (int u = 0; u < kUnrollSym; u++) f += mark_cslot<W>(cs[u], kk[u], p.xptr, p.xcol, flags);
      }
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

static __global__ void __launch_bounds__(kScanThreads) k_scan_down(const int32_t* __restrict__ in, int64_t n,
                                                            const int64_t* __restrict__ part,
                                                            int64_t* __restrict__ out) {
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
    if (j < n) out[j + 1] = run;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = 0;
}

// ---------------------------------------------------------------------------
// K_numeric
// ---------------------------------------------------------------------------
template <class V, class IdxT>
struct NumArgs {
  const uint64_t* aptr;
  uint64_t abase;
  const IdxT* acol;
  const V* aval;
  int64_t rows;
  XView<V> x;
  int32_t region_elems;  // per-warp accumulator elements (>= n_cols)
  const int32_t* cnt;
  const int64_t* cptr;
  const int64_t* rflops;
  const int64_t* num_heavy;
  int64_t heavy_flops;
  IdxT* ccol;
  V* cval;
  int64_t* fix_rows;
  Ctl* ctl;
};

// Warp emission of a dense accumulator in ascending column order; resets the
// touched cells to the marker.  Returns the number of cells emitted.
template <class V, class IdxT>
__device__ __forceinline__ int64_t emit_warp(V* acc, int n_cols, int64_t out, IdxT* __restrict__ ccol,
                                             V* __restrict__ cval) {
  const int lane = lane_id();
  int64_t n = 0;
  for (int c0 = 0; c0 < n_cols; c0 += 32) {
    int c = c0 + lane;
    V v = c < n_cols ? acc[c] : Sentinel<V>::value();
    bool t = !Sentinel<V>::is(v);
    unsigned b = __ballot_sync(kFull, t);
    if (t) {
      int64_t pos = out + n + __popc(b & ((1u << lane) - 1));
      ccol[pos] = static_cast<IdxT>(c);
      cval[pos] = v;
      acc[c] = Sentinel<V>::value();
    }
    n += __popc(b);
  }
  return n;
}

template <class V>
__device__ __forceinline__ typename SlotOf<V>::type load_slot(const typename SlotOf<V>::type* __restrict__ slots,
                                                              uint64_t i) {
  using S = typename SlotOf<V>::type;
  S s;
  if constexpr (sizeof(S) == 8) {
    uint2 v = __ldg(reinterpret_cast<const uint2*>(slots + i));
    s.col = v.x;
    s.val = __uint_as_float(v.y);
  } else {
    uint4 v = __ldg(reinterpret_cast<const uint4*>(slots + i));
    s.col = v.x;
    s.pad = v.y;
    s.val = __longlong_as_double(static_cast<long long>((static_cast<unsigned long long>(v.w) << 32) | v.z));
  }
  return s;
}

template <class V>
__device__ __forceinline__ typename SlotOf<V>::type empty_slot() {
  typename SlotOf<V>::type s;
  s.col = kSlotEmpty;
  s.val = V(0);
  return s;
}

__device__ __forceinline__ void acc_add(float* p, float v) { atomicAdd(p, v); }

// fp32, order-free: every lane of every group applies its entry at once (CAS add).
template <class IdxT>
__device__ __forceinline__ void apply_f32(const SlotF& en, float a, const XView<float>& x, float* acc) {
  if (en.col < kSlotOvf) {
    acc_add(&acc[en.col], a * en.val);
  } else if (en.col != kSlotEmpty) {
    int64_t off = slot_ovf_offset(en);
    int64_t n = en.col & 0x7fffffffu;
    for (int64_t t = 0; t < n; t++) acc_add(&acc[x.col[off + t]], a * x.val[off + t]);
  }
}

// Group-strided product loop of one row for fp32.  `G` groups of W lanes; group g
// handles A entries b + g, b + g + G, ...
template <class IdxT, int W>
__device__ __forceinline__ void row_products_f32(const NumArgs<float, IdxT>& p, uint64_t s, uint64_t e,
                                                 int gid, int G, int ent, float* acc) {
  for (uint64_t b = s; b < e; b += static_cast<uint64_t>(G) * kUnrollNum) {
    uint64_t kk[kUnrollNum];
    float aa[kUnrollNum];
#pragma unroll
    for (int u = 0; u < kUnrollNum; u++) {
      uint64_t i = b + static_cast<uint64_t>(u) * G + gid;
      kk[u] = ~0ull;
      aa[u] = 0.f;
      if (i < e) {
        kk[u] = static_cast<uint64_t>(p.acol[i]);
        aa[u] = p.aval[i];
      }
    }
    SlotF en[kUnrollNum];
#pragma unroll
    for (int u = 0; u < kUnrollNum; u++)
      en[u] = kk[u] < static_cast<uint64_t>(p.x.K) ? load_slot<float>(p.x.slots, kk[u] * W + ent)
                                                  : empty_slot<float>();
#pragma unroll
    for (int u = 0; u < kUnrollNum; u++) apply_f32<IdxT>(en[u], aa[u], p.x, acc);
  }
}

template <class IdxT, int W>
__global__ void __launch_bounds__(256) k_numeric_f32(NumArgs<float, IdxT> p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float* accs = reinterpret_cast<float*>(smem_raw);
  __shared__ unsigned long long s_ticket;
  const int lane = lane_id(), warp = warp_id(), nw = blockDim.x >> 5;
  for (int i = threadIdx.x; i < nw * p.region_elems; i += blockDim.x) accs[i] = Sentinel<float>::value();
  __syncthreads();
  const unsigned long long n_heavy = p.ctl->n_num_heavy;

  // Phase 1: heavy rows, one CTA per row, groups across the CTA, shared accumulator.
  for (;;) {
    if (threadIdx.x == 0) s_ticket = atomicAdd(&p.ctl->num_heavy_next, 1ull);
    __syncthreads();
    const unsigned long long h = s_ticket;
    __syncthreads();
    if (h >= n_heavy) break;
    const int64_t r = p.num_heavy[h];
    const uint64_t s = p.aptr[r] - p.abase, e = p.aptr[r + 1] - p.abase;
    row_products_f32<IdxT, W>(p, s, e, threadIdx.x / W, blockDim.x / W, threadIdx.x % W, accs);
    __syncthreads();
    if (warp == 0) {
      int64_t n = emit_warp<float, IdxT>(accs, p.x.n_cols, p.cptr[r], p.ccol, p.cval);
      warp_append(lane == 0 && n != p.cnt[r], r, p.fix_rows, &p.ctl->n_fix);
    }
    __syncthreads();
  }

  // Phase 2: light rows, one warp per row.
  float* acc = accs + static_cast<int64_t>(warp) * p.region_elems;
  for (;;) {
    unsigned long long r0 = 0;
    if (lane == 0) r0 = atomicAdd(&p.ctl->num_light_next, static_cast<unsigned long long>(kLightBatch));
    r0 = __shfl_sync(kFull, r0, 0);
    if (r0 >= static_cast<unsigned long long>(p.rows)) break;
    const int64_t r1 = min(static_cast<int64_t>(r0) + kLightBatch, p.rows);
    for (int64_t r = static_cast<int64_t>(r0); r < r1; r++) {
      if (p.rflops[r] > p.heavy_flops) continue;
      const uint64_t s = p.aptr[r] - p.abase, e = p.aptr[r + 1] - p.abase;
      row_products_f32<IdxT, W>(p, s, e, lane / W, 32 / W, lane % W, acc);
      __syncwarp();
      int64_t n = emit_warp<float, IdxT>(acc, p.x.n_cols, p.cptr[r], p.ccol, p.cval);
      warp_append(lane == 0 && n != p.cnt[r], r, p.fix_rows, &p.ctl->n_fix);
      __syncwarp();
    }
  }
}

// fp64 exact: within a group step, groups apply their entries one group at a time
// (ascending A entry == ascending k), so every cell is summed in ascending k with one
// IEEE multiply and one IEEE add per term (no FMA): bit-identical to dot_row_col.
// Lanes whose column is outside [c_lo, c_hi) skip (column-owner split of heavy rows).
template <int W>
__device__ __forceinline__ void apply_f64_ordered(const SlotD& en, double a, const XView<double>& x,
                                                  double* acc, int c_lo, int c_hi) {
  if (en.col < kSlotOvf) {
    int c = static_cast<int>(en.col);
    if (c >= c_lo && c < c_hi) acc[c] = __dadd_rn(acc[c], __dmul_rn(a, en.val));
  } else if (en.col != kSlotEmpty) {
    int64_t off = slot_ovf_offset(en);
    int64_t n = en.col & 0x7fffffffu;
    for (int64_t t = 0; t < n; t++) {
      int c = x.col[off + t];
      if (c >= c_lo && c < c_hi) acc[c] = __dadd_rn(acc[c], __dmul_rn(a, x.val[off + t]));
    }
  }
}

template <class IdxT, int W>
__device__ __forceinline__ void row_products_f64(const NumArgs<double, IdxT>& p, uint64_t s, uint64_t e,
                                                 double* acc, int c_lo, int c_hi) {
  constexpr int G = 32 / W;
  const int lane = lane_id(), gid = lane / W, ent = lane % W;
  for (uint64_t b = s; b < e; b += static_cast<uint64_t>(G) * kUnrollNum) {
    uint64_t kk[kUnrollNum];
    double aa[kUnrollNum];
#pragma unroll
    for (int u = 0; u < kUnrollNum; u++) {
      uint64_t i = b + static_cast<uint64_t>(u) * G + gid;
      kk[u] = ~0ull;
      aa[u] = 0.0;
      if (i < e) {
        kk[u] = static_cast<uint64_t>(p.acol[i]);
        aa[u] = p.aval[i];
      }
    }
    SlotD en[kUnrollNum];
#pragma unroll
    for (int u = 0; u < kUnrollNum; u++)
      en[u] = kk[u] < static_cast<uint64_t>(p.x.K) ? load_slot<double>(p.x.slots, kk[u] * W + ent)
                                                  : empty_slot<double>();
#pragma unroll
    for (int u = 0; u < kUnrollNum; u++) {
#pragma unroll
      for (int g = 0; g < G; g++) {
        if (gid == g) apply_f64_ordered<W>(en[u], aa[u], p.x, acc, c_lo, c_hi);
        __syncwarp();
      }
    }
  }
}

template <class IdxT, int W>
__global__ void __launch_bounds__(256) k_numeric_f64(NumArgs<double, IdxT> p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* accs = reinterpret_cast<double*>(smem_raw);
  __shared__ unsigned long long s_ticket;
  __shared__ int64_t s_cnt[32];
  const int lane = lane_id(), warp = warp_id(), nw = blockDim.x >> 5;
  for (int i = threadIdx.x; i < nw * p.region_elems; i += blockDim.x) accs[i] = Sentinel<double>::value();
  __syncthreads();
  const unsigned long long n_heavy = p.ctl->n_num_heavy;
  const int n_cols = p.x.n_cols;

  // Phase 1: heavy rows.  Column-owner split: warp w owns a contiguous column range of
  // the shared accumulator and walks every A entry of the row in order, so each cell is
  // still accumulated in ascending k by exactly one warp.
  const int span = ((n_cols + nw - 1) / nw + 31) & ~31;
  const int c_lo = min(warp * span, n_cols), c_hi = min(c_lo + span, n_cols);
  for (;;) {
    if (threadIdx.x == 0) s_ticket = atomicAdd(&p.ctl->num_heavy_next, 1ull);
    __syncthreads();
    const unsigned long long h = s_ticket;
    __syncthreads();
    if (h >= n_heavy) break;
    const int64_t r = p.num_heavy[h];
    const uint64_t s = p.aptr[r] - p.abase, e = p.aptr[r + 1] - p.abase;
    if (c_lo < c_hi) row_products_f64<IdxT, W>(p, s, e, accs, c_lo, c_hi);
    __syncthreads();
    if (warp == 0) {
      int64_t n = emit_warp<double, IdxT>(accs, n_cols, p.cptr[r], p.ccol, p.cval);
      warp_append(lane == 0 && n != p.cnt[r], r, p.fix_rows, &p.ctl->n_fix);
    }
    __syncthreads();
  }
  (void)s_cnt;

  // Phase 2: light rows, one warp per row.
  double* acc = accs + static_cast<int64_t>(warp) * p.region_elems;
  for (;;) {
    unsigned long long r0 = 0;
    if (lane == 0) r0 = atomicAdd(&p.ctl->num_light_next, static_cast<unsigned long long>(kLightBatch));
    r0 = __shfl_sync(kFull, r0, 0);
    if (r0 >= static_cast<unsigned long long>(p.rows)) break;
    const int64_t r1 = min(static_cast<int64_t>(r0) + kLightBatch, p.rows);
    for (int64_t r = static_cast<int64_t>(r0); r < r1; r++) {
      if (p.rflops[r] > p.heavy_flops) continue;
      const uint64_t s = p.aptr[r] - p.abase, e = p.aptr[r + 1] - p.abase;
      row_products_f64<IdxT, W>(p, s, e, acc, 0, n_cols);
      __syncwarp();
      int64_t n = emit_warp<double, IdxT>(acc, n_cols, p.cptr[r], p.ccol, p.cval);
      warp_append(lane == 0 && n != p.cnt[r], r, p.fix_rows, &p.ctl->n_fix);
      __syncwarp();
    }
  }
}

// ---------------------------------------------------------------------------
// K_fix: rows whose marker count disagreed (all-(-0.0) cells).  One warp per row,
// explicit byte marks, +0.0 start, A entries applied one k at a time in ascending
// order from the plain CSR copy of X.  Rare; correctness path only.
// ---------------------------------------------------------------------------
template <class V, class IdxT>
__global__ void __launch_bounds__(32) k_fix_rows(NumArgs<V, IdxT> p, int64_t n_fix) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  V* acc = reinterpret_cast<V*>(smem_raw);
  unsigned char* mark = smem_raw + static_cast<size_t>(p.region_elems) * sizeof(V);
  const int lane = lane_id();
  const int n_cols = p.x.n_cols;
  for (int64_t q = blockIdx.x; q < n_fix; q += gridDim.x) {
    const int64_t r = p.fix_rows[q];
    for (int c = lane; c < n_cols; c += 32) {
      acc[c] = V(0);
      mark[c] = 0;
    }
    __syncwarp();
    const uint64_t s = p.aptr[r] - p.abase, e = p.aptr[r + 1] - p.abase;
    for (uint64_t i = s; i < e; i++) {
      uint64_t k = static_cast<uint64_t>(p.acol[i]);
      if (k >= static_cast<uint64_t>(p.x.K)) continue;
      V a = p.aval[i];
      for (int64_t t = p.x.ptr[k] + lane; t < p.x.ptr[k + 1]; t += 32) {
        int c = p.x.col[t];
        V prod;
        if constexpr (sizeof(V) == 8) {
          prod = __dmul_rn(a, p.x.val[t]);
          acc[c] = __dadd_rn(acc[c], prod);
        } else {
          prod = __fmul_rn(a, p.x.val[t]);
          acc[c] = __fadd_rn(acc[c], prod);
        }
        mark[c] = 1;
      }
      __syncwarp();
    }
    int64_t out = p.cptr[r], n = 0;
    for (int c0 = 0; c0 < n_cols; c0 += 32) {
      int c = c0 + lane;
      bool t = c < n_cols && mark[c];
      unsigned b = __ballot_sync(kFull, t);
      if (t) {
        int64_t pos = out + n + __popc(b & ((1u << lane) - 1));
        p.ccol[pos] = static_cast<IdxT>(c);
        p.cval[pos] = acc[c];
      }
      n += __popc(b);
    }
    __syncwarp();
  }
}

}  // namespace ab2
