// ab2_numeric.cuh -- the A·X product pass of the B200 SpGEMM (spgemm.hpp:60-132), sm_100a.
//
// Single pass over A: each row is accumulated once into a dense shared-memory accumulator,
// counted, and written once (ascending columns, canonical per sparse.hpp:26-28) into a
// bump-allocated staging area; K_place then streams the rows into their exact CSR offsets
// (row_ptr = exclusive scan of the counts, spgemm.hpp:107/:111-112).
//   Why not two passes: a symbolic pass re-walks every A entry and gathers X's column slots
//   (L1-wavefront bound, ~1.1 ms at the Reddit shape on B200), while this pass leaves HBM
//   mostly idle, so one extra streaming copy of C (~2 bytes moved per C byte at full HBM
//   bandwidth) is the cheaper way to the exact layout.
//   Why not a row-level decoupled look-back: with heavy-tailed row costs it serialises warps
//   behind slow rows (measured 10 s at the Reddit shape).
//
// Mapping (light rows, one warp per row):
//   * X rows live in W-entry slots (ab2_operand.cuh); a group of W lanes takes one A entry
//     (k, a) and each lane one slot entry, so a warp step covers G = 32/W A entries.
//   * A entries are read 32 at a time, coalesced, and handed to groups by shuffles.
//   * Unused slot entries and padding A entries hit the accumulator's trash column, so
//     the step is unpredicated: SHFL k, SHFL a, LDG slot, FMUL, LDS, FADD, STS.
//   * fp32: every group owns a private accumulator copy, so no two lanes of a warp step
//     ever touch the same shared word (smem CAS add measured 11.7 SM-cycles per warp op on
//     B200 vs 6.7 for a plain RMW).  Copies are summed when the row is counted.
//   * fp64-exact: one accumulator; the G groups of a step apply their entries one group at
//     a time, so each cell is summed in ascending k with one IEEE mul and one IEEE add per
//     term -- bit-identical to dot_row_col (spgemm.hpp:21-42).
// Heavy rows (A-degree > heavy_deg) are claimed first, one CTA per row: fp32 warps split
// the row's entries and the CTA sums all copies; fp64 warps split the columns (each warp
// walks every entry in order and redirects columns outside its range to the trash column).
//
// Marker: accumulator cells start at -0.0 (-0.0 + p == p unless p == -0.0).  Any product
// that is exactly zero sends the row through the explicit-mark path (start +0.0, byte
// marks), the reference's `sum = 0.0; if (hit)` semantics (spgemm.hpp:27-41, :58-59).
#pragma once
#include <type_traits>

#ifndef AB2_NUM_BATCH
#define AB2_NUM_BATCH 8
#endif
// resident CTAs per SM the register budget is sized for: 128 threads x 6 CTAs -> 80 registers
// for the fp32 16-entry-slot walk and the fp64 walks (two load buffers in flight), 64 otherwise
#ifndef AB2_NUM_MINB
#define AB2_NUM_MINB 8
#endif
#ifndef AB2_NUM_MINB_WIDE
#define AB2_NUM_MINB_WIDE 6
#endif
#ifndef AB2_NUM_MAXT
#define AB2_NUM_MAXT 128
#endif

#include "ab2_kernels.cuh"

namespace ab2 {


template <class V, class IdxT>
struct Num3Args {
  const uint64_t* aptr;
  uint64_t abase;
  const IdxT* acol;
  const V* aval;
  int64_t rows;
  XView<V> x;
  int32_t stride;      // accumulator elements per copy (>= n_cols + 1, multiple of 32)
  int32_t copies;      // accumulator copies per warp
  int32_t warp_bytes;  // shared bytes per warp: copies*stride*sizeof(V) + stride marks + chunk table
  int32_t pad0;          // rows with <= 32 terms: 1 register sort (short_row), 2 dense cells (<= 256 columns)
  const int64_t* heavy;  // heavy rows (A-degree > heavy_deg)
  int64_t heavy_deg;
  uint32_t* cnt;         // per-row nnz
  uint64_t* toff;        // per-row staging offset
  IdxT* tcol;            // staging area
  V* tval;
  uint64_t t_cap;
  const uint16_t* xlen;  // X row lengths (K+1, dummy row 0), for the MAC count
  V tiny;                // |a| threshold of the per-chunk zero-product check
  uint32_t stage_block;  // staging entries a warp reserves at a time (>= 8 * stride)
  uint32_t pad1;
  Ctl* ctl;
  const int64_t* cpos;  // direct mode: exact C row offsets (symbolic pass), else staging
  int64_t cbase;
};

// Per-warp chunk table in shared memory (32 entries of up to 16 bytes: {slot index k*W, a}).
using ChunkPair = uint4;

// Shared-memory read-modify-write at a 32-bit shared address.
__device__ __forceinline__ void smem_fma(uint32_t addr, float a, float x) {
  asm volatile(
      "{\n\t.reg .f32 t;\n\tld.shared.f32 t, [%0];\n\tfma.rn.f32 t, %1, %2, t;\n\tst.shared.f32 [%0], t;\n\t}" ::"r"(addr),
      "f"(a), "f"(x)
      : "memory");
}
// fp64 exact: one IEEE multiply, one IEEE add (no contraction).
__device__ __forceinline__ void smem_mul_add(uint32_t addr, double a, double x) {
  asm volatile(
      "{\n\t.reg .f64 t, p;\n\tmul.rn.f64 p, %1, %2;\n\tld.shared.f64 t, [%0];\n\tadd.rn.f64 t, t, p;\n\tst.shared.f64 [%0], t;\n\t}" ::"r"(addr),
      "d"(a), "d"(x)
      : "memory");
}

template <class V>
__device__ __forceinline__ void smem_acc(uint32_t addr, V a, V x) {
  if constexpr (sizeof(V) == 8)
    smem_mul_add(addr, a, x);
  else
    smem_fma(addr, a, x);
}

// ---- the group-strided walk over a contiguous range of A entries (W-lane slot groups) --------
// Entries [0, n) of ac/av in chunks of 32 (one coalesced load each); chunk c is handled iff
// c == chunk0 (mod chunk_stride), which lets a CTA's warps interleave over one heavy row.
// Columns outside [c_lo, c_hi) are skipped (the fp64 column-owner split).  The chunk's entries
// {k*W, a} go to a per-warp shared table once; each step reads its group's entry with one
// broadcast LDS.  Slots are loaded whole (entries past the row's length hold the trash column
// and are skipped without touching shared memory); MACs are counted from the real entries.
//
// Zero products (which need the explicit-mark path) are detected per chunk, not per step:
// a product can only round to zero if |a| * min|x| < 2^-148 (fp32) / 2^-1073 (fp64), or if
// X stores an exact zero (operand flag XZ: then every product is checked).
template <class V, class IdxT, int W, bool EXACT, bool RANGE, bool XZ>
__device__ __forceinline__ uint32_t walk_slots(const Num3Args<V, IdxT>& p, const IdxT* __restrict__ ac,
                                                  const V* __restrict__ av, uint32_t n, uint32_t chunk0,
                                                  uint32_t chunk_stride, V* acc, ChunkPair* tab, uint32_t c_lo,
                                                  uint32_t c_hi, bool& zero) {
  constexpr int G = 32 / W;
  constexpr int B = W < AB2_NUM_BATCH ? W : AB2_NUM_BATCH;  // group steps per batch (loads in flight)
  constexpr uint32_t VS = sizeof(V);
  const int lane = lane_id(), gid = lane / W, ent = lane % W;
  const int mlane = gid * W + (W - 1);  // the group's marker lane
  const uint32_t K = static_cast<uint32_t>(p.x.K);
  const uint32_t trash = static_cast<uint32_t>(p.x.n_cols);
  const int32_t* __restrict__ xcol = p.x.col;
  const V* __restrict__ xval = p.x.val;
  const V tiny = p.tiny;
  const uint32_t copy_s = static_cast<uint32_t>(__cvta_generic_to_shared(EXACT ? acc : acc + gid * p.stride));
  const uint32_t tab_s = static_cast<uint32_t>(__cvta_generic_to_shared(tab));
  uint32_t macs = 0;
  auto add = [&](uint32_t c, V a, V x) {
    if constexpr (XZ) {
      if constexpr (EXACT)
        zero |= __dmul_rn(a, x) == 0.0;
      else
        zero |= a * x == 0.f;
    }
    smem_acc<V>(copy_s + c * VS, a, x);
  };
  const uint32_t step = chunk_stride * 32;
  auto load_ka = [&](uint32_t bb, uint32_t& k, V& a) {
    const uint32_t i = bb + lane;
    k = K;  // dummy row: an all-trash slot
    a = V(1);
    if (i < n) {
      const uint64_t kk = static_cast<uint64_t>(ac[i]);
      k = kk < K ? static_cast<uint32_t>(kk) : K;
      a = av[i];
    }
  };
  // two chunks of (k, a) in flight ahead of the one being accumulated
  uint32_t k1, k2;
  V a1, a2;
  load_ka(chunk0 * 32, k1, a1);
  load_ka(chunk0 * 32 + step, k2, a2);
  for (uint32_t b = chunk0 * 32; b < n; b += step) {
    const uint32_t kw = k1 * W;
    const V a = a1;
    if (b + lane < n) zero |= !(fabs(a) >= tiny);  // zero, tiny, or NaN weight: take the explicit path
    k1 = k2;
    a1 = a2;
    load_ka(b + 2 * step, k2, a2);
    // one broadcast LDS per step (1 wavefront) instead of two SHFLs (~2.6 wavefronts measured)
    __syncwarp();
    if constexpr (sizeof(V) == 4)
      asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(tab_s + lane * 8u), "r"(kw), "r"(__float_as_uint(a))
                   : "memory");
    else
      asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(tab_s + lane * 16u), "r"(kw), "r"(0u),
                   "r"(__double2loint(a)), "r"(__double2hiint(a))
                   : "memory");
    __syncwarp();
    const uint32_t steps = (min(32u, n - b) + G - 1) / G;
#pragma unroll 1
    for (uint32_t u0 = 0; u0 < steps; u0 += B) {
      uint32_t col[B];
      V xv[B], aa[B];
      uint32_t any = 0;
#pragma unroll
      for (int u = 0; u < B; u++) {
        const int src = static_cast<int>(((u0 + u) * G + gid) & 31u);
        uint32_t skw;
        if constexpr (sizeof(V) == 4) {
          uint32_t ab;
          asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(skw), "=r"(ab) : "r"(tab_s + src * 8u) : "memory");
          aa[u] = __uint_as_float(ab);
        } else {
          uint32_t z, lo, hi;
          asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(skw), "=r"(z), "=r"(lo), "=r"(hi)
                       : "r"(tab_s + src * 16u)
                       : "memory");
          aa[u] = __hiloint2double(hi, lo);
        }
        if constexpr (sizeof(V) == 4) {
          const uint2 e = __ldg(reinterpret_cast<const uint2*>(p.x.slots) + (skw + ent));
          col[u] = e.x;
          xv[u] = __uint_as_float(e.y);
        } else {
          const uint4 e = __ldg(reinterpret_cast<const uint4*>(p.x.slots) + (skw + ent));
          col[u] = e.x;
          xv[u] = __hiloint2double(e.w, e.z);
          if (e.x & kSlotOvf) xv[u] = __longlong_as_double(static_cast<long long>(e.y));
        }
        if ((u0 + u) * G >= 32u) col[u] = trash;  // steps past the chunk (only when G does not divide 32)
        any |= col[u];
      }
      if (!__any_sync(kFull, (any & kSlotOvf) != 0)) {
        // fast path: no marker in the batch; trash entries touch nothing
#pragma unroll
        for (int u = 0; u < B; u++) {
          const bool real = col[u] != trash;
          macs += real;
          // (column-owner split: a column outside this warp's range is not touched at all, so no
          // two warps ever share a cell -- not even a trash cell)
          const uint32_t c = col[u];
          const bool mine = real && (!RANGE || (c >= c_lo && c < c_hi));
          if constexpr (EXACT) {
#pragma unroll
            for (int g = 0; g < G; g++) {
              if (gid == g && mine) add(c, aa[u], xv[u]);
              __syncwarp();
            }
          } else {
            if (mine) add(c, aa[u], xv[u]);
            __syncwarp();  // steps u and u+1 of one group may hit the same cell (different X rows)
          }
        }
        __syncwarp();
      } else {
#pragma unroll
        for (int u = 0; u < B; u++) {
          // marker lane: col = kSlotOvf | tail<<16 | trash; the tail offset rides in the value
          // bits (fp32: 1.0f + offset ulps) or the pad word (fp64, stashed in xv above)
          uint32_t moff;
          if constexpr (sizeof(V) == 4)
            moff = __float_as_uint(xv[u]) - kOneBits;
          else
            moff = static_cast<uint32_t>(__double_as_longlong(xv[u]));
          const uint32_t mc = __shfl_sync(kFull, col[u], mlane);
          const uint32_t mo = __shfl_sync(kFull, moff, mlane);
          const uint32_t tn = (mc & kSlotOvf) ? (mc >> 16) & kMaxTail : 0;
          const bool real = col[u] != trash && !(col[u] & kSlotOvf);
          macs += real;
          for (uint32_t t = ent; t < tn; t += W) macs++;
          auto mine = [&](uint32_t c) { return !RANGE || (c >= c_lo && c < c_hi); };
          if constexpr (EXACT) {
#pragma unroll
            for (int g = 0; g < G; g++) {
              if (gid == g) {
                if (real && mine(col[u] & kSlotColMask)) add(col[u] & kSlotColMask, aa[u], xv[u]);
                for (uint32_t t = ent; t < tn; t += W) {
                  const uint32_t c = static_cast<uint32_t>(xcol[mo + t]);
                  if (mine(c)) add(c, aa[u], xval[mo + t]);
                }
              }
              __syncwarp();
            }
          } else {
            if (real && mine(col[u] & kSlotColMask)) add(col[u] & kSlotColMask, aa[u], xv[u]);
            for (uint32_t t = ent; t < tn; t += W) {
              const uint32_t c = static_cast<uint32_t>(xcol[mo + t]);
              if (mine(c)) add(c, aa[u], xval[mo + t]);
            }
            __syncwarp();
          }
        }
      }
    }
  }
  return macs;
}

// ---- fp32 walk over 16-entry slots: two 16-lane groups, column-interleaved copies -----------
// Group g takes A entries 2u+g (step u) of a 32-entry chunk and adds the X row's slot entries into
// its copy of the accumulator; the two copies are interleaved per column (cell 2c + g), so group g
// only touches banks of parity g -- the two groups never conflict and a group's conflicts come
// from its own X row alone (simulated: 1.69 vs 2.03 wavefronts per RMW with copies side by side);
// the fold reads a column's two copies with one LDS.64.  The chunk's {k*16} and {a} go to two
// small tables laid out so that a group reads four steps' entries with one LDS.128, and the slot
// loads of the next eight steps are in flight while the current eight are added (two register
// buffers; the next chunk's table is written while the current one is consumed).
template <class IdxT, bool XZ>
__device__ __forceinline__ uint32_t walk_pair(const Num3Args<float, IdxT>& p, const IdxT* __restrict__ ac,
                                              const float* __restrict__ av, uint32_t n, uint32_t chunk0,
                                              uint32_t chunk_stride, float* acc, ChunkPair* tab, bool& zero) {
  const int lane = lane_id(), gid = lane >> 4, ent = lane & 15;
  const uint32_t K = static_cast<uint32_t>(p.x.K);
  const uint32_t trash = static_cast<uint32_t>(p.x.n_cols);
  const uint2* __restrict__ sl = reinterpret_cast<const uint2*>(p.x.slots) + ent;  // this lane's entry of a slot
  auto slot_at = [&](uint32_t kw) {  // sl + kw in one IMAD.WIDE.U32
    const uint2* q;
    asm("mad.wide.u32 %0, %1, 8, %2;" : "=l"(q) : "r"(kw), "l"(sl));
    return q;
  };
  const float tiny = p.tiny;
  const uint32_t copy_s = static_cast<uint32_t>(__cvta_generic_to_shared(acc)) + gid * 4u;
  // table buffer t: kw words at tk(t) + 4*pos, a words at tk(t) + 144 + 4*pos, pos(j) = (j & 1) * 20 + (j >> 1)
  const uint32_t tab_s = static_cast<uint32_t>(__cvta_generic_to_shared(tab));
  const uint32_t my_pos = (lane & 1) * 20u + (lane >> 1);
  const uint32_t grp_pos = gid * 20u;
  uint32_t macs = 0;
  const uint32_t step = chunk_stride * 32;
  uint64_t kr = K;  // raw (k, a) of the next chunk to stage
  float ar = 1.f;
  auto load_ka = [&](uint32_t bb) {
    const uint32_t i = bb + lane;
    kr = K;  // dummy row: an all-trash slot
    ar = 1.f;
    if (i < n) {
      kr = static_cast<uint64_t>(ac[i]);
      ar = av[i];
    }
  };
  auto stage = [&](uint32_t b, uint32_t t) {
    const uint32_t kw = (kr < K ? static_cast<uint32_t>(kr) : K) * 16u;
    if (b + lane < n) zero |= !(fabsf(ar) >= tiny);  // zero, tiny, or NaN weight: take the explicit path
    const uint32_t tk = tab_s + t * 288u + my_pos * 4u;
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(tk), "r"(kw) : "memory");
    asm volatile("st.shared.f32 [%0], %1;" ::"r"(tk + 144u), "f"(ar) : "memory");
  };
  // slot loads of steps 8h .. 8h+7 of the chunk in table t (steps past the chunk: the dummy row)
  auto issue = [&](uint32_t t, uint32_t h, uint2 (&e)[8]) {
#pragma unroll
    for (int q = 0; q < 2; q++) {
      uint32_t k0, k1, k2, k3;
      asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(k0), "=r"(k1), "=r"(k2), "=r"(k3)
                   : "r"(tab_s + t * 288u + (grp_pos + 8u * h + 4u * q) * 4u)
                   : "memory");
      e[4 * q + 0] = __ldg(slot_at(k0));
      e[4 * q + 1] = __ldg(slot_at(k1));
      e[4 * q + 2] = __ldg(slot_at(k2));
      e[4 * q + 3] = __ldg(slot_at(k3));
    }
  };
  auto consume = [&](uint32_t t, uint32_t h, const uint2 (&e)[8]) {
    float aa[8];
#pragma unroll
    for (int q = 0; q < 2; q++)
      asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                   : "=f"(aa[4 * q]), "=f"(aa[4 * q + 1]), "=f"(aa[4 * q + 2]), "=f"(aa[4 * q + 3])
                   : "r"(tab_s + t * 288u + 144u + (grp_pos + 8u * h + 4u * q) * 4u)
                   : "memory");
    uint32_t any = 0;
#pragma unroll
    for (int u = 0; u < 8; u++) any |= e[u].x;
    if (!__any_sync(kFull, (any & kSlotOvf) != 0u)) {
      // Steps u and u+1 of one group may hit the same cell (different X rows): a __syncwarp
      // between the steps orders one step's stores before the next step's loads for every lane
      // (racecheck-clean; the lanes of a step never share a cell).
#pragma unroll
      for (int u = 0; u < 8; u++) {
        const uint32_t c = e[u].x;
        const bool real = c != trash;
        if (real) {
          if constexpr (XZ) zero |= aa[u] * __uint_as_float(e[u].y) == 0.f;
          smem_fma(copy_s + (c << 3), aa[u], __uint_as_float(e[u].y));
        }
        macs += real;
        __syncwarp();
      }
      return;
    }
    // a row longer than 16: entry 15 is col = kSlotOvf | tail << 16 | trash with the tail's CSR
    // offset in the value bits (1.0f + offset ulps); the group adds the tail after the entry
#pragma unroll
    for (int u = 0; u < 8; u++) {
      const int ml = (gid << 4) | 15;
      const uint32_t mc = __shfl_sync(kFull, e[u].x, ml);
      const uint32_t mo = __shfl_sync(kFull, e[u].y - kOneBits, ml);
      const uint32_t tn = (mc & kSlotOvf) ? (mc >> 16) & kMaxTail : 0u;
      const uint32_t c = e[u].x;
      if (c != trash && !(c & kSlotOvf)) {
        smem_fma(copy_s + (c << 3), aa[u], __uint_as_float(e[u].y));
        if constexpr (XZ) zero |= aa[u] * __uint_as_float(e[u].y) == 0.f;
        macs++;
      }
      for (uint32_t t2 = ent; t2 < tn; t2 += 16) {
        const float x = p.x.val[mo + t2];
        smem_fma(copy_s + (static_cast<uint32_t>(p.x.col[mo + t2]) << 3), aa[u], x);
        if constexpr (XZ) zero |= aa[u] * x == 0.f;
        macs++;
      }
      __syncwarp();
    }
  };
  uint32_t b = chunk0 * 32;
  if (b >= n) return 0;
  load_ka(b);
  stage(b, 0);
  load_ka(b + step);
  uint2 e0[8], e1[8];
  __syncwarp();
  issue(0, 0, e0);
  for (uint32_t t = 0;; t ^= 1u) {
    const bool two = n - b > 16;  // the chunk has steps 8..15
    if (two) issue(t, 1, e1);
    consume(t, 0, e0);
    const uint32_t bn = b + step;
    if (bn < n) {
      stage(bn, t ^ 1u);
      load_ka(bn + step);
      __syncwarp();
      issue(t ^ 1u, 0, e0);
    }
    if (two) consume(t, 1, e1);
    b = bn;
    if (b >= n) break;
    __syncwarp();  // table t is free again
  }
  return macs;
}

// Explicit-mark slow path (rows with a zero product): one k at a time in ascending order,
// +0.0 start, byte marks; leaves copy 0 holding values for marked cells and the marker
// everywhere else (other copies reset), so the common fold / emit path applies.
template <class V, class IdxT, int CS = 1>
__device__ void slow_row(const Num3Args<V, IdxT>& p, const IdxT* __restrict__ ac, const V* __restrict__ av,
                         uint32_t n, V* acc, unsigned char* mark) {
  // (CS: cell stride of copy 0 -- 2 for the column-interleaved copies of walk_pair)
  const int lane = lane_id();
  const int n_cols = p.x.n_cols;
  for (int c = lane; c < p.stride * p.copies; c += 32) acc[c] = Sentinel<V>::value();
  for (int c = lane; c < p.stride; c += 32) mark[c] = 0;
  __syncwarp();
  for (int c = lane; c < n_cols; c += 32) acc[c * CS] = V(0);
  __syncwarp();
  for (uint32_t i = 0; i < n; i++) {
    const uint64_t k = static_cast<uint64_t>(ac[i]);
    if (k >= static_cast<uint64_t>(p.x.K)) continue;
    const V a = av[i];
    for (int64_t t = p.x.ptr[k] + lane; t < p.x.ptr[k + 1]; t += 32) {
      const int c = p.x.col[t];
      if constexpr (sizeof(V) == 8)
        acc[c * CS] = __dadd_rn(acc[c * CS], __dmul_rn(a, p.x.val[t]));
      else
        acc[c * CS] = __fadd_rn(acc[c * CS], __fmul_rn(a, p.x.val[t]));
      mark[c] = 1;
    }
    __syncwarp();
  }
  for (int c = lane; c < n_cols; c += 32)
    if (!mark[c]) acc[c * CS] = Sentinel<V>::value();
  __syncwarp();
}

// Folds the copies into copy 0 (resetting the others and the trash column) and returns
// the row nnz.
template <class V>
__device__ __forceinline__ uint32_t fold_count(V* acc, int stride, int copies, int n_cols) {
  const int lane = lane_id();
  uint32_t cnt = 0;
  for (int c0 = 0; c0 < stride; c0 += 32) {
    const int c = c0 + lane;
    V v = acc[c];
    for (int g = 1; g < copies; g++) {
      v += acc[g * stride + c];  // -0.0 is the identity for every operand but +0.0 (stays +0.0)
      acc[g * stride + c] = Sentinel<V>::value();
    }
    if (c >= n_cols) v = Sentinel<V>::value();  // trash column / padding
    acc[c] = v;
    cnt += __popc(__ballot_sync(kFull, !Sentinel<V>::is(v)));
  }
  __syncwarp();
  return cnt;
}

// Writes copy 0 (ascending columns) to ccol/cval and resets it.
template <class V, class IdxT>
__device__ __forceinline__ void emit_copy0(V* acc, int n_cols, IdxT* __restrict__ ccol, V* __restrict__ cval) {
  const int lane = lane_id();
  uint32_t n = 0;
  for (int c0 = 0; c0 < n_cols; c0 += 32) {
    const int c = c0 + lane;
    const V v = c < n_cols ? acc[c] : Sentinel<V>::value();
    const bool t = !Sentinel<V>::is(v);
    const unsigned b = __ballot_sync(kFull, t);
    if (t) {
      const uint32_t pos = n + __popc(b & ((1u << lane) - 1));
      ccol[pos] = static_cast<IdxT>(c);
      cval[pos] = v;
      acc[c] = Sentinel<V>::value();
    }
    n += __popc(b);
  }
  __syncwarp();  // the next row's accumulation reads these cells from other lanes
}

// Warp-level bump allocation in the staging area.
// Each reservation wastes less than one row (< stride entries) out of >= 8*stride, so the
// host sizes the staging area as bound * 8/7 + one block per warp; a reservation past the
// end sets ctl->bad_row and the row is dropped (reported as capacity_exceeded).
struct StageCursor {
  unsigned long long cur = 0, end = 0;
  __device__ __forceinline__ unsigned long long take(uint32_t cnt, Ctl* ctl, uint32_t block) {
    if (cur + cnt > end) {
      const unsigned long long want = cnt > block ? cnt : block;
      unsigned long long base = 0;
      if (lane_id() == 0) base = atomicAdd(&ctl->n_fix, want);  // n_fix doubles as the stage counter
      base = __shfl_sync(kFull, base, 0);
      cur = base;
      end = base + want;
    }
    const unsigned long long o = cur;
    cur += cnt;
    return o;
  }
  // room for up to `most` entries at the cursor (a new block if needed); commit() keeps `cnt`
  __device__ __forceinline__ unsigned long long reserve(uint32_t most, Ctl* ctl, uint32_t block) {
    const unsigned long long o = take(most, ctl, block);
    cur = o;
    return o;
  }
  __device__ __forceinline__ void commit(uint32_t cnt) { cur += cnt; }
};

// Output offset of row r: the exact CSR position when the row counts are known in advance
// (out-of-core tiles, cpos = C row_ptr from the symbolic pass; a count that disagrees flags
// ctl->bad_row = 2), else a bump allocation in the staging area.
template <class P>
__device__ __forceinline__ unsigned long long out_offset(const P& p, int64_t r, uint32_t cnt, StageCursor& stage) {
  if (p.cpos != nullptr) {
    const int64_t o = p.cpos[r] - p.cbase;
    if (p.cpos[r + 1] - p.cpos[r] != static_cast<int64_t>(cnt)) {
      if (lane_id() == 0) atomicMax(&p.ctl->bad_row, 2ull);
      return ~0ull;
    }
    return static_cast<unsigned long long>(o);
  }
  return stage.take(cnt, p.ctl, p.stage_block);
}

// Fold + count + emit in one pass over the accumulator: the copies are summed into the output
// cells (all copies reset on the way), the row's entries are written in ascending column order,
// and the count comes out at the end.  The position is fixed before the count is known: the
// exact CSR offset in direct mode (a count that disagrees flags ctl->bad_row = 2), else room for
// a full row (n_cols entries) at the warp's staging cursor, of which the row keeps its count.
// Writes past the capacity are dropped and flag ctl->bad_row = 1.  Returns the count.
template <class V, int CS, class P>
__device__ __forceinline__ uint32_t fold_emit(const P& p, V* acc, int copies, int64_t r, StageCursor& stage,
                                              unsigned long long& off) {
  // CS = 2: two column-interleaved fp32 copies (cell 2c + g), read and reset with one LDS.64 /
  // STS.64 per column; CS = 1: `copies` copies of `stride` cells each
  const int lane = lane_id();
  const int n_cols = p.x.n_cols, stride = p.stride;
  unsigned long long cap;
  if (p.cpos != nullptr) {
    off = static_cast<unsigned long long>(p.cpos[r] - p.cbase);
    cap = static_cast<unsigned long long>(p.cpos[r + 1] - p.cpos[r]);
  } else {
    off = stage.reserve(static_cast<uint32_t>(n_cols), p.ctl, p.stage_block);
    cap = static_cast<unsigned long long>(n_cols);
  }
  const bool ok = off <= p.t_cap && off + cap <= p.t_cap;
  uint32_t cnt = 0;
  for (int c0 = 0; c0 < stride; c0 += 32) {
    const int c = c0 + lane;
    V v;
    if constexpr (CS == 2) {
      const uint32_t a2 = static_cast<uint32_t>(__cvta_generic_to_shared(acc + 2 * c));
      float x0, x1;
      asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(x0), "=f"(x1) : "r"(a2) : "memory");
      const uint32_t s = 0x80000000u;
      asm volatile("st.shared.v2.u32 [%0], {%1, %1};" ::"r"(a2), "r"(s) : "memory");
      v = x0 + x1;  // -0.0 is the identity for every operand but +0.0 (stays +0.0)
    } else {
      v = acc[c];
      for (int g = 1; g < copies; g++) {
        v += acc[g * stride + c];
        acc[g * stride + c] = Sentinel<V>::value();
      }
      acc[c] = Sentinel<V>::value();
    }
    if (c >= n_cols) v = Sentinel<V>::value();  // trash column / padding
    const bool t = !Sentinel<V>::is(v);
    const unsigned b = __ballot_sync(kFull, t);
    const uint32_t pos = cnt + __popc(b & ((1u << lane) - 1));
    if (t && ok && pos < cap) {
      p.tcol[off + pos] = static_cast<decltype(+p.tcol[0])>(c);
      p.tval[off + pos] = v;
    }
    cnt += __popc(b);
  }
  __syncwarp();  // the next row's accumulation reads these cells from other lanes
  if (p.cpos != nullptr) {
    if (cnt != cap && lane == 0) atomicMax(&p.ctl->bad_row, 2ull);
  } else {
    stage.commit(cnt);
  }
  if (!ok && lane == 0) atomicMax(&p.ctl->bad_row, 1ull);
  return cnt;
}

// Rows whose products fit one warp (<= 32 terms; degree <= 32): the terms are formed one per lane,
// sorted by (column, order of arrival) with a bitonic network over shuffles, and each column's terms
// are summed left to right from +0.0 -- dot_row_col's arithmetic (spgemm.hpp:21-42), so fp64 stays
// bit-exact, and every column with a term is kept (structural zeros included).  No shared-memory
// accumulator, no fold: for short rows (the ogbn-products shape averages ~26 terms per row) the
// copies' fold was a third of the kernel.  Returns false (nothing done) when the row has more terms.
template <class V>
__device__ __forceinline__ V mul_rn(V a, V b) {
  if constexpr (sizeof(V) == 8)
    return __dmul_rn(a, b);
  else
    return __fmul_rn(a, b);
}
template <class V>
__device__ __forceinline__ V add_rn(V a, V b) {
  if constexpr (sizeof(V) == 8)
    return __dadd_rn(a, b);
  else
    return __fadd_rn(a, b);
}

//
// Narrow outputs (<= 256 columns, e.g. the ogbn-products features): instead of the 32-key sort, lanes
// holding the same column are grouped with match.any, each group's lowest lane sums the group's
// terms in lane (= arrival) order and writes the sum into the warp's accumulator cell, the touched
// columns are collected as bitmaps with redux.or, and the row is emitted in column order from the
// bitmaps (the cells are reset to the sentinel as they are read).  Same sums, same order, same
// structural zeros as the sorted form.
template <class V, class IdxT, int CS = 1>
__device__ __forceinline__ bool short_row(const Num3Args<V, IdxT>& p, const IdxT* __restrict__ ac,
                                          const V* __restrict__ av, uint32_t n, int64_t r, StageCursor& stage,
                                          unsigned long long& my_nnz, unsigned long long& my_macs,
                                          V* acc = nullptr) {
  const int lane = lane_id();
  const uint64_t K = static_cast<uint64_t>(p.x.K);
  int64_t xs = 0;
  uint32_t len = 0;
  V a = V(0);
  if (static_cast<uint32_t>(lane) < n) {
    const uint64_t k = static_cast<uint64_t>(ac[lane]);
    a = av[lane];
    if (k < K) {
      xs = p.x.ptr[k];
      len = static_cast<uint32_t>(p.x.ptr[k + 1] - xs);
    }
  }
  const uint32_t incl = warp_incl_scan(len);
  const uint32_t T = __shfl_sync(kFull, incl, 31);
  if (T > 32) return false;
  const uint32_t excl = incl - len;
  // owner of term t = lane: the last entry j with excl_j <= t (it has len_j > 0 when t < T)
  const uint32_t t = static_cast<uint32_t>(lane);
  int j = 0;
#pragma unroll
  for (int step = 16; step >= 1; step >>= 1) {
    const int cand = j + step;
    const uint32_t ec = __shfl_sync(kFull, excl, cand & 31);
    if (cand < 32 && ec <= t) j = cand;
  }
  const int64_t xs_j = __shfl_sync(kFull, xs, j);
  const uint32_t ex_j = __shfl_sync(kFull, excl, j);
  const V a_j = __shfl_sync(kFull, a, j);
  uint32_t key = 0xffffffffu;
  V v = V(0);
  if (t < T) {
    const int64_t q = xs_j + static_cast<int64_t>(t - ex_j);
    key = (static_cast<uint32_t>(p.x.col[q]) << 5) | t;
    v = mul_rn<V>(a_j, p.x.val[q]);
  }
  if (acc != nullptr) {  // narrow output: group by column, dense cells, bitmap emission
    const bool real = t < T;
    const uint32_t col = key >> 5;
    const unsigned grp = __match_any_sync(kFull, real ? col : 0xffffffffu);
    const bool lead = real && lane == __ffs(grp) - 1;
    V sum = add_rn<V>(V(0), v);  // sum = 0.0; sum += term, then the group's later terms in order
    unsigned rest = lead ? grp & (grp - 1) : 0u;
    while (__any_sync(kFull, rest != 0)) {
      const V ov = __shfl_sync(kFull, v, rest ? __ffs(rest) - 1 : lane);
      if (rest) {
        sum = add_rn<V>(sum, ov);
        rest &= rest - 1;
      }
    }
    if (lead) acc[CS * col] = sum;
    const int nw = (p.x.n_cols + 31) >> 5;  // <= 8
    unsigned bits[8];
    uint32_t cnt = 0;
#pragma unroll
    for (int w = 0; w < 8; w++) {
      bits[w] = 0;
      if (w < nw) bits[w] = __reduce_or_sync(kFull, lead && (col >> 5) == static_cast<uint32_t>(w) ? 1u << (col & 31) : 0u);
      cnt += __popc(bits[w]);
    }
    const unsigned long long off = out_offset(p, r, cnt, stage);
    __syncwarp();
    const bool fits = off <= p.t_cap && off + cnt <= p.t_cap;
    uint32_t base = 0;
#pragma unroll
    for (int w = 0; w < 8; w++) {
      if ((bits[w] >> lane) & 1u) {
        const uint32_t c = 32 * w + lane;
        if (fits) {
          const unsigned long long pos = off + base + __popc(bits[w] & ((1u << lane) - 1));
          p.tcol[pos] = static_cast<IdxT>(c);
          p.tval[pos] = acc[CS * c];
        }
        acc[CS * c] = Sentinel<V>::value();
      }
      base += __popc(bits[w]);
    }
    __syncwarp();
    if (!fits && lane == 0) atomicMax(&p.ctl->bad_row, 1ull);
    if (lane == 0) {
      p.cnt[r] = cnt;
      p.toff[r] = off;
      my_nnz += cnt;
      my_macs += T;
    }
    return true;
  }
  // bitonic sort of the 32 (key, value) pairs, ascending
#pragma unroll
  for (int kk = 2; kk <= 32; kk <<= 1) {
#pragma unroll
    for (int jj = kk >> 1; jj > 0; jj >>= 1) {
      const uint32_t ok = __shfl_xor_sync(kFull, key, jj);
      const V ov = __shfl_xor_sync(kFull, v, jj);
      const bool keep_min = ((lane & kk) == 0) == ((lane & jj) == 0);
      if (keep_min ? ok < key : ok > key) {
        key = ok;
        v = ov;
      }
    }
  }
  const bool real = key != 0xffffffffu;
  const uint32_t col = key >> 5;
  const uint32_t pcol = __shfl_up_sync(kFull, col, 1);
  const bool head = real && (lane == 0 || pcol != col);
  V sum = add_rn<V>(V(0), v);  // sum = 0.0; sum += term (a -0.0 term gives +0.0, as in the reference)
  for (int d = 1; d < 32; d++) {
    const uint32_t ncol = __shfl_down_sync(kFull, col, d);
    const V nv = __shfl_down_sync(kFull, v, d);
    const bool cont = head && lane + d < 32 && ncol == col;
    if (!__any_sync(kFull, cont)) break;
    if (cont) sum = add_rn<V>(sum, nv);
  }
  const unsigned hm = __ballot_sync(kFull, head);
  const uint32_t cnt = __popc(hm);
  const unsigned long long off = out_offset(p, r, cnt, stage);
  if (off <= p.t_cap && off + cnt <= p.t_cap) {
    if (head) {
      const unsigned long long pos = off + __popc(hm & ((1u << lane) - 1));
      p.tcol[pos] = static_cast<IdxT>(col);
      p.tval[pos] = sum;
    }
  } else if (lane == 0) {
    atomicMax(&p.ctl->bad_row, 1ull);
  }
  if (lane == 0) {
    p.cnt[r] = cnt;
    p.toff[r] = off;
    my_nnz += cnt;
    my_macs += T;
  }
  return true;
}

// fp32 over 16-entry slots: walk_pair (two column-interleaved copies); otherwise W-lane groups.
template <class V, class IdxT, int W>
constexpr bool kPairWalk = sizeof(V) == 4 && W == 16;

template <class V, class IdxT, int W, bool XZ>
__device__ __forceinline__ uint32_t walk(const Num3Args<V, IdxT>& p, const IdxT* __restrict__ ac,
                                         const V* __restrict__ av, uint32_t n, uint32_t chunk0, uint32_t chunk_stride,
                                         V* acc, ChunkPair* tab, bool& zero) {
  if constexpr (kPairWalk<V, IdxT, W>)
    return walk_pair<IdxT, XZ>(p, ac, av, n, chunk0, chunk_stride, acc, tab, zero);
  else
    return walk_slots<V, IdxT, W, sizeof(V) == 8, false, XZ>(p, ac, av, n, chunk0, chunk_stride, acc, tab, 0, 0, zero);
}

template <class V, class IdxT, int W, bool XZ>
__global__ void __launch_bounds__(AB2_NUM_MAXT, (sizeof(V) == 8 || W == 16) ? AB2_NUM_MINB_WIDE : AB2_NUM_MINB)
    k_numeric3(Num3Args<V, IdxT> p) {
  constexpr bool EXACT = sizeof(V) == 8;
  constexpr int CS = kPairWalk<V, IdxT, W> ? 2 : 1;  // cell stride of a warp's copies (walk_pair)
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ unsigned long long s_ticket;
  __shared__ int s_zero;
  const int lane = lane_id(), warp = warp_id(), nw = blockDim.x >> 5;
  const int n_cols = p.x.n_cols;
  const int acc_elems = p.stride * p.copies;
  auto warp_acc = [&](int w) { return reinterpret_cast<V*>(smem_raw + static_cast<size_t>(w) * p.warp_bytes); };
  auto warp_mark = [&](int w) {
    return smem_raw + static_cast<size_t>(w) * p.warp_bytes + static_cast<size_t>(acc_elems) * sizeof(V);
  };
  auto warp_tab = [&](int w) {
    return reinterpret_cast<ChunkPair*>(smem_raw + static_cast<size_t>(w) * p.warp_bytes +
                                           static_cast<size_t>(acc_elems) * sizeof(V) + p.stride);
  };
  for (int w = 0; w < nw; w++)
    for (int i = threadIdx.x; i < acc_elems; i += blockDim.x) warp_acc(w)[i] = Sentinel<V>::value();
  __syncthreads();
  StageCursor stage;
  unsigned long long my_nnz = 0, my_macs = 0;
  const unsigned long long n_heavy = p.ctl->n_sym_heavy;

  // ---- Phase 1: heavy rows first (the long tail would otherwise finish last) ----
  // fp64-exact: one warp per heavy row.  Each cell's terms must be added in ascending k, so a CTA
  // could only split a row's columns -- every warp then walks (loads and steps over) every entry of
  // the row; at cfg2 that replication made the pass 7.5 ms instead of 5.1 ms.
  if constexpr (EXACT) {
    V* hacc = warp_acc(warp);
    for (;;) {
      unsigned long long h = 0;
      if (lane == 0) h = atomicAdd(&p.ctl->heavy_next, 1ull);
      h = __shfl_sync(kFull, h, 0);
      if (h >= n_heavy) break;
      const int64_t r = p.heavy[h];
      const uint64_t s = p.aptr[r] - p.abase, e = p.aptr[r + 1] - p.abase;
      const uint32_t n = static_cast<uint32_t>(e - s);
      bool zero = false;
      my_macs += walk<V, IdxT, W, XZ>(p, p.acol + s, p.aval + s, n, 0, 1, hacc, warp_tab(warp), zero);
      if (__any_sync(kFull, zero)) slow_row<V, IdxT, CS>(p, p.acol + s, p.aval + s, n, hacc, warp_mark(warp));
      unsigned long long off;
      const uint32_t cnt = fold_emit<V, CS>(p, hacc, 1, r, stage, off);
      if (lane == 0) {
        p.cnt[r] = cnt;
        p.toff[r] = off;
        my_nnz += cnt;
      }
    }
  }
  // fp32: one CTA per heavy row, the row's entries split over the warps (each its own copies)
  for (; !EXACT;) {
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
    const V* av = p.aval + s;
    bool zero = false;
    my_macs += walk<V, IdxT, W, XZ>(p, ac, av, n, warp, nw, warp_acc(warp), warp_tab(warp), zero);
    if (zero) s_zero = 1;
    __syncthreads();
    if (s_zero) {
      if (warp == 0) slow_row<V, IdxT, CS>(p, ac, av, n, warp_acc(0), warp_mark(0));
      if (!EXACT && warp != 0)
        for (int i = lane; i < acc_elems; i += 32) warp_acc(warp)[i] = Sentinel<V>::value();
    } else if constexpr (!EXACT) {
      // CTA fold: every warp's copies into warp 0's copy 0
      for (int c = threadIdx.x; c < p.stride; c += blockDim.x) {
        V v = Sentinel<V>::value();
        for (int w = 0; w < nw; w++)
          for (int g = 0; g < p.copies; g++) {
            V* q = warp_acc(w) + (CS == 2 ? 2 * c + g : g * p.stride + c);
            v += *q;
            *q = Sentinel<V>::value();
          }
        warp_acc(0)[CS * c] = v;
      }
    }
    __syncthreads();
    if (warp == 0) {
      unsigned long long off;
      const uint32_t cnt = fold_emit<V, CS>(p, warp_acc(0), CS, r, stage, off);
      if (lane == 0) {
        p.cnt[r] = cnt;
        p.toff[r] = off;
        my_nnz += cnt;
      }
    }
    __syncthreads();
  }

  // ---- Phase 2: light rows, one warp per row ----
  V* acc = warp_acc(warp);
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
      const V* av = p.aval + s;
      if (p.pad0 && n <= 32 &&
          short_row<V, IdxT, CS>(p, ac, av, n, r, stage, my_nnz, my_macs, p.pad0 == 2 ? acc : nullptr))
        continue;
      bool zero = false;
      my_macs += walk<V, IdxT, W, XZ>(p, ac, av, n, 0, 1, acc, warp_tab(warp), zero);
      if (__any_sync(kFull, zero)) slow_row<V, IdxT, CS>(p, ac, av, n, acc, warp_mark(warp));
      unsigned long long off;
      const uint32_t cnt = fold_emit<V, CS>(p, acc, EXACT ? 1 : p.copies, r, stage, off);
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

// K_place: staging -> exact CSR offsets.  One warp per row, 16-byte vector copies when the
// source and destination share alignment.
template <class V, class IdxT>
__global__ void __launch_bounds__(256) k_place(const uint32_t* __restrict__ cnt, const uint64_t* __restrict__ toff,
                                               const int64_t* __restrict__ cptr, const IdxT* __restrict__ tcol,
                                               const V* __restrict__ tval, int64_t rows, IdxT* __restrict__ ccol,
                                               V* __restrict__ cval) {
  const int lane = lane_id();
  const int64_t wid = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r = wid; r < rows; r += nwarps) {
    const uint32_t n = cnt[r];
    const uint64_t src = toff[r];
    const int64_t dst = cptr[r];
    for (uint32_t i = lane; i < n; i += 32) {
      ccol[dst + i] = tcol[src + i];
      cval[dst + i] = tval[src + i];
    }
  }
}

}  // namespace ab2
