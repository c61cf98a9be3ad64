// ab2_operand.cuh -- the B200 layout of the right operand X (features).
//
// Gustavson row-wise SpGEMM gathers one X row per A entry (667 M
// gathers of a 13 MB X at the Reddit shape).  Measured on B200
// (tools/microbench/smem_accum.cu): per-lane pointer-chasing gathers of CSR rows
// are L1-wavefront bound at ~65 G rows/s.  So X is re-laid out once per operand
// into fixed-width, aligned *slots*: row k occupies W consecutive entries at
// k*W, loaded by a W-lane group with one 8 B (fp32) / 16 B (fp64) load per lane
// -- no row-pointer lookup on the hot path, one cache line (or less) per row.
// Rows longer than W keep W-1 entries inline; the last entry is an overflow
// marker pointing at the tail of the row in the plain CSR copy.
// A second, column-only slot array (u16 per entry) serves the symbolic pass.
#pragma once
#include <cstdint>

namespace ab2 {

constexpr uint32_t kSlotEmpty = 0xffffffffu;  // entry unused
constexpr uint32_t kSlotOvf = 0x80000000u;    // col field of an overflow marker | count
constexpr uint16_t kCEmpty = 0xffff;          // column-only slot: unused
constexpr uint16_t kCOvf = 0xfffe;            // column-only slot: overflow marker

// fp32 slot entry: 8 bytes
struct __align__(8) SlotF {
  uint32_t col;  // column, kSlotEmpty, or kSlotOvf|count
  float val;     // value, or (bit-cast) CSR offset of the overflow tail
};
// fp64 slot entry: 16 bytes
struct __align__(16) SlotD {
  uint32_t col;
  uint32_t pad;
  double val;  // value, or (bit-cast int64) CSR offset of the overflow tail
};

template <class V>
struct SlotOf;
template <>
struct SlotOf<float> {
  using type = SlotF;
};
template <>
struct SlotOf<double> {
  using type = SlotD;
};

__device__ __forceinline__ int64_t slot_ovf_offset(const SlotF& s) {
  return static_cast<int64_t>(__float_as_uint(s.val));
}
__device__ __forceinline__ int64_t slot_ovf_offset(const SlotD& s) {
  return static_cast<int64_t>(__double_as_longlong(s.val));
}

// Device view of a prepared operand (owned by XOperand in ab2_internal.h).
template <class V>
struct XView {
  int64_t K;        // rows of X (inner dimension)
  int32_t n_cols;   // columns of X (= columns of C)
  int32_t W;        // slot width
  const int64_t* ptr;   // plain CSR (K+1), rebased to 0
  const int32_t* col;   // plain CSR columns (sorted per row)
  const V* val;         // plain CSR values
  const typename SlotOf<V>::type* slots;  // K*W
  const uint16_t* cslots;                 // K*W (column-only)
};

}  // namespace ab2
