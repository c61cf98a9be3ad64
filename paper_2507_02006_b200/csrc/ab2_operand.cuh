// ab2_operand.cuh -- the B200 layout of the right operand X (features).
//
// Gustavson row-wise SpGEMM gathers one X row per A entry (~0.7 G gathers
// of a 13 MB X at the Reddit shape).  Measured on B200 (tools/microbench/smem_accum.cu):
// per-lane pointer-chasing gathers of CSR rows are L1-wavefront bound at ~65 G rows/s.
// So X is re-laid out once per operand into fixed-width, aligned *slots*: row k occupies
// W consecutive entries at k*W, loaded by a W-lane group with one 8 B (fp32) / 16 B (fp64)
// load per lane -- no row-pointer lookup on the hot path, one cache line (or less) per row.
//
// Entry encoding (branch-free hot loop):
//   * column field low 16 bits = the accumulator column to add into.  Unused entries
//     point at the "trash" column n_cols (every accumulator has one spare column) with
//     value 1.0, so every lane always performs its read-modify-write; the trash column is
//     never emitted.
//   * rows longer than W keep W-1 entries inline; entry W-1 is an overflow marker:
//     col = kSlotOvf | (tail_len << 16) | trash, and the CSR offset of the tail (entries
//     W-1 .. len-1 of the row in the plain CSR copy) is kept in the value bits as
//     1.0f + offset ulps (fp32, so the marker's harmless trash add never multiplies by a
//     zero/denormal) or in the pad word (fp64).
//   * a dummy row K (all unused entries) absorbs out-of-range / padding A entries.
// A second, column-only slot array (16 x u16 = one 32 B sector per row) serves the
// symbolic row-nnz pass, where one lane handles one A entry: 16 wide so that overflow is
// negligible across 32 lanes (with 8-wide column slots ~99% of symbolic warp steps ran
// the serial tail path on the Reddit shape).
#pragma once
#include <cstdint>

namespace ab2 {

constexpr uint32_t kSlotOvf = 0x80000000u;    // overflow marker flag in the column field
constexpr uint32_t kSlotColMask = 0xffffu;    // accumulator column bits
constexpr uint32_t kOneBits = 0x3f800000u;    // 1.0f
constexpr uint16_t kCEmpty = 0xffff;          // column-only slot: unused
constexpr uint16_t kCOvf = 0xfffe;            // column-only slot: overflow marker
constexpr int kCSlotW = 16;                   // column-only slot width: 32 B = one L2 sector
constexpr int kMaxTail = 0x7fff;              // tail length field width (15 bits)

// fp32 slot entry: 8 bytes
struct __align__(8) SlotF {
  uint32_t col;
  float val;
};
// fp64 slot entry: 16 bytes
struct __align__(16) SlotD {
  uint32_t col;
  uint32_t pad;  // marker: CSR offset of the tail
  double val;
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

// CSR offset of an overflow marker's tail.
__device__ __forceinline__ uint32_t slot_tail_off(const SlotF& s) { return __float_as_uint(s.val) - kOneBits; }
__device__ __forceinline__ uint32_t slot_tail_off(const SlotD& s) { return s.pad; }

// Device view of a prepared operand (owned by XOperand in ab2_internal.h).
template <class V>
struct XView {
  int64_t K;        // rows of X (inner dimension); slot row K is the dummy row
  int32_t n_cols;   // columns of X (= columns of C); also the trash column index
  int32_t W;        // slot width
  const int64_t* ptr;   // plain CSR (K+1), rebased to 0
  const int32_t* col;   // plain CSR columns (sorted per row)
  const V* val;         // plain CSR values
  const typename SlotOf<V>::type* slots;  // (K+1)*W
  const uint16_t* cslots;                 // K*kCSlotW (column-only)
};

}  // namespace ab2
