// ab2_host.cpp -- host-side parts of the boundary that need no device.
//
// aires_b200_checksum: the reference's C checksum (serialize.hpp:22-59), FNV-1a 64 over the
// canonical little-endian stream n_rows, n_cols, nnz, row_ptr, col_idx (as u64) and values (as
// f64 bit patterns).  It is byte-serial by definition (one dependent multiply per byte), so it runs
// on the host and never inside a timed region; narrow widths are widened exactly as the reference's
// u64/f64 containers would hold them.
//
// A zero byte leaves FNV-1a's xor step unchanged (s ^= 0), so a run of k zero bytes is one multiply
// by P^k.  Column indices and row offsets are small integers (high bytes zero) and fp32-widened
// values have zero low bytes, so the dependent chain is 3-6 multiplies per word instead of 8; the
// result is bit-identical to the byte loop.
#include <cstdint>
#include <cstring>

#include "aires_b200.h"

namespace {
constexpr uint64_t kPrime = 1099511628211ULL;
struct PowTable {
  uint64_t p[9];
  constexpr PowTable() : p() {
    p[0] = 1;
    for (int i = 1; i <= 8; i++) p[i] = p[i - 1] * kPrime;
  }
};
constexpr PowTable kPow;

struct Fnv {
  uint64_t s = 14695981039346656037ULL;
  inline void byte(uint64_t v, int i) {
    s ^= static_cast<unsigned char>(v >> (8 * i));
    s *= kPrime;
  }
  inline void u64(uint64_t v) {
    for (int i = 0; i < 8; i++) byte(v, i);
  }
  // small integers (row offsets, column indices): the high zero bytes are one multiply; the
  // branch follows the data's width, which is uniform within an array
  inline void small(uint64_t v) {
    if (v < (uint64_t(1) << 16)) {
      byte(v, 0);
      byte(v, 1);
      s *= kPow.p[6];
    } else if (v < (uint64_t(1) << 32)) {
      byte(v, 0);
      byte(v, 1);
      byte(v, 2);
      byte(v, 3);
      s *= kPow.p[4];
    } else {
      u64(v);
    }
  }
  // f64 bit patterns: fp32-widened values have their three low bytes zero (one multiply)
  inline void f64bits(uint64_t v) {
    if ((v & 0xffffffu) == 0) {
      s *= kPow.p[3];
      for (int i = 3; i < 8; i++) byte(v, i);
    } else {
      u64(v);
    }
  }
};
}  // namespace

extern "C" uint64_t aires_b200_checksum(uint64_t n_rows, uint64_t n_cols, uint64_t nnz, const uint64_t* row_ptr,
                                        const void* col_idx, uint32_t idx_bytes, const void* values,
                                        uint32_t val_bytes) {
  Fnv h;
  h.u64(n_rows);
  h.u64(n_cols);
  h.u64(nnz);
  const uint64_t base = row_ptr ? row_ptr[0] : 0;
  for (uint64_t r = 0; r <= n_rows && row_ptr; r++) h.small(row_ptr[r] - base);
  if (idx_bytes == 4) {
    const auto* c = static_cast<const uint32_t*>(col_idx);
    for (uint64_t i = 0; i < nnz; i++) h.small(c[i]);
  } else {
    const auto* c = static_cast<const uint64_t*>(col_idx);
    for (uint64_t i = 0; i < nnz; i++) h.small(c[i]);
  }
  if (val_bytes == 4) {
    const auto* f = static_cast<const float*>(values);
    for (uint64_t i = 0; i < nnz; i++) {
      const double v = static_cast<double>(f[i]);
      uint64_t b;
      std::memcpy(&b, &v, 8);
      h.f64bits(b);
    }
  } else {
    const auto* d = static_cast<const uint64_t*>(values);
    for (uint64_t i = 0; i < nnz; i++) h.f64bits(d[i]);
  }
  return h.s;
}
