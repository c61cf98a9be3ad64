// ab2_host.cpp -- host-side parts of the boundary that need no device.
//
// aires_b200_checksum: the reference's C checksum (serialize.hpp:22-59), FNV-1a 64 over the
// canonical little-endian stream n_rows, n_cols, nnz, row_ptr, col_idx (as u64) and values (as
// f64 bit patterns).  It is byte-serial by definition (0.63 GB/s measured), so it
// runs on the host and never inside a timed region; narrow widths are widened exactly as the
// reference's u64/f64 containers would hold them.
#include <cstdint>
#include <cstring>

#include "aires_b200.h"

namespace {
struct Fnv {
  uint64_t s = 14695981039346656037ULL;
  inline void u64(uint64_t v) {
    for (int i = 0; i < 8; i++) {
      s ^= static_cast<unsigned char>(v >> (8 * i));
      s *= 1099511628211ULL;
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
  for (uint64_t r = 0; r <= n_rows && row_ptr; r++) h.u64(row_ptr[r] - base);
  for (uint64_t i = 0; i < nnz; i++)
    h.u64(idx_bytes == 4 ? static_cast<const uint32_t*>(col_idx)[i] : static_cast<const uint64_t*>(col_idx)[i]);
  for (uint64_t i = 0; i < nnz; i++) {
    const double v = val_bytes == 4 ? static_cast<double>(static_cast<const float*>(values)[i])
                                    : static_cast<const double*>(values)[i];
    uint64_t b;
    std::memcpy(&b, &v, 8);
    h.u64(b);
  }
  return h.s;
}
