// b200_glue.hpp -- C++ side of the drop-in: reference containers <-> the C ABI of aires_b200.h.
//
// Used by the drop-in headers in this directory (spgemm.hpp, partition.hpp, scheduler.hpp).  The
// reference's own containers and error type are used unchanged (they come from the reference
// headers, reached with #include_next), so CsrMatrix / CscMatrix / RobwSegment / RunResult are
// the reference's structs byte for byte.
#ifndef AIRES_B200_GLUE_HPP
#define AIRES_B200_GLUE_HPP

#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "aires/error.hpp"
#include "aires/sparse.hpp"
#include "aires_b200.h"

namespace aires::b200 {

/// Throws the reference's exception for a C-ABI status (1 + errc, error.hpp:9-27); device and
/// runtime failures (>= 100) have no errc and surface as std::runtime_error.
inline void check(int status) {
  if (status == AIRES_B200_OK) return;
  const std::string msg = aires_b200_last_error();
  if (status >= 1 && status <= 17) throw aires::error(static_cast<errc>(status - 1), msg);
  throw std::runtime_error("aires_b200 status " + std::to_string(status) + ": " + msg);
}

/// Output allocator adopting std::vector storage (the exact allocation of spgemm.hpp:111-112).
struct VectorOut {
  CsrMatrix* c;
  static int alloc(void* user, uint64_t n_rows, uint64_t nnz, void** ptr, void** idx, void** val) {
    auto* self = static_cast<VectorOut*>(user);
    try {
      self->c->row_ptr.assign(n_rows + 1, 0);
      self->c->col_idx.resize(nnz);
      self->c->values.resize(nnz);
    } catch (const std::bad_alloc&) {
      return 1 + static_cast<int>(errc::capacity_exceeded);
    }
    *ptr = self->c->row_ptr.data();
    *idx = self->c->col_idx.data();
    *val = self->c->values.data();
    return 0;
  }
  aires_b200_output out() {
    aires_b200_output o{};
    o.location = AIRES_B200_HOST;
    o.idx_bytes = sizeof(index_t);
    o.val_bytes = sizeof(value_t);
    o.alloc = &VectorOut::alloc;
    o.user = this;
    return o;
  }
};

inline aires_b200_matrix csr_rows_view(std::span<const index_t> row_ptr, std::span<const index_t> col_idx,
                                       std::span<const value_t> values, index_t rows, index_t n_cols) {
  aires_b200_matrix m{};
  m.n_rows = rows;
  m.n_cols = n_cols;
  m.layout = AIRES_B200_CSR;
  m.location = AIRES_B200_HOST;
  m.idx_bytes = sizeof(index_t);
  m.val_bytes = sizeof(value_t);
  m.ptr = row_ptr.data();
  m.idx = col_idx.data();
  m.val = values.data();
  m.span = std::min<uint64_t>(col_idx.size(), values.size());
  return m;
}

inline aires_b200_matrix view(const CsrMatrix& a) {
  return csr_rows_view(a.row_ptr, a.col_idx, a.values, a.n_rows, a.n_cols);
}

inline aires_b200_matrix view(const CscMatrix& b) {
  aires_b200_matrix m{};
  m.n_rows = b.n_rows;
  m.n_cols = b.n_cols;
  m.layout = AIRES_B200_CSC;
  m.location = AIRES_B200_HOST;
  m.idx_bytes = sizeof(index_t);
  m.val_bytes = sizeof(value_t);
  m.ptr = b.col_ptr.data();
  m.idx = b.row_idx.data();
  m.val = b.values.data();
  m.span = std::min<uint64_t>(b.row_idx.size(), b.values.size());
  return m;
}

}  // namespace aires::b200

#endif  // AIRES_B200_GLUE_HPP
