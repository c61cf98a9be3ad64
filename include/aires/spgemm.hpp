// aires/spgemm.hpp -- drop-in replacement of the reference's spgemm.hpp (proj/include/aires/
// spgemm.hpp) for the B200.  Put this directory BEFORE the reference's include directory:
//   -I<repo>/include -I<reference>/proj/include   and link libaires_b200.so.
//
// The reference header is still compiled (#include_next) for everything that is not the hot
// path -- CsrBlockResult, assemble_blocks, dense_oracle, kDefaultColTile -- with its own
// spgemm_block / spgemm_full renamed to *_cpu_reference, and these declarations take the
// original names with identical signatures, defaults and semantics (spgemm.hpp:60-151):
//   * dimension check -> errc::dimension_mismatch (spgemm.hpp:66-68); tile_cols == 0 means the
//     default; tile width never changes bits (the B200 kernels do not tile columns);
//   * row_ptr may be absolute (spgemm.hpp:79-84);
//   * output canonical (ascending columns), computed structural zeros kept (:58-59);
//   * fp64 values summed per cell in ascending k with one IEEE multiply and one IEEE add per
//     term (no FMA): bit-identical to dot_row_col (:21-42);
//   * flops == the structural MAC count (:51).
#ifndef AIRES_B200_SPGEMM_DROPIN_HPP
#define AIRES_B200_SPGEMM_DROPIN_HPP

#include "aires/partition.hpp"  // the drop-in partition.hpp (device RoBW cuts)

#define spgemm_block spgemm_block_cpu_reference
#define spgemm_full spgemm_full_cpu_reference
#include_next "aires/spgemm.hpp"
#undef spgemm_block
#undef spgemm_full

#include "aires/b200_glue.hpp"

namespace aires {

/// spgemm.hpp:60-132 on the B200 (aires_b200_spgemm, FP64_EXACT).
inline CsrBlockResult spgemm_block(std::span<const index_t> row_ptr, std::span<const index_t> col_idx,
                                   std::span<const value_t> values, index_t rows, index_t a_n_cols,
                                   const CscMatrix& b, index_t start_row = 0,
                                   index_t tile_cols = kDefaultColTile) {
  (void)tile_cols;
  if (a_n_cols != b.n_rows)
    fail(errc::dimension_mismatch,
         "inner dimensions " + std::to_string(a_n_cols) + " and " + std::to_string(b.n_rows) + " differ");
  CsrBlockResult res;
  res.start_row = start_row;
  res.end_row = start_row + rows;
  res.fragment.n_rows = rows;
  res.fragment.n_cols = b.n_cols;
  if (rows == 0) {
    res.fragment.row_ptr.assign(1, 0);
    return res;
  }
  aires_b200_matrix a = b200::csr_rows_view(row_ptr, col_idx, values, rows, a_n_cols);
  aires_b200_matrix bm = b200::view(b);
  b200::VectorOut vo{&res.fragment};
  aires_b200_output out = vo.out();
  b200::check(aires_b200_spgemm(&a, &bm, AIRES_B200_MODE_FP64_EXACT, &out));
  res.fragment.n_rows = rows;
  res.fragment.n_cols = b.n_cols;
  res.flops = out.flops;
  return res;
}

/// spgemm.hpp:134-139
inline CsrBlockResult spgemm_block(const RobwSegment& seg, index_t a_n_cols, const CscMatrix& b,
                                   index_t tile_cols = kDefaultColTile) {
  return spgemm_block(seg.row_ptr_local, seg.col_idx, seg.values, seg.rows(), a_n_cols, b, seg.start_row,
                      tile_cols);
}

/// spgemm.hpp:142-146
inline CsrMatrix spgemm_full(const CsrMatrix& a, const CscMatrix& b, index_t tile_cols = kDefaultColTile) {
  return spgemm_block(a.row_ptr, a.col_idx, a.values, a.n_rows, a.n_cols, b, 0, tile_cols).fragment;
}

/// spgemm.hpp:148-151: X as CSR goes to the device as is (no host csr_to_csc).
inline CsrMatrix spgemm_full(const CsrMatrix& a, const CsrMatrix& b, index_t tile_cols = kDefaultColTile) {
  (void)tile_cols;
  if (a.n_cols != b.n_rows)
    fail(errc::dimension_mismatch,
         "inner dimensions " + std::to_string(a.n_cols) + " and " + std::to_string(b.n_rows) + " differ");
  CsrMatrix c;
  c.n_rows = a.n_rows;
  c.n_cols = b.n_cols;
  if (a.n_rows == 0) {
    c.row_ptr.assign(1, 0);
    return c;
  }
  aires_b200_matrix am = b200::view(a), bm = b200::view(b);
  b200::VectorOut vo{&c};
  aires_b200_output out = vo.out();
  b200::check(aires_b200_spgemm(&am, &bm, AIRES_B200_MODE_FP64_EXACT, &out));
  c.n_rows = a.n_rows;
  c.n_cols = b.n_cols;
  return c;
}

}  // namespace aires

#endif  // AIRES_B200_SPGEMM_DROPIN_HPP
