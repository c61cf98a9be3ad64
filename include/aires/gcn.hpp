// aires/gcn.hpp -- drop-in for the reference's gcn.hpp: the steps either side of A·X on the B200.
//
// normalize_adjacency (gcn.hpp:29-72) and combine (gcn.hpp:90-116) forward to the C ABI
// (aires_b200_normalize_adjacency / aires_b200_combine, fp64, bit-identical to the reference);
// aggregate and layer_forward are the reference's own code (#include_next), so a whole
// layer_forward -- normalize, A·H through run_strategy, combine -- now runs on the device.
#ifndef AIRES_B200_GCN_DROPIN_HPP
#define AIRES_B200_GCN_DROPIN_HPP

#include "aires/scheduler.hpp"
#include "aires/spgemm.hpp"

#define normalize_adjacency normalize_adjacency_cpu_reference
#define combine combine_cpu_reference
#include_next "aires/gcn.hpp"
#undef normalize_adjacency
#undef combine

#include "aires/b200_glue.hpp"

namespace aires {

inline NormalizedAdjacency normalize_adjacency(const CsrMatrix& a) {
  if (a.n_rows != a.n_cols)
    fail(errc::non_square, std::to_string(a.n_rows) + "x" + std::to_string(a.n_cols) + " adjacency is not square");
  NormalizedAdjacency out;
  out.a_tilde.n_rows = out.a_tilde.n_cols = a.n_rows;
  aires_b200_matrix am = b200::view(a);
  b200::VectorOut vo{&out.a_tilde};
  aires_b200_output o = vo.out();
  b200::check(aires_b200_normalize_adjacency(&am, &o));
  out.a_tilde.n_rows = out.a_tilde.n_cols = a.n_rows;
  return out;
}

inline CsrMatrix combine(const CsrMatrix& x, const DenseMatrix& w) {
  if (x.n_cols != w.n_rows)
    fail(errc::dimension_mismatch,
         "feature width " + std::to_string(x.n_cols) + " does not match weight rows " + std::to_string(w.n_rows));
  CsrMatrix h;
  h.n_rows = x.n_rows;
  h.n_cols = w.n_cols;
  aires_b200_matrix xm = b200::view(x);
  b200::VectorOut vo{&h};
  aires_b200_output o = vo.out();
  b200::check(aires_b200_combine(&xm, w.data.data(), w.n_rows, w.n_cols, AIRES_B200_HOST, &o));
  h.n_rows = x.n_rows;
  h.n_cols = w.n_cols;
  return h;
}

}  // namespace aires

#endif  // AIRES_B200_GCN_DROPIN_HPP
