// aires/partition.hpp -- drop-in replacement of the reference's partition.hpp for the B200.
//
// robw_partition (Alg. 1, partition.hpp:52-74) takes its cuts from the device tiler
// (aires_b200_robw_cuts: search over F(r) = r*I + row_ptr[r]*(I+V), bit-identical cuts and the
// same row_too_large row); the segments are then sliced by the reference's own slice_rows.
// Everything else (RobwSegment, slice_rows and the MaxMemory baseline) is the reference's,
// compiled through #include_next with its robw_partition renamed to robw_partition_cpu_reference.
#ifndef AIRES_B200_PARTITION_DROPIN_HPP
#define AIRES_B200_PARTITION_DROPIN_HPP

#define robw_partition robw_partition_cpu_reference
#include_next "aires/partition.hpp"
#undef robw_partition

#include "aires/b200_glue.hpp"

namespace aires {

inline std::vector<RobwSegment> robw_partition(const CsrMatrix& a, std::uint64_t m_a, ElementSizes s = {}) {
  std::vector<RobwSegment> segs;
  if (a.n_rows == 0) return segs;
  std::vector<std::uint64_t> cuts(a.n_rows + 1);
  std::uint64_t n_segs = 0, bad = 0;
  const int rc = aires_b200_robw_cuts(a.row_ptr.data(), a.n_rows, m_a, s.index_bytes, s.value_bytes,
                                      AIRES_B200_HOST, cuts.data(), cuts.size(), &n_segs, &bad);
  if (rc == AIRES_B200_ROW_TOO_LARGE)
    fail(errc::row_too_large, "row " + std::to_string(bad) + " needs " +
                                  std::to_string(calc_mem(1, a.row_ptr[bad + 1] - a.row_ptr[bad], s)) +
                                  " bytes, block budget is " + std::to_string(m_a));
  b200::check(rc);
  segs.reserve(n_segs);
  for (std::uint64_t j = 0; j < n_segs; j++) segs.push_back(slice_rows(a, cuts[j], cuts[j + 1], j, s));
  return segs;
}

}  // namespace aires

#endif  // AIRES_B200_PARTITION_DROPIN_HPP
