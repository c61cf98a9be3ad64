// The real out-of-core run behind the drop-in C++ headers (include/aires/scheduler.hpp:
// aires::b200::run_aires_real / run_maxmemory_real over aires_b200_run), checked bit-exactly
// (fp64-exact mode, CsrMatrix operator==, sparse.hpp:38) against the drop-in in-core product
// spgemm_full (spgemm.hpp:148-151), which the reference's own spgemm_test.cpp pins to the reference.
// Inputs come from the reference's generators (synth.hpp:26-78).  Results must not depend on the
// budget, the tile count, the ring depth, the strategy or the output protocol (partition
// independence, spgemm_test.cpp:97-115).  Test infrastructure: built by oracle/Makefile (dropin).
#include "aires/scheduler.hpp"

#include <gtest/gtest.h>

#include "aires/synth.hpp"

namespace aires {
namespace {

struct Case {
  CsrMatrix a;
  CsrMatrix x;
  CsrMatrix want;
  std::uint64_t bytes_a = 0, bytes_c = 0;
};

Case make_case(index_t n, double density, index_t dim, std::uint64_t seed) {
  Case c;
  c.a = gen_symmetric(n, density, seed);
  c.x = gen_features(n, dim, 95.0, seed + 1);
  c.want = spgemm_full(c.a, c.x);
  c.bytes_a = calc_mem(c.a.n_rows, c.a.nnz());
  c.bytes_c = calc_mem(c.want.n_rows, c.want.nnz());
  return c;
}

TEST(RealRun, UncappedExactAndStreamedMatchInCore) {
  const Case c = make_case(3000, 0.01, 64, 11);
  const CscMatrix b = csr_to_csc(c.x);
  for (std::uint32_t nbuf : {2u, 3u}) {
    RunResult exact = b200::run_aires_real(c.a, b, MemoryBudget{0}, SimConfig{}, nbuf, false);
    EXPECT_TRUE(exact.c == c.want);
    EXPECT_EQ(exact.report.c_checksum, checksum(c.want));
    RunResult streamed = b200::run_aires_real(c.a, b, MemoryBudget{0}, SimConfig{}, nbuf, true);
    EXPECT_TRUE(streamed.c == c.want);
    EXPECT_EQ(streamed.report.c_checksum, checksum(c.want));
    EXPECT_GE(streamed.report.segments, 1u);
  }
}

TEST(RealRun, CappedBudgetsMatchInCore) {
  const Case c = make_case(4000, 0.008, 64, 21);
  const CscMatrix b = csr_to_csc(c.x);
  for (double frac : {1.0, 0.5, 0.25}) {
    const std::uint64_t budget = 4'000'000 + static_cast<std::uint64_t>(frac * (c.bytes_a + c.bytes_c));
    RunResult r = b200::run_aires_real(c.a, b, MemoryBudget{budget}, SimConfig{}, 3, false);
    EXPECT_TRUE(r.c == c.want) << "budget fraction " << frac;
    if (frac < 1.0) EXPECT_GE(r.report.segments, 2u);
    // a capped budget keeps the exact protocol even when streamed output is asked for
    RunResult s = b200::run_aires_real(c.a, b, MemoryBudget{budget}, SimConfig{}, 3, true);
    EXPECT_TRUE(s.c == c.want) << "budget fraction " << frac;
  }
}

TEST(RealRun, MaxMemoryBaselineMatchesInCore) {
  const Case c = make_case(4000, 0.008, 64, 31);
  const CscMatrix b = csr_to_csc(c.x);
  const std::uint64_t budget = 4'000'000 + (c.bytes_a + c.bytes_c) / 3;
  RunResult r = b200::run_maxmemory_real(c.a, b, MemoryBudget{budget}, SimConfig{}, 2);
  EXPECT_TRUE(r.c == c.want);
  EXPECT_EQ(r.report.strategy, Strategy::maxmemory);
  EXPECT_GE(r.report.segments, 2u);
}

TEST(RealRun, DimensionMismatchThrows) {
  const Case c = make_case(500, 0.02, 16, 41);
  const CsrMatrix wrong = gen_features(499, 16, 95.0, 3);
  EXPECT_THROW(b200::run_aires_real(c.a, csr_to_csc(wrong), MemoryBudget{0}, SimConfig{}), error);
}

}  // namespace
}  // namespace aires
