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

// The real run's measured trace replays through the reference's own auditor (tiered_sim.hpp:344-420):
// per-channel transfer counts and bytes equal the ledger, timestamps and phases are monotone, every
// free matches an alloc, and the device occupancy it implies stays inside the budget.  (The auditor's
// seconds come from the cost model, so only counts and bytes are compared.)
void expect_audited(const RunResult& r, std::uint64_t budget, const char* what) {
  ASSERT_FALSE(r.trace.empty()) << what;
  const AuditResult au = audit_trace(r.trace, SimConfig{}, budget ? budget : ~std::uint64_t(0));
  EXPECT_EQ(au.h2d.count, r.report.ledger.h2d.count) << what;
  EXPECT_EQ(au.h2d.bytes, r.report.ledger.h2d.bytes) << what;
  EXPECT_EQ(au.d2h.count, r.report.ledger.d2h.count) << what;
  EXPECT_EQ(au.d2h.bytes, r.report.ledger.d2h.bytes) << what;
  EXPECT_TRUE(au.timestamps_monotone) << what;
  EXPECT_TRUE(au.phases_monotone) << what;
  EXPECT_TRUE(au.frees_matched) << what;
  EXPECT_TRUE(au.within_capacity) << what;
  if (budget) EXPECT_LE(r.report.ledger.peak_device_occupancy, budget) << what;
  EXPECT_GT(r.report.ledger.h2d.seconds, 0.0) << what;
  EXPECT_GT(r.report.ledger.d2h.seconds, 0.0) << what;
  EXPECT_GE(r.report.ledger.h2d.count, r.report.segments) << what;
  EXPECT_DOUBLE_EQ(r.report.total_s, r.report.phase1_s + r.report.phase2_s + r.report.phase3_s) << what;
}

TEST(RealRun, TraceAndLedgerAuditEveryProtocol) {
  const Case c = make_case(4000, 0.008, 64, 51);
  const CscMatrix b = csr_to_csc(c.x);
  const std::uint64_t capped = 4'000'000 + (c.bytes_a + c.bytes_c) / 3;
  const std::uint64_t macs = [&] {
    std::uint64_t m = 0;
    for (index_t i = 0; i < c.a.nnz(); i++) {
      const index_t k = c.a.col_idx[i];
      m += c.x.row_ptr[k + 1] - c.x.row_ptr[k];
    }
    return m;
  }();
  struct P {
    const char* what;
    std::uint64_t budget;
    bool stream;
  };
  for (const P& p : {P{"uncapped exact", 0, false}, P{"uncapped streamed", 0, true}, P{"capped exact", capped, false},
                     P{"capped streamed", capped, true}}) {
    RunResult r = b200::run_aires_real(c.a, b, MemoryBudget{p.budget}, SimConfig{}, 3, p.stream);
    EXPECT_TRUE(r.c == c.want) << p.what;
    expect_audited(r, p.budget, p.what);
    std::uint64_t flops = 0;
    for (const TraceEvent& e : r.trace)
      if (e.kind == EventKind::compute) flops += e.flops;
    // streamed/capped-streamed and exact tiles carry the product's MACs; the exact protocol's sizing
    // chunks carry none
    EXPECT_EQ(flops, macs) << p.what;
    EXPECT_EQ(r.report.ledger.merge_bytes, 0u) << p.what;
    EXPECT_DOUBLE_EQ(r.report.merge_seconds, 0.0) << p.what;
  }
  RunResult mm = b200::run_maxmemory_real(c.a, b, MemoryBudget{capped}, SimConfig{}, 2);
  EXPECT_TRUE(mm.c == c.want);
  expect_audited(mm, capped, "maxmemory");
  if (mm.report.ledger.merge_bytes > 0) EXPECT_GT(mm.report.merge_seconds, 0.0);
}

// The default flavour of the drop-in: aires::run_aires / run_maxmemory / run_strategy /
// compare_strategies are the real pipeline (scheduler.hpp:72-324 signatures).
TEST(RealDefault, ReferenceEntryPointsRunTheRealPipeline) {
  const Case c = make_case(3000, 0.01, 64, 61);
  const CscMatrix b = csr_to_csc(c.x);
  const std::uint64_t capped = 4'000'000 + (c.bytes_a + c.bytes_c) / 4;
  RunResult r = run_aires(c.a, b, MemoryBudget{capped}, SimConfig{});
  EXPECT_TRUE(r.c == c.want);
  EXPECT_EQ(r.report.c_checksum, checksum(c.want));
  EXPECT_GE(r.report.segments, 2u);
  // A crosses the link once: the ledger's upload bytes are A's and X's canonical bytes + one row
  // pointer per extra tile
  RunResult m = run_strategy(Strategy::maxmemory, c.a, b, MemoryBudget{capped}, SimConfig{});
  EXPECT_TRUE(m.c == c.want);
  EXPECT_EQ(m.report.strategy, Strategy::maxmemory);
  std::vector<RunReport> rows = compare_strategies(c.a, b, {capped, 50'000}, SimConfig{});
  ASSERT_EQ(rows.size(), 4u);
  EXPECT_FALSE(rows[0].oom);
  EXPECT_FALSE(rows[1].oom);
  EXPECT_TRUE(rows[2].oom);
  EXPECT_TRUE(rows[3].oom);
  EXPECT_EQ(rows[0].c_checksum, rows[1].c_checksum);
}

TEST(RealDefault, EmptyOperandsStillProduceC) {
  CsrMatrix a;
  a.n_rows = 5;
  a.n_cols = 5;
  a.row_ptr.assign(6, 0);
  CscMatrix b;
  b.n_rows = 5;
  b.n_cols = 3;
  b.col_ptr.assign(4, 0);
  for (Strategy st : {Strategy::aires, Strategy::maxmemory}) {
    RunResult r = run_strategy(st, a, b, MemoryBudget{0}, SimConfig{});
    EXPECT_EQ(r.c.n_rows, 5u);
    EXPECT_EQ(r.c.n_cols, 3u);
    EXPECT_EQ(r.c.nnz(), 0u);
    EXPECT_EQ(r.c.row_ptr.size(), 6u);
  }
}

// X wider than the fp64 device accumulator (4096 columns): the pipeline's tiles hold whole C rows,
// so the default run_aires falls back to the reference scheduler with the B200 spgemm_block (which
// tiles B's columns) -- same C as the in-core product.
TEST(RealDefault, WideFeaturesFallBackToTheColumnTiledScheduler) {
  CsrMatrix a = gen_symmetric(300, 0.03, 71);
  CsrMatrix x = gen_features(300, 5000, 99.0, 72);
  const CsrMatrix want = spgemm_full(a, x);
  const CscMatrix b = csr_to_csc(x);
  EXPECT_THROW(b200::run_aires_real(a, b, MemoryBudget{0}, SimConfig{}, 3, true), error);
  SimConfig cfg;
  RunResult r = run_aires(a, b, cfg.budget(), cfg);
  EXPECT_TRUE(r.c == want);
  EXPECT_EQ(r.report.c_checksum, checksum(want));
}

TEST(RealRun, DimensionMismatchThrows) {
  const Case c = make_case(500, 0.02, 16, 41);
  const CsrMatrix wrong = gen_features(499, 16, 95.0, 3);
  EXPECT_THROW(b200::run_aires_real(c.a, csr_to_csc(wrong), MemoryBudget{0}, SimConfig{}), error);
}

}  // namespace
}  // namespace aires
