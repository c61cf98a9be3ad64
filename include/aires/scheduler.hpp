// aires/scheduler.hpp -- drop-in for the reference's scheduler.hpp on the B200.
//
// Two run_aires flavours (scheduler.hpp:72-168):
//   * default (real): run_aires / run_maxmemory / run_strategy / compare_strategies run the real
//     out-of-core pipeline (aires_b200_run): A streamed from host memory through a ring of device
//     slots sized by A + C bytes under budget.device_total (0 = no cap), C drained tile by tile, the
//     RunReport filled with measured phase times, ChannelTotals {count, bytes, seconds} of the real
//     copies (CUDA events), merge_seconds (MaxMemory), and RunResult::trace with the measured
//     TraceEvents (transfers, computes, allocs, frees) -- audit_trace (tiered_sim.hpp:344-420)
//     replays it (counts, bytes, monotone timestamps and phases, matched frees, capacity);
//   * AIRES_B200_SIMULATED_RUN: the reference's own three-phase scheduler over its TieredSystem
//     accounting, compiled through #include_next; because spgemm.hpp in this directory replaces
//     spgemm_block, every segment it multiplies runs on the B200 (bit-identical fp64), while the
//     simulator identities of scheduler_test.cpp:39-66 / :197-211 (modelled seconds, gds/s2h
//     channels, byte-identical reruns) hold exactly as in the reference.
// aires::b200::run_aires_real / run_maxmemory_real are available in both flavours.
#ifndef AIRES_B200_SCHEDULER_DROPIN_HPP
#define AIRES_B200_SCHEDULER_DROPIN_HPP

#include "aires/partition.hpp"
#include "aires/spgemm.hpp"

#ifndef AIRES_B200_SIMULATED_RUN
#define run_aires run_aires_simulated
#define run_maxmemory run_maxmemory_simulated
#define run_strategy run_strategy_simulated
#define compare_strategies compare_strategies_simulated
#endif
#include_next "aires/scheduler.hpp"
#ifndef AIRES_B200_SIMULATED_RUN
#undef run_aires
#undef run_maxmemory
#undef run_strategy
#undef compare_strategies
#endif

#include "aires/b200_glue.hpp"

namespace aires::b200 {

/// The measured trace of a real run as the reference's TraceEvents (tiered_sim.hpp:60-68).
inline void append_trace(void* user, const aires_b200_trace_event* ev, uint64_t n) {
  auto* out = static_cast<std::vector<TraceEvent>*>(user);
  static const char* const kCh[] = {"gds", "s2h", "h2d", "d2h"};
  static const char* const kTier[] = {"device", "host", "storage"};
  out->reserve(out->size() + n);
  for (uint64_t i = 0; i < n; i++) {
    const aires_b200_trace_event& e = ev[i];
    TraceEvent t;
    t.timestamp = e.timestamp_ms * 1e-3;
    t.kind = static_cast<EventKind>(e.kind);
    t.phase = static_cast<Phase>(e.phase);
    t.where = e.kind == AIRES_B200_EV_TRANSFER ? kCh[e.where & 3] : kTier[e.where % 3];
    switch (e.buffer) {
      case AIRES_B200_BUF_B: t.buffer = "B"; break;
      case AIRES_B200_BUF_A_TILE: t.buffer = "a_tile_" + std::to_string(e.index); break;
      case AIRES_B200_BUF_C_BLOCK: t.buffer = "C"; break;
      case AIRES_B200_BUF_FRAGMENT: t.buffer = "frag_" + std::to_string(e.index); break;
      default: t.buffer = "A"; break;
    }
    t.bytes = e.bytes;
    t.flops = e.flops;
    out->push_back(std::move(t));
  }
}

inline RunResult run_real(const CsrMatrix& a, const CscMatrix& b, const MemoryBudget& budget, const SimConfig& cfg,
                          std::uint32_t n_buffers, std::uint32_t strategy /* 1 AIRES, 2 MaxMemory */,
                          bool stream_out = false) {
  (void)cfg;  // cost-model parameters of the simulator; the real run measures instead
  if (a.n_cols != b.n_rows)
    fail(errc::dimension_mismatch,
         "inner dimensions " + std::to_string(a.n_cols) + " and " + std::to_string(b.n_rows) + " differ");
  RunResult res;
  res.c.n_rows = a.n_rows;
  res.c.n_cols = b.n_cols;
  aires_b200_matrix am = view(a), bm = view(b);
  VectorOut vo{&res.c};
  aires_b200_output out = vo.out();
  aires_b200_run_config rc{};
  rc.device_budget = budget.device_total;
  rc.mode = AIRES_B200_MODE_FP64_EXACT;
  rc.c_aware = strategy;
  rc.n_buffers = n_buffers;
  rc.flags = stream_out ? AIRES_B200_RUN_STREAM_OUT : 0u;
  rc.trace = &append_trace;
  rc.trace_user = &res.trace;
  aires_b200_run_report rep{};
  check(aires_b200_run(&am, &bm, &rc, &out, &rep));
  res.c.col_idx.resize(out.nnz);  // streamed output: the vectors were sized to the nnz bound
  res.c.values.resize(out.nnz);
  res.c.n_rows = a.n_rows;
  res.c.n_cols = b.n_cols;
  RunReport& r = res.report;
  r.strategy = strategy == 2 ? Strategy::maxmemory : Strategy::aires;
  r.budget_bytes = budget.device_total;
  r.phase1_s = rep.phase1_ms * 1e-3;
  r.phase2_s = rep.phase2_ms * 1e-3;
  r.phase3_s = rep.phase3_ms * 1e-3;
  r.total_s = r.phase1_s + r.phase2_s + r.phase3_s;
  r.ledger.h2d = ChannelTotals{rep.h2d_count, rep.h2d_bytes, rep.h2d_ms * 1e-3};
  r.ledger.d2h = ChannelTotals{rep.d2h_count, rep.d2h_bytes, rep.d2h_ms * 1e-3};
  r.ledger.peak_device_occupancy = rep.peak_device_bytes;
  r.ledger.merge_bytes = rep.merge_bytes;
  r.merge_seconds = rep.merge_ms * 1e-3;
#ifndef AIRES_B200_NO_RUN_CHECKSUM
  // serialize.hpp:50-59 (byte-serial FNV-1a; AIRES_B200_NO_RUN_CHECKSUM leaves it 0 for callers that
  // hash the result themselves)
  r.c_checksum = checksum(res.c);
#endif
  r.segments = rep.segments;
  return res;
}

/// run_aires (scheduler.hpp:72-168) as the real out-of-core pipeline.  stream_out: each tile is
/// sized on the device after its upload (capped budgets) or not at all (uncapped: the vectors are
/// sized to an upper bound of nnz(C), then trimmed), so A crosses the link once and C drains while A
/// still uploads; without it the reference's exact-allocation protocol (a sizing pass first).
inline RunResult run_aires_real(const CsrMatrix& a, const CscMatrix& b, const MemoryBudget& budget,
                                const SimConfig& cfg, std::uint32_t n_buffers = 2, bool stream_out = false) {
  return run_real(a, b, budget, cfg, n_buffers, 1, stream_out);
}

/// run_maxmemory (scheduler.hpp:174-293) for real: fixed byte tiles, split rows' fragments returned
/// to the host and re-sent with the next tile.
inline RunResult run_maxmemory_real(const CsrMatrix& a, const CscMatrix& b, const MemoryBudget& budget,
                                    const SimConfig& cfg, std::uint32_t n_buffers = 2) {
  return run_real(a, b, budget, cfg, n_buffers, 2);
}

}  // namespace aires::b200

#ifndef AIRES_B200_SIMULATED_RUN
namespace aires {
/// scheduler.hpp:72-168 -- the real pipeline, streamed output, ring of 3.  Feature matrices wider
/// than the device accumulator (aires_b200_run reports unsupported_format: the pipeline's tiles hold
/// whole C rows) run on the reference scheduler with the B200 spgemm_block, which tiles B's columns.
inline RunResult run_aires(const CsrMatrix& a, const CscMatrix& b, const MemoryBudget& budget,
                           const SimConfig& cfg) {
  try {
    return b200::run_aires_real(a, b, budget, cfg, 3, true);
  } catch (const error& e) {
    if (e.code() != errc::unsupported_format) throw;
    return run_aires_simulated(a, b, budget, cfg);
  }
}

/// scheduler.hpp:174-293 -- the real MaxMemory baseline (wide features: as run_aires).
inline RunResult run_maxmemory(const CsrMatrix& a, const CscMatrix& b, const MemoryBudget& budget,
                               const SimConfig& cfg) {
  try {
    return b200::run_maxmemory_real(a, b, budget, cfg, 2);
  } catch (const error& e) {
    if (e.code() != errc::unsupported_format) throw;
    return run_maxmemory_simulated(a, b, budget, cfg);
  }
}

/// scheduler.hpp:295-299
inline RunResult run_strategy(Strategy st, const CsrMatrix& a, const CscMatrix& b, const MemoryBudget& budget,
                              const SimConfig& cfg) {
  return st == Strategy::aires ? run_aires(a, b, budget, cfg) : run_maxmemory(a, b, budget, cfg);
}

/// scheduler.hpp:303-324 -- out-of-memory outcomes recorded as flagged rows, not raised.
inline std::vector<RunReport> compare_strategies(const CsrMatrix& a, const CscMatrix& b,
                                                 const std::vector<std::uint64_t>& budgets, const SimConfig& cfg) {
  std::vector<RunReport> rows;
  for (std::uint64_t bytes : budgets) {
    for (Strategy st : {Strategy::aires, Strategy::maxmemory}) {
      MemoryBudget budget{bytes, cfg.host_bytes, cfg.sizes};
      try {
        rows.push_back(run_strategy(st, a, b, budget, cfg).report);
      } catch (const error& e) {
        if (e.code() != errc::insufficient_device_memory && e.code() != errc::row_too_large) throw;
        RunReport r;
        r.strategy = st;
        r.budget_bytes = bytes;
        r.oom = true;
        rows.push_back(r);
      }
    }
  }
  return rows;
}
}  // namespace aires
#endif

#endif  // AIRES_B200_SCHEDULER_DROPIN_HPP
