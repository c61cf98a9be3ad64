// ref_shim.cpp -- TEST/BASELINE INFRASTRUCTURE ONLY.
//
// Compiles the UNMODIFIED reference headers from /root/reference/proj/include
// (header-only C++20; nothing is copied into this repo) into
// oracle/_ref/libaires_ref.so and exposes a C ABI so the tests can pin the C
// oracle (aires_oracle.c) against the reference itself, and bench.py can time
// the reference's own CPU spgemm_block as the cpu_baseline / --impl reference arm.
//
// Build recipe: oracle/Makefile (reference flags -std=c++20 -O3 -DNDEBUG, no -march,
// -ffp-contract=off; proj/CMakeLists.txt:3,8-10).
#include <atomic>
#include <fstream>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <span>
#include <thread>
#include <vector>

#include "aires/gcn.hpp"
#include "aires/memory_model.hpp"
#include "aires/partition.hpp"
#include "aires/scheduler.hpp"
#include "aires/serialize.hpp"
#include "aires/spgemm.hpp"
#include "aires/synth.hpp"
#include "../oracle/aires_oracle.h"

using namespace aires;

namespace {

template <class T>
T* dup(const std::vector<T>& v) {
  T* p = static_cast<T*>(std::malloc(v.size() ? v.size() * sizeof(T) : 1));
  if (!v.empty()) std::memcpy(p, v.data(), v.size() * sizeof(T));
  return p;
}

void export_csr(const CsrMatrix& m, ao_csr* out) {
  out->n_rows = m.n_rows;
  out->n_cols = m.n_cols;
  out->nnz = m.nnz();
  out->ptr = dup(m.row_ptr);
  out->idx = dup(m.col_idx);
  out->val = dup(m.values);
}

CscMatrix make_csc(uint64_t n_rows, uint64_t n_cols, const uint64_t* col_ptr,
                   const uint64_t* row_idx, const double* vals) {
  CscMatrix b;
  b.n_rows = n_rows;
  b.n_cols = n_cols;
  b.col_ptr.assign(col_ptr, col_ptr + n_cols + 1);
  b.row_idx.assign(row_idx, row_idx + col_ptr[n_cols]);
  b.values.assign(vals, vals + col_ptr[n_cols]);
  return b;
}

CsrMatrix make_csr(uint64_t n_rows, uint64_t n_cols, const uint64_t* row_ptr,
                   const uint64_t* col_idx, const double* vals) {
  CsrMatrix a;
  a.n_rows = n_rows;
  a.n_cols = n_cols;
  a.row_ptr.assign(row_ptr, row_ptr + n_rows + 1);
  a.col_idx.assign(col_idx, col_idx + row_ptr[n_rows]);
  a.values.assign(vals, vals + row_ptr[n_rows]);
  return a;
}

int code_of(const error& e) { return 1 + static_cast<int>(e.code()); }

}  // namespace

extern "C" {

// spgemm.hpp:60-132 called verbatim. col/val spans are [0, nnz_span).
int ref_spgemm_block(const uint64_t* row_ptr, const uint64_t* col_idx, const double* values,
                     uint64_t nnz_span, uint64_t rows, uint64_t a_n_cols, uint64_t b_n_rows,
                     uint64_t b_n_cols, const uint64_t* b_col_ptr, const uint64_t* b_row_idx,
                     const double* b_values, uint64_t start_row, uint64_t tile_cols,
                     ao_csr* out, uint64_t* macs) {
  try {
    CscMatrix b = make_csc(b_n_rows, b_n_cols, b_col_ptr, b_row_idx, b_values);
    CsrBlockResult r = spgemm_block(std::span<const index_t>(row_ptr, rows + 1),
                                    std::span<const index_t>(col_idx, nnz_span),
                                    std::span<const value_t>(values, nnz_span), rows,
                                    a_n_cols, b, start_row, tile_cols);
    export_csr(r.fragment, out);
    *macs = r.flops;
    return 0;
  } catch (const error& e) {
    return code_of(e);
  }
}

int ref_csr_to_csc(uint64_t n_rows, uint64_t n_cols, const uint64_t* row_ptr,
                   const uint64_t* col_idx, const double* values, ao_csr* out) {
  CscMatrix b = csr_to_csc(make_csr(n_rows, n_cols, row_ptr, col_idx, values));
  out->n_rows = b.n_rows;
  out->n_cols = b.n_cols;
  out->nnz = b.nnz();
  out->ptr = dup(b.col_ptr);
  out->idx = dup(b.row_idx);
  out->val = dup(b.values);
  return 0;
}

int ref_robw_cuts(const uint64_t* row_ptr, uint64_t n_rows, uint64_t m_a, uint64_t I,
                  uint64_t V, uint64_t* cuts, uint64_t* n_segs, uint64_t* seg_bytes) {
  CsrMatrix a;
  a.n_rows = n_rows;
  a.n_cols = 1;
  a.row_ptr.assign(row_ptr, row_ptr + n_rows + 1);
  a.col_idx.assign(row_ptr[n_rows], 0);
  a.values.assign(row_ptr[n_rows], 1.0);
  try {
    std::vector<RobwSegment> segs = robw_partition(a, m_a, ElementSizes{I, V});
    cuts[0] = 0;
    for (std::size_t s = 0; s < segs.size(); s++) {
      cuts[s + 1] = segs[s].end_row;
      if (seg_bytes) seg_bytes[s] = segs[s].byte_size;
    }
    *n_segs = segs.size();
    return 0;
  } catch (const error& e) {
    return code_of(e);
  }
}

uint64_t ref_checksum(uint64_t n_rows, uint64_t n_cols, uint64_t nnz, const uint64_t* row_ptr,
                      const uint64_t* col_idx, const double* values) {
  CsrMatrix a;
  a.n_rows = n_rows;
  a.n_cols = n_cols;
  a.row_ptr.assign(row_ptr, row_ptr + n_rows + 1);
  a.col_idx.assign(col_idx, col_idx + nnz);
  a.values.assign(values, values + nnz);
  return checksum(a);
}

uint64_t ref_fnv1a64(const void* data, uint64_t n) { return fnv1a64(data, n); }

uint64_t ref_estimate_output_memory(uint64_t aa, double sa, uint64_t ab, double sb) {
  return estimate_output_memory(aa, sa, ab, sb);
}

int ref_gen_features(uint64_t n, uint64_t dim, double sparsity, uint64_t seed, ao_csr* out) {
  try {
    export_csr(gen_features(n, dim, sparsity, seed), out);
    return 0;
  } catch (const error& e) {
    return code_of(e);
  }
}

int ref_gen_sparse(uint64_t rows, uint64_t cols, double density, uint64_t seed, double lo,
                   double hi, ao_csr* out) {
  try {
    export_csr(gen_sparse(rows, cols, density, seed, lo, hi), out);
    return 0;
  } catch (const error& e) {
    return code_of(e);
  }
}

int ref_gen_symmetric(uint64_t n, double density, uint64_t seed, ao_csr* out) {
  try {
    export_csr(gen_symmetric(n, density, seed), out);
    return 0;
  } catch (const error& e) {
    return code_of(e);
  }
}

int ref_normalize_adjacency(uint64_t n, const uint64_t* row_ptr, const uint64_t* col_idx,
                            const double* values, ao_csr* out) {
  try {
    export_csr(normalize_adjacency(make_csr(n, n, row_ptr, col_idx, values)).a_tilde, out);
    return 0;
  } catch (const error& e) {
    return code_of(e);
  }
}

// robw_partition + write_segments (partition.hpp:52-74, serialize.hpp:148-174) to a file.
int ref_write_segments(const char* path, uint64_t n_rows, uint64_t n_cols, const uint64_t* row_ptr,
                       const uint64_t* col_idx, const double* values, uint64_t m_a, uint64_t I, uint64_t V) {
  try {
    ElementSizes s{I, V};
    std::vector<RobwSegment> segs = robw_partition(make_csr(n_rows, n_cols, row_ptr, col_idx, values), m_a, s);
    std::ofstream out(path, std::ios::binary);
    write_segments(out, segs, s);
    return out ? 0 : 1 + static_cast<int>(errc::io_error);
  } catch (const error& e) {
    return code_of(e);
  }
}

int ref_gen_weights(uint64_t in_dim, uint64_t out_dim, uint64_t seed, double* out) {
  DenseMatrix w = gen_weights(in_dim, out_dim, seed);
  std::memcpy(out, w.data.data(), w.data.size() * sizeof(double));
  return 0;
}

int ref_combine(uint64_t rows, uint64_t x_cols, const uint64_t* row_ptr, const uint64_t* col_idx,
                const double* values, const double* w, uint64_t w_rows, uint64_t w_cols, ao_csr* out) {
  try {
    DenseMatrix wd{w_rows, w_cols, std::vector<value_t>(w, w + w_rows * w_cols)};
    export_csr(combine(make_csr(rows, x_cols, row_ptr, col_idx, values), wd), out);
    return 0;
  } catch (const error& e) {
    return code_of(e);
  }
}

// run_aires (scheduler.hpp:72-168) verbatim; returns the report fields the
// B200 drop-in must reproduce.  rep: [segments, gds.count, gds.bytes, s2h.count,
// s2h.bytes, h2d.count, h2d.bytes, d2h.count, d2h.bytes, merge_bytes,
// peak_device_occupancy, c_checksum]
int ref_run_aires(uint64_t n_rows, uint64_t n_cols, const uint64_t* row_ptr,
                  const uint64_t* col_idx, const double* values, uint64_t b_n_rows,
                  uint64_t b_n_cols, const uint64_t* b_col_ptr, const uint64_t* b_row_idx,
                  const double* b_values, uint64_t device_total, uint64_t I, uint64_t V,
                  ao_csr* out, uint64_t* rep, double* secs) {
  try {
    CsrMatrix a = make_csr(n_rows, n_cols, row_ptr, col_idx, values);
    CscMatrix b = make_csc(b_n_rows, b_n_cols, b_col_ptr, b_row_idx, b_values);
    SimConfig cfg;
    MemoryBudget budget{device_total, cfg.host_bytes, ElementSizes{I, V}};
    RunResult r = run_aires(a, b, budget, cfg);
    export_csr(r.c, out);
    const IoLedger& l = r.report.ledger;
    uint64_t v[12] = {r.report.segments, l.gds.count, l.gds.bytes, l.s2h.count,
                      l.s2h.bytes,       l.h2d.count, l.h2d.bytes, l.d2h.count,
                      l.d2h.bytes,       l.merge_bytes, l.peak_device_occupancy,
                      r.report.c_checksum};
    std::memcpy(rep, v, sizeof v);
    if (secs) {
      secs[0] = r.report.phase1_s;
      secs[1] = r.report.phase2_s;
      secs[2] = r.report.phase3_s;
      secs[3] = r.report.total_s;
    }
    return 0;
  } catch (const error& e) {
    return code_of(e);
  }
}

// CPU baseline: the reference's spgemm_block, unmodified, applied to a row
// sample (each sampled row passed as an absolute 2-entry row_ptr sub-span,
// legal per spgemm.hpp:79-84), split over nthreads host threads.  Rows are
// independent, so each row's output is exactly the reference's.  Returns wall
// seconds; *macs / *c_nnz are the sample's totals, *row_hash an order-
// independent sum of per-row FNV hashes of (col_idx, value bits).
double ref_spgemm_rows_timed(const uint64_t* row_ptr, const uint64_t* col_idx,
                             const double* values, uint64_t nnz, uint64_t a_n_cols,
                             const uint64_t* rows, uint64_t n_sample, uint64_t b_n_rows,
                             uint64_t b_n_cols, const uint64_t* b_col_ptr,
                             const uint64_t* b_row_idx, const double* b_values, int nthreads,
                             uint64_t* macs, uint64_t* c_nnz, uint64_t* row_hash) {
  CscMatrix b = make_csc(b_n_rows, b_n_cols, b_col_ptr, b_row_idx, b_values);
  std::atomic<uint64_t> next{0}, tot_macs{0}, tot_nnz{0}, tot_hash{0};
  auto t0 = std::chrono::steady_clock::now();
  auto work = [&] {
    uint64_t m = 0, z = 0, h = 0;
    for (;;) {
      uint64_t i = next.fetch_add(1);
      if (i >= n_sample) break;
      uint64_t r = rows[i];
      CsrBlockResult res = spgemm_block(std::span<const index_t>(row_ptr + r, 2),
                                        std::span<const index_t>(col_idx, nnz),
                                        std::span<const value_t>(values, nnz), 1, a_n_cols,
                                        b, r);
      m += res.flops;
      z += res.fragment.nnz();
      Fnv1a64 f;
      f.update_u64(r);
      for (index_t c : res.fragment.col_idx) f.update_u64(c);
      for (value_t v : res.fragment.values) f.update_f64(v);
      h += f.state;
    }
    tot_macs += m;
    tot_nnz += z;
    tot_hash += h;
  };
  std::vector<std::thread> th;
  for (int t = 1; t < nthreads; t++) th.emplace_back(work);
  work();
  for (auto& t : th) t.join();
  double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  *macs = tot_macs;
  *c_nnz = tot_nnz;
  *row_hash = tot_hash;
  return s;
}

void ref_free(ao_csr* m) {
  std::free(m->ptr);
  std::free(m->idx);
  std::free(m->val);
  m->ptr = nullptr;
  m->idx = nullptr;
  m->val = nullptr;
}

}  // extern "C"
