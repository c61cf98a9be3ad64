/*
 * aires_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference AIRES hot path (arxiv 2507.02006,
 * /root/reference/proj/include/aires/ headers).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this library, and
 * only as the checker or the CPU baseline -- never as the product path.
 *
 * Parity pinning: every function below is checked in tests/test_oracle.py against
 *   (1) the known-answer values of the reference's own unit tests (cited per test), and
 *   (2) the reference itself compiled from /root/reference (oracle/_ref/libaires_ref.so,
 *       built by oracle/Makefile) through the committed golden fixtures in tests/golden/.
 *
 * Widths follow the reference API: index_t = uint64_t, value_t = double
 * (sparse.hpp:15-16).  Status codes: 0 = ok, otherwise 1 + (int)aires::errc
 * (error.hpp:9-27).
 */
#ifndef AIRES_ORACLE_H
#define AIRES_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* 1 + errc (error.hpp:9-27) */
enum {
  AO_OK = 0,
  AO_INDEX_OUT_OF_RANGE = 1,
  AO_INSUFFICIENT_DEVICE_MEMORY = 5,
  AO_ROW_TOO_LARGE = 6,
  AO_DIMENSION_MISMATCH = 8,
  AO_INVALID_DENSITY = 13,
  AO_NON_SQUARE = 14,
  AO_NEGATIVE_WEIGHT = 15,
};

/* A CSR (or CSC, with the roles of rows/cols swapped) owned by the oracle. */
typedef struct ao_csr {
  uint64_t n_rows, n_cols, nnz;
  uint64_t* ptr;   /* n_rows+1 (CSR) or n_cols+1 (CSC) */
  uint64_t* idx;   /* nnz */
  double* val;     /* nnz */
} ao_csr;

void ao_free(ao_csr* m);

/* sparse.hpp:119-140 csr_to_csc (counting sort, stable in row order). */
int ao_csr_to_csc(uint64_t n_rows, uint64_t n_cols, const uint64_t* row_ptr,
                  const uint64_t* col_idx, const double* values, ao_csr* out_csc);
/* sparse.hpp:142-163 csc_to_csr. */
int ao_csc_to_csr(uint64_t n_rows, uint64_t n_cols, const uint64_t* col_ptr,
                  const uint64_t* row_idx, const double* values, ao_csr* out_csr);

/*
 * spgemm.hpp:60-132 spgemm_block, restated literally: inner-product two-pointer
 * walk of every row against every column of B (CSC), symbolic pass, exact
 * allocation, numeric pass.  row_ptr may be absolute (spgemm.hpp:79-84).
 * out->ptr is the local (rebased) row pointer of the fragment.  *macs = flops.
 */
int ao_spgemm_inner(const uint64_t* row_ptr, const uint64_t* col_idx, const double* values,
                    uint64_t rows, uint64_t a_n_cols, uint64_t b_n_rows, uint64_t b_n_cols,
                    const uint64_t* b_col_ptr, const uint64_t* b_row_idx,
                    const double* b_values, uint64_t tile_cols, ao_csr* out,
                    uint64_t* macs);

/*
 * Same result bits as ao_spgemm_inner, computed row-wise (Gustavson) from B in CSR:
 * each output cell is the sum of a_ik*b_kj in ascending k starting from +0.0
 * (dot_row_col, spgemm.hpp:21-42), cells with a structural hit are kept even
 * if the sum is zero (spgemm.hpp:58-59).  nthreads>1 splits rows (rows are
 * independent, so bits do not change).
 */
int ao_spgemm_rowwise(const uint64_t* row_ptr, const uint64_t* col_idx, const double* values,
                      uint64_t rows, uint64_t a_n_cols, uint64_t b_n_rows, uint64_t b_n_cols,
                      const uint64_t* b_row_ptr, const uint64_t* b_col_idx,
                      const double* b_values, int nthreads, ao_csr* out, uint64_t* macs);

/* memory_model.hpp:84-86 */
uint64_t ao_calc_mem(uint64_t k, uint64_t q, uint64_t index_bytes, uint64_t value_bytes);
/* memory_model.hpp:61-74 */
uint64_t ao_estimate_output_memory(uint64_t alpha_a, double s_a, uint64_t alpha_b, double s_b);
/* memory_model.hpp:32-36 */
double ao_sparsity_percent(uint64_t n_rows, uint64_t n_cols, uint64_t nnz);
/* memory_model.hpp:90-106: returns AO_INSUFFICIENT_DEVICE_MEMORY or fills p, m_a. */
int ao_block_budget(uint64_t device_total, uint64_t m_c, uint64_t m_b, uint64_t* p,
                    uint64_t* m_a);

/*
 * partition.hpp:52-74 robw_partition (Alg. 1): greedy maximal whole-row segments
 * with calc_mem(k,q) <= m_a.  cuts[0..*n_segs] receives the segment boundaries
 * (cuts[0]=0, cuts[n_segs]=n_rows; capacity n_rows+1).  On row_too_large the
 * offending row is written to *bad_row.
 */
int ao_robw_cuts(const uint64_t* row_ptr, uint64_t n_rows, uint64_t m_a,
                 uint64_t index_bytes, uint64_t value_bytes, uint64_t* cuts,
                 uint64_t* n_segs, uint64_t* bad_row);

/* serialize.hpp:22-59 */
uint64_t ao_fnv1a64(const void* data, uint64_t n);
uint64_t ao_checksum(uint64_t n_rows, uint64_t n_cols, uint64_t nnz, const uint64_t* row_ptr,
                     const uint64_t* col_idx, const double* values);

/* synth.hpp:14-16, 49-69, 73-78 (std::mt19937_64 restated). */
int ao_gen_sparse(uint64_t rows, uint64_t cols, double density, uint64_t seed, double lo,
                  double hi, ao_csr* out);
int ao_gen_features(uint64_t n_nodes, uint64_t dim, double sparsity_pct, uint64_t seed,
                    ao_csr* out);

/* gcn.hpp:29-72 normalize_adjacency */
int ao_normalize_adjacency(uint64_t n, const uint64_t* row_ptr, const uint64_t* col_idx,
                           const double* values, ao_csr* out);

/* synth.hpp:81-86 */
int ao_gen_weights(uint64_t in_dim, uint64_t out_dim, uint64_t seed, double* out);
/* gcn.hpp:90-116 (row_ptr rebased: row_ptr[0] == 0) */
int ao_combine(uint64_t rows, uint64_t x_cols, const uint64_t* row_ptr, const uint64_t* col_idx,
               const double* values, const double* w, uint64_t w_rows, uint64_t w_cols, ao_csr* out);

/* Benchmark inputs for the reference arm: restatement of aires_b200_synth_graph
 * (paper_2507_02006_b200/csrc/ab2_synth.cpp), byte-identical output at API widths (u64/f64).
 * stats (8 doubles, may be NULL): nnz(A) before self-loops, max degree, mean degree, rounds, 0, i0. */
int ao_synth_graph(uint64_t n, uint64_t target_nnz, double alpha, uint64_t degree_cap, uint64_t seed,
                   uint64_t relabel_seed, int relabel, int normalize, int threads, ao_csr* out, double* stats);

/* Sum over rows[] of FNV-1a 64 of (row id, columns, value bits): the row hash the reference arm's
 * ref_spgemm_rows_timed (oracle/ref_shim.cpp) reports for its sampled rows. */
uint64_t ao_rows_hash(const uint64_t* row_ptr, const uint64_t* col_idx, const double* values,
                      const uint64_t* rows, uint64_t n_sample);

#ifdef __cplusplus
}
#endif
#endif
