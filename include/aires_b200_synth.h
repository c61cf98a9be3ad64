/*
 * aires_b200_synth.h -- seeded synthetic inputs for the benchmark shapes (host, C++ threads).
 *
 * Not part of the reference hot path: these generate the inputs BASELINE.md §4 names.
 *   aires_b200_synth_graph    : Chung-Lu power-law adjacency, symmetrized, self-loops
 *                               dropped, duplicates merged (value 1), seeded relabel; with
 *                               normalize=1 it returns Ã = D̂^-½(A+I)D̂^-½ with the exact
 *                               arithmetic of normalize_adjacency (gcn.hpp:29-72).
 *   aires_b200_synth_features : the reference's gen_features (synth.hpp:73-78) draw for draw
 *                               (std::mt19937_64), so X is byte-identical to the reference's.
 *   aires_b200_synth_weights  : the reference's gen_weights (synth.hpp:81-86), same draws.
 * Outputs go through the aires_b200_output allocator (location must be HOST).
 */
#ifndef AIRES_B200_SYNTH_H
#define AIRES_B200_SYNTH_H

#include <stdint.h>

#include "aires_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct aires_b200_graph_spec {
  uint64_t n;            /* nodes */
  uint64_t target_nnz;   /* stored nnz of A before self-loops ("edges", both directions) */
  double alpha;          /* Chung-Lu weight exponent: w_i = (i + i0)^-alpha */
  uint64_t degree_cap;   /* expected degree of the heaviest node (sets i0) */
  uint64_t seed;         /* edge sampling seed */
  uint64_t relabel_seed; /* node permutation seed */
  int32_t relabel;       /* 1 = apply the seeded permutation */
  int32_t normalize;     /* 1 = return Ã (self-loops added, symmetric normalization) */
  int32_t threads;       /* host threads (0 = all) */
  int32_t reserved;
} aires_b200_graph_spec;

/* stats (optional, 8 doubles): [nnz(A) before self-loops, max degree, mean degree,
   rounds, seconds, i0, 0, 0] */
int aires_b200_synth_graph(const aires_b200_graph_spec* spec, aires_b200_output* out, double* stats);

int aires_b200_synth_features(uint64_t n, uint64_t dim, double sparsity_pct, uint64_t seed,
                              aires_b200_output* out);

/* the reference's gen_weights (synth.hpp:81-86): row-major in_dim x out_dim, U[0,1) - 0.5 */
int aires_b200_synth_weights(uint64_t in_dim, uint64_t out_dim, uint64_t seed, double* out);

#ifdef __cplusplus
}
#endif
#endif
