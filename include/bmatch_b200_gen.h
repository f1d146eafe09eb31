/*
 * bmatch_b200_gen.h — host-side synthetic graph generators and CSC helpers
 * for the five BASELINE configs. Not on the matching hot
 * path; they replace the reference's single-threaded generate_random_bipartite
 * + from_edge_list (csr_graph.cpp:10-43, 92-112), which take ~400 s at 1.6e9
 * edges.
 *
 * Protocol: the caller allocates cxadj[nc+1] and cadj[capacity] (capacity from
 * the matching *_capacity function, an upper bound on the edge count before
 * de-duplication); the generator writes a sorted, duplicate-free CSC and
 * returns the edge count in *nedges. `threads` <= 0 uses every host core.
 */
#ifndef BMATCH_B200_GEN_H
#define BMATCH_B200_GEN_H

#include <stdint.h>

#include "bmatch_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Bit-identical to the reference's generate_random_bipartite(nc, nr,
 * avg_degree, seed) (csr_graph.cpp:92-112): libstdc++ mt19937_64 +
 * uniform_int_distribution<int>, llround(nc*avg_degree) candidates, then sort +
 * unique. The sequential random stream is replayed from per-chunk engine
 * snapshots so counting and scattering run on all cores. */
int64_t   bm_gen_uniform_capacity(int32_t nc, double avg_degree);
bm_status bm_gen_uniform(int32_t nc, int32_t nr, double avg_degree, uint64_t seed, int32_t threads,
                         int64_t* cxadj, int32_t* cadj, int64_t* nedges);

/* C2: n x n with a planted perfect matching (c, pi(c)) for a keyed Feistel
 * permutation pi, plus llround((avg_degree-1)*n) uniform (c, r) pairs drawn
 * with replacement from a counter-based splitmix64 stream. Maximum = n. */
int64_t   bm_gen_planted_capacity(int32_t n, double avg_degree);
bm_status bm_gen_planted(int32_t n, double avg_degree, uint64_t seed, int32_t threads,
                         int64_t* cxadj, int32_t* cadj, int64_t* nedges);

/* C3: bipartite R-MAT, nc = nr = 2^scale, llround(edge_factor*2^scale)
 * candidates; per bit level the quadrant is drawn with probabilities
 * (a, b, c, 1-a-b-c) (Graph500: 0.57, 0.19, 0.19); row bit = q>>1, column
 * bit = q&1. permute != 0 relabels rows and columns with independent keyed
 * permutations (the RCP experiments). */
int64_t   bm_gen_rmat_capacity(int32_t scale, double edge_factor);
bm_status bm_gen_rmat(int32_t scale, double edge_factor, double a, double b, double c, uint64_t seed,
                      int32_t permute, int32_t threads, int64_t* cxadj, int32_t* cadj, int64_t* nedges);

/* C4: banded, structurally deficient: column c -> rows {c, ..., c+band-1}
 * within [0, n), minus every row of a seeded delete_frac share of rows.
 * Maximum = number of live rows (returned in *live_rows). */
int64_t   bm_gen_banded_capacity(int32_t n, int32_t band);
bm_status bm_gen_banded(int32_t n, int32_t band, double delete_frac, uint64_t seed, int32_t permute,
                        int32_t threads, int64_t* cxadj, int32_t* cadj, int64_t* nedges,
                        int64_t* live_rows);

/* The column and row permutations of the reference's permute_random(g, seed)
 * (csr_graph.cpp:68-90): one mt19937_64, columns drawn first. */
bm_status bm_permutation_pair(int32_t nc, int32_t nr, uint64_t seed, int32_t* cperm, int32_t* rperm);

/* Structural check of a CSC (check_csr, csr_graph.cpp:45-64): returns BM_OK or
 * BM_ERR_INVALID_ARG with the first violation in bm_last_error(). */
bm_status bm_check_csc(int32_t nc, int32_t nr, const int64_t* cxadj, const int32_t* cadj);

/* 64-bit FNV-1a style digest of (nc, nr, cxadj, cadj), used by golden fixtures. */
uint64_t  bm_csc_digest(int32_t nc, int32_t nr, const int64_t* cxadj, const int32_t* cadj);

#ifdef __cplusplus
}
#endif

#endif /* BMATCH_B200_GEN_H */
