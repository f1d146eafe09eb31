/*
 * bm_oracle.h — CPU restatement of the reference's matching path, in plain C.
 *
 * TEST INFRASTRUCTURE ONLY. This is the parity checker for the B200 engine:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load it, and only to check or to time the CPU side. The product path
 * (paper_1303_1379_b200) never calls it and fails loudly without its CUDA
 * library.
 *
 * Each function names the reference code it restates (paths relative to
 * /root/reference/proj). The grid functions reproduce the reference's
 * *Serial* schedule exactly (virtual threads tid = 0..tot-1 in order, each
 * visiting vertices i*tot + tid, kernel_grid.hpp:117-126, 166-170), so their
 * traces and counters are bit-identical to the reference's on the same
 * inputs; the pinning tests check that against fixtures produced by the
 * reference itself (tests/golden/).
 */
#ifndef BM_ORACLE_H
#define BM_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct or_graph {
  int32_t nc, nr;
  const int64_t* cxadj; /* nc + 1 */
  const int32_t* cadj;  /* cxadj[nc] */
} or_graph;

/* PhaseCounters (gpu_match.hpp:39-52); launches[] optional. */
typedef struct or_counters {
  int64_t outer_iterations;
  int64_t columns_scanned;
  int64_t alternations_attempted;
  int64_t fix_resets;
  int64_t serial_retries;
  int64_t bfs_launches_total;
  int64_t* launches;      /* caller buffer, one entry per outer iteration (may be NULL) */
  int64_t launches_cap;
} or_counters;

/* matching.cpp:13-26 */
void    or_cheap_matching(const or_graph* g, int32_t* rmatch, int32_t* cmatch);
/* matching.cpp:28-31 */
int64_t or_cardinality(int32_t nr, const int32_t* rmatch);
/* matching.cpp:70-104: number of violations (0 = valid). */
int64_t or_validate(const or_graph* g, const int32_t* rmatch, const int32_t* cmatch);
/* matching.cpp:106-131: 1 maximum, 0 not maximum, -1 invalid state. */
int32_t or_is_maximum(const or_graph* g, const int32_t* rmatch, const int32_t* cmatch);
/* matching.cpp:133-172 (small graphs only: recursion depth <= nc). */
int64_t or_brute_force_maximum(const or_graph* g);
/* baselines.cpp:17-93: Hopcroft-Karp from the given matching (in/out). */
void    or_hopcroft_karp(const or_graph* g, int32_t* rmatch, int32_t* cmatch);
/* tests/oracles.hpp:16-37: hop depth from the nearest unmatched column, -1 unreachable. */
void    or_alternating_bfs_depths(const or_graph* g, const int32_t* rmatch, const int32_t* cmatch,
                                  int32_t* depth);

/* gpu_match.cpp:8-21 */
void    or_init_bfs_array(int32_t nc, const int32_t* cmatch, int32_t start_level, int32_t* bfs);
void    or_init_root(int32_t nc, const int32_t* cmatch, int32_t* root);

/* One level, Serial schedule over tot virtual threads (gpu_match.cpp:23-72 /
 * 74-135). flags[0] = vertex_inserted, flags[1] = augmenting_path_found
 * (raised, never cleared). Returns columns scanned. root may be NULL for
 * the plain kernel. improved requires start_level == 2 (returns -1 otherwise). */
int64_t or_gpubfs(const or_graph* g, int32_t tot, int32_t bfs_level, int32_t start_level,
                  int32_t* bfs, int32_t* pred, int32_t* rmatch, int32_t* flags);
int64_t or_gpubfs_wr(const or_graph* g, int32_t tot, int32_t bfs_level, int32_t start_level,
                     int32_t improved, int32_t* bfs, int32_t* pred, int32_t* root, int32_t* rmatch,
                     int32_t* flags);
/* gpu_match.cpp:158-186 / 188-218; return walks attempted. */
int64_t or_alternate(const or_graph* g, int32_t tot, const int32_t* pred, int32_t* rmatch, int32_t* cmatch);
int64_t or_alternate_wr(const or_graph* g, int32_t tot, const int32_t* bfs, const int32_t* pred,
                        int32_t* rmatch, int32_t* cmatch);
/* gpu_match.cpp:220-245; returns resets. */
int64_t or_fix_matching(int32_t nc, int32_t nr, int32_t* rmatch, int32_t* cmatch);

/* Whole driver, Serial schedule (gpu_match.cpp:306-376). tot = grid threads
 * (GridConfig::threads_for). kernel: 0 GPUBFS, 1 WR. rmatch/cmatch in/out.
 * Returns 0 ok, 2 logic error (improved without WR), 3 bound exceeded. */
int32_t or_driver(const or_graph* g, int32_t tot, int32_t shortest, int32_t kernel, int32_t improved,
                  int32_t* rmatch, int32_t* cmatch, or_counters* counters);

#ifdef __cplusplus
}
#endif

#endif /* BM_ORACLE_H */
