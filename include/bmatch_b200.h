/*
 * bmatch_b200.h — C ABI of the B200-native maximum-cardinality bipartite
 * matching engine (APFB/APsB x GPUBFS/GPUBFS-WR, ALTERNATE + FIXMATCHING,
 * arXiv 1303.1379).
 *
 * This is the drop-in boundary for the reference's hot path. Every entry
 * point names the reference interface it replaces (paths relative to
 * /root/reference/proj). Plain C types only: int32/int64 arrays, sizes,
 * opaque handles. Host buffers are always caller-owned; the library never
 * retains a host pointer after a call returns.
 *
 * Reference interfaces replaced:
 *   apfb(g, init, grid, schedule, kernel, observer)        include/bmatch/gpu_match.hpp:133-135
 *   apsb(g, init, grid, schedule, kernel, improved, obs)   include/bmatch/gpu_match.hpp:141-144
 *   DriverResult{matching, counters}                       include/bmatch/gpu_match.hpp:126-129
 *   PhaseCounters                                          include/bmatch/gpu_match.hpp:39-52
 *   PhaseEvent / PhaseObserver                             include/bmatch/gpu_match.hpp:115-124
 *   BipartiteCsr{nc,nr,cxadj(int64),cadj(int32)}           include/bmatch/csr_graph.hpp:18-31
 *   MatchingState{rmatch,cmatch}                           include/bmatch/matching.hpp:15-25
 *   cheap_matching (init)                                  src/matching.cpp:13-26
 *   registry ids {apfb,apsb}-{gpubfs,wr}                   src/algorithms.cpp:19-27
 *
 * Error model (mirrors the reference's exceptions, see bm_status):
 *   std::invalid_argument  -> BM_ERR_INVALID_ARG  (e.g. matching.cpp:71-73)
 *   std::logic_error       -> BM_ERR_LOGIC        (gpu_match.cpp:77-80, 272-274)
 *   std::runtime_error     -> BM_ERR_BOUND_EXCEEDED (nc+1 phase bound, gpu_match.cpp:317-320)
 *   ParseError{line}       -> BM_ERR_PARSE        (matrix_market.cpp:29-99; bmatch_b200_io.h)
 *   "cannot open" etc.     -> BM_ERR_IO           (matrix_market.cpp:103-104)
 * The message of the last failure on the calling thread is bm_last_error().
 * There is no CPU fallback: without a usable sm_100 device every compute
 * entry point fails with BM_ERR_CUDA.
 *
 * Tuning environment variables (read at upload / launch; defaults are the
 * measured best): BM_ROW_LAYOUT=plain|interleave (row-state
 * layout, default by rmatch size), BM_BU_FRAC (share of the edges a frontier
 * must hold to be pulled: default 0.45, or 0.2 once the row state is
 * interleaved, i.e. far beyond L2), BM_BU_AUTO
 * (0|1: overrides the AUTO decision), BM_SOLO_EDGES
 * (widest level run by one CTA, default 1024), BM_PERSIST_MB (L2 persisting
 * window on the row state, default off), BM_LATE=0|1 (late phases: phases
 * with at most BM_LATE_ROOTS roots, default max(65536, nc / 200), first try a bounded
 * meet-in-the-middle search; default on for pulling runs of graphs with at
 * least 2^22 columns; bounds BM_LATE_BCAP, BM_LATE_FCAP, BM_LATE_FPER,
 * BM_LATE_BLV, BM_LATE_FLV).
 */
#ifndef BMATCH_B200_H
#define BMATCH_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BM_ABI_VERSION 1

typedef enum bm_status {
  BM_OK = 0,
  BM_ERR_INVALID_ARG = 1,
  BM_ERR_LOGIC = 2,
  BM_ERR_BOUND_EXCEEDED = 3,
  BM_ERR_CUDA = 4,
  BM_ERR_OOM = 5,
  BM_ERR_NCCL = 6,
  BM_ERR_PARSE = 7,  /* malformed input file: the reference's ParseError (parse_error.hpp:9-14) */
  BM_ERR_IO = 8      /* a file cannot be opened, read or written */
} bm_status;

/* Driver: APFB = augment along every path found per phase (gpu_match.hpp:131-135);
 * APSB = break the level loop at the first level that finds a path (gpu_match.hpp:137-144). */
typedef enum bm_driver { BM_DRIVER_APFB = 0, BM_DRIVER_APSB = 1 } bm_driver;

/* BFS kernel: GPUBFS (Alg. 2, gpu_match.cpp:23-72) or GPUBFS-WR (Alg. 4, gpu_match.cpp:74-135). */
typedef enum bm_bfs_kernel { BM_BFS_GPUBFS = 0, BM_BFS_WR = 1 } bm_bfs_kernel;

/* Initial matching: GIVEN = use the caller's rmatch/cmatch (the reference's
 * methodology: cheap_matching on the host, bench.cpp:52-63); GPU_GREEDY =
 * parallel first-fit on the device; GPU_KS = degree-1 columns first, then
 * parallel first-fit (one-sided Karp-Sipser priority). */
typedef enum bm_init { BM_INIT_GIVEN = 0, BM_INIT_GPU_GREEDY = 1, BM_INIT_GPU_KS = 2 } bm_init;

typedef struct bm_match_opts {
  int32_t driver;            /* bm_driver */
  int32_t bfs_kernel;        /* bm_bfs_kernel */
  int32_t improved;          /* endpoint-encoded WR + alternate_wr (requires BM_BFS_WR),
                                gpu_match.cpp:188-218; algorithms.cpp:19-27 enables it for apsb-wr */
  int32_t init;              /* bm_init */
  int32_t max_phases;        /* 0 = run to the maximum (bound nc+1); >0 = stop after that many
                                outer iterations and return with *done = 0 (resumable) */
  int32_t claim_policy;      /* bm_claim_policy (WR only): which trees may claim a column */
  int32_t endpoint_policy;   /* bm_endpoint_policy (WR only): how many free rows a tree may hold */
  int32_t bottom_up;         /* bm_bottom_up: whether levels whose frontier holds >= 45% of
                                the edges (20% once the row state is interleaved) are pulled
                                (direction-optimised); they need a row index
                                of the graph (E ints), built by bm_prepare_row_index or the
                                first such run after an upload */
} bm_match_opts;

/* OFF: push every level. ON: pull dense levels (builds the row index on the
 * first run after an upload). AUTO: pull them on graphs of the kind where that
 * pays (bm_bottom_up_auto: >= 2M rows, so the row state outgrows what L2 keeps
 * close; >= 75% non-empty columns; average degree >= 8 over those, i.e. a BFS
 * whose middle levels cover most columns), once the row index exists
 * (bm_prepare_row_index) or right away at >= 2^26 rows, where one run repays
 * building it. Measured on B200: -20% per run on C2, -45% on C5; C1, C3 and
 * C4 do not qualify. BM_BU_AUTO=0|1 overrides the graph test. */
typedef enum bm_bottom_up { BM_BU_OFF = 0, BM_BU_ON = 1, BM_BU_AUTO = 2 } bm_bottom_up;

/* Column claims under GPUBFS-WR. REFERENCE: a tree whose root already found a
 * path keeps claiming columns at discovery; they are skipped at expansion
 * (gpu_match.cpp:106-108). AT_DISCOVERY: such a tree also stops claiming, which
 * leaves the columns to live trees (one coherent root-mark read per claim). */
typedef enum bm_claim_policy { BM_CLAIM_REFERENCE = 0, BM_CLAIM_AT_DISCOVERY = 1 } bm_claim_policy;

/* Free-row (endpoint) claims under GPUBFS-WR. AUTO = ONE_PER_TREE for the WR
 * kernels. EVERY: every free row a tree reaches is flagged -2 (gpu_match.cpp:
 * 120-125); all but one are wasted, since a tree augments along one path, and
 * they are unavailable to other trees until FIX. ONE_PER_TREE: the first free
 * row a tree claims is recorded at its root (atomic CAS on bfs_array[root]);
 * a tree that already holds one releases any further row it flagged, so the
 * row stays available to other trees in the same phase. Correctness does not
 * depend on it (ALTERNATE's claim check + FIX do; the last phase is still a
 * full BFS that finds no path). GPUBFS has no roots and always uses EVERY. */
typedef enum bm_endpoint_policy {
  BM_EP_AUTO = 0,
  BM_EP_EVERY = 1,
  BM_EP_ONE_PER_TREE = 2
} bm_endpoint_policy;

/* PhaseCounters (gpu_match.hpp:39-52) plus the device-side work counters the
 * roofline accounting needs. */
typedef struct bm_counters {
  int64_t outer_iterations;
  int64_t bfs_launches_total;      /* sum of bfs_launches_per_iteration (BFS levels expanded) */
  int64_t columns_scanned;         /* columns expanded (passed level + WR tests): reference counter */
  int64_t alternations_attempted;  /* walks started */
  int64_t fix_resets;
  int64_t serial_retries;
  int64_t edges_traversed;         /* E_trav: adjacency entries read by expanded columns */
  int64_t columns_visited;         /* N_vis: columns newly labelled (bitmap claims) */
  int64_t walk_steps;              /* L_walk: pair swaps performed by ALTERNATE */
  int64_t frontier_entries;        /* frontier entries processed (incl. WR-skipped) */
  int64_t cardinality;             /* final cardinality (count of rmatch >= 0) */
  int64_t initial_cardinality;     /* cardinality of the (given or GPU-built) initial matching */
  int64_t n_phase_records;         /* number of valid entries written to bfs_launches_per_iteration */
  int64_t reserved[3];
} bm_counters;

/* PhaseEvent (gpu_match.hpp:115-123). rmatch/cmatch point at a host snapshot
 * valid only during the callback. Return nonzero to abort the run
 * (bm_run then returns BM_ERR_INVALID_ARG with "aborted by observer"). */
typedef struct bm_phase_event {
  int64_t iteration;
  int32_t augmenting_path_found;
  int32_t serial_retry;
  int64_t cardinality_before;
  int64_t cardinality_after;
  int64_t bfs_launches;
  const int32_t* rmatch; int32_t nr;
  const int32_t* cmatch; int32_t nc;
} bm_phase_event;

typedef int (*bm_phase_cb)(const bm_phase_event* ev, void* user);

typedef struct bm_handle bm_handle;

/* ---- lifecycle ------------------------------------------------------- */
int32_t     bm_abi_version(void);
const char* bm_last_error(void);                       /* thread-local message of the last failure */
const char* bm_status_string(int32_t status);
int32_t     bm_device_count(void);                     /* 0 when no CUDA device is usable */
bm_status   bm_create(int32_t device, bm_handle** out);
bm_status   bm_destroy(bm_handle* h);
/* Use an external CUDA stream (cudaStream_t passed as void*; NULL = the handle's own). */
bm_status   bm_set_stream(bm_handle* h, void* stream);

/* ---- graph: device-resident CSC (replaces BipartiteCsr, csr_graph.hpp:18-31) ----
 * Copies cxadj[nc+1] (int64, cxadj[0]=0, non-decreasing) and cadj[E]
 * (int32 row ids in [0,nr)) to HBM. Validation (check_csr, csr_graph.cpp:45-64,
 * minus the per-column sortedness rule the kernels do not rely on) runs on the
 * device; a violation returns BM_ERR_INVALID_ARG. E must be < 2^32. */
bm_status   bm_upload_csc(bm_handle* h, int32_t nc, int32_t nr,
                          const int64_t* cxadj, const int32_t* cadj);
bm_status   bm_graph_info(bm_handle* h, int32_t* nc, int32_t* nr, int64_t* nedges);
/* BM_BU_AUTO for the resident graph: 0 = pushes; 1 = pulls its dense levels
 * once the row index is prepared; 2 = pulls them from the first run. */
bm_status   bm_bottom_up_auto(bm_handle* h, int32_t* enabled);
/* Builds the row index the pulled levels read (4E + 8E bytes of device
 * memory; about 6 ms for 1.6e8 edges), so that BM_BU_AUTO pulls from the next
 * run on. Call it once per upload when the same graph is matched repeatedly;
 * a single match of a graph below 2^26 rows does not repay it and pushes. */
bm_status   bm_prepare_row_index(bm_handle* h);
/* The row index as the pulled levels read it: roffs[nr + 1] (uint32) and
 * radj[E] (int32), the columns of row r in radj[roffs[r], roffs[r + 1]) in no
 * particular order. BM_ERR_INVALID_ARG when it has not been built. Either
 * pointer may be NULL. (Diagnostics and tests: the one-pass build and the
 * build that bm_upload_csc overlaps with the copy must agree.)
 *
 * bm_upload_csc builds the row index while it copies the adjacency (chunk by
 * chunk, on a second stream; only the final scatter is left when the copy
 * ends, and the next run waits for it) on graphs where AUTO pulls from the
 * first run (>= 2^26 rows and E >= 6 nc), or of >= 2^22 rows whose sampled
 * columns pass AUTO's test (late phases). BM_PREBUILD=1|0 forces it on|off. */
bm_status   bm_download_row_index(bm_handle* h, uint32_t* roffs, int32_t* radj);

/* ---- matching: the reference-shaped one-call entry ----------------------
 * Replaces apfb()/apsb() (gpu_match.hpp:133-144): rmatch[nr]/cmatch[nc] are
 * the initial matching on input when opts->init == BM_INIT_GIVEN (ignored
 * otherwise) and the maximum matching on output. bfs_launches_per_iteration
 * (nullable) receives one entry per outer iteration, up to `cap` entries;
 * counters->n_phase_records says how many were written. */
bm_status   bm_match(bm_handle* h, const bm_match_opts* opts,
                     int32_t* rmatch, int32_t* cmatch,
                     int64_t* cardinality, bm_counters* counters,
                     int64_t* bfs_launches_per_iteration, int64_t cap,
                     bm_phase_cb cb, void* user);

/* ---- device-resident path (inputs already in HBM; used by the bench) ---- */
bm_status   bm_load_matching(bm_handle* h, const int32_t* rmatch, const int32_t* cmatch);
/* Runs from the loaded initial matching (a device-to-device copy, so repeated
 * runs start from the same state); the result stays on the device. *done is
 * 1 when the matching is maximum, 0 when max_phases stopped it early
 * (call bm_resume to continue). */
bm_status   bm_run(bm_handle* h, const bm_match_opts* opts, int64_t* cardinality,
                   bm_counters* counters, int64_t* bfs_launches_per_iteration,
                   int64_t cap, bm_phase_cb cb, void* user, int32_t* done);
bm_status   bm_resume(bm_handle* h, const bm_match_opts* opts, int64_t* cardinality,
                      bm_counters* counters, int64_t* bfs_launches_per_iteration,
                      int64_t cap, bm_phase_cb cb, void* user, int32_t* done);
bm_status   bm_download_matching(bm_handle* h, int32_t* rmatch, int32_t* cmatch);
/* Device time (ms, CUDA events on the handle's stream) of the driver kernel
 * launches of the last bm_run/bm_resume/bm_match, and how many kernels that
 * run launched (driver launches plus the initial-state copy kernel). */
bm_status   bm_last_kernel_time(bm_handle* h, double* ms, int32_t* launches);
/* BFS launches (levels) of every outer iteration of the last bm_run / bm_resume /
 * bm_match (PhaseCounters::bfs_launches_per_iteration): *n receives the count,
 * out (nullable) up to cap entries. Lets a caller pass a small per_iter buffer
 * to bm_match and fetch the rest only when the run had more phases. */
bm_status   bm_last_phase_launches(bm_handle* h, int64_t* out, int64_t cap, int64_t* n);

/* Fault injection for the failure-path tests (no reference counterpart; every
 * key defaults to off). PHASE_BOUND: replaces the nc+1 termination bound of
 * run_driver (gpu_match.cpp:313-320) by `value` phases (0 = nc+1), so a run
 * that needs more phases fails with BM_ERR_BOUND_EXCEEDED. SKIP_ALTERNATE_PHASE:
 * outer iteration `value` (1-based; 0 = none) runs its raced ALTERNATE as a
 * no-op, i.e. finds paths but augments none, which forces the serial retry of
 * gpu_match.cpp:328-343 (serial_retries = 1). */
typedef enum bm_debug_key { BM_DEBUG_PHASE_BOUND = 1, BM_DEBUG_SKIP_ALTERNATE_PHASE = 2 } bm_debug_key;
bm_status   bm_debug_set(bm_handle* h, int32_t key, int64_t value);

/* Stage timeline of the last bm_run/bm_resume/bm_match: `n` records of two
 * uint64 each, (tag, device %globaltimer in ns). tag = (kind << 32) | arg with
 * kind 0 start, 1 init pass, 2 setup, 3 BFS level (arg = frontier entries),
 * 4 ALTERNATE, 5 FIX rows, 6 FIX columns, 7 roots of the next phase, 8 end,
 * 9 the preceding level's frontier edges (arg; same timestamp), 10 the
 * preceding pushed level's pairs turned into entries (materialize), 11 the
 * preceding pulled level's frontier bitmap built (pull prep), 12 the
 * preceding bucketed pushed level's partition pass done, 13 a late phase's
 * level (arg = entries; top bit set: backward), 14 a late phase's end
 * (arg = paths flipped).
 * Written by one thread after each grid barrier (a few ns per stage). */
bm_status   bm_timeline(bm_handle* h, uint64_t* out, int64_t cap, int64_t* n);

/* Raw device counters of the last run (profiling): edges traversed, columns
 * expanded/visited, frontier entries, walks, walk steps, FIX resets, levels,
 * serial retries, dense-FIX fallbacks, then per-part CTA cycle totals
 * (tile fetch, window setup, rounds, flush, grid barrier, other). */
bm_status   bm_debug_stats(bm_handle* h, uint64_t* out, int64_t cap, int64_t* n);

/* ---- one BFS phase without ALTERNATE/FIX (parity probes) ----------------
 * Mirrors run_phase up to expand_bfs (gpu_match.cpp:268-290) from the given
 * matching and returns the phase arrays: bfs_array[nc] (levels, L0 = 2),
 * predecessor[nr], and rmatch[nr] with -2 endpoint flags. Any pointer may be
 * NULL. *launches receives the number of levels expanded. */
bm_status   bm_bfs_phase(bm_handle* h, int32_t driver, int32_t bfs_kernel, int32_t improved,
                         const int32_t* rmatch_in, const int32_t* cmatch_in,
                         int32_t* bfs_array, int32_t* predecessor, int32_t* rmatch_out,
                         int64_t* launches, int32_t* path_found);

/* ---- GPU Berge certificate (replaces validate + is_maximum, matching.cpp:70-131) ----
 * Runs on the device against the uploaded graph. *violations = number of
 * validity violations (pending -2, asymmetry, non-edge, out of range);
 * *is_max = 1 when no augmenting path exists (only meaningful when
 * *violations == 0). */
bm_status   bm_verify(bm_handle* h, const int32_t* rmatch, const int32_t* cmatch,
                      int64_t* violations, int32_t* is_max, int64_t* cardinality);

/* ---- random relabelling on the device (permute_random, csr_graph.cpp:80-90) ----
 * Relabels the uploaded graph: column c becomes cperm[c], row r becomes
 * rperm[r], and each column's rows are re-sorted (the RCP experiments,
 * PAPER.md:444-445). With the permutations of bm_permutation_pair(seed) the
 * result is bit-identical to the reference's permute_random(g, seed). Any
 * loaded initial matching is dropped. bm_download_csc returns the resident
 * graph (cxadj[nc+1], cadj[E]). */
bm_status   bm_permute_random(bm_handle* h, const int32_t* cperm, const int32_t* rperm);
bm_status   bm_download_csc(bm_handle* h, int64_t* cxadj, int32_t* cadj);

/* ---- multi-GPU engine: one persistent kernel per rank over peer memory ----
 * (the reference has no multi-device path, its only
 * parallelism is the emulated grid, kernel_grid.hpp:161-222.)
 * 1-D partition: rank q owns columns [cb[q], cb[q+1]) with their CSC slice,
 * cmatch and root marks, and rows [rb[q], rb[q+1]) with their row state and
 * (pulled levels) their slice of the row index. The whole APFB/APsB driver
 * (run_driver, gpu_match.cpp:306-376) runs as ONE cooperative launch per rank:
 * claims are system-scope atomics at the row's owner, winner columns are
 * stored into their owner's inbox, and the level barrier spans the team,
 * all over peer memory (CUDA IPC / NVLink; plain pointers for ranks of one
 * process). No host round trip per level, no collective on the data path.
 * Protocol (every rank):
 *   bm_mg_create(device, rank, world, share)   share = ranks on this device
 *   bm_mg_upload(slice)                        bounds from bm_mg_partition
 *   bm_mg_export(blob) -> all-gather blobs -> bm_mg_import(all blobs)
 *   [bm_mg_row_index_begin, host barrier, bm_mg_row_index_end]  pulled levels
 *   bm_mg_load_matching(own rows, own columns), host barrier
 *   bm_mg_launch (every rank) then bm_mg_finish  (= bm_mg_run)
 *   bm_mg_download(own rows, own columns)
 * Status codes as for the single-GPU engine; BM_ERR_BOUND_EXCEEDED for the
 * nc + 1 bound (gpu_match.cpp:313-320). */
typedef struct bm_mg bm_mg;
bm_status   bm_mg_partition(int32_t n, int32_t world, int32_t* bounds /* world + 1 */);
bm_status   bm_mg_create(int32_t device, int32_t rank, int32_t world, int32_t share, bm_mg** out);
bm_status   bm_mg_destroy(bm_mg* h);
bm_status   bm_mg_set_stream(bm_mg* h, void* stream);
/* cxadj[cb[rank+1]-cb[rank]+1] rebased to 0, cadj its rows (global ids) */
bm_status   bm_mg_upload(bm_mg* h, int32_t nc, int32_t nr, int64_t e_total, const int32_t* cb,
                         const int32_t* rb, const int64_t* cxadj, const int32_t* cadj);
bm_status   bm_mg_blob_size(int64_t* bytes);
bm_status   bm_mg_export(bm_mg* h, void* blob);
bm_status   bm_mg_import(bm_mg* h, const void* blobs /* world blobs, rank order */);
bm_status   bm_mg_row_index_begin(bm_mg* h);
bm_status   bm_mg_row_index_end(bm_mg* h);
bm_status   bm_mg_load_matching(bm_mg* h, const int32_t* rmatch_slice, const int32_t* cmatch_slice);
bm_status   bm_mg_launch(bm_mg* h, const bm_match_opts* opts);
bm_status   bm_mg_finish(bm_mg* h, int64_t* cardinality, bm_counters* counters /* this rank's work */);
bm_status   bm_mg_run(bm_mg* h, const bm_match_opts* opts, int64_t* cardinality, bm_counters* counters);
bm_status   bm_mg_download(bm_mg* h, int32_t* rmatch_slice, int32_t* cmatch_slice);
bm_status   bm_mg_kernel_time(bm_mg* h, double* ms);
bm_status   bm_mg_info(bm_mg* h, int64_t* local_edges, int64_t* row_index_edges, int32_t* pulled_capable);

#ifdef __cplusplus
}
#endif

#endif /* BMATCH_B200_H */
