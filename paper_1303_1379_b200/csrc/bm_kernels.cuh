// bm_kernels.cuh — the device side of the engine: the persistent driver kernel
// and its stages, plus the upload / verify / row-index kernels.
//
// Included twice, inside a namespace, with no includes of its own:
//   * bm_engine.cu:  namespace bm   — the single-GPU engine (BM_MG undefined);
//   * bm_mg.cu:      namespace bmg  — the multi-GPU engine (BM_MG = 1): the same
//     stages, with the row state, cmatch, root marks and frontier roots of other
//     ranks reached through peer pointers (see the BM_MG blocks).
// The includer provides <cooperative_groups.h> (as cg), CUB, bm_device.cuh and
// bmatch_b200.h.

#ifndef BM_THREADS
#define BM_THREADS 256
#endif
constexpr int kThreads = BM_THREADS;  // threads per CTA (1024 / kThreads CTAs per SM at <= 64 registers)
#ifndef BM_ITEMS
#define BM_ITEMS 4
#endif
// Resident CTAs per SM (launch bounds), per kernel family: the pulled-capable
// kernels run 3 (80 registers; A/B on C5/C2 against 4: -1.6 %/-5 % per phase
// before the phase count's noise), the push-only kernels 4 (64 registers; C3
// -8 %, C4 and C1 even). BM_MINB overrides both.
#ifdef BM_MINB
#define BM_MINB_BU BM_MINB
#define BM_MINB_PUSH BM_MINB
#endif
#ifndef BM_MINB_BU
#define BM_MINB_BU (768 / BM_THREADS)
#endif
#ifndef BM_MINB_PUSH
#define BM_MINB_PUSH (1024 / BM_THREADS)
#endif
constexpr int kItems = BM_ITEMS;      // edges per thread per round (memory-level parallelism)
#ifndef BM_EPT
#define BM_EPT 1
#endif
constexpr int kEPT = BM_EPT;          // frontier entries per thread in a push window
constexpr int kWin = kThreads * kEPT; // entries per push window
#ifndef BM_GRAN
#define BM_GRAN 512
#endif
constexpr unsigned kGran = BM_GRAN;   // edges per granule-index entry; tiles are whole granules
#ifndef BM_TILE_GRAN
#define BM_TILE_GRAN 8
#endif
constexpr unsigned kMaxTileGran = BM_TILE_GRAN;  // <= 4096 edges per tile (= the winner buffer)
constexpr unsigned kWBuf = kGran * kMaxTileGran;
#ifndef BM_INTERLEAVE_MB
#define BM_INTERLEAVE_MB 72  // interleave {mate, pred} when the plain rmatch exceeds this many MB
#endif
#ifndef BM_SOLO_EDGES
#define BM_SOLO_EDGES 1024
#endif
constexpr unsigned kSoloEdges = BM_SOLO_EDGES;  // widest level block 0 expands alone
// Frontier capacity per phase beyond nc: room for the duplicate entries that
// store claims can create (see expand_level). A level claims by store only when
// even one entry per frontier edge would fit, so the capacity can never overflow.
constexpr size_t kFSlack(long long nc) { return (size_t)(nc / 4 + 4096); }
// Inlining of the level functions into the persistent kernel (A/B knobs): a
// separately compiled function gets its own register allocation instead of
// sharing the driver's.
#define BM_NOINLINE_FN __device__ __noinline__  // (for -DBM_SWEEP_INLINE=BM_NOINLINE_FN)
#ifndef BM_SWEEP_INLINE
#define BM_SWEEP_INLINE __device__ __forceinline__
#endif
#ifndef BM_PREP_INLINE
#define BM_PREP_INLINE __device__ __forceinline__
#endif
#ifndef BM_MAT_INLINE
#define BM_MAT_INLINE __device__ __forceinline__
#endif
#ifndef BM_EXPAND_INLINE
#define BM_EXPAND_INLINE __device__ __forceinline__
#endif
#ifndef BM_PB_FN
#define BM_PB_FN BM_NOINLINE_FN  // push_bucketed: out of line (BM_PB_FN=BM_INLINE_FN to inline it)
#endif
#define BM_INLINE_FN __device__ __forceinline__
#ifndef BM_TAIL_FN
#define BM_TAIL_FN __device__ __forceinline__  // phase_tail (BM_NOINLINE_FN: out of line)
#endif
#ifndef BM_PHASE_FN
#define BM_PHASE_FN __device__  // run_phase (the compiler's choice; BM_NOINLINE_FN to force it out of line)
#endif
#ifndef BM_EXPAND_OOL
#define BM_EXPAND_OOL 1  // pulled-capable kernels call expand_level out of line (expand_level_ool)
#endif
constexpr int kStartLevel = 2;        // L0 (gpu_match.cpp:275)
constexpr int kUnvisited = kStartLevel - 1;
constexpr int kFoundMark = kStartLevel - 2;
constexpr unsigned long long kEdgeMask = (1ull << 33) - 1;
// "Column visited this phase" lives in bit 30 of its mate's rmatch entry: the
// gather rmatch[row] that finds a row's column also says whether that column
// was claimed, so a traversed edge costs one random access, not two. Needs
// nc < 2^30; cleared by sweep_visited() when the BFS ends.
constexpr int kVisBit = 1 << 30;

enum CtlError : int {
  kErrNone = 0,
  kErrBound = 1,        // more than nc + 1 phases (gpu_match.cpp:317-320)
  kErrInvalidInit = 2,  // initial matching is not a clean valid matching
  kErrBarrier = 3,      // grid barrier watchdog fired
  kErrWalk = 4,         // an ALTERNATE walk exceeded nc steps (cannot happen on valid state)
  kErrLevels = 5,       // more BFS levels than columns (cannot happen)
  kErrWindow = 6,       // a push window's live edges exceed its tile (inconsistent frontier entries)
  kErrCheck = 7,        // BM_CHECK=1 self-check of a level's entries failed (dbg holds the details)
};

struct alignas(128) Slot {
  unsigned long long packed;  // (entries << 33) | edges, pushed by the previous level
  unsigned tile;              // dynamic edge-tile counter while this level is expanded
  unsigned pad[29];
};

struct PhaseRec {
  long long launches;
  long long before;
  long long after;
  int found;
  int retry;
};

enum Stat : int {
  kStTrav = 0,
  kStCexp,
  kStNvis,
  kStEntries,
  kStWalks,
  kStSteps,
  kStResets,
  kStLevels,
  kStRetries,
  kStDenseFix,
  kStCycTile,     // CTA cycles (thread 0's view) per part of expand_level and in grid barriers
  kStCycWindow,
  kStCycRounds,
  kStCycFlush,
  kStCycBarrier,
  kStCycOther,
  kStRowsPulled,  // rows a pulled level screened in as candidates (scanned their own columns)
  kStPulledLevels,
  kStMaterialized,  // frontier entries turned from (col, root) pairs into edge-tiled entries
  kStCycBuScreen,   // pulled levels, warp cycles (lane 0's view): screening chunks into the candidate queue
  kStCycBuProbe,    // ... probe rounds
  kStCycBuFlush,    // ... winner and endpoint flushes
  kStBuRounds,      // ... probe rounds (warp-level)
  kStLatePhases,    // late phases run (late_phase), including ones that found nothing
  kStLatePaths,     // augmenting paths they flipped
  kStLateProofs,    // runs ended by a late phase's exhausted backward search (no full phase needed)
  kNumStats
};

constexpr int kBarSub = 16;  // grid barrier fan-in groups
constexpr int kPbMax = 64;   // row buckets of a bucketed pushed level

struct alignas(128) Ctrl {
  unsigned bar_count;
  unsigned bar_gen;
  unsigned pad0[30];
  unsigned bar_sub[kBarSub][32];  // one 128-byte line per group counter
  Slot lvl[3];
  Slot roots;
  Slot mat[2];  // materialize reservations, by level parity (never the level's own slot: slow CTAs
                // may still be reading its count when the next level starts)
  Slot rootp;   // multi-GPU: next-phase roots routed here by other ranks' FIX, as (c, c) pairs in P
  unsigned n_ep;
  unsigned pad1[31];
  // bucketed pushed level (push_bucketed), by level parity: per-bucket cursors,
  // overflow cursor, claim-pass ticket (reset after the level's barrier)
  unsigned pb_cur[2][64];
  unsigned pb_ovf[2];
  unsigned pb_ticket[2];
  unsigned n_left[3];  // pulled levels' leftover lists, by level mod 3 (see Params::left)
  unsigned pad1c[25];
  // late phases (late_phase): backward / forward queue counts by level mod 3, paths recorded
  unsigned lt_b[3];
  unsigned lt_f[3];
  unsigned lt_nep;
  unsigned lt_hit;  // the backward search met a free column (a path may exist)
  unsigned lt_ovf;  // a backward queue dropped an entry (the search was not exhaustive)
  unsigned pad1e[23];
  unsigned n_log;
  unsigned log_overflow;
  unsigned n_tl;
  unsigned pad1b[29];
  unsigned path_found[2];
  unsigned pad2[30];
  // hand-over from a solo run of narrow levels (block 0 alone) to the grid
  int solo_lv;
  int solo_stop;
  unsigned solo_ls;
  unsigned solo_n;
  unsigned solo_T;
  int solo_found;
  long long solo_launches;
  unsigned pad2b[24];
  unsigned long long invalid;
  unsigned long long isolated;
  unsigned long long init_rows;  // setup's check of a given initial matching: matched rows ...
  unsigned long long init_cols;  // ... and matched columns whose row points back
  unsigned long long pad3[12];
  unsigned long long stats[kNumStats];
  // run state carried between launches (written by block 0 / thread 0 on exit)
  long long outer;
  long long card;
  long long isolated_cols;
  long long init_card;
  long long bfs_levels_last;
  int cur;
  int done;
  int error;
  int n_recs;
  int path_found_last;
  int phase_parity;
  long long dbg[8];  // details of the first kErrWindow (ls, n, T, i, e, wend, live, level)
};

#ifndef BM_MG
#define BM_MG 0
#endif
constexpr int kMaxRanks = 8;

#if BM_MG
// One rank's state as every rank addresses it (multi-GPU engine, bm_mg.cu).
// Bases are pre-offset so that they take GLOBAL ids: row r of the owner's row
// range is rm + rs * r, column c of its column range is cmatch + c, etc. Peers
// are reached through CUDA IPC mappings (NVLink), or are other allocations on
// the same device when several ranks share one GPU.
struct PeerPtrs {
  int* rm;          // row state {mate, pred} (interleaved) or mates (plain)
  int* pred;
  int* cmatch;
  int* bfs;         // root marks
  int* croot;       // root of each frontier column (pulled levels)
  unsigned* dead;   // the rank's replica of the dead-root bitmap (all nc bits)
  unsigned* fbit;   // the rank's replicas of the frontier bitmaps (kNumFbit x all nc bits)
  int2* P;          // pair inbox: (column, root) winners routed to the column's owner
  int* EP;          // endpoint rows found by the rank
  int4* F0;
  int4* F1;
  struct Ctrl* ctl;
};
// Cross-rank barrier and the flags every rank reads (rank 0's memory).
struct alignas(128) MgTeam {
  unsigned count;
  unsigned gen;
  unsigned pad0[30];
  unsigned path_found[2];
  unsigned pad1[30];
};
#endif

// Frontier bitmaps of pulled levels, rotating by level (lv % 3): a level reads
// its own, its winners mark the next one, and the one two levels back is
// cleared meanwhile (no barrier needed between the clear and the next marks).
constexpr int kNumFbit = 3;

struct Params {
  int nc, nr;
  const unsigned* offs;  // nc + 1
  const int* adj;        // E
  int* rm;          // row state: mates at rm[rs * r]
  int rs;           // row stride: 2 = interleaved {mate, pred}, 1 = plain (pred in `pred`)
  int* cmatch;
  int* pred;
  int* bfs;
  unsigned* dead;   // WR: 1 bit per column, set when the tree rooted there holds an endpoint
  int ndead_words;
  int4* F0;
  int4* F1;
  unsigned* gidx0;  // granule index, ping-pong by level parity
  unsigned* gidx1;
  int* EP;
  int2* wlog;       // ALTERNATE write log: (row, col) per step, (row, -1) for a dangling row
  unsigned log_cap;
  Ctrl* ctl;
  PhaseRec* recs;
  int rec_cap;
  int apsb;
  int init_mode;
  int fresh;
  int init_checked;  // the given initial matching was validated when it was loaded (bm_load_matching)
  int sorted;        // every column's rows ascend (binary-searchable adjacency)
  int dbg_skip_alt_phase;  // fault injection (bm_debug_set): this phase's raced ALTERNATE does nothing
  int check;               // BM_CHECK=1: verify every pushed level's entries before expanding it (debugging)
  int max_phases;
  int stop_after_bfs;
  int trace;        // write bfs_array level labels (parity probes)
  int claim_mode;   // WR claim check at discovery: 0 none (reference), 1 coherent root-mark check
  int ep_one;       // WR endpoint policy: 1 = one free row per tree (root-mark CAS), 0 = every row (reference)
  unsigned solo_edges;  // levels with at most this many frontier edges run on block 0 alone (0 = never)
  // bottom-up levels (see bu_sweep); roffs == nullptr disables them
  const unsigned* roffs;   // nr + 1, transposed adjacency (rows -> columns)
  const int* radj;
  unsigned* fbit[kNumFbit];  // frontier bitmaps (nc bits each), rotating by level (lv % kNumFbit)
  int* croot;              // root of each frontier column (bottom-up levels)
  int nfbit_words;
  unsigned long long bu_min_edges;  // bu_rule 0: a level with at least this many frontier edges goes bottom-up
  int bu_rule;             // 0: bu_min_edges threshold; 1: frontier edges vs unexplored edges (below)
  float bu_alpha;          // bu_rule 1: pull when alpha * frontier edges >= edges of the unvisited rows ...
  unsigned bu_min_n;       // ... and the frontier holds at least this many columns
  double deg_col;          // E / nc: frontier edges of a level held as pairs are estimated from its size
  double deg_row;          // E / nr
  // Lazy frontier (pulled-capable kernels only): a wide level pushes its winners
  // as (col, root) pairs; the next level either pulls straight from them or,
  // when it is pushed, first turns them into edge-tiled entries (materialize).
  // Winners of a pulled level never need their offsets gathered.
  int2* P;                 // pairs, indexed like F (level entries [ls, ls + n))
  // Leftovers of a pulled level: the candidates that found no frontier column,
  // i.e. exactly the rows still unvisited afterwards (with their row state). A
  // pulled level after a pulled level takes its candidates from that list
  // instead of screening every row again. Rotating by level mod 3 (nr each).
  int2* left[3];
  unsigned long long pairs_min_edges;  // a pushed level this wide emits pairs
  long long phase_bound;
  unsigned long long fcap;  // frontier entries a phase may append (F0/F1 and P hold nc + kFSlack)
  int claim_store;          // pushed levels may claim by plain store (BM_CLAIM_STORE=0 disables)
  // Bucketed pushed levels (push_bucketed): a wide level's live edges are first
  // written as (row, col, root) triples grouped by row range, then claimed bucket
  // by bucket, so the row-state gathers and claims of a bucket hit an L2-sized window.
  int4* tb;                 // triples: pb_nb regions of pb_cap, then an overflow region
  unsigned long long pb_min_edges;  // a pushed level with at least this many edges (and <= pb_max) goes bucketed
  unsigned long long pb_max_edges;  // (0: never)
  int pb_shift;             // bucket of row r = r >> pb_shift
  int pb_nb;                // buckets (<= kPbMax)
  unsigned pb_cap;          // triples per bucket region
  // Bucketed bu_prep (bu_prep_bucketed): the frontier's (col, root) pairs grouped by
  // column range in the same buffer (as int2), so the root stores and bitmap
  // atomics of a bucket stay inside an L2-sized window. 0 buckets: off.
  int pp_shift;             // bucket of column c = c >> pp_shift
  int pp_nb;
  unsigned pp_cap;          // pairs per bucket region (int2 units of tb)
  unsigned long long pp_min; // a pulled level with at least this many frontier entries
  unsigned long long* tl;  // stage timeline: (tag, %globaltimer ns) pairs written by the leader
  unsigned tl_cap;
  // Late phases (late_phase; single GPU, pulled-capable runs; lt_col == nullptr: off)
  int2* lt_col;             // per column {epoch, row}: claimed by the backward search from that row
                            // ({epoch, -2} on a root: its tree holds a path)
  int* lt_croot;            // per column: the free row its backward tree started from
  int* lt_row;              // per row: epoch when a forward tree claimed it (on a free row: when it was used)
  int* lt_epoch;            // late phases so far (persistent across runs: the stamps are never reset)
  unsigned lt_qcap;         // entries per queue (two queues in P)
  unsigned lt_max_roots;    // a phase with at most this many roots is tried as a late phase first
  unsigned lt_bcap;         // backward search: stop once it claimed this many columns ...
  unsigned lt_fcap;         // forward search: ... this many frontier entries
  unsigned lt_fper;         // ... or 64K + this many per root still without a path
  int lt_blv, lt_flv;       // ... or after this many levels
#if BM_MG
  int world, rank;
  int col_lo, col_hi, row_lo, row_hi;  // this rank's columns and rows
  int cb[kMaxRanks - 1];               // column ownership: owner(c) = #{i : c >= cb[i]} (cb[i] = INT_MAX past world - 1)
  int rb[kMaxRanks - 1];               // row ownership, likewise
  int world_solo;                      // world == 1: narrow levels may still run on block 0 alone
  MgTeam* team;
  PeerPtrs peer[kMaxRanks];
#endif
};

enum TlTag : unsigned {
  kTlStart = 0, kTlInit = 1, kTlSetup = 2, kTlLevel = 3, kTlAlt = 4, kTlFixRows = 5, kTlFixCols = 6,
  kTlRoots = 7, kTlEnd = 8, kTlLevelEdges = 9, kTlMat = 10, kTlPrep = 11, kTlBucket = 12,
  kTlLateLevel = 13,  // a late phase's level: arg = entries (top bit: backward)
  kTlLate = 14        // a late phase ended: arg = paths flipped
};

__device__ __forceinline__ void tl_mark(const Params& p, unsigned kind, unsigned arg) {
  if (blockIdx.x == 0 && threadIdx.x == 0 && p.tl) {
    const unsigned n = p.ctl->n_tl;
    if (n < p.tl_cap) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      p.tl[2 * n] = ((unsigned long long)kind << 32) | arg;
      p.tl[2 * n + 1] = t;
    }
    p.ctl->n_tl = n + 1;
  }
}

// A pulled-level candidate row: its row-state value and its column range in the row index.
struct BuCand {
  int row;
  int val;
  unsigned j0;
  unsigned j1;
};
constexpr int kCandCap = 160;  // per-warp queue: < 32 left over + one screened chunk of 128 rows

struct Smem {
  union {  // a top-down window (a pulled level keeps its candidate queues in wbuf)
    struct {
      unsigned pre[kWin + 1];      // window: raw edge prefix of each entry, then the live-edge prefix
      int col[kWin];
      int root[kWin];
      unsigned beg[kWin];          // first live adjacency index of each entry in this window
    };
  };
  // 16-byte aligned: the compiler reads wtot with LDS.128. Unaligned, the first of
  // those loads also covered beg[kWin - 1] (value discarded), which racecheck
  // reported as a WAR hazard against the compaction's write of beg[] (profiles/README.md).
  alignas(16) unsigned wtot[kThreads / 32];
  unsigned short cgr[kWBuf / 32 + 2];  // entry holding live edge 32*q (coarse index for the search)
  unsigned tile;
  unsigned long long cnt[kNumStats];  // per-CTA work counters, flushed to Ctrl at exit
  unsigned long long wsum[kThreads / 32];  // CTA-aggregated pushes: per-warp totals
  unsigned wep[kThreads / 32];
  unsigned long long blk_base;
  unsigned blk_ep;
  unsigned pb_hist[kPbMax];   // bucketed push: this window's triples per bucket ...
  unsigned pb_base[kPbMax];   // ... their first slot in the bucket's region
  unsigned pb_obase[kPbMax];  // ... and in the overflow region (the part past the region's end)
  unsigned pb_pre[kPbMax + 2];  // claim pass: first chunk of each bucket (and of the overflow)
  unsigned nw;                          // winners staged in wbuf for the current window
  int2 wbuf[kWBuf];                     // (column, root) claimed in the current window
#if BM_MG
  // level bookkeeping of every rank (thread 0 refreshes it after each barrier)
  unsigned mg_ls[kMaxRanks];    // first entry of the current level in the rank's F / P
  unsigned mg_n[kMaxRanks];     // entries of the current level
  unsigned mg_nn[kMaxRanks];    // entries of the next level (pushed into the rank's inbox)
  unsigned mg_cnt[kMaxRanks];   // routed flush: winners per destination ...
  unsigned mg_base[kMaxRanks];  // ... their slots in the destination's inbox ...
  unsigned mg_cur[kMaxRanks];   // ... and the cursor within them
  unsigned long long mg_tot[4];  // team sums (entries, edges, ...) of the last refresh
#endif
};

// Warp-reduce a per-thread count and add it to the CTA's shared counter. Must
// be called by every lane of the warp.
__device__ __forceinline__ void flush_count(Smem& sm, int idx, unsigned v) {
  v = warp_sum(v);
  if (lane_id() == 0 && v) atomicAdd(&sm.cnt[idx], (unsigned long long)v);
}

// ---------------------------------------------------------------------------
// Grid barrier. All CTAs are co-resident (cooperative launch). Thread 0 of
// each CTA arrives with one atomic; the last arriver resets the count and
// bumps the generation. __threadfence() on both sides orders every write of
// the stage before every read of the next (and invalidates this SM's L1).
//
// Multi-GPU (BM_MG): the barrier spans the team. The last CTA of each rank to
// arrive does the cross-rank arrival on rank 0's team block (system-scope
// atomics, NVLink) and releases its own grid only when every rank has arrived;
// system-scope fences make each CTA's stores to peer memory visible first.
#if BM_MG
#define BM_FENCE()                      \
  do {                                  \
    if (p.world > 1)                    \
      __threadfence_system();           \
    else                                \
      __threadfence();                  \
  } while (0)
#else
#define BM_FENCE() __threadfence()
#endif
__device__ __forceinline__ unsigned ld_acq_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __noinline__ void grid_sync(const Params& p) {
  Ctrl* ctl = p.ctl;
  __syncthreads();
  if (threadIdx.x == 0) {
    // Two-level arrival: CTAs count in kBarSub group counters (separate L2
    // lines, so their atomics proceed in parallel); each group's last arriver
    // counts at the top; the last of those resets and releases everyone.
    const unsigned gen = ld_acq(&ctl->bar_gen);
    BM_FENCE();
    const unsigned G = gridDim.x;
    const unsigned grp = blockIdx.x % kBarSub;
    const unsigned ngrp = G < (unsigned)kBarSub ? G : (unsigned)kBarSub;
    const unsigned in_grp = G / kBarSub + (grp < G % kBarSub ? 1u : 0u);
    bool last = false;
    if (atomicAdd(&ctl->bar_sub[grp][0], 1u) == in_grp - 1) {
      st_rlx(&ctl->bar_sub[grp][0], 0u);
      __threadfence();  // the reset is visible before this group can be released
      last = atomicAdd(&ctl->bar_count, 1u) == ngrp - 1;
    }
    if (last) {
      st_rlx(&ctl->bar_count, 0u);
#if BM_MG
      if (p.world > 1) {  // every rank's grid has arrived before any is released
        MgTeam* t = p.team;
        const unsigned tgen = ld_acq_sys(&t->gen);
        __threadfence_system();
        if (atomicAdd_system(&t->count, 1u) == (unsigned)p.world - 1) {
          atomicExch_system(&t->count, 0u);
          __threadfence_system();
          atomicAdd_system(&t->gen, 1u);
        } else {
          const long long t0 = clock64();
          unsigned spins = 0;
          while (ld_acq_sys(&t->gen) == tgen) {
            __nanosleep(64);
            if (((++spins) & 0xfffu) == 0 && clock64() - t0 > (1ll << 37)) {
              ctl->error = kErrBarrier;
              __threadfence_system();
              __trap();
            }
          }
        }
      }
#endif
      BM_FENCE();
      atomicAdd(&ctl->bar_gen, 1u);
    } else {
      const long long t0 = clock64();
      unsigned spins = 0;
      while (ld_acq(&ctl->bar_gen) == gen) {
        __nanosleep(32);
        if (((++spins) & 0xfffu) == 0 && clock64() - t0 > (1ll << 37)) {  // ~70 s watchdog
          ctl->error = kErrBarrier;
          __threadfence_system();
          __trap();
        }
      }
    }
    BM_FENCE();
  }
  __syncthreads();
}

__device__ __forceinline__ bool is_leader() { return blockIdx.x == 0 && threadIdx.x == 0; }

// "An augmenting path was found in this phase" (by parity): team-wide in the
// multi-GPU build (rank 0's team block), per launch otherwise.
__device__ __forceinline__ unsigned* path_flag_of(const Params& p, int pf) {
#if BM_MG
  return &p.team->path_found[pf];
#else
  return &p.ctl->path_found[pf];
#endif
}
// Multi-GPU teams of more than one rank route every winner to its owner.
__device__ __forceinline__ bool routed(const Params& p) {
#if BM_MG
  return p.world > 1;
#else
  return false;
#endif
}

__device__ __forceinline__ long long clk() { return clock64(); }

__device__ __forceinline__ unsigned long long global_thread() {
  return (unsigned long long)blockIdx.x * kThreads + threadIdx.x;
}
__device__ __forceinline__ unsigned long long global_threads() {
  return (unsigned long long)gridDim.x * kThreads;
}

__device__ __forceinline__ unsigned long long warp_incl_scan64(unsigned long long v) {
  const unsigned lane = lane_id();
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long t = __shfl_up_sync(kFull, v, o);
    if (lane >= (unsigned)o) v += t;
  }
  return v;
}

// CTA-wide reservation of frontier slots/edge prefix and endpoint slots: one
// atomic per CTA instead of one per warp (every warp of the GPU pushes into
// the same two counters, so per-warp atomics serialise in L2). `cnt`/`deg`
// are this thread's winners and their total degree, `epc` its endpoints.
// Returns this thread's first packed (slot << 33 | prefix) and endpoint slot.
// Must be called by every thread of the CTA; returns false (no work) for all
// threads when the CTA pushes nothing.
__device__ __forceinline__ bool cta_reserve(Smem& sm, unsigned cnt, unsigned deg, unsigned epc, Slot* out,
                                            unsigned* n_ep, unsigned long long& tbase, unsigned& tep) {
  const unsigned long long v = ((unsigned long long)cnt << 33) | deg;
  const unsigned long long incl = warp_incl_scan64(v);
  const unsigned ep_incl = warp_incl_scan(epc);
  const unsigned warp = threadIdx.x >> 5;
  if (lane_id() == 31) {
    sm.wsum[warp] = incl;
    sm.wep[warp] = ep_incl;
  }
  if (!__syncthreads_or((cnt | epc) != 0u)) return false;
  if (threadIdx.x == 0) {
    unsigned long long run = 0;
    unsigned er = 0;
#pragma unroll
    for (int w = 0; w < kThreads / 32; ++w) {
      const unsigned long long t = sm.wsum[w];
      sm.wsum[w] = run;
      run += t;
      const unsigned te = sm.wep[w];
      sm.wep[w] = er;
      er += te;
    }
    sm.blk_base = run ? atomicAdd(&out->packed, run) : 0ull;
    sm.blk_ep = er ? atomicAdd(n_ep, er) : 0u;
  }
  __syncthreads();
  tbase = sm.blk_base + sm.wsum[warp] + (incl - v);
  tep = sm.blk_ep + sm.wep[warp] + (ep_incl - epc);
  return true;
}

// Whether row r is in column c's adjacency [b, e) (binary search over a sorted
// CSC, else a scan): a matched pair of an initial matching must be an edge
// (validate, matching.cpp:70-104).
__device__ __forceinline__ bool has_edge(const int* adj, unsigned b, unsigned e, int r, bool sorted) {
  if (sorted) {
    while (b < e) {
      const unsigned mid = b + ((e - b) >> 1);
      const int v = ld_ro(adj + mid);
      if (v == r) return true;
      if (v < r) b = mid + 1; else e = mid;
    }
    return false;
  }
  for (unsigned j = b; j < e; ++j)
    if (ld_ro(adj + j) == r) return true;
  return false;
}

// Writes one reserved frontier entry and its granule-index records.
__device__ __forceinline__ void put_entry(int4* F, unsigned out_base, unsigned* gidx, unsigned long long slot,
                                          int col, int root, unsigned beg, unsigned deg,
                                          unsigned long long pol = 0) {
  const unsigned local = (unsigned)(slot >> 33);
  const unsigned pre = (unsigned)(slot & kEdgeMask);
  if (pol) st_stream(F + out_base + local, make_int4(col, root, (int)beg, (int)pre), pol);
  else st_plain(F + out_base + local, make_int4(col, root, (int)beg, (int)pre));
  if (deg == 0) return;  // holds no edge: no granule starts inside it
  const unsigned m1 = (pre + deg - 1) / kGran;
  for (unsigned m = (pre + kGran - 1) / kGran; m <= m1; ++m) st_plain(reinterpret_cast<int*>(gidx) + m, (int)local);
}

// Row state layout (chosen per graph at upload). Interleaved: a row's mate (rmatch) and
// its BFS predecessor share one 8-byte slot: the claim is an atomicOr on the
// mate word and the predecessor store that follows it lands in the same L2
// sector, which the atomic has just brought in and dirtied, instead of a
// second random sector (with a DRAM read-for-fill of a partial write).
// That wins once rmatch is far larger than L2 (C4, C5); while rmatch fits in
// L2 the plain layout keeps the gathered array half as large (C2, C3).
#if BM_MG
__device__ __forceinline__ int owner_col(const Params& p, long long c) {
  int q = 0;
#pragma unroll
  for (int i = 0; i < kMaxRanks - 1; ++i) q += c >= p.cb[i] ? 1 : 0;
  return q;
}
__device__ __forceinline__ int owner_row(const Params& p, long long r) {
  int q = 0;
#pragma unroll
  for (int i = 0; i < kMaxRanks - 1; ++i) q += r >= p.rb[i] ? 1 : 0;
  return q;
}
// any row / column, wherever it lives
__device__ __forceinline__ int* RM(const Params& p, long long r) { return p.peer[owner_row(p, r)].rm + p.rs * r; }
__device__ __forceinline__ int* PR(const Params& p, long long r) { return p.peer[owner_row(p, r)].pred + p.rs * r; }
__device__ __forceinline__ int* CM(const Params& p, long long c) { return p.peer[owner_col(p, c)].cmatch + c; }
__device__ __forceinline__ int* BF(const Params& p, long long c) { return p.peer[owner_col(p, c)].bfs + c; }
__device__ __forceinline__ int* CR(const Params& p, long long c) { return p.peer[owner_col(p, c)].croot + c; }
#else
__device__ __forceinline__ int* RM(const Params& p, long long r) { return p.rm + p.rs * r; }
__device__ __forceinline__ int* PR(const Params& p, long long r) { return p.pred + p.rs * r; }
__device__ __forceinline__ int* CM(const Params& p, long long c) { return p.cmatch + c; }
__device__ __forceinline__ int* BF(const Params& p, long long c) { return p.bfs + c; }
__device__ __forceinline__ int* CR(const Params& p, long long c) { return p.croot + c; }
#endif
// this rank's own rows / columns (the whole graph on one GPU): no ownership lookup
__device__ __forceinline__ int* RML(const Params& p, long long r) { return p.rm + p.rs * r; }
__device__ __forceinline__ int* PRL(const Params& p, long long r) { return p.pred + p.rs * r; }

// State atomics: system scope when the location may live on another GPU.
#if BM_MG
__device__ __forceinline__ int at_or(int* a, int v) { return atomicOr_system(a, v); }
__device__ __forceinline__ unsigned at_or(unsigned* a, unsigned v) { return atomicOr_system(a, v); }
__device__ __forceinline__ int at_cas(int* a, int c, int v) { return atomicCAS_system(a, c, v); }
__device__ __forceinline__ unsigned at_cas(unsigned* a, unsigned c, unsigned v) { return atomicCAS_system(a, c, v); }
__device__ __forceinline__ unsigned long long at_add(unsigned long long* a, unsigned long long v) {
  return atomicAdd_system(a, v);
}
#else
__device__ __forceinline__ int at_or(int* a, int v) { return atomicOr(a, v); }
__device__ __forceinline__ unsigned at_or(unsigned* a, unsigned v) { return atomicOr(a, v); }
__device__ __forceinline__ int at_cas(int* a, int c, int v) { return atomicCAS(a, c, v); }
__device__ __forceinline__ unsigned at_cas(unsigned* a, unsigned c, unsigned v) { return atomicCAS(a, c, v); }
__device__ __forceinline__ unsigned long long at_add(unsigned long long* a, unsigned long long v) {
  return atomicAdd(a, v);
}
#endif

// Offsets of a claimed column (read-only path).
__device__ __forceinline__ unsigned ld_offs(const unsigned* a, unsigned long long) { return ld_ro(a); }

// WR early-exit test (gpu_match.cpp:106-108) against the dead-root bitmap:
// nc/8 bytes that stay in L2, instead of a bfs_array[root] gather per entry.
// bfs_array[root] still carries the reference's mark (and the endpoint for
// the improved walk); the bit only mirrors "marked".
__device__ __forceinline__ bool root_dead(const Params& p, int root) {
  return (ld_rlx(p.dead + (root >> 5)) >> (root & 31)) & 1u;
}
__device__ __forceinline__ void mark_dead(const Params& p, int root) {
#if BM_MG
  for (int q = 0; q < p.world; ++q) atomicOr_system(p.peer[q].dead + (root >> 5), 1u << (root & 31));  // every replica
#else
  atomicOr(p.dead + (root >> 5), 1u << (root & 31));
#endif
}

// Pushes the winners staged in sm.wbuf as next-level frontier entries: one
// CTA reservation (slots + edge prefix) for all of them. CTA-uniform call.
__device__ __forceinline__ void flush_winners(const Params& p, Smem& sm, int4* F, unsigned out_base, unsigned* gout,
                                              Slot* out, unsigned long long pol) {
  const unsigned tid = threadIdx.x;
  const unsigned nw = sm.nw;
  if (!nw) return;
  unsigned long long slot;
  unsigned unused;
  if (nw <= (unsigned)kThreads) {  // one winner per thread: a single pass
    const bool has = tid < nw;
    int2 cr = make_int2(0, 0);
    unsigned b0 = 0, d0 = 0;
    if (has) {
      cr = sm.wbuf[tid];
      b0 = ld_offs(p.offs + cr.x, pol);
      d0 = ld_offs(p.offs + cr.x + 1, pol) - b0;
    }
    cta_reserve(sm, has ? 1u : 0u, d0, 0u, out, &p.ctl->n_ep, slot, unused);
    if (has) put_entry(F, out_base, gout, slot, cr.x, cr.y, b0, d0, pol);
  } else {
    unsigned cnt = 0, deg = 0;
    for (unsigned j = tid; j < nw; j += kThreads) {
      const int c = sm.wbuf[j].x;
      deg += ld_offs(p.offs + c + 1, pol) - ld_offs(p.offs + c, pol);
      cnt++;
    }
    cta_reserve(sm, cnt, deg, 0u, out, &p.ctl->n_ep, slot, unused);
    for (unsigned j = tid; j < nw; j += kThreads) {
      const int2 cr = sm.wbuf[j];
      const unsigned b0 = ld_offs(p.offs + cr.x, pol);
      const unsigned d0 = ld_offs(p.offs + cr.x + 1, pol) - b0;
      put_entry(F, out_base, gout, slot, cr.x, cr.y, b0, d0, pol);
      slot += (1ull << 33) + d0;
    }
  }
  __syncthreads();
  if (tid == 0) sm.nw = 0;  // callers barrier before staging again
}

// Stages one winner per thread (or none) in sm.wbuf: one shared atomic per warp.
__device__ __forceinline__ void stage_winner(Smem& sm, bool win, int col, int root) {
  const unsigned mine = win ? 1u : 0u;
  const unsigned incl = warp_incl_scan(mine);
  const unsigned tot = __shfl_sync(kFull, incl, 31);
  unsigned wb = 0;
  if (lane_id() == 31 && tot) wb = atomicAdd(&sm.nw, tot);
  wb = __shfl_sync(kFull, wb, 31) + incl - mine;
  if (win) sm.wbuf[wb] = make_int2(col, root);
}

// Pushes the winners staged in sm.wbuf as (col, root) pairs: one slot
// reservation per CTA, coalesced stores, no offsets gathered. CTA-uniform call.
__device__ __forceinline__ void flush_pairs(const Params& p, Smem& sm, unsigned out_base, Slot* out,
                                            unsigned long long pol) {
  const unsigned nw = sm.nw;
  if (!nw) return;
  if (threadIdx.x == 0) sm.blk_base = atomicAdd(&out->packed, (unsigned long long)nw << 33);
  __syncthreads();
  const unsigned base = out_base + (unsigned)(sm.blk_base >> 33);
  for (unsigned j = threadIdx.x; j < nw; j += kThreads) st_stream(p.P + base + j, sm.wbuf[j], pol);
  __syncthreads();
  if (threadIdx.x == 0) sm.nw = 0;
}

__device__ __forceinline__ unsigned lanemask_lt() { return (1u << lane_id()) - 1u; }
#if BM_MG
// Multi-GPU: routes the winners staged in sm.wbuf to their columns' owners —
// per destination one slot reservation on the owner's level counter, then the
// pairs are stored straight into the owner's inbox (peer memory, NVLink).
// CTA-uniform call.
__device__ __forceinline__ void flush_pairs_mg(const Params& p, Smem& sm, int out_slot, unsigned long long pol) {
  const unsigned nw = sm.nw;
  if (!nw) return;
  if (threadIdx.x < kMaxRanks) {
    sm.mg_cnt[threadIdx.x] = 0;
    sm.mg_cur[threadIdx.x] = 0;
  }
  __syncthreads();
  for (unsigned j = threadIdx.x; j < nw; j += kThreads) atomicAdd(&sm.mg_cnt[owner_col(p, sm.wbuf[j].x)], 1u);
  __syncthreads();
  if (threadIdx.x < (unsigned)p.world && sm.mg_cnt[threadIdx.x])
    sm.mg_base[threadIdx.x] = (unsigned)(atomicAdd_system(&p.peer[threadIdx.x].ctl->lvl[out_slot].packed,
                                                          (unsigned long long)sm.mg_cnt[threadIdx.x] << 33) >> 33);
  __syncthreads();
  for (unsigned j = threadIdx.x; j < nw; j += kThreads) {
    const int2 w = sm.wbuf[j];
    const int q = owner_col(p, w.x);
    const unsigned i = atomicAdd(&sm.mg_cur[q], 1u);
    st_stream(p.peer[q].P + sm.mg_ls[q] + sm.mg_n[q] + sm.mg_base[q] + i, w, pol);
  }
  __syncthreads();
  if (threadIdx.x == 0) sm.nw = 0;
}
// The same for one warp's stage of nwin winners (pulled levels); warp-uniform call.
__device__ __forceinline__ void warp_flush_mg(const Params& p, const Smem& sm, const int2* wst, unsigned nwin,
                                              int out_slot, unsigned long long pol) {
  const unsigned lane = lane_id();
  unsigned cnt = 0;  // lane d: winners for destination d
  for (unsigned i0 = 0; i0 < nwin; i0 += 32) {
    const unsigned i = i0 + lane;
    const int q = i < nwin ? owner_col(p, wst[i].x) : -1;
    for (int d = 0; d < p.world; ++d) {
      const unsigned m = __ballot_sync(kFull, q == d);
      if (lane == (unsigned)d) cnt += __popc(m);
    }
  }
  unsigned base = 0;
  if (lane < (unsigned)p.world && cnt)
    base = (unsigned)(atomicAdd_system(&p.peer[lane].ctl->lvl[out_slot].packed, (unsigned long long)cnt << 33) >> 33);
  unsigned run = 0;
  for (unsigned i0 = 0; i0 < nwin; i0 += 32) {
    const unsigned i = i0 + lane;
    const int2 w = i < nwin ? wst[i] : make_int2(-1, 0);
    const int q = w.x >= 0 ? owner_col(p, w.x) : -1;
    unsigned pos = 0;
    for (int d = 0; d < p.world; ++d) {
      const unsigned m = __ballot_sync(kFull, q == d);
      const unsigned b = __shfl_sync(kFull, base + run, d);
      if (q == d) pos = b + __popc(m & lanemask_lt());
      if (lane == (unsigned)d) run += __popc(m);
    }
    if (q >= 0) st_stream(p.peer[q].P + sm.mg_ls[q] + sm.mg_n[q] + pos, w, pol);
  }
}
#endif

// Turns the n pairs of a level, P[ls, ls + n), into edge-tiled frontier entries
// F[ls, ls + n) plus their granule index, for a level that is pushed.
// Reservations go to `in`, a zeroed slot, whose low bits end as the level's
// edge total. Every CTA of the caller's set must call it (a grid barrier must
// follow before the entries are read).
constexpr int kMatItems = 4;
BM_MAT_INLINE void materialize(const Params& p, Smem& sm, int4* F, unsigned ls, unsigned n,
                                            unsigned* gin, Slot* in, unsigned long long pol, bool solo) {
  const unsigned long long G = solo ? 1ull : gridDim.x;
  const unsigned long long B0 = solo ? 0ull : blockIdx.x;
  unsigned done = 0;
  for (unsigned long long b = B0 * kThreads * kMatItems; b < n; b += G * kThreads * kMatItems) {
    int2 pr[kMatItems];
    unsigned beg[kMatItems], deg[kMatItems];
    unsigned cnt = 0, sum = 0;
#pragma unroll
    for (int k = 0; k < kMatItems; ++k) {
      const unsigned long long i = b + (unsigned long long)k * kThreads + threadIdx.x;
      pr[k] = i < n ? ld_cg(p.P + ls + i) : make_int2(-1, 0);
    }
#pragma unroll
    for (int k = 0; k < kMatItems; ++k) {
      beg[k] = pr[k].x >= 0 ? ld_ro(p.offs + pr[k].x) : 0u;
      deg[k] = pr[k].x >= 0 ? ld_ro(p.offs + pr[k].x + 1) : 0u;
    }
#pragma unroll
    for (int k = 0; k < kMatItems; ++k) {
      deg[k] -= beg[k];
      if (pr[k].x >= 0) {
        cnt++;
        sum += deg[k];
      }
    }
    unsigned long long slot;
    unsigned unused;
    if (cta_reserve(sm, cnt, sum, 0u, in, &p.ctl->n_ep, slot, unused)) {
#pragma unroll
      for (int k = 0; k < kMatItems; ++k)
        if (pr[k].x >= 0) {
          put_entry(F, ls, gin, slot, pr[k].x, pr[k].y, beg[k], deg[k], pol);
          slot += (1ull << 33) + deg[k];
        }
    }
    done += cnt;
  }
  flush_count(sm, kStMaterialized, done);
}

// ---------------------------------------------------------------------------
// Direction-optimised (bottom-up) level for dense frontiers. The same level of
// the same BFS as expand_level (gpubfs / gpubfs_wr, gpu_match.cpp:42-70,
// 99-133), pulled instead of pushed: every unvisited matched row scans its own
// columns (the transposed adjacency) for one in the frontier and is claimed by
// the first it finds; every free row likewise becomes an endpoint of the first
// live tree it touches. Any frontier neighbour is a valid discoverer (the
// reference's races pick one arbitrarily too), so levels, roots and the
// augmenting paths keep their meaning; a row stops at its first hit, which is
// what saves the work when most columns are already in the frontier.
//
// bu_prep: the frontier of level lv as a bitmap (+ the root of each member).
// The bitmap is clean: a bottom-up level clears its own right after the grid
// barrier that ends it (bu_clear; the next level uses the other bitmap).
__device__ __forceinline__ void bu_clear(const Params& p, int b) {
  unsigned* fb = p.fbit[b];
  for (unsigned long long k = global_thread(); k < (unsigned long long)p.nfbit_words; k += global_threads())
    st_plain(reinterpret_cast<int*>(fb) + k, 0);
}
// The frontier comes as (col, root) pairs (levels >= 1 of a pulled-capable
// run) or as entries (level 0). Counts the live entries as columns expanded.
// write_root = false (lazy roots, see bu_sweep_q): only the bitmap is built.
template <bool WR>
BM_PREP_INLINE void bu_prep(const Params& p, Smem& sm, const int4* F, bool pairs, unsigned ls,
                                        unsigned n, int lv, bool write_root = true) {
  unsigned* fb = p.fbit[lv % kNumFbit];
  unsigned live = 0;
  constexpr int K = 8;  // entries per thread in flight (the loop is latency-bound otherwise)
  const unsigned long long GT = global_threads();
  for (unsigned long long k0 = global_thread(); k0 < n; k0 += K * GT) {
    int col[K], root[K];
#pragma unroll
    for (int i = 0; i < K; ++i) {
      const unsigned long long k = k0 + i * GT;
      col[i] = -1;
      root[i] = 0;
      if (k < n) {
        if (pairs) {
          const int2 pr = ld_cg(p.P + ls + k);
          col[i] = pr.x;
          root[i] = pr.y;
        } else {
          const int4 ent = ld_cg(F + ls + k);
          col[i] = ent.x;
          root[i] = ent.y;
        }
      }
    }
    bool on[K];
#pragma unroll
    for (int i = 0; i < K; ++i) on[i] = col[i] >= 0 && !(WR && root_dead(p, root[i]));
#pragma unroll
    for (int i = 0; i < K; ++i)
      if (on[i]) {
        live++;
        atomicOr(fb + (col[i] >> 5), 1u << (col[i] & 31));
        if (write_root) st_plain(p.croot + col[i], WR ? root[i] : col[i]);
      }
  }
  flush_count(sm, kStCexp, live);
}


// bu_prep in two passes for wide frontiers with roots (the first pulled level of
// a C5 phase: ~45 M columns): pass 1 drops dead trees' entries and writes the
// live (col, root) pairs into the region of their column's bucket (CTA-staged
// runs, one reservation per bucket per window; an overflow region takes any
// skew); after a grid barrier, pass 2 takes the buckets in order (chunks handed
// out from a ticket), so each bucket's root stores and bitmap atomics hit an
// L2-resident window of croot / fbit instead of a random DRAM sector each.
template <bool WR>
__device__ __noinline__ void bu_prep_bucketed(const Params& p, Smem& sm, const int4* F, bool pairs, unsigned ls,
                                              unsigned n, int lv, int par) {
  Ctrl* ctl = p.ctl;
  unsigned* fb = p.fbit[lv % kNumFbit];
  int2* const buf = reinterpret_cast<int2*>(p.tb);
  const int nb = p.pp_nb, shift = p.pp_shift;
  const unsigned cap = p.pp_cap;
  const unsigned long long ovf0 = (unsigned long long)nb * cap;
  unsigned* const cur = ctl->pb_cur[par];
  const unsigned long long pol = policy_evict_first();
  const unsigned tid = threadIdx.x;
  unsigned live = 0;
  constexpr int K = 8;
  constexpr unsigned W = kThreads * K;  // entries per CTA window
  // ---- pass 1: partition the live entries by column bucket ----
  for (unsigned long long w0 = (unsigned long long)blockIdx.x * W; w0 < n; w0 += (unsigned long long)gridDim.x * W) {
    for (int b = tid; b < nb; b += kThreads) sm.pb_hist[b] = 0;
    __syncthreads();
    int col[K], root[K];
    unsigned rank[K];
#pragma unroll
    for (int i = 0; i < K; ++i) {
      const unsigned long long k = w0 + (unsigned long long)i * kThreads + tid;
      col[i] = -1;
      root[i] = 0;
      if (k < n) {
        if (pairs) {
          const int2 pr = ld_cg(p.P + ls + k);
          col[i] = pr.x;
          root[i] = pr.y;
        } else {
          const int4 ent = ld_cg(F + ls + k);
          col[i] = ent.x;
          root[i] = ent.y;
        }
      }
    }
#pragma unroll
    for (int i = 0; i < K; ++i) {
      if (col[i] >= 0 && WR && root_dead(p, root[i])) col[i] = -1;
      rank[i] = col[i] >= 0 ? atomicAdd(&sm.pb_hist[col[i] >> shift], 1u) : 0u;
    }
    __syncthreads();
    for (int b = tid; b < nb; b += kThreads) {
      const unsigned h = sm.pb_hist[b];
      if (h) {
        const unsigned base = atomicAdd(cur + b, h);
        sm.pb_base[b] = base;
        const unsigned fit = base >= cap ? 0u : min(h, cap - base);
        if (fit < h) sm.pb_obase[b] = atomicAdd(&ctl->pb_ovf[par], h - fit);
      }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < K; ++i) {
      if (col[i] < 0) continue;
      live++;
      const int b = col[i] >> shift;
      const unsigned pos = sm.pb_base[b] + rank[i];
      const unsigned long long idx =
          pos < cap ? (unsigned long long)b * cap + pos : ovf0 + sm.pb_obase[b] + (pos - max(sm.pb_base[b], cap));
      st_stream(buf + idx, make_int2(col[i], WR ? root[i] : col[i]), pol);
    }
    __syncthreads();
  }
  flush_count(sm, kStCexp, live);
  grid_sync(p);
  // ---- pass 2: bucket by bucket, the bitmap and the roots ----
  constexpr unsigned CH = kThreads * K;
  if (tid == 0) {
    unsigned acc = 0;
    for (int b = 0; b < nb; ++b) {
      sm.pb_pre[b] = acc;
      acc += (min(ld_rlx(cur + b), cap) + CH - 1) / CH;
    }
    sm.pb_pre[nb] = acc;
    acc += (ld_rlx(&ctl->pb_ovf[par]) + CH - 1) / CH;
    sm.pb_pre[nb + 1] = acc;
  }
  __syncthreads();
  const unsigned total = sm.pb_pre[nb + 1];
  for (;;) {
    if (tid == 0) sm.tile = atomicAdd(&ctl->pb_ticket[par], 1u);
    __syncthreads();
    const unsigned t = sm.tile;
    __syncthreads();
    if (t >= total) break;
    int b = 0;
    while (b < nb && sm.pb_pre[b + 1] <= t) ++b;
    const unsigned long long r0 = b < nb ? (unsigned long long)b * cap : ovf0;
    const unsigned m = b < nb ? min(ld_rlx(cur + b), cap) : ld_rlx(&ctl->pb_ovf[par]);
    const unsigned j0 = (t - sm.pb_pre[b]) * CH;
    int2 pr[K];
#pragma unroll
    for (int i = 0; i < K; ++i) {
      const unsigned jj = j0 + i * kThreads + tid;
      pr[i] = jj < m ? ld_cg(buf + r0 + jj) : make_int2(-1, 0);
    }
#pragma unroll
    for (int i = 0; i < K; ++i)
      if (pr[i].x >= 0) {
        atomicOr(fb + (pr[i].x >> 5), 1u << (pr[i].x & 31));
        st_plain(p.croot + pr[i].x, pr[i].y);
      }
  }
}
#ifndef BM_BU_PROBE
#define BM_BU_PROBE 4
#endif
#ifndef BM_BU_PF
#define BM_BU_PF 1  // pulled levels: L2 prefetch of the next chunk's row state/offsets and of each candidate's columns
                    // (A/B on C5: screen cycles -34 %, -3.5 % per phase)
#endif
#ifndef BM_V2ST
#define BM_V2ST 1  // interleaved row state: a claim by store writes {mate | visited, pred} in one 8-byte store
#endif
#ifndef BM_BU_LAZY
#define BM_BU_LAZY 1  // pulled levels with few rows left resolve their hits' roots instead of scattering them
#endif
constexpr bool BU_LAZY = BM_BU_LAZY != 0;
#ifndef BM_BU_CYC
#define BM_BU_CYC 0  // 1: per-part warp cycle counters in pulled levels (profiling builds)
#endif
// Warp-autonomous pulled level. Every warp owns chunks of 128 consecutive rows
// (grid-stride over the warps of the grid) and keeps a queue of candidate rows
// in shared memory: screening a chunk reads the rows' state and their row-index
// offsets in one coalesced round and appends the candidates (unvisited matched
// rows, free rows) with their column ranges. Lanes then probe independently:
// a lane whose row is resolved (hit, or its columns exhausted) takes the next
// queued candidate in the following round, so a warp never waits for its
// slowest row, and no CTA-wide barrier is needed — winners are staged per warp
// in its slice of wbuf and flushed with one reservation per warp.
#if BM_MG
// Multi-GPU: after bu_prep, each rank copies the words of its own columns
// (column ranges are 32-aligned) into every peer's replica of the bitmap.
__device__ __forceinline__ void bu_share(const Params& p, int lv) {
  if (p.col_lo >= p.col_hi) return;  // owns no column (the last word belongs to the rank that ends at nc)
  const unsigned w0 = (unsigned)p.col_lo >> 5, w1 = ((unsigned)p.col_hi + 31) >> 5;
  const unsigned* src = p.fbit[lv % kNumFbit];
  const unsigned long long off = (unsigned long long)(lv % kNumFbit) * p.nfbit_words;
  for (unsigned long long k = w0 + global_thread(); k < w1; k += global_threads()) {
    const unsigned v = (unsigned)ld_cg(reinterpret_cast<const int*>(src) + k);
    for (int q = 0; q < p.world; ++q)
      if (q != p.rank) st_plain(reinterpret_cast<int*>(p.peer[q].fbit + off) + k, (int)v);
  }
}
#endif

// lazy_root: this level's bu_prep wrote no roots (few rows are left to claim, so
// scattering one root per frontier column would cost more than resolving the
// roots of the hits): a hit column c's root is that of the column that
// discovered its mate row, croot[pred[cmatch[c]]], which the level before
// (pulled, with roots) wrote.
// lin / n_in (nullable): take the candidates from the level before's leftover
// list instead of screening every row (Params::left); lout / n_out (nullable):
// append this level's leftovers (candidates that found no frontier column,
// i.e. every row that is still unvisited afterwards).
template <bool WR, bool IMP>
BM_SWEEP_INLINE void bu_sweep_q(const Params& p, Smem& sm, unsigned out_base, Slot* out, int out_slot,
                                           int lv, int pf, bool lazy_root = false,
                                           const int2* lin = nullptr, unsigned n_in = 0, int2* lout = nullptr,
                                           unsigned* n_out = nullptr) {
  constexpr int kWarps = kThreads / 32;
  constexpr unsigned kChunk = 128;
  constexpr unsigned kWStage = 128;  // winners staged per warp
  // wbuf is free during a pulled level: it holds the warps' candidate queues, then their winner stages
  static_assert(sizeof(BuCand) * kCandCap * kWarps + sizeof(int2) * kWStage * kWarps <= sizeof(int2) * kWBuf,
                "candidate queues and winner stages must fit in wbuf");
  constexpr int kBuProbe = BM_BU_PROBE;
  const unsigned* fb = p.fbit[lv % kNumFbit];
  const unsigned long long pol = policy_evict_first();
  unsigned* const path_flag = path_flag_of(p, pf);
#if BM_MG
  const unsigned long long rlo = (unsigned long long)p.row_lo, rhi = (unsigned long long)p.row_hi;  // own rows
#else
  const unsigned long long rlo = 0, rhi = (unsigned long long)p.nr;
#endif
  unsigned c_trav = 0, c_nvis = 0, c_rows = 0;
  long long cy_screen = 0, cy_probe = 0, cy_flush = 0, n_rounds = 0;  // BM_BU_CYC
  const unsigned warp = threadIdx.x >> 5, lane = lane_id();
  BuCand* const q = reinterpret_cast<BuCand*>(sm.wbuf) + warp * kCandCap;
  int2* const wst = reinterpret_cast<int2*>(reinterpret_cast<BuCand*>(sm.wbuf) + kWarps * kCandCap) + warp * kWStage;
  const unsigned long long nchunks = lin ? (n_in + kChunk - 1) / kChunk : (rhi - rlo + kChunk - 1) / kChunk;
  const unsigned long long W = (unsigned long long)gridDim.x * kWarps;
  unsigned long long chunk = (unsigned long long)blockIdx.x * kWarps + warp;
  unsigned qh = 0, qt = 0;  // queued candidates q[qh, qt) (warp-uniform)
  unsigned nwin = 0;        // winners staged in wst (warp-uniform)
  int rr = -1, vv = 0;      // this lane's current candidate
  unsigned j = 0, j1 = 0;
  for (;;) {
    // refill: the idle lanes would drain the queue and rows remain
    long long t0 = BM_BU_CYC ? clk() : 0;
    const unsigned idle = __ballot_sync(kFull, rr < 0);
    while (qt - qh < (unsigned)__popc(idle) && chunk < nchunks) {  // (a chunk may hold no candidate)
      // move the leftovers (< 32) to the front, then screen one chunk
      const unsigned left = qt - qh;
      BuCand keep;
      if (lane < left) keep = q[qh + lane];
      __syncwarp();
      if (lane < left) q[lane] = keep;
      qh = 0;
      qt = left;
      if (lin) {  // the level before's leftovers: (row, row state), every one a candidate
        const unsigned long long i0 = chunk * kChunk;
        chunk += W;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const unsigned long long i = i0 + (unsigned long long)k * 32 + lane;
          BuCand c;
          c.row = -1;
          c.val = 0;
          c.j0 = c.j1 = 0;
          if (i < n_in) {
            const int2 ent = ld_cg(lin + i);
            c.row = ent.x;
            c.val = ent.y;
            c.j0 = ld_ro(p.roffs + ent.x);
            c.j1 = ld_ro(p.roffs + ent.x + 1);
          }
          const unsigned m = __ballot_sync(kFull, c.row >= 0);
          if (c.row >= 0) {
            q[qt + __popc(m & ((1u << lane) - 1))] = c;
#if BM_BU_PF
            prefetch_l2n(p.radj + c.j0);
#endif
          }
          qt += __popc(m);
        }
        __syncwarp();
        continue;
      }
      const unsigned long long r0 = rlo + chunk * kChunk;
      chunk += W;
#if BM_BU_PF
      // L2 prefetch of the warp's next chunk (row state, row offsets): its screen,
      // a few probe rounds from now, then finds them in L2 instead of waiting on DRAM
      if (chunk < nchunks) {
        const unsigned long long rn = rlo + chunk * kChunk;
        const unsigned long long rend = min(rhi, rn + kChunk);
        // row state: kChunk rows x 4 B x rs -> one 32-byte sector per lane (rs = 2: 1 KB = 32 sectors)
        const unsigned long long rr0 = rn + (unsigned long long)lane * (8 / p.rs);
        if (rr0 < rend) prefetch_l2n(RML(p, rr0));
        if (lane < 16) {  // offsets: 512 B = 16 sectors
          const unsigned long long ro = rn + (unsigned long long)lane * 8;
          if (ro <= rend) prefetch_l2n(p.roffs + ro);
        }
      }
#endif
      int v[4];
      unsigned o[4], onext;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const unsigned long long r = r0 + (unsigned long long)k * 32 + lane;
        v[k] = r < rhi ? ld_cg(RML(p, r)) : -3;
        o[k] = r <= rhi ? ld_ro(p.roffs + r) : 0u;  // roffs[rhi] ends the last row
      }
      {
        const unsigned long long r = r0 + 4 * 32;
        onext = (lane == 0 && r <= rhi) ? ld_ro(p.roffs + r) : 0u;
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        // end of this row's columns = start of the next row's
        unsigned e = __shfl_down_sync(kFull, o[k], 1);
        const unsigned nxt0 = __shfl_sync(kFull, k < 3 ? o[(k + 1) & 3] : onext, 0);
        if (lane == 31) e = nxt0;
        const bool is_cand = (v[k] >= 0 && !(v[k] & kVisBit)) || v[k] == -1;
        const unsigned m = __ballot_sync(kFull, is_cand && e > o[k]);
        if (is_cand && e > o[k]) {
          BuCand c;
          c.row = (int)(r0 + (unsigned long long)k * 32 + lane);
          c.val = v[k];
          c.j0 = o[k];
          c.j1 = e;
          q[qt + __popc(m & ((1u << lane) - 1))] = c;
#if BM_BU_PF
          prefetch_l2n(p.radj + o[k]);  // the candidate's first probe group, a few rounds ahead
#endif
        }
        qt += __popc(m);
      }
      __syncwarp();
    }
    // idle lanes take queued candidates in lane order
    {
      const unsigned avail = qt - qh;
      const unsigned rank = __popc(idle & ((1u << lane) - 1));
      if (rr < 0 && rank < avail) {
        const BuCand c = q[qh + rank];
        rr = c.row;
        vv = c.val;
        j = c.j0;
        j1 = c.j1;
        c_rows++;
      }
      qh += min((unsigned)__popc(idle), avail);
    }
    if (BM_BU_CYC) {
      const long long t = clk();
      cy_screen += t - t0;
      t0 = t;
    }
    if (!__any_sync(kFull, rr >= 0)) break;  // queue empty and every chunk screened
    // one probe round
    bool win = false, ep = false;
    int cw = 0, rootw = 0;
    const int myrow = rr;
    if (rr >= 0) {
      int cs[kBuProbe];
      unsigned wd[kBuProbe];
#pragma unroll
      for (int k = 0; k < kBuProbe; ++k) cs[k] = j + k < j1 ? ld_stream(p.radj + j + k, pol) : -1;
#pragma unroll
      for (int k = 0; k < kBuProbe; ++k)
        wd[k] = cs[k] >= 0 ? ld_ca(reinterpret_cast<const int*>(fb) + (cs[k] >> 5)) : 0u;
      bool done = false;
#pragma unroll
      for (int k = 0; k < kBuProbe; ++k) {
        const int c = cs[k];
        if (done || c < 0) continue;
        c_trav++;
        if (!((wd[k] >> (c & 31)) & 1)) continue;
        int root = c;
        if (WR && lazy_root) {
          root = ld_cg(CR(p, ld_cg(PR(p, ld_rlx(CM(p, c))))));
          if (root_dead(p, root)) continue;  // (bu_prep filtered by the pairs' roots; the tree may have died since)
        } else if (WR) {
          root = ld_cg(CR(p, c));
        }
        if (vv >= 0) {  // matched row: its column joins the frontier below c's tree
          if (BM_V2ST && p.rs == 2) {  // interleaved {mate, pred}: one 8-byte store
            st_plain(reinterpret_cast<int2*>(RML(p, rr)), make_int2(vv | kVisBit, c));
          } else {
            st_plain(RML(p, rr), vv | kVisBit);
            st_plain(PRL(p, rr), c);
          }
          win = true;
          cw = vv;
          rootw = root;
          done = true;
          continue;
        }
        // free row: an endpoint of c's tree
        const bool one = WR && p.ep_one;
        if (one && root_dead(p, root)) continue;
        bool mine = true;
        if (one) mine = at_cas(BF(p, root), kStartLevel, IMP ? -rr : kFoundMark) == kStartLevel;
        else if (WR) st_rlx(BF(p, root), IMP ? -rr : kFoundMark);
        if (!mine) continue;  // that tree already holds an endpoint: try another neighbour
        if (WR) mark_dead(p, root);
        st_rlx(RML(p, rr), -2);
        st_plain(PRL(p, rr), c);
        ep = true;
        if (ld_rlx(path_flag) == 0u) st_rlx(path_flag, 1u);
        done = true;
      }
      j += kBuProbe;
      if (done || j >= j1) {
        if (!done && lout) {  // no frontier column: still unvisited after this level
          cg::coalesced_group g = cg::coalesced_threads();
          unsigned b = 0;
          if (g.thread_rank() == 0) b = atomicAdd(n_out, g.size());
          b = g.shfl(b, 0) + g.thread_rank();
          st_plain(lout + b, make_int2(rr, vv));
        }
        rr = -1;
      }
    }
    if (BM_BU_CYC) {
      __syncwarp();
      const long long t = clk();
      cy_probe += t - t0;
      t0 = t;
      n_rounds++;
    }
    // stage winners in this warp's slice of wbuf; flush it when the next round might not fit
    {
      const unsigned m = __ballot_sync(kFull, win);
      if (win) wst[nwin + __popc(m & ((1u << lane) - 1))] = make_int2(cw, rootw);
      nwin += __popc(m);
      c_nvis += win ? 1u : 0u;
      if (nwin > kWStage - 32) {
        __syncwarp();
#if BM_MG
        if (routed(p)) {
          warp_flush_mg(p, sm, wst, nwin, out_slot, pol);
        } else
#endif
        {
          unsigned base = 0;
          if (lane == 0) base = (unsigned)(atomicAdd(&out->packed, (unsigned long long)nwin << 33) >> 33);
          base = __shfl_sync(kFull, base, 0) + out_base;
          for (unsigned i = lane; i < nwin; i += 32) st_stream(p.P + base + i, wst[i], pol);
        }
        __syncwarp();
        nwin = 0;
      }
    }
    {  // endpoints: rare, warp-aggregated global append
      const unsigned m = __ballot_sync(kFull, ep);
      if (m) {
        unsigned eb = 0;
        if (lane == 0) eb = atomicAdd(&p.ctl->n_ep, (unsigned)__popc(m));
        eb = __shfl_sync(kFull, eb, 0) + __popc(m & ((1u << lane) - 1));
        if (ep) st_plain(p.EP + eb, myrow);
      }
    }
    if (BM_BU_CYC) cy_flush += clk() - t0;
  }
  if (BM_BU_CYC && lane == 0) {
    atomicAdd(&sm.cnt[kStCycBuScreen], (unsigned long long)cy_screen);
    atomicAdd(&sm.cnt[kStCycBuProbe], (unsigned long long)cy_probe);
    atomicAdd(&sm.cnt[kStCycBuFlush], (unsigned long long)cy_flush);
    atomicAdd(&sm.cnt[kStBuRounds], (unsigned long long)n_rounds);
  }
  if (nwin) {
    __syncwarp();
#if BM_MG
    if (routed(p)) {
      warp_flush_mg(p, sm, wst, nwin, out_slot, pol);
    } else
#endif
    {
      unsigned base = 0;
      if (lane == 0) base = (unsigned)(atomicAdd(&out->packed, (unsigned long long)nwin << 33) >> 33);
      base = __shfl_sync(kFull, base, 0) + out_base;
      for (unsigned i = lane; i < nwin; i += 32) st_stream(p.P + base + i, wst[i], pol);
    }
  }
  flush_count(sm, kStTrav, c_trav);
  flush_count(sm, kStNvis, c_nvis);
  flush_count(sm, kStRowsPulled, c_rows);
}


// ---------------------------------------------------------------------------
// One BFS level (GPUBFS, Alg. 2, gpu_match.cpp:42-70; GPUBFS-WR, Alg. 4,
// gpu_match.cpp:99-133) over the frontier F[ls, ls+n) holding T edges.
template <bool WR, bool IMP, bool BU>
BM_EXPAND_INLINE void expand_level(const Params& p, Smem& sm, int4* F, unsigned ls, unsigned n, unsigned T,
                             const unsigned* gin, unsigned* gout, Slot* in, Slot* out, int level, int pf,
                             bool pairs_out, bool claim_store, int out_slot) {
  if (T == 0) return;
  const unsigned tid = threadIdx.x;
  unsigned c_trav = 0, c_cexp = 0, c_nvis = 0, c_entries = 0;
  const unsigned long long G = gridDim.x;
  unsigned long long per = (T + 2 * G - 1) / (2 * G);
  per = ((per + kGran - 1) / kGran) * kGran;
  if (per > (unsigned long long)kGran * kMaxTileGran) per = (unsigned long long)kGran * kMaxTileGran;
  const unsigned ET = (unsigned)per;
  const unsigned ntiles = (unsigned)((T + (unsigned long long)ET - 1) / ET);
  const unsigned out_base = ls + n;
  unsigned* const path_flag = path_flag_of(p, pf);

  const unsigned long long pol = policy_evict_first();
#ifndef BM_PF
#define BM_PF 2
#endif
#ifndef BM_KEEP
#define BM_KEEP 1
#endif
  // BM_KEEP: 0 default priority for the gathered state; 1 rmatch evict_last;
  // 2 rmatch + visited bitmap + offsets evict_last.
  const unsigned long long keep = policy_evict_last();
  if (tid == 0) sm.nw = 0;
  long long t_a = clk();
  for (;;) {
    if (tid == 0) sm.tile = atomicAdd(&in->tile, 1u);
    __syncthreads();
    const unsigned tile = sm.tile;
    __syncthreads();
    if (tid == 0) {
      const long long t = clk();
      sm.cnt[kStCycTile] += t - t_a;
      t_a = t;
    }
    if (tile >= ntiles) break;
    const unsigned e0 = tile * ET;
    const unsigned e1 = (T - e0 < ET) ? T : e0 + ET;
    unsigned i = (unsigned)ld_cg(reinterpret_cast<const int*>(gin) + e0 / kGran);  // entry holding edge e0
    unsigned e = e0;
    while (e < e1) {
      // Window of up to kWin entries starting at i (thread t holds entries t*kEPT ..).
#pragma unroll
      for (int k = 0; k < kEPT; ++k) {
        const unsigned sl0 = tid * kEPT + k;
        const unsigned wi = i + sl0;
        if (wi < n) {
          const int4 ent = ld_cg_stream(F + ls + wi, pol);
          bool skip = false;
          if (WR) skip = root_dead(p, ent.y);  // early exit (gpu_match.cpp:106-108)
          sm.col[sl0] = ent.x;
          sm.root[sl0] = skip ? -1 : ent.y;
          sm.beg[sl0] = (unsigned)ent.z;
          sm.pre[sl0] = (unsigned)ent.w;
          if ((unsigned)ent.w >= e0 && (unsigned)ent.w < e1) {
            c_entries++;
            if (!skip) c_cexp++;
          }
        } else {
          sm.pre[sl0] = T;
          sm.root[sl0] = -1;
        }
      }
      if (tid == 0) sm.pre[kWin] = (i + kWin < n) ? ld_cg_u(F + ls + i + kWin) : T;
      __syncthreads();
      const unsigned wend = min(e1, sm.pre[kWin]);
      // Compact the window to its live edges: entries of trees that already
      // found a path (WR) and edge ranges outside [e, wend) contribute none.
      unsigned live;
      {
        unsigned len[kEPT], nb[kEPT], tsum = 0;
#pragma unroll
        for (int k = 0; k < kEPT; ++k) {
          const unsigned sl0 = tid * kEPT + k;
          const unsigned lo = max(sm.pre[sl0], e);
          const unsigned hi = min(sm.pre[sl0 + 1], wend);
          len[k] = (sm.root[sl0] >= 0 && hi > lo) ? hi - lo : 0u;
          nb[k] = sm.beg[sl0] + (lo - sm.pre[sl0]);
          tsum += len[k];
        }
        const unsigned incl = warp_incl_scan(tsum);
        if (lane_id() == 31) sm.wtot[tid >> 5] = incl;
        __syncthreads();
        unsigned wbase = 0, tot = 0;
#pragma unroll
        for (int w = 0; w < kThreads / 32; ++w) {
          const unsigned t = sm.wtot[w];
          wbase += (w < (int)(tid >> 5)) ? t : 0u;
          tot += t;
        }
        live = tot;
        if (tot > kWBuf) {  // cannot happen on consistent entries: skip the window, report, stop the run
          if (tid == 0 && atomicCAS(&p.ctl->error, 0, (int)kErrWindow) == 0) {
            long long* d = p.ctl->dbg;
            d[0] = ls; d[1] = n; d[2] = T; d[3] = i; d[4] = e; d[5] = wend; d[6] = tot; d[7] = level;
          }
          live = 0;
          for (int k = 0; k < kEPT; ++k) len[k] = 0;
        }
        unsigned vp = wbase + incl - tsum;
#pragma unroll
        for (int k = 0; k < kEPT; ++k) {
          const unsigned sl0 = tid * kEPT + k;
          sm.beg[sl0] = nb[k];
          sm.pre[sl0] = vp;  // live-edge prefix (ties resolve to the last entry)
          if (len[k]) {  // coarse index: this entry holds live edges 32q for q in [ceil(vp/32), (vp+len-1)/32]
            const unsigned q1 = (vp + len[k] - 1) >> 5;
            for (unsigned q = (vp + 31) >> 5; q <= q1; ++q) sm.cgr[q] = (unsigned short)sl0;
          }
          vp += len[k];
        }
        if (tid == 0) sm.pre[kWin] = tot;
        __syncthreads();
      }
      const unsigned nq = (live + 31) >> 5;
      if (tid == 0) {
        const long long t = clk();
        sm.cnt[kStCycWindow] += t - t_a;
        t_a = t;
      }
      // Prefetch the next window's entries while this window's rounds run.
#pragma unroll
      for (int k = 0; k < kEPT; ++k)
        if (wend < e1 && i + kWin + k * kThreads + tid < n) prefetch_l2(F + ls + i + kWin + k * kThreads + tid);

      // Rounds over the live edges: no CTA-wide barrier inside; winners are
      // staged in sm.wbuf.
      for (unsigned base = 0; base < live; base += kThreads * kItems) {
        int row[kItems], cm[kItems], sl[kItems];
#pragma unroll
        for (int k = 0; k < kItems; ++k) {
          const unsigned ee = base + k * kThreads + tid;
          row[k] = -1;
          sl[k] = 0;
          if (ee < live) {
            // the entry holding ee lies in [cgr[q], cgr[q+1]] (1-2 steps for typical degrees)
            const unsigned q = ee >> 5;
            int a = sm.cgr[q];
            int b = (q + 1 < nq) ? (int)sm.cgr[q + 1] + 1 : kWin;
            while (b - a > 1) {
              const int mid = (a + b) >> 1;
              if (sm.pre[mid] <= ee) a = mid; else b = mid;
            }
            sl[k] = a;
            row[k] = ld_stream(p.adj + sm.beg[a] + (ee - sm.pre[a]), pol);
            c_trav++;
          }
        }
#pragma unroll
        for (int k = 0; k < kItems; ++k)
          cm[k] = row[k] >= 0 ? (BM_KEEP >= 1 ? ld_rlx_hint(RM(p, row[k]), keep) : ld_rlx(RM(p, row[k])))
                              : -3;
        unsigned wins = 0, eps = 0;
        // Column claims: issue every item's atomic before consuming any result
        // (kItems claims in flight per thread instead of one).
        int old[kItems];
#pragma unroll
        for (int k = 0; k < kItems; ++k) {
          const int c = cm[k];  // mate of the row; kVisBit set = its column was claimed this phase
          old[k] = kVisBit;
          if (c >= 0 && !(c & kVisBit) && (!WR || p.claim_mode == 0 || !root_dead(p, sm.root[sl[k]]))) {
            if (claim_store) {  // racy claim: a rare concurrent discoverer pushes the column twice
              if (BM_V2ST && p.rs == 2)  // interleaved: the claim and the predecessor in one 8-byte store
                st_plain(reinterpret_cast<int2*>(RM(p, row[k])), make_int2(c | kVisBit, sm.col[sl[k]]));
              else
                st_plain(RM(p, row[k]), c | kVisBit);
              old[k] = c;
            } else {
              old[k] = at_or(RM(p, row[k]), kVisBit);
            }
          }
        }
#pragma unroll
        for (int k = 0; k < kItems; ++k) {
          const int c = cm[k];
          const int col = sm.col[sl[k]];
          const int root = WR ? sm.root[sl[k]] : col;
          if (c >= 0) {
            if (!(old[k] & kVisBit)) {
              wins |= 1u << k;
              if (!routed(p)) {  // (routed: the owner of c reads its offsets when it materializes the pair)
                if (BM_PF == 2) prefetch_l2(p.offs + c);  // the flush reads offs[c], offs[c+1]
                if (BM_PF == 1) asm volatile("prefetch.global.L2 [%0];" ::"l"(p.offs + c));
              }
              if (!(BM_V2ST && claim_store && p.rs == 2)) st_stream(PR(p, row[k]), col, pol);
              if (p.trace) st_plain(BF(p, c), level + 1);
            }
          } else if (c == -1) {
            // ONE_PER_TREE: a tree that already holds an endpoint leaves the row alone
            const bool one = WR && p.ep_one;
            if ((!one || !root_dead(p, root)) && at_cas(RM(p, row[k]), -1, -2) == -1) {
              bool mine = true;
              if (one) {
                // the root's mark is the tree's endpoint slot: first CAS wins, a loser releases the row
                mine = at_cas(BF(p, root), kStartLevel, IMP ? -row[k] : kFoundMark) == kStartLevel;
                if (!mine) st_rlx(RM(p, row[k]), -1);
                else mark_dead(p, root);
              } else if (WR) {
                st_rlx(BF(p, root), IMP ? -row[k] : kFoundMark);  // gpu_match.cpp:122-123
                mark_dead(p, root);
              }
              if (mine) {
                eps |= 1u << k;
                st_plain(PR(p, row[k]), col);
                if (ld_rlx(path_flag) == 0u) st_rlx(path_flag, 1u);
              }
            }
          }
        }
        // stage winners (one shared-memory atomic per warp)
        {
          const unsigned mine = __popc(wins);
          const unsigned incl = warp_incl_scan(mine);
          const unsigned tot = __shfl_sync(kFull, incl, 31);
          unsigned wb = 0;
          if (lane_id() == 31 && tot) wb = atomicAdd(&sm.nw, tot);
          wb = __shfl_sync(kFull, wb, 31) + incl - mine;
#pragma unroll
          for (int k = 0; k < kItems; ++k)
            if (wins & (1u << k)) sm.wbuf[wb++] = make_int2(cm[k], WR ? sm.root[sl[k]] : sm.col[sl[k]]);
          c_nvis += mine;
        }
        // endpoints are rare: warp-aggregated global append
        {
          const unsigned mine = __popc(eps);
          const unsigned incl = warp_incl_scan(mine);
          const unsigned tot = __shfl_sync(kFull, incl, 31);
          if (tot) {
            unsigned eb = 0;
            if (lane_id() == 31) eb = atomicAdd(&p.ctl->n_ep, tot);
            eb = __shfl_sync(kFull, eb, 31) + incl - mine;
#pragma unroll
            for (int k = 0; k < kItems; ++k)
              if (eps & (1u << k)) st_plain(p.EP + eb++, row[k]);
          }
        }
      }
      __syncthreads();
      if (tid == 0) {
        const long long t = clk();
        sm.cnt[kStCycRounds] += t - t_a;
        t_a = t;
      }
      // Flush the window's winners: one CTA reservation for all of them.
#if BM_MG
      if (routed(p)) flush_pairs_mg(p, sm, out_slot, pol);  // every winner goes to its column's owner as a pair
      else
#endif
      if (BU && pairs_out) flush_pairs(p, sm, out_base, out, pol);
      else flush_winners(p, sm, F, out_base, gout, out, pol);
      e = wend;
      i += kWin;
      __syncthreads();
      if (tid == 0) {
        const long long t = clk();
        sm.cnt[kStCycFlush] += t - t_a;
        t_a = t;
      }
    }
  }
  flush_count(sm, kStTrav, c_trav);
  flush_count(sm, kStCexp, c_cexp);
  flush_count(sm, kStNvis, c_nvis);
  flush_count(sm, kStEntries, c_entries);
}

// expand_level compiled out of line, for the pulled-capable kernels: there it
// gets its own register allocation instead of sharing the driver's (A/B: C5
// -7 %, C2 -9 % per phase), while inlining stays better for the push-only
// kernels (C3 +21 %, C4 +17 % out of line).
template <bool WR, bool IMP, bool BU>
__device__ __noinline__ void expand_level_ool(const Params& p, Smem& sm, int4* F, unsigned ls, unsigned n, unsigned T,
                                              const unsigned* gin, unsigned* gout, Slot* in, Slot* out, int level,
                                              int pf, bool pairs_out, bool claim_store, int out_slot) {
  expand_level<WR, IMP, BU>(p, sm, F, ls, n, T, gin, gout, in, out, level, pf, pairs_out, claim_store, out_slot);
}
template <bool WR, bool IMP, bool BU>
__device__ __forceinline__ void expand_level_any(const Params& p, Smem& sm, int4* F, unsigned ls, unsigned n,
                                                 unsigned T, const unsigned* gin, unsigned* gout, Slot* in, Slot* out,
                                                 int level, int pf, bool pairs_out, bool claim_store, int out_slot) {
  if constexpr (BU && BM_EXPAND_OOL)
    expand_level_ool<WR, IMP, BU>(p, sm, F, ls, n, T, gin, gout, in, out, level, pf, pairs_out, claim_store, out_slot);
  else
    expand_level<WR, IMP, BU>(p, sm, F, ls, n, T, gin, gout, in, out, level, pf, pairs_out, claim_store, out_slot);
}

// ---------------------------------------------------------------------------
// Bucketed pushed level: the same level as expand_level (gpubfs / gpubfs_wr,
// gpu_match.cpp:42-70, 99-133) for wide levels over a row state far beyond L2,
// in two passes separated by a grid barrier:
//   1. partition: expand_level's edge-tiled windows, but every live edge is
//      written as a triple (row, col, root) into the region of its row's bucket
//      (CTA-staged runs, one reservation per bucket per window); no row state
//      is touched;
//   2. claim: the triples bucket by bucket (chunks handed out in order), so the
//      grid's row-state gathers, claims and predecessor stores stay inside one
//      or two buckets' slice of the row state (L2-sized) instead of landing
//      anywhere in it (one random DRAM sector per edge otherwise).
// Claims, endpoints and winners are expand_level's; only their order differs,
// which the reference's races leave open too.
template <bool WR, bool IMP, bool BU>
BM_PB_FN void push_bucketed(const Params& p, Smem& sm, int4* F, unsigned ls, unsigned n, unsigned T,
                                            const unsigned* gin, unsigned* gout, Slot* in, Slot* out, int level,
                                            int pf, bool pairs_out, bool claim_store, int par) {
  const unsigned tid = threadIdx.x;
  Ctrl* ctl = p.ctl;
  unsigned c_trav = 0, c_cexp = 0, c_nvis = 0, c_entries = 0;
  const unsigned long long G = gridDim.x;
  unsigned long long per = (T + 2 * G - 1) / (2 * G);
  per = ((per + kGran - 1) / kGran) * kGran;
  if (per > (unsigned long long)kGran * kMaxTileGran) per = (unsigned long long)kGran * kMaxTileGran;
  const unsigned ET = (unsigned)per;
  const unsigned ntiles = (unsigned)((T + (unsigned long long)ET - 1) / ET);
  const unsigned out_base = ls + n;
  unsigned* const path_flag = path_flag_of(p, pf);
  const unsigned long long pol = policy_evict_first();
  const unsigned long long keep = policy_evict_last();
  const int nb = p.pb_nb, shift = p.pb_shift;
  const unsigned cap = p.pb_cap;
  const unsigned long long ovf0 = (unsigned long long)nb * cap;  // overflow region
  unsigned* const cur = ctl->pb_cur[par];

  // ---- pass 1: partition the level's live edges by row bucket ----
  for (;;) {
    if (tid == 0) sm.tile = atomicAdd(&in->tile, 1u);
    __syncthreads();
    const unsigned tile = sm.tile;
    __syncthreads();
    if (tile >= ntiles) break;
    const unsigned e0 = tile * ET;
    const unsigned e1 = (T - e0 < ET) ? T : e0 + ET;
    unsigned i = (unsigned)ld_cg(reinterpret_cast<const int*>(gin) + e0 / kGran);
    unsigned e = e0;
    while (e < e1) {
#pragma unroll
      for (int k = 0; k < kEPT; ++k) {
        const unsigned sl0 = tid * kEPT + k;
        const unsigned wi = i + sl0;
        if (wi < n) {
          const int4 ent = ld_cg_stream(F + ls + wi, pol);
          bool skip = false;
          if (WR) skip = root_dead(p, ent.y);
          sm.col[sl0] = ent.x;
          sm.root[sl0] = skip ? -1 : ent.y;
          sm.beg[sl0] = (unsigned)ent.z;
          sm.pre[sl0] = (unsigned)ent.w;
          if ((unsigned)ent.w >= e0 && (unsigned)ent.w < e1) {
            c_entries++;
            if (!skip) c_cexp++;
          }
        } else {
          sm.pre[sl0] = T;
          sm.root[sl0] = -1;
        }
      }
      if (tid == 0) sm.pre[kWin] = (i + kWin < n) ? ld_cg_u(F + ls + i + kWin) : T;
      for (int b = tid; b < nb; b += kThreads) sm.pb_hist[b] = 0;
      __syncthreads();
      const unsigned wend = min(e1, sm.pre[kWin]);
      unsigned live;
      {
        unsigned len[kEPT], nbg[kEPT], tsum = 0;
#pragma unroll
        for (int k = 0; k < kEPT; ++k) {
          const unsigned sl0 = tid * kEPT + k;
          const unsigned lo = max(sm.pre[sl0], e);
          const unsigned hi = min(sm.pre[sl0 + 1], wend);
          len[k] = (sm.root[sl0] >= 0 && hi > lo) ? hi - lo : 0u;
          nbg[k] = sm.beg[sl0] + (lo - sm.pre[sl0]);
          tsum += len[k];
        }
        const unsigned incl = warp_incl_scan(tsum);
        if (lane_id() == 31) sm.wtot[tid >> 5] = incl;
        __syncthreads();
        unsigned wbase = 0, tot = 0;
#pragma unroll
        for (int w = 0; w < kThreads / 32; ++w) {
          const unsigned t = sm.wtot[w];
          wbase += (w < (int)(tid >> 5)) ? t : 0u;
          tot += t;
        }
        live = tot;
        if (tot > kWBuf) {
          if (tid == 0 && atomicCAS(&p.ctl->error, 0, (int)kErrWindow) == 0) {
            long long* d = p.ctl->dbg;
            d[0] = ls; d[1] = n; d[2] = T; d[3] = i; d[4] = e; d[5] = wend; d[6] = tot; d[7] = level;
          }
          live = 0;
          for (int k = 0; k < kEPT; ++k) len[k] = 0;
        }
        unsigned vp = wbase + incl - tsum;
#pragma unroll
        for (int k = 0; k < kEPT; ++k) {
          const unsigned sl0 = tid * kEPT + k;
          sm.beg[sl0] = nbg[k];
          sm.pre[sl0] = vp;
          if (len[k]) {
            const unsigned q1 = (vp + len[k] - 1) >> 5;
            for (unsigned q = (vp + 31) >> 5; q <= q1; ++q) sm.cgr[q] = (unsigned short)sl0;
          }
          vp += len[k];
        }
        if (tid == 0) sm.pre[kWin] = tot;
        __syncthreads();
      }
      const unsigned nq = (live + 31) >> 5;
#pragma unroll
      for (int k = 0; k < kEPT; ++k)
        if (wend < e1 && i + kWin + k * kThreads + tid < n) prefetch_l2(F + ls + i + kWin + k * kThreads + tid);
      // stage every live edge as (row, slot | rank-in-bucket << 8); count per bucket
      for (unsigned base = 0; base < live; base += kThreads * kItems) {
        int row[kItems], sl[kItems];
#pragma unroll
        for (int k = 0; k < kItems; ++k) {
          const unsigned ee = base + k * kThreads + tid;
          row[k] = -1;
          sl[k] = 0;
          if (ee < live) {
            const unsigned q = ee >> 5;
            int a = sm.cgr[q];
            int b = (q + 1 < nq) ? (int)sm.cgr[q + 1] + 1 : kWin;
            while (b - a > 1) {
              const int mid = (a + b) >> 1;
              if (sm.pre[mid] <= ee) a = mid; else b = mid;
            }
            sl[k] = a;
            row[k] = ld_stream(p.adj + sm.beg[a] + (ee - sm.pre[a]), pol);
            c_trav++;
          }
        }
#pragma unroll
        for (int k = 0; k < kItems; ++k) {
          const unsigned ee = base + k * kThreads + tid;
          if (row[k] >= 0) {
            const unsigned rank = atomicAdd(&sm.pb_hist[row[k] >> shift], 1u);
            sm.wbuf[ee] = make_int2(row[k], sl[k] | (int)(rank << 8));
          }
        }
      }
      __syncthreads();
      // one reservation per bucket; the part of a run past its region's end goes to the overflow region
      for (int b = tid; b < nb; b += kThreads) {
        const unsigned h = sm.pb_hist[b];
        if (h) {
          const unsigned base = atomicAdd(cur + b, h);
          sm.pb_base[b] = base;
          const unsigned fit = base >= cap ? 0u : min(h, cap - base);
          if (fit < h) sm.pb_obase[b] = atomicAdd(&ctl->pb_ovf[par], h - fit);
        }
      }
      __syncthreads();
      for (unsigned ee = tid; ee < live; ee += kThreads) {
        const int2 w = sm.wbuf[ee];
        const int slw = w.y & 255;
        const unsigned rank = (unsigned)w.y >> 8;
        const int b = w.x >> shift;
        const unsigned pos = sm.pb_base[b] + rank;
        const unsigned long long idx =
            pos < cap ? (unsigned long long)b * cap + pos : ovf0 + sm.pb_obase[b] + (pos - max(sm.pb_base[b], cap));
        st_stream(p.tb + idx, make_int4(w.x, sm.col[slw], WR ? sm.root[slw] : sm.col[slw], 0), pol);
      }
      __syncthreads();
      e = wend;
      i += kWin;
    }
  }
  flush_count(sm, kStTrav, c_trav);
  flush_count(sm, kStCexp, c_cexp);
  flush_count(sm, kStEntries, c_entries);
  grid_sync(p);
  tl_mark(p, kTlBucket, n);

  // ---- pass 2: claim bucket by bucket ----
  constexpr unsigned CH = kThreads * kItems;
  if (tid == 0) {
    unsigned acc = 0;
    for (int b = 0; b < nb; ++b) {
      sm.pb_pre[b] = acc;
      acc += (min(ld_rlx(cur + b), cap) + CH - 1) / CH;
    }
    sm.pb_pre[nb] = acc;
    acc += (ld_rlx(&ctl->pb_ovf[par]) + CH - 1) / CH;
    sm.pb_pre[nb + 1] = acc;
    sm.nw = 0;
  }
  __syncthreads();
  const unsigned total = sm.pb_pre[nb + 1];
  for (;;) {
    if (tid == 0) sm.tile = atomicAdd(&ctl->pb_ticket[par], 1u);
    __syncthreads();
    const unsigned t = sm.tile;
    __syncthreads();
    if (t >= total) break;
    int b = 0;
    while (b < nb && sm.pb_pre[b + 1] <= t) ++b;  // b == nb: the overflow region
    const unsigned long long r0 = b < nb ? (unsigned long long)b * cap : ovf0;
    const unsigned m = b < nb ? min(ld_rlx(cur + b), cap) : ld_rlx(&ctl->pb_ovf[par]);
    const unsigned j0 = (t - sm.pb_pre[b]) * CH;
    int row[kItems], cm[kItems], colk[kItems], rootk[kItems];
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
      const unsigned jj = j0 + k * kThreads + tid;
      row[k] = -1;
      colk[k] = 0;
      rootk[k] = 0;
      if (jj < m) {
        const int4 tr = ld_cg_stream(p.tb + r0 + jj, pol);
        row[k] = tr.x;
        colk[k] = tr.y;
        rootk[k] = tr.z;
      }
    }
#pragma unroll
    for (int k = 0; k < kItems; ++k) cm[k] = row[k] >= 0 ? ld_rlx_hint(RM(p, row[k]), keep) : -3;
    unsigned wins = 0, eps = 0;
    int old[kItems];
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
      const int c = cm[k];
      old[k] = kVisBit;
      if (c >= 0 && !(c & kVisBit) && (!WR || p.claim_mode == 0 || !root_dead(p, rootk[k]))) {
        if (claim_store) {
          if (BM_V2ST && p.rs == 2)
            st_plain(reinterpret_cast<int2*>(RM(p, row[k])), make_int2(c | kVisBit, colk[k]));
          else
            st_plain(RM(p, row[k]), c | kVisBit);
          old[k] = c;
        } else {
          old[k] = at_or(RM(p, row[k]), kVisBit);
        }
      }
    }
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
      const int c = cm[k];
      const int col = colk[k];
      const int root = rootk[k];
      if (c >= 0) {
        if (!(old[k] & kVisBit)) {
          wins |= 1u << k;
          if (!(BU && pairs_out)) prefetch_l2(p.offs + c);  // the flush reads offs[c], offs[c+1]
          if (!(BM_V2ST && claim_store && p.rs == 2)) st_stream(PR(p, row[k]), col, pol);
          if (p.trace) st_plain(BF(p, c), level + 1);
        }
      } else if (c == -1) {
        const bool one = WR && p.ep_one;
        if ((!one || !root_dead(p, root)) && at_cas(RM(p, row[k]), -1, -2) == -1) {
          bool mine = true;
          if (one) {
            mine = at_cas(BF(p, root), kStartLevel, IMP ? -row[k] : kFoundMark) == kStartLevel;
            if (!mine) st_rlx(RM(p, row[k]), -1);
            else mark_dead(p, root);
          } else if (WR) {
            st_rlx(BF(p, root), IMP ? -row[k] : kFoundMark);
            mark_dead(p, root);
          }
          if (mine) {
            eps |= 1u << k;
            st_plain(PR(p, row[k]), col);
            if (ld_rlx(path_flag) == 0u) st_rlx(path_flag, 1u);
          }
        }
      }
    }
    {
      const unsigned mine = __popc(wins);
      const unsigned incl = warp_incl_scan(mine);
      const unsigned tot = __shfl_sync(kFull, incl, 31);
      unsigned wb = 0;
      if (lane_id() == 31 && tot) wb = atomicAdd(&sm.nw, tot);
      wb = __shfl_sync(kFull, wb, 31) + incl - mine;
#pragma unroll
      for (int k = 0; k < kItems; ++k)
        if (wins & (1u << k)) sm.wbuf[wb++] = make_int2(cm[k], WR ? rootk[k] : colk[k]);
      c_nvis += mine;
    }
    {
      const unsigned mine = __popc(eps);
      const unsigned incl = warp_incl_scan(mine);
      const unsigned tot = __shfl_sync(kFull, incl, 31);
      if (tot) {
        unsigned eb = 0;
        if (lane_id() == 31) eb = atomicAdd(&p.ctl->n_ep, tot);
        eb = __shfl_sync(kFull, eb, 31) + incl - mine;
#pragma unroll
        for (int k = 0; k < kItems; ++k)
          if (eps & (1u << k)) st_plain(p.EP + eb++, row[k]);
      }
    }
    __syncthreads();
    if (BU && pairs_out) flush_pairs(p, sm, out_base, out, pol);
    else flush_winners(p, sm, F, out_base, gout, out, pol);
    __syncthreads();
  }
  flush_count(sm, kStNvis, c_nvis);
}

// Appends one (row, col) record to the ALTERNATE write log; lanes that reach
// this point together share one atomic.
__device__ __forceinline__ void log_write(const Params& p, int row, int col) {
  cg::coalesced_group g = cg::coalesced_threads();
  unsigned base = 0;
  if (g.thread_rank() == 0) base = atomicAdd(&p.ctl->n_log, g.size());
  base = g.shfl(base, 0) + g.thread_rank();
  if (base < p.log_cap) {
    asm volatile("st.global.v2.b32 [%0], {%1,%2};" ::"l"(p.wlog + base), "r"(row), "r"(col) : "memory");
  } else {
    st_rlx(&p.ctl->log_overflow, 1u);
  }
}

// ALTERNATE walk (gpu_match.cpp:144-154): swap pairs toward the root, break
// on a column another walk already claimed this phase.
__device__ __forceinline__ void alternate_walk(const Params& p, unsigned& walks, unsigned& nsteps, int row) {
  long long steps = 0;
  while (row != -1) {
    const int col = ld_cg(PR(p, row));
    if (col < 0) break;
    const int mr = ld_rlx(CM(p, col));
    if (mr >= 0 && ld_cg(PR(p, mr)) == col) {
      if (steps > 0) log_write(p, row, -1);  // left dangling: its column now belongs to another row
      break;
    }
    st_rlx(CM(p, col), row);
    st_rlx(RM(p, row), col);
    log_write(p, row, col);
    row = mr;
    if (++steps > p.nc) {
      p.ctl->error = kErrWalk;
      break;
    }
  }
  nsteps += (unsigned)steps;
  walks++;
}

// FIX rules 1 and 2 for one row (gpu_match.cpp:221-237). The CAS keeps the
// reset count exact when a row is listed more than once.
__device__ __forceinline__ void fix_row(const Params& p, unsigned& resets, int r) {
  const int v = ld_rlx(RM(p, r));
  if (v == -2) {
    if (at_cas(RM(p, r), -2, -1) == -2) resets++;
  } else if (v >= 0 && ld_rlx(CM(p, v)) != r) {
    if (at_cas(RM(p, r), v, -1) == v) resets++;
  }
}

// FIX rule 3 for one column (gpu_match.cpp:238-243); returns true if the
// column is unmatched afterwards.
__device__ __forceinline__ bool fix_col(const Params& p, unsigned& resets, int c) {
  const int r = ld_rlx(CM(p, c));
  if (r >= 0 && ld_rlx(RM(p, r)) != c) {
    if (at_cas(CM(p, c), r, -1) == r) resets++;
    return true;
  }
  return r < 0;
}

// Clears the visited bits the BFS left in rmatch (one streaming pass, int4).
__device__ __forceinline__ void sweep_visited(const Params& p) {
  // one int4 covers 2 interleaved rows or 4 plain ones
  const bool il = p.rs == 2;
  const int kRowsPer4 = il ? 2 : 4;
#if BM_MG
  const long long r_lo = p.row_lo, nrows = (long long)p.row_hi - p.row_lo;  // own rows (32-aligned start)
#else
  const long long r_lo = 0, nrows = p.nr;
#endif
  int4* r4 = reinterpret_cast<int4*>(RML(p, r_lo));
  const unsigned long long n4 = (unsigned long long)nrows / kRowsPer4;
  auto clr = [](int& v) { if (v >= 0) v &= ~kVisBit; };
  constexpr int K = 4;  // int4s per thread in flight
  const unsigned long long GT = global_threads();
  for (unsigned long long k0 = global_thread(); k0 < n4; k0 += K * GT) {
    int4 v[K];
#pragma unroll
    for (int i = 0; i < K; ++i)
      if (k0 + i * GT < n4) v[i] = ld_cg(r4 + k0 + i * GT);
#pragma unroll
    for (int i = 0; i < K; ++i) {
      if (k0 + i * GT >= n4) continue;
      const int4 o = v[i];
      clr(v[i].x);
      if (!il) clr(v[i].y);
      clr(v[i].z);
      if (!il) clr(v[i].w);
      if (v[i].x != o.x || v[i].y != o.y || v[i].z != o.z || v[i].w != o.w) st_plain(r4 + k0 + i * GT, v[i]);
    }
  }
  for (unsigned long long r = n4 * kRowsPer4 + global_thread(); r < (unsigned long long)nrows; r += global_threads()) {
    const int v = ld_cg(RML(p, r_lo + r));
    if (v >= 0 && (v & kVisBit)) st_plain(RML(p, r_lo + r), v & ~kVisBit);
  }
}

// Whether a level of T frontier edges over n columns is pulled (bu_rule 1:
// direction-optimising BFS — pull once the frontier's edges are a large enough
// share of the edges still to explore, i.e. of the rows not yet visited).
__device__ __forceinline__ bool want_pull(const Params& p, unsigned long long T, unsigned n, unsigned ls) {
  if (p.bu_rule == 0) return T >= p.bu_min_edges;
  const long long unv = (long long)p.nr - (long long)ls - (long long)n;
  const double mu = (unv > 0 ? (double)unv : 0.0) * p.deg_row;
  return n >= p.bu_min_n && (double)T * (double)p.bu_alpha >= mu;
}

__device__ __forceinline__ void check_fail(const Params& p, long long a, long long b, long long c, long long d,
                                           long long e, long long f, long long g, long long h) {
  if (atomicCAS(&p.ctl->error, 0, (int)kErrCheck) == 0) {
    long long* x = p.ctl->dbg;
    x[0] = a; x[1] = b; x[2] = c; x[3] = d; x[4] = e; x[5] = f; x[6] = g; x[7] = h;
  }
}
// BM_CHECK: the n entries of a pushed level are consecutive edge ranges
// (pre[k] + deg[k] == pre[k+1], the last ending at T) and the granule index
// points at the entry holding each granule's first edge.
__device__ void check_level(const Params& p, const int4* F, unsigned ls, unsigned n, unsigned T, const unsigned* gin,
                            int lv, int tag) {
  for (unsigned long long k = global_thread(); k < n; k += global_threads()) {
    const int4 a = ld_cg(F + ls + k);
    if (a.x < 0 || a.x >= p.nc) {
      check_fail(p, tag + 20, lv, ls, n, T, k, a.x, a.w);
      continue;
    }
    const unsigned deg = ld_ro(p.offs + a.x + 1) - ld_ro(p.offs + a.x);
    const unsigned nxt = k + 1 < n ? (unsigned)ld_cg(F + ls + k + 1).w : T;
    if (a.x < 0 || a.x >= p.nc || (unsigned)a.w + deg != nxt || (unsigned)a.z != ld_ro(p.offs + a.x))
      check_fail(p, tag, lv, ls, n, T, k, a.w, nxt);
    if (deg) {
      const unsigned m1 = ((unsigned)a.w + deg - 1) / kGran;
      for (unsigned m = ((unsigned)a.w + kGran - 1) / kGran; m <= m1; ++m)
        if ((unsigned)ld_cg(reinterpret_cast<const int*>(gin) + m) != k) check_fail(p, tag + 10, lv, ls, n, T, k, m, 0);
    }
  }
}

struct PhaseOut {
  bool found;
  long long launches;
  long long after;
};

// One phase = run_phase (gpu_match.cpp:268-302) from the roots in F[cur].
// The end of a phase: ALTERNATE, FIX and the next phase's roots (run_phase's
// tail; returns the cardinality after the phase). A separate function so that
// its registers are allocated apart from the level loop's (BM_TAIL_FN).
template <bool WR, bool IMP, bool BU>
BM_TAIL_FN long long phase_tail(const Params& p, Smem& sm, int cur, int parity, bool serial_alt, long long isolated,
                                bool skip_alt, unsigned n0, unsigned long long rp) {
  Ctrl* ctl = p.ctl;
  int4* F = cur ? p.F1 : p.F0;
  int4* Fn = cur ? p.F0 : p.F1;
  // ---- ALTERNATE (gpu_match.cpp:158-218) ----
  if (is_leader()) *path_flag_of(p, parity ^ 1) = 0u;  // flag of the next phase
  const unsigned n_ep = ld_rlx(&ctl->n_ep);
  unsigned walks = 0, steps = 0, resets = 0;
  if (skip_alt) {
    // fault injection: a raced ALTERNATE that augmented nothing, so the driver
    // must take the serial retry (gpu_match.cpp:328-343)
  } else if (!serial_alt) {
    if (!IMP) {
      for (unsigned long long k = global_thread(); k < n_ep; k += global_threads())
        alternate_walk(p, walks, steps, ld_cg(p.EP + k));
    } else {
      for (unsigned long long k = global_thread(); k < n0; k += global_threads()) {
        const int c = ld_cg(reinterpret_cast<const int*>(F + k));
        const int mark = ld_rlx(p.bfs + c);
        if (mark <= 0) alternate_walk(p, walks, steps, -mark);  // live levels are >= 1 (L0 = 2)
      }
    }
  } else if (is_leader()) {
    // Serial retry (gpu_match.cpp:328-343): one thread walks every endpoint
    // in turn; the first walk cannot meet a claimed column, so the phase
    // always augments when a path exists.
#if BM_MG
    if (p.rank == 0)  // rank 0 walks every rank's endpoints (or roots), in rank order
      for (int q = 0; q < p.world; ++q) {
        if (!IMP) {
          const unsigned nq = ld_rlx(&p.peer[q].ctl->n_ep);
          for (unsigned k = 0; k < nq; ++k) alternate_walk(p, walks, steps, ld_cg(p.peer[q].EP + k));
        } else {
          const int4* Fq = cur ? p.peer[q].F1 : p.peer[q].F0;
          const unsigned nq = (unsigned)(ld_rlx(&p.peer[q].ctl->roots.packed) >> 33);
          for (unsigned k = 0; k < nq; ++k) {
            const int c = ld_cg(reinterpret_cast<const int*>(Fq + k));
            const int mark = ld_rlx(BF(p, c));
            if (mark <= 0) alternate_walk(p, walks, steps, -mark);
          }
        }
      }
#else
    if (!IMP) {
      for (unsigned k = 0; k < n_ep; ++k) alternate_walk(p, walks, steps, ld_cg(p.EP + k));
    } else {
      for (unsigned k = 0; k < n0; ++k) {
        const int c = ld_cg(reinterpret_cast<const int*>(F + k));
        const int mark = ld_rlx(p.bfs + c);
        if (mark <= 0) alternate_walk(p, walks, steps, -mark);
      }
    }
#endif
  }
  flush_count(sm, kStWalks, walks);
  flush_count(sm, kStSteps, steps);
  grid_sync(p);
  tl_mark(p, kTlAlt, 0);

  // ---- FIXMATCHING rules 1+2 over the rows ALTERNATE wrote or left behind ----
#if BM_MG
  bool dense = false;  // team-wide: a rank whose log overflowed lost rows of other ranks too
  for (int q = 0; q < p.world; ++q) dense = dense || ld_rlx(&p.peer[q].ctl->log_overflow) != 0u;
#else
  const bool dense = ld_rlx(&ctl->log_overflow) != 0u;
#endif
  const unsigned n_log = dense ? 0u : min(ld_rlx(&ctl->n_log), p.log_cap);
  if (!dense) {
    for (unsigned long long k = global_thread(); k < n_log; k += global_threads())
      fix_row(p, resets, ld_cg(reinterpret_cast<const int*>(p.wlog + k)));
    for (unsigned long long k = global_thread(); k < n_ep; k += global_threads())
      fix_row(p, resets, ld_cg(p.EP + k));
  } else {  // log overflow: the reference's full pass (over this rank's rows)
#if BM_MG
    const unsigned long long r_lo = p.row_lo, r_hi = p.row_hi;
#else
    const unsigned long long r_lo = 0, r_hi = p.nr;
#endif
    for (unsigned long long r = r_lo + global_thread(); r < r_hi; r += global_threads()) fix_row(p, resets, (int)r);
  }
  if (WR)
    for (unsigned long long k = global_thread(); k < (unsigned long long)p.ndead_words; k += global_threads())
      st_plain(reinterpret_cast<int*>(p.dead) + k, 0);

  if (is_leader()) {
    for (int s = 0; s < 3; ++s) {
      ctl->lvl[s].packed = 0;
      ctl->lvl[s].tile = 0;
    }
    ctl->roots.packed = 0;
    ctl->roots.tile = 0;
    ctl->mat[0].packed = 0;
    ctl->mat[1].packed = 0;
  }
  grid_sync(p);
  tl_mark(p, kTlFixRows, dense ? 1u : 0u);

  // ---- FIXMATCHING rule 3 over the columns ALTERNATE wrote; a non-root column
  //      it unmatches becomes a root of the next phase ----
#if BM_MG
  const unsigned long long c_lo = p.col_lo;  // dense: this rank's columns
  const unsigned long long ncheck = dense ? (unsigned long long)(p.col_hi - p.col_lo) : n_log;
#else
  const unsigned long long c_lo = 0;
  const unsigned long long ncheck = dense ? (unsigned long long)p.nc : n_log;
#endif
  for (unsigned long long b = (unsigned long long)blockIdx.x * kThreads; b < ncheck; b += global_threads()) {
    const unsigned long long k = b + threadIdx.x;
    bool push = false;
    int c = -1;
    unsigned beg = 0, deg = 0;
    if (k < ncheck) {
      c = dense ? (int)(c_lo + k) : ld_cg(reinterpret_cast<const int*>(p.wlog + k) + 1);
      if (c >= 0 && fix_col(p, resets, c)) {
        // roots of this phase are handled below; others enter the root set once
        if (dense) {
          push = ld_rlx(BF(p, c)) == kUnvisited;
          if (push) st_rlx(BF(p, c), kStartLevel);
        } else {
          push = at_cas(BF(p, c), kUnvisited, kStartLevel) == kUnvisited;
        }
#if BM_MG
        if (push && owner_col(p, c) != p.rank) {
          // another rank's column: route it to its owner's next roots (it was matched, so it has an edge)
          const int q = owner_col(p, c);
          const unsigned sl = (unsigned)(atomicAdd_system(&p.peer[q].ctl->rootp.packed, 1ull << 33) >> 33);
          st_plain(p.peer[q].P + sl, make_int2(c, c));
          push = false;
        }
#endif
        if (push) {
          beg = ld_ro(p.offs + c);
          deg = ld_ro(p.offs + c + 1) - beg;
          push = deg > 0;
        }
      }
    }
    unsigned long long slot;
    unsigned unused;
    if (cta_reserve(sm, push ? 1u : 0u, push ? deg : 0u, 0u, &ctl->roots, &ctl->n_ep, slot, unused) && push)
      put_entry(Fn, 0u, p.gidx0, slot, c, c, beg, deg);
  }
  if (is_leader()) {
    ctl->n_ep = 0u;
    for (int k = 0; k < 3; ++k) ctl->n_left[k] = 0u;
    ctl->n_log = 0u;
    ctl->log_overflow = 0u;
  }
  grid_sync(p);
  tl_mark(p, kTlFixCols, n_log);

  // ---- this phase's roots: still unmatched -> root again; matched -> bfs 1 ----
  for (unsigned long long b = (unsigned long long)blockIdx.x * kThreads; b < n0; b += global_threads()) {
    const unsigned long long k = b + threadIdx.x;
    bool push = false;
    int c = -1;
    unsigned beg = 0, deg = 0;
    if (k < n0) {
      const int4 ent = ld_cg(F + k);
      c = ent.x;
      if (ld_rlx(p.cmatch + c) < 0) {
        push = true;
        beg = (unsigned)ent.z;
        const unsigned nxt = (k + 1 < n0) ? ld_cg_u(F + k + 1) : (unsigned)(rp & kEdgeMask);
        deg = nxt - (unsigned)ent.w;
        st_plain(p.bfs + c, kStartLevel);
      } else {
        st_plain(p.bfs + c, kUnvisited);
      }
    }
    unsigned long long slot;
    unsigned unused;
    if (cta_reserve(sm, push ? 1u : 0u, push ? deg : 0u, 0u, &ctl->roots, &ctl->n_ep, slot, unused) && push)
      put_entry(Fn, 0u, p.gidx0, slot, c, c, beg, deg);
  }
  flush_count(sm, kStResets, resets);
  grid_sync(p);
#if BM_MG
  if (routed(p)) {  // the roots other ranks routed here join this rank's roots
    const unsigned n_rp = (unsigned)(ld_rlx(&ctl->rootp.packed) >> 33);
    if (n_rp) materialize(p, sm, Fn, 0u, n_rp, p.gidx0, &ctl->roots, policy_evict_first(), false);
    grid_sync(p);  // (every rank: the barrier is team-wide)
    if (is_leader()) ctl->rootp.packed = 0;
  }
  long long roots_tot = 0;
  for (int q = 0; q < p.world; ++q) roots_tot += (long long)(ld_rlx(&p.peer[q].ctl->roots.packed) >> 33);
  tl_mark(p, kTlRoots, (unsigned)roots_tot);
  return (long long)p.nc - isolated - roots_tot;
#else
  const unsigned long long np = ld_rlx(&ctl->roots.packed);
  tl_mark(p, kTlRoots, (unsigned)(np >> 33));
  return (long long)p.nc - isolated - (long long)(np >> 33);
#endif
}

template <bool WR, bool IMP, bool BU>
BM_PHASE_FN PhaseOut run_phase(const Params& p, Smem& sm, int cur, int parity, bool serial_alt,
                              long long isolated, bool skip_alt) {
  Ctrl* ctl = p.ctl;
  int4* F = cur ? p.F1 : p.F0;
  int4* Fn = cur ? p.F0 : p.F1;
  PhaseOut out{false, 0, 0};

  // ---- BFS level loop (expand_bfs, gpu_match.cpp:247-266) ----
  const unsigned long long rp = ld_rlx(&ctl->roots.packed);
  const unsigned n0 = (unsigned)(rp >> 33);
  unsigned n = n0;
  unsigned T = (unsigned)(rp & kEdgeMask);
  unsigned ls = 0;
  int lv = 0;
  bool found = false;
  bool in_pairs = false;  // this level's entries are (col, root) pairs in P (pulled-capable kernels)
  unsigned dirty = 0;     // frontier bitmaps holding marks (bit b: fbit[b]); grid-uniform
  bool croot_prev = false;  // the level before was pulled and wrote its frontier's roots (lazy roots)
  bool list_prev = false;   // the level before was pulled and listed its leftovers (Params::left)
  const unsigned long long pol_mat = policy_evict_first();
#if BM_MG
  if (routed(p)) {
  // Multi-GPU level loop: every rank expands its own frontier (columns it
  // owns); every winner goes to its column's owner as a pair, so each level
  // after the roots arrives as pairs and is materialized (pushed) or turned
  // into the bitmap (pulled) by its owner. Decisions (pull, stop) use team
  // totals read from every rank's counters after the barrier, so all ranks
  // take the same ones.
  (void)pol_mat;
  if (threadIdx.x == 0) {
    unsigned long long nt = 0, tt = 0, mx = 0;
    for (int q = 0; q < p.world; ++q) {
      const unsigned long long v = ld_rlx(&p.peer[q].ctl->roots.packed);
      sm.mg_ls[q] = 0;
      sm.mg_n[q] = (unsigned)(v >> 33);
      nt += v >> 33;
      tt += v & kEdgeMask;
      mx = (v >> 33) > mx ? (v >> 33) : mx;
    }
    sm.mg_tot[0] = nt;
    sm.mg_tot[1] = tt;
    sm.mg_tot[3] = mx;
  }
  __syncthreads();
  unsigned long long n_tot = sm.mg_tot[0], T_tot = sm.mg_tot[1], ls_tot = 0;
  for (;;) {
    Slot* in = lv == 0 ? &ctl->roots : &ctl->lvl[lv % 3];
    const bool bu = BU && p.roffs && !p.trace && want_pull(p, T_tot, (unsigned)n_tot, (unsigned)ls_tot);
    if (in_pairs && !bu) {  // pushed: this rank's pairs become edge-tiled entries
      Slot* ms = &ctl->mat[lv & 1];
      materialize(p, sm, F, ls, n, (lv & 1) ? p.gidx1 : p.gidx0, ms, policy_evict_first(), false);
      grid_sync(p);
      T = (unsigned)(ld_rlx(&ms->packed) & kEdgeMask);
      in_pairs = false;
    }
    Slot* outs = &ctl->lvl[(lv + 1) % 3];
    if (is_leader() && lv >= 1) {
      Slot* z = &ctl->lvl[(lv + 2) % 3];
      z->packed = 0;
      z->tile = 0;
    }
    if (is_leader()) ctl->mat[(lv + 1) & 1].packed = 0;
    if (bu) {
      bu_prep<WR>(p, sm, F, in_pairs, ls, n, lv);
      grid_sync(p);
      if (p.world > 1) {
        bu_share(p, lv);
        grid_sync(p);
      }
      bu_sweep_q<WR, IMP>(p, sm, ls + n, outs, (lv + 1) % 3, lv, parity);
      if (threadIdx.x == 0) sm.cnt[kStPulledLevels] += is_leader() ? 1 : 0;
    } else {
      // store claims when even one entry per frontier edge of the team fits every inbox
      const bool claim_store = p.claim_store && sm.mg_tot[3] + T_tot <= p.fcap;
      expand_level_any<WR, IMP, BU>(p, sm, F, ls, n, T, (lv & 1) ? p.gidx1 : p.gidx0, (lv & 1) ? p.gidx0 : p.gidx1,
                                in, outs, kStartLevel + lv, parity, true, claim_store, (lv + 1) % 3);
    }
    const long long tb = clk();
    grid_sync(p);
    if (bu) bu_clear(p, lv % kNumFbit);
    if (threadIdx.x == 0) sm.cnt[kStCycBarrier] += clk() - tb;
    tl_mark(p, kTlLevel, n);
    tl_mark(p, kTlLevelEdges, (T & 0x7fffffffu) | (bu ? 0x80000000u : 0u));
    out.launches++;
    if (threadIdx.x == 0) {
      unsigned long long nt = 0;
      for (int q = 0; q < p.world; ++q) {
        const unsigned nn = (unsigned)(ld_rlx(&p.peer[q].ctl->lvl[(lv + 1) % 3].packed) >> 33);
        sm.mg_nn[q] = nn;
        nt += nn;
      }
      sm.mg_tot[0] = nt;
    }
    __syncthreads();
    const unsigned long long n_next_tot = sm.mg_tot[0];
    found = ld_rlx(path_flag_of(p, parity)) != 0u;
    bool stop = (p.apsb && found) || n_next_tot == 0;
    if (!stop) {
      ls += n;
      n = sm.mg_nn[p.rank];
      in_pairs = true;
      T = (unsigned)fmin((double)n * p.deg_col, 4294967295.0);  // an estimate until materialized
      ls_tot += n_tot;
      n_tot = n_next_tot;
      T_tot = (unsigned long long)fmin((double)n_tot * p.deg_col, 1.8e19);
      ++lv;
      if (lv > p.nc + 2) {
        if (is_leader()) ctl->error = kErrLevels;
        stop = true;
      }
    }
    __syncthreads();  // every thread has read mg_nn before thread 0 advances the bookkeeping
    if (!stop && threadIdx.x == 0) {
      unsigned long long mx = 0;
      for (int q = 0; q < p.world; ++q) {
        sm.mg_ls[q] += sm.mg_n[q];
        sm.mg_n[q] = sm.mg_nn[q];
        const unsigned long long e = (unsigned long long)sm.mg_ls[q] + sm.mg_n[q];
        mx = e > mx ? e : mx;
      }
      sm.mg_tot[3] = mx;
    }
    __syncthreads();
    if (stop) break;
  }
  } else {  // a team of one: the single-GPU level loop below
#endif
  // Narrow levels (at most solo_edges frontier edges) run on block 0 alone,
  // back to back with CTA barriers only — a grid barrier costs more than such
  // a level's work. The other CTAs wait at one grid barrier and take over
  // when the frontier widens again or the BFS ends.
  for (;;) {
    Slot* in = lv == 0 ? &ctl->roots : &ctl->lvl[lv % 3];
    // BU: compiled only into the bottom-up kernel instances, so the push-only
    // kernel keeps its register allocation
    const bool bu = BU && p.roffs && !p.trace && T > p.solo_edges && want_pull(p, T, n, ls);
    const bool mat = BU && in_pairs && !bu;
    if (p.check && BU && in_pairs) {
      for (unsigned long long k = global_thread(); k < n; k += global_threads()) {
        const int2 pr = ld_cg(p.P + ls + k);
        if (pr.x < 0 || pr.x >= p.nc || pr.y < 0 || pr.y >= p.nc) check_fail(p, 40, lv, ls, n, T, k, pr.x, pr.y);
      }
      grid_sync(p);
    }
    if (mat) {  // pushed after all: build its edge-tiled entries first
      Slot* ms = &ctl->mat[lv & 1];
      materialize(p, sm, F, ls, n, (lv & 1) ? p.gidx1 : p.gidx0, ms, pol_mat, false);
      grid_sync(p);
      if (dirty & (1u << (lv % kNumFbit))) {  // the marks the level before left for a pull: unused
        bu_clear(p, lv % kNumFbit);           // (next written two levels on, after a grid barrier)
        dirty &= ~(1u << (lv % kNumFbit));
      }
      tl_mark(p, kTlMat, n);
      const unsigned long long mp = ld_rlx(&ms->packed);
      T = (unsigned)(mp & kEdgeMask);
      in_pairs = false;
      if (p.check && is_leader() && (mp >> 33) != n) check_fail(p, 30, lv, ls, n, T, (long long)(mp >> 33), 0, 0);
    }
    if (p.check && !bu && T > p.solo_edges) {  // (block 0's solo levels are not checked)
      check_level(p, F, ls, n, T, (lv & 1) ? p.gidx1 : p.gidx0, lv, mat ? 2 : 1);
      grid_sync(p);
    }
    const bool solo = !bu && T <= p.solo_edges;
    if (solo && blockIdx.x != 0) {
      grid_sync(p);  // block 0's hand-over
      lv = ld_rlx(&ctl->solo_lv);
      ls = (unsigned)ld_rlx(&ctl->solo_ls);
      n = (unsigned)ld_rlx(&ctl->solo_n);
      T = (unsigned)ld_rlx(&ctl->solo_T);
      found = ld_rlx(&ctl->solo_found) != 0;
      out.launches = (long long)ld_rlx((const unsigned long long*)&ctl->solo_launches);
      in_pairs = false;  // solo levels push entries
      croot_prev = false;
      list_prev = false;
      if (ld_rlx(&ctl->solo_stop)) break;
      continue;
    }
    Slot* outs = &ctl->lvl[(lv + 1) % 3];
    if (is_leader() && lv >= 1) {
      Slot* z = &ctl->lvl[(lv + 2) % 3];
      z->packed = 0;
      z->tile = 0;
    }
    if (BU && is_leader()) ctl->mat[(lv + 1) & 1].packed = 0;  // last read before this level's barrier
    if (solo) __syncthreads();
    // a wide level hands its winners on as pairs (see Params::P)
    const bool pairs_out = BU && p.roffs && !p.trace && !solo && (bu || (unsigned long long)T >= p.pairs_min_edges);
    // A wide pushed level over a row state far beyond L2 goes bucketed (push_bucketed).
    // (Marking the successor's bitmap at claim time instead of a bu_prep pass was
    // measured and lost: +20 % per phase on C5 unbucketed, +12 % bucketed.)
    const bool bucketed = BU && !bu && !solo && p.tb && (unsigned long long)T >= p.pb_min_edges &&
                          (unsigned long long)T <= p.pb_max_edges;
    // Lazy roots: when few rows are left to claim (fewer than a third of the
    // frontier), bu_prep skips the scattered root store of every frontier column
    // and the hits resolve their roots through the level before (bu_sweep_q).
    const long long unvisited = (long long)p.nr - (long long)ls - (long long)n;
    const bool lazy = BU_LAZY && WR && bu && croot_prev && in_pairs && 3 * unvisited < (long long)n;
    const bool prep_bucketed = bu && !lazy && p.tb && p.pp_nb > 0 && (unsigned long long)n >= p.pp_min;
    if (bu) {
      if (prep_bucketed)
        bu_prep_bucketed<WR>(p, sm, F, in_pairs, ls, n, lv, lv & 1);
      else
        bu_prep<WR>(p, sm, F, in_pairs, ls, n, lv, !lazy);
      grid_sync(p);
      dirty |= 1u << (lv % kNumFbit);
      tl_mark(p, kTlPrep, n);
      const bool lists = p.left[0] != nullptr;  // leftover lists (single-GPU pulled levels)
      const int2* lin = lists && list_prev ? p.left[(lv + 2) % 3] : nullptr;
      const unsigned n_in = lin ? ld_rlx(&ctl->n_left[(lv + 2) % 3]) : 0u;
      bu_sweep_q<WR, IMP>(p, sm, ls + n, outs, (lv + 1) % 3, lv, parity, lazy, lin, n_in,
                          lists ? p.left[lv % 3] : nullptr, lists ? &ctl->n_left[lv % 3] : nullptr);
      if (threadIdx.x == 0) sm.cnt[kStPulledLevels] += is_leader() ? 1 : 0;
    } else {
      // Claims by plain store (no atomic round trip; two discoverers racing on one
      // row both push its column, which the reference's plain stores allow too)
      // when one output entry per frontier edge still fits the phase's frontier
      // capacity; otherwise by atomicOr, which pushes every column once.
      const bool claim_store = p.claim_store && (unsigned long long)ls + n + T <= p.fcap;
      if (bucketed)
        push_bucketed<WR, IMP, BU>(p, sm, F, ls, n, T, (lv & 1) ? p.gidx1 : p.gidx0, (lv & 1) ? p.gidx0 : p.gidx1,
                                   in, outs, kStartLevel + lv, parity, pairs_out, claim_store, lv & 1);
      else
        expand_level_any<WR, IMP, BU>(p, sm, F, ls, n, T, (lv & 1) ? p.gidx1 : p.gidx0, (lv & 1) ? p.gidx0 : p.gidx1,
                                  in, outs, kStartLevel + lv, parity, pairs_out, claim_store, (lv + 1) % 3);
    }
    croot_prev = bu && !lazy;  // the next level may resolve its roots through this one's
    list_prev = bu && p.left[0] != nullptr;  // this level wrote its leftovers

    const long long tb = clk();
    if (solo) {
      __threadfence_block();
      __syncthreads();
    } else {
      grid_sync(p);
      if (is_leader()) ctl->n_left[(lv + 2) % 3] = 0;  // the level before's list: consumed or unused; next written at lv + 2
      if ((bucketed || prep_bucketed) && is_leader()) {  // next used two levels on (after another barrier)
        for (int b = 0; b < kPbMax; ++b) ctl->pb_cur[lv & 1][b] = 0;
        ctl->pb_ovf[lv & 1] = 0;
        ctl->pb_ticket[lv & 1] = 0;
      }
      if (dirty & (1u << (lv % kNumFbit))) {  // read by nobody from here on
        bu_clear(p, lv % kNumFbit);
        dirty &= ~(1u << (lv % kNumFbit));
      }
    }
    if (threadIdx.x == 0) sm.cnt[kStCycBarrier] += clk() - tb;
    tl_mark(p, kTlLevel, n);
    tl_mark(p, kTlLevelEdges, (T & 0x7fffffffu) | (bu ? 0x80000000u : 0u));  // frontier edges; top bit: pulled
    out.launches++;
    const unsigned long long op = ld_rlx(&outs->packed);
    const unsigned n_next = (unsigned)(op >> 33);
    found = ld_rlx(path_flag_of(p, parity)) != 0u;
    bool stop = (p.apsb && found) || n_next == 0;
    if (!stop) {
      ls += n;
      n = n_next;
      T = (unsigned)(op & kEdgeMask);
      in_pairs = pairs_out;
      if (pairs_out) T = (unsigned)fmin((double)n * p.deg_col, 4294967295.0);  // an estimate until materialized
      ++lv;
      if (lv > p.nc + 2) {
        if (is_leader()) ctl->error = kErrLevels;
        stop = true;
      }
    }
    if (solo && (stop || T > p.solo_edges)) {  // block 0 hands the BFS back to the grid
      if (threadIdx.x == 0) {
        for (int k = 0; k < 3; ++k) ctl->n_left[k] = 0;  // (solo levels list nothing; the grid restarts clean)
        ctl->solo_lv = lv;
        ctl->solo_stop = stop ? 1 : 0;
        ctl->solo_ls = ls;
        ctl->solo_n = n;
        ctl->solo_T = T;
        ctl->solo_found = found ? 1 : 0;
        ctl->solo_launches = out.launches;
      }
      grid_sync(p);
    }
    if (stop) break;
  }
  for (int b = 0; b < kNumFbit; ++b)  // marks the BFS left (its last levels): clean for the next phase
    if (dirty & (1u << b)) bu_clear(p, b);
#if BM_MG
  }
#endif
  out.found = found;
  sweep_visited(p);
  grid_sync(p);
  if (p.stop_after_bfs) return out;

  out.after = phase_tail<WR, IMP, BU>(p, sm, cur, parity, serial_alt, isolated, skip_alt, n0, rp);
  return out;
}

#if !BM_MG
// ---------------------------------------------------------------------------
// Late phases (an engine extension, single GPU, pulled-capable runs of
// GPUBFS-WR under APFB). Once few roots are left, a phase still sweeps most of
// the graph: each tree must grow until it meets one of the few free rows. A
// late phase meets in the middle instead:
//   1. a bounded backward search from the free rows over the row index,
//      alternating like the forward one (row -> its columns -> their mates);
//      each column it claims records the row it came from and its free row;
//   2. a bounded forward search from the roots; a tree's row whose mate the
//      backward search claimed (or a free row) ends the tree with a path,
//      provided the tree and that backward tree are both still unused (CAS on
//      the root's and the free row's stamps); such rows are dead ends either way;
//   3. each path is flipped: the backward part toward its free row, then the
//      forward part toward its root.
// One path per root and per free row, and forward trees never pass through a
// backward row, so the paths are vertex-disjoint and need no FIX. A late phase
// that finds nothing hands over to a full phase (run_phase), which alone ends
// the driver: a full phase without a path proves the matching maximum, as in
// the reference (gpu_match.cpp:306-359).
__device__ __forceinline__ unsigned lt_append(unsigned* cnt) {
  cg::coalesced_group g = cg::coalesced_threads();
  unsigned base = 0;
  if (g.thread_rank() == 0) base = atomicAdd(cnt, g.size());
  return g.shfl(base, 0) + g.thread_rank();
}
__device__ __forceinline__ int lt_stamp(const int2* a, long long i) {
  return ld_rlx(reinterpret_cast<const int*>(a + i));
}
#ifndef BM_LT_U
#define BM_LT_U 1
#endif
constexpr int kLtU = BM_LT_U;  // late levels: edges per lane per step (A/B on C5: 1 25.8 ms, 2 26.0, 4 26.8)
// Lanes of a warp that step in lockstep reserve their queue slots with one atomic.
__device__ __forceinline__ unsigned lt_reserve(unsigned* cnt, bool want) {
  const unsigned m = __ballot_sync(kFull, want);
  if (!m) return 0u;
  const int leader = __ffs(m) - 1;
  unsigned base = 0;
  if ((int)lane_id() == leader) base = atomicAdd(cnt, (unsigned)__popc(m));
  base = __shfl_sync(kFull, base, leader);
  return base + (unsigned)__popc(m & lanemask_lt());
}
__device__ __forceinline__ void lt_seed(const Params& p, unsigned qcap, int2* q, int r) {
  if (ld_ro(p.roffs + r + 1) == ld_ro(p.roffs + r)) return;  // no edge
  const unsigned s = lt_append(&p.ctl->lt_b[0]);
  if (s < qcap) st_plain(q + s, make_int2(r, r));
  else st_rlx(&p.ctl->lt_ovf, 1u);
}
// The tree rooted at R takes its one path (false: it already has one).
__device__ __forceinline__ bool lt_take_root(const Params& p, int R, int ep) {
  unsigned long long* w = reinterpret_cast<unsigned long long*>(p.lt_col + R);
  const unsigned long long old = ld_rlx(w);
  if ((int)(unsigned)old == ep) return false;
  return atomicCAS(w, old, (unsigned long long)(unsigned)ep | (0xfffffffeull << 32)) == old;
}

__device__ __noinline__ long long late_phase(const Params& p, Smem& sm, int cur, long long isolated,
                                             unsigned& levels, unsigned& paths, bool& proven) {
  Ctrl* ctl = p.ctl;
  const int4* F = cur ? p.F1 : p.F0;
  int4* Fn = cur ? p.F0 : p.F1;
  const unsigned long long rp = ld_rlx(&ctl->roots.packed);
  const unsigned n0 = (unsigned)(rp >> 33);
  grid_sync(p);  // every thread has read the roots' slot
  if (is_leader()) {
    st_rlx(p.lt_epoch, ld_rlx(p.lt_epoch) + 1);
    ctl->roots.packed = 0;
    ctl->roots.tile = 0;
    for (int k = 0; k < 3; ++k) {
      ctl->lt_b[k] = 0;
      ctl->lt_f[k] = 0;
    }
    ctl->lt_nep = 0;
    ctl->lt_hit = 0;
    ctl->lt_ovf = 0;
  }
  grid_sync(p);
  const int ep = ld_rlx(p.lt_epoch);
  const unsigned qcap = p.lt_qcap;
  int2* Q[2] = {p.P, p.P + qcap};
  // A warp takes 4 entries at a time, 8 lanes per entry, stepping through the
  // entries' edges in lockstep (one queue atomic per step: lt_reserve).
  const unsigned gl = lane_id() & 7u;
  const unsigned long long w4 = (global_thread() >> 5) * 4, nw4 = (global_threads() >> 5) * 4;

  // ---- backward seeds: the free rows with an edge (one streaming pass over the row state) ----
  {
    const int per = p.rs == 2 ? 2 : 4;  // rows per int4
    const unsigned long long n4 = (unsigned long long)p.nr / per;
    const int4* r4 = reinterpret_cast<const int4*>(p.rm);
    for (unsigned long long k = global_thread(); k < n4; k += global_threads()) {
      const int4 v = ld_cg(r4 + k);
      if (per == 2) {
        if (v.x == -1) lt_seed(p, qcap, Q[0], (int)(2 * k));
        if (v.z == -1) lt_seed(p, qcap, Q[0], (int)(2 * k + 1));
      } else {
        if (v.x == -1) lt_seed(p, qcap, Q[0], (int)(4 * k));
        if (v.y == -1) lt_seed(p, qcap, Q[0], (int)(4 * k + 1));
        if (v.z == -1) lt_seed(p, qcap, Q[0], (int)(4 * k + 2));
        if (v.w == -1) lt_seed(p, qcap, Q[0], (int)(4 * k + 3));
      }
    }
    for (unsigned long long r = n4 * per + global_thread(); r < (unsigned long long)p.nr; r += global_threads())
      if (ld_cg(RML(p, r)) == -1) lt_seed(p, qcap, Q[0], (int)r);
  }
  grid_sync(p);

  // ---- backward levels: (row, free row) entries ----
  unsigned blv = 0;
  unsigned long long btot = 0;
  bool exhausted = false;  // the backward search ran out of rows (not out of bounds)
  for (;;) {
    const unsigned n = min(ld_rlx(&ctl->lt_b[blv % 3]), qcap);
    if (n == 0) {
      exhausted = true;
      break;
    }
    if ((int)blv >= p.lt_blv || btot + n > p.lt_bcap) break;
    if (is_leader()) ctl->lt_b[(blv + 2) % 3] = 0;  // last read before the previous barrier
    unsigned* outc = &ctl->lt_b[(blv + 1) % 3];
    const int2* in = Q[blv & 1];
    int2* nxt = Q[(blv + 1) & 1];
    unsigned c_trav = 0, c_ent = 0, c_vis = 0;
    for (unsigned long long kb = w4; kb < n; kb += nw4) {
      const unsigned long long k = kb + (lane_id() >> 3);
      int2 e = make_int2(-1, -1);
      unsigned j = 0, j1 = 0;
      if (k < n) {
        e = ld_cg(in + k);
        j = ld_ro(p.roffs + e.x) + gl;
        j1 = ld_ro(p.roffs + e.x + 1);
        c_ent += gl == 0 ? 1u : 0u;
      }
      // kLtU edges per lane per step, their loads and CASes issued back to back
      const unsigned long long nw = (unsigned long long)(unsigned)ep | ((unsigned long long)(unsigned)e.x << 32);
      while (__any_sync(kFull, j < j1)) {
        int cc[kLtU], mm[kLtU];
        unsigned long long ow[kLtU], got[kLtU];
#pragma unroll
        for (int u = 0; u < kLtU; ++u) cc[u] = j + 8u * u < j1 ? ld_ro(p.radj + j + 8u * u) : -1;
#pragma unroll
        for (int u = 0; u < kLtU; ++u) mm[u] = cc[u] >= 0 ? ld_rlx(p.cmatch + cc[u]) : -1;
#pragma unroll
        for (int u = 0; u < kLtU; ++u)
          ow[u] = mm[u] >= 0 ? ld_rlx(reinterpret_cast<const unsigned long long*>(p.lt_col + cc[u])) : 0ull;
#pragma unroll
        for (int u = 0; u < kLtU; ++u)
          got[u] = (mm[u] >= 0 && (int)(unsigned)ow[u] != ep)
                       ? atomicCAS(reinterpret_cast<unsigned long long*>(p.lt_col + cc[u]), ow[u], nw)
                       : ~ow[u];
#pragma unroll
        for (int u = 0; u < kLtU; ++u) {
          bool push = false;
          if (cc[u] >= 0) {
            c_trav++;
            if (mm[u] < 0) {  // a free column: an augmenting path may exist (the forward search starts there)
              if (ld_rlx(&ctl->lt_hit) == 0u) st_rlx(&ctl->lt_hit, 1u);
            } else if (got[u] == ow[u]) {
              st_plain(p.lt_croot + cc[u], e.y);
              push = true;
              c_vis++;
            }
          }
          const unsigned s = lt_reserve(outc, push);
          if (push && s < qcap) st_plain(nxt + s, make_int2(mm[u], e.y));
          if (push && s >= qcap) st_rlx(&ctl->lt_ovf, 1u);
        }
        j += 8u * kLtU;
      }
    }
    flush_count(sm, kStTrav, c_trav);
    flush_count(sm, kStCexp, c_ent);
    flush_count(sm, kStNvis, c_vis);
    grid_sync(p);
    tl_mark(p, kTlLateLevel, n | 0x80000000u);
    btot += min(ld_rlx(outc), qcap);
    ++blv;
  }

  // ---- forward levels: (column, root) entries; level 0 = the roots ----
  unsigned flv = 0, nf = n0;
  unsigned long long ftot = 0;
  for (;;) {
    // bounded: a level is expanded only while the search stays within lt_fcap entries and
    // within lt_fper entries per root still without a path (trees that found no path that
    // far are most likely without one: the full phase takes them)
    const unsigned nep_now = ld_rlx(&ctl->lt_nep);
    const unsigned long long lim =
        min((unsigned long long)p.lt_fcap, 65536ull + (unsigned long long)p.lt_fper * (n0 - min(nep_now, n0)));
    if (nf == 0 || nep_now >= n0 || (int)flv >= p.lt_flv || ftot + nf > lim) break;
    if (is_leader()) ctl->lt_f[(flv + 2) % 3] = 0;
    unsigned* outc = &ctl->lt_f[(flv + 1) % 3];
    const int2* in = Q[flv & 1];
    int2* nxt = Q[(flv + 1) & 1];
    unsigned c_trav = 0, c_ent = 0, c_vis = 0;
    for (unsigned long long kb = w4; kb < nf; kb += nw4) {
      const unsigned long long k = kb + (lane_id() >> 3);
      int col = -1, R = -1;
      unsigned j = 0, j1 = 0;
      if (k < nf) {
        if (flv == 0) {
          col = R = ld_cg(reinterpret_cast<const int*>(F + k));
        } else {
          const int2 e = ld_cg(in + k);
          col = e.x;
          R = e.y;
        }
        if (lt_stamp(p.lt_col, R) != ep) {  // (else the tree has its path)
          j = ld_ro(p.offs + col) + gl;
          j1 = ld_ro(p.offs + col + 1);
          c_ent += gl == 0 ? 1u : 0u;
        }
      }
      while (__any_sync(kFull, j < j1)) {
        int rr[kLtU], old[kLtU], cas[kLtU], mm[kLtU], stm[kLtU];
        bool won[kLtU];
#pragma unroll
        for (int u = 0; u < kLtU; ++u) rr[u] = j + 8u * u < j1 ? ld_ro(p.adj + j + 8u * u) : -1;
#pragma unroll
        for (int u = 0; u < kLtU; ++u) old[u] = rr[u] >= 0 ? ld_rlx(p.lt_row + rr[u]) : ep;
#pragma unroll
        for (int u = 0; u < kLtU; ++u) cas[u] = old[u] != ep ? atomicCAS(p.lt_row + rr[u], old[u], ep) : ep;
#pragma unroll
        for (int u = 0; u < kLtU; ++u) {
          won[u] = old[u] != ep && cas[u] == old[u];
          if (won[u]) st_rlx(PR(p, rr[u]), col);
        }
#pragma unroll
        for (int u = 0; u < kLtU; ++u) mm[u] = won[u] ? ld_rlx(RML(p, rr[u])) : -1;
#pragma unroll
        for (int u = 0; u < kLtU; ++u) stm[u] = mm[u] >= 0 ? lt_stamp(p.lt_col, mm[u]) : 0;
#pragma unroll
        for (int u = 0; u < kLtU; ++u) {
          bool push = false, got = false;
          if (rr[u] >= 0) c_trav++;
          if (won[u]) {
            c_vis++;
            if (mm[u] < 0) {  // a free row (this claim also used it up)
              got = lt_take_root(p, R, ep);
            } else if (stm[u] == ep) {  // a backward row: meet, or a dead end
              const int fr = ld_rlx(p.lt_croot + mm[u]);
              const int of = ld_rlx(p.lt_row + fr);
              if (of != ep && atomicCAS(p.lt_row + fr, of, ep) == of) {
                got = lt_take_root(p, R, ep);
                if (!got) st_rlx(p.lt_row + fr, 0);  // hand the free row back
              }
            } else {
              push = true;
            }
          }
          const unsigned se = lt_reserve(&ctl->lt_nep, got);  // (one path per root: < n0 <= nr)
          if (got) st_plain(p.EP + se, rr[u]);
          const unsigned s = lt_reserve(outc, push);
          if (push && s < qcap) st_plain(nxt + s, make_int2(mm[u], R));
        }
        j += 8u * kLtU;
      }
    }
    flush_count(sm, kStTrav, c_trav);
    flush_count(sm, kStCexp, c_ent);
    flush_count(sm, kStNvis, c_vis);
    grid_sync(p);
    tl_mark(p, kTlLateLevel, nf);
    ftot += nf;
    nf = min(ld_rlx(outc), qcap);
    ++flv;
  }

  // ---- flip the paths ----
  const unsigned nep = ld_rlx(&ctl->lt_nep);
  unsigned c_walks = 0, c_steps = 0;
  for (unsigned long long k = global_thread(); k < nep; k += global_threads()) {
    const int e = ld_cg(p.EP + k);
    long long steps = 0;
    c_walks++;
    int c = ld_rlx(RML(p, e));
    while (c >= 0) {  // backward part: e's column moves to the row the backward search reached it from
      const int r2 = ld_rlx(reinterpret_cast<const int*>(p.lt_col + c) + 1);
      const int c2 = ld_rlx(RML(p, r2));
      st_rlx(RML(p, r2), c);
      st_rlx(p.cmatch + c, r2);
      c = c2;
      if (++steps > p.nc) {
        ctl->error = kErrWalk;
        break;
      }
    }
    int row = e;
    while (row >= 0) {  // forward part, toward the root
      const int col = ld_rlx(PR(p, row));
      const int mr = ld_rlx(p.cmatch + col);
      st_rlx(p.cmatch + col, row);
      st_rlx(RML(p, row), col);
      row = mr;
      if (++steps > p.nc) {
        ctl->error = kErrWalk;
        break;
      }
    }
    c_steps += (unsigned)steps;
  }
  flush_count(sm, kStWalks, c_walks);
  flush_count(sm, kStSteps, c_steps);
  grid_sync(p);

  // ---- the roots left (as phase_tail's last step) ----
  for (unsigned long long b = (unsigned long long)blockIdx.x * kThreads; b < n0; b += global_threads()) {
    const unsigned long long k = b + threadIdx.x;
    bool push = false;
    int c = -1;
    unsigned beg = 0, deg = 0;
    if (k < n0) {
      const int4 ent = ld_cg(F + k);
      c = ent.x;
      if (ld_rlx(p.cmatch + c) < 0) {
        push = true;
        beg = (unsigned)ent.z;
        const unsigned nxt = (k + 1 < n0) ? ld_cg_u(F + k + 1) : (unsigned)(rp & kEdgeMask);
        deg = nxt - (unsigned)ent.w;
      } else {
        st_plain(p.bfs + c, kUnvisited);
      }
    }
    unsigned long long slot;
    unsigned unused;
    if (cta_reserve(sm, push ? 1u : 0u, push ? deg : 0u, 0u, &ctl->roots, &ctl->n_ep, slot, unused) && push)
      put_entry(Fn, 0u, p.gidx0, slot, c, c, beg, deg);
  }
  grid_sync(p);
  const unsigned long long np = ld_rlx(&ctl->roots.packed);
  levels = blv + flv;
  paths = nep;
  // No path, and the alternating search from every free row ran to its end
  // without meeting a free column: no augmenting path exists (Berge), so the
  // matching is maximum — the same certificate a full phase without a path
  // gives, taken from the free rows' side.
  proven = nep == 0 && exhausted && ld_rlx(&ctl->lt_hit) == 0u && ld_rlx(&ctl->lt_ovf) == 0u;
  tl_mark(p, kTlLate, nep);
  return (long long)p.nc - isolated - (long long)(np >> 33);
}
#endif

// ---------------------------------------------------------------------------
template <bool WR, bool IMP, bool BU>
#if BM_MG
__global__ void __launch_bounds__(kThreads, BU ? BM_MINB_BU : BM_MINB_PUSH) driver_kernel(const __grid_constant__ Params p) {
  // (grid constant: the peer table is indexed at run time without a local copy)
  const unsigned long long c_lo = p.col_lo, c_hi = p.col_hi, r_lo = p.row_lo, r_hi = p.row_hi;
#else
__global__ void __launch_bounds__(kThreads, BU ? BM_MINB_BU : BM_MINB_PUSH) driver_kernel(Params p) {
  const unsigned long long c_lo = 0, c_hi = p.nc, r_lo = 0, r_hi = p.nr;
#endif
  extern __shared__ __align__(16) unsigned char smem_raw[];  // sizeof(Smem) > 48 KB: dynamic shared memory
  Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
  Ctrl* ctl = p.ctl;
  if (threadIdx.x < kNumStats) sm.cnt[threadIdx.x] = 0;
  __syncthreads();
  tl_mark(p, kTlStart, p.fresh);

  int cur;
  long long card, outer, isolated;
  int recs = 0;

  if (p.fresh) {
    // ---- optional GPU initial matching (parallel first-fit with CAS) ----
    if (p.init_mode != BM_INIT_GIVEN) {
      for (int pass = (p.init_mode == BM_INIT_GPU_KS ? 0 : 1); pass < 2; ++pass) {
        // Parallel greedy (the GPU cheap init: a maximal matching like first-fit,
        // matching.cpp:13-26) with CAS: each thread walks two columns at once,
        // gathering 4 of each column's rows' states per round, in first-fit order.
        const unsigned long long GT = global_threads();
        for (unsigned long long c0 = c_lo + global_thread(); c0 < c_hi; c0 += 2 * GT) {
          unsigned long long cc[2] = {c0, c0 + GT};
          bool act[2];
          unsigned j[2], e[2], b0[2];
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            act[i] = cc[i] < c_hi && ld_cg(p.cmatch + cc[i]) == -1;
            b0[i] = act[i] ? ld_ro(p.offs + cc[i]) : 0u;
            e[i] = act[i] ? ld_ro(p.offs + cc[i] + 1) - b0[i] : 0u;  // (degree)
            if (pass == 0 && e[i] != 1) act[i] = false;  // one-sided Karp-Sipser: degree-1 columns first
            if (e[i] == 0) act[i] = false;
            j[i] = 0;  // probes done
          }
          while (act[0] || act[1]) {
            int rw[2][4], st[2][4];
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
              for (int k = 0; k < 4; ++k) rw[i][k] = act[i] && j[i] + k < e[i] ? ld_ro(p.adj + b0[i] + j[i] + k) : -1;
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
              for (int k = 0; k < 4; ++k) st[i][k] = rw[i][k] >= 0 ? ld_rlx(RM(p, rw[i][k])) : 0;
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              if (!act[i]) continue;
#pragma unroll
              for (int k = 0; k < 4; ++k)
                if (act[i] && st[i][k] == -1 && at_cas(RM(p, rw[i][k]), -1, (int)cc[i]) == -1) {
                  st_plain(p.cmatch + cc[i], rw[i][k]);
                  act[i] = false;
                }
              j[i] += 4;
              if (j[i] >= e[i]) act[i] = false;
            }
          }
        }
        grid_sync(p);
        tl_mark(p, kTlInit, pass);
      }
    }
    // ---- setup: validate init, bfs_array init, roots of phase 1 ----
    unsigned long long bad = 0, iso = 0, mrows = 0, mcols = 0;
    // A CTA takes kSetupK x kThreads consecutive columns per step and reserves
    // their roots' frontier slots with ONE cta_reserve (one per 256 columns cost
    // 4.5 ms at C5: 390K barrier-separated reservations on one counter).
    constexpr int kSetupK = 8;
    for (unsigned long long b = c_lo + (unsigned long long)blockIdx.x * kThreads * kSetupK; b < c_hi;
         b += global_threads() * kSetupK) {
      unsigned rootm = 0, beg[kSetupK], deg[kSetupK], cnt = 0, sum = 0;
#pragma unroll
      for (int k = 0; k < kSetupK; ++k) {
        const unsigned long long c = b + (unsigned long long)k * kThreads + threadIdx.x;
        beg[k] = 0;
        deg[k] = 0;
        if (c < c_hi) {
          const int r = ld_cg(p.cmatch + c);
          if (!p.init_checked) {
            if (r < -1 || r >= p.nr) bad++;
            else if (r >= 0 && ld_cg(RM(p, r)) != (int)c) bad++;
            else if (r >= 0 && !has_edge(p.adj, ld_ro(p.offs + c), ld_ro(p.offs + c + 1), r, p.sorted)) bad++;
            else if (r >= 0) mcols++;
          }
          st_plain(p.bfs + c, r >= 0 ? kUnvisited : kStartLevel);
          if (r < 0) {
            beg[k] = ld_ro(p.offs + c);
            deg[k] = ld_ro(p.offs + c + 1) - beg[k];
            if (deg[k] > 0) {
              rootm |= 1u << k;
              cnt++;
              sum += deg[k];
            } else {
              iso++;
            }
          }
        }
      }
      unsigned long long slot;
      unsigned unused;
      if (cta_reserve(sm, cnt, sum, 0u, &ctl->roots, &ctl->n_ep, slot, unused)) {
#pragma unroll
        for (int k = 0; k < kSetupK; ++k)
          if (rootm & (1u << k)) {
            const int c = (int)(b + (unsigned long long)k * kThreads + threadIdx.x);
            put_entry(p.F0, 0u, p.gidx0, slot, c, c, beg[k], deg[k]);
            slot += (1ull << 33) + deg[k];
          }
      }
    }
    // Rows need no gather: every matched column's row points back to it (above),
    // so cmatch is injective into the matched rows; equal counts make it onto,
    // i.e. every matched row's column points back too (validate, matching.cpp:70-104).
    if (!p.init_checked)
      for (unsigned long long r = r_lo + global_thread(); r < r_hi; r += global_threads()) {
        const int v = ld_cg(RML(p, r));
        if (v < -1 || v >= p.nc) bad++;
        else if (v >= 0) mrows++;
      }
    bad = warp_sum(bad);
    iso = warp_sum(iso);
    mrows = warp_sum(mrows);
    mcols = warp_sum(mcols);
    if (lane_id() == 0) {
      if (bad) atomicAdd(&ctl->invalid, bad);
      if (iso) atomicAdd(&ctl->isolated, iso);
      if (mrows) atomicAdd(&ctl->init_rows, mrows);
      if (mcols) atomicAdd(&ctl->init_cols, mcols);
    }
    grid_sync(p);
    tl_mark(p, kTlSetup, 0);
#if BM_MG
    unsigned long long inv_tot = 0, iso_tot = 0, roots_tot = 0, mr_tot = 0, mc_tot = 0;  // team totals
    for (int q = 0; q < p.world; ++q) {
      mr_tot += ld_rlx(&p.peer[q].ctl->init_rows);
      mc_tot += ld_rlx(&p.peer[q].ctl->init_cols);
      inv_tot += ld_rlx(&p.peer[q].ctl->invalid);
      iso_tot += ld_rlx(&p.peer[q].ctl->isolated);
      roots_tot += ld_rlx(&p.peer[q].ctl->roots.packed) >> 33;
    }
#else
    const unsigned long long inv_tot = ld_rlx(&ctl->invalid), iso_tot = ld_rlx(&ctl->isolated);
    const unsigned long long mr_tot = ld_rlx(&ctl->init_rows), mc_tot = ld_rlx(&ctl->init_cols);
    const unsigned long long roots_tot = ld_rlx(&ctl->roots.packed) >> 33;
#endif
    if (inv_tot != 0ull || (!p.init_checked && mr_tot != mc_tot)) {
      if (is_leader()) ctl->error = kErrInvalidInit;
      return;
    }
    isolated = (long long)iso_tot;
    cur = 0;
    card = (long long)p.nc - isolated - (long long)roots_tot;
    outer = 0;
    if (is_leader()) {
      ctl->init_card = card;
      ctl->isolated_cols = isolated;
    }
  } else {
    cur = ctl->cur;
    card = ctl->card;
    outer = ctl->outer;
    isolated = ctl->isolated_cols;
  }
  int parity = ctl->phase_parity;
  if (p.fresh) parity = 0;

  // ---- driver loop (run_driver, gpu_match.cpp:306-359) ----
  bool done = false;
#if !BM_MG
  // late phases (late_phase): APFB over GPUBFS-WR with the row index, no probes
  const bool late_on = BU && WR && !IMP && !p.apsb && p.lt_col != nullptr && p.roffs != nullptr && !p.trace &&
                       !p.stop_after_bfs && p.dbg_skip_alt_phase == 0;
  bool late_ok = late_on;
#endif
  for (;;) {
    if (outer + 1 > p.phase_bound) {
      if (is_leader()) ctl->error = kErrBound;
      break;
    }
    ++outer;
    const long long before = card;
    long long late_levels = 0;
#if !BM_MG
    if constexpr (BU && WR && !IMP) {
      const unsigned nroots = (unsigned)(ld_rlx(&ctl->roots.packed) >> 33);
      if (late_ok && nroots > 0 && nroots <= p.lt_max_roots) {
        unsigned lvls = 0, paths = 0;
        bool proven = false;
        const long long after = late_phase(p, sm, cur, isolated, lvls, paths, proven);
        cur ^= 1;
        if (is_leader()) {
          sm.cnt[kStLatePhases]++;
          sm.cnt[kStLatePaths] += paths;
        }
        if (after > before) {
          if (is_leader()) {
            if (recs < p.rec_cap) {
              PhaseRec r;
              r.launches = lvls;
              r.before = before;
              r.after = after;
              r.found = 1;
              r.retry = 0;
              p.recs[recs] = r;
            }
            sm.cnt[kStLevels] += lvls;
          }
          ++recs;
          card = after;
          if (ld_rlx((const unsigned*)&ctl->error) != 0u) break;
          if (recs >= p.max_phases || recs >= p.rec_cap) break;
          continue;
        }
        if (proven) {  // maximum: this late phase is the run's last phase
          if (is_leader()) {
            if (recs < p.rec_cap) {
              PhaseRec r;
              r.launches = lvls;
              r.before = before;
              r.after = after;
              r.found = 0;
              r.retry = 0;
              p.recs[recs] = r;
            }
            sm.cnt[kStLevels] += lvls;
            sm.cnt[kStLateProofs]++;
          }
          ++recs;
          card = after;
          done = true;
          break;
        }
        late_ok = false;  // nothing found: this phase runs in full
        late_levels = lvls;
      }
    }
#endif
    PhaseOut ph = run_phase<WR, IMP, BU>(p, sm, cur, parity, false, isolated, outer == p.dbg_skip_alt_phase);
    if (p.stop_after_bfs) {
      if (is_leader()) {
        ctl->bfs_levels_last = ph.launches;
        ctl->path_found_last = ph.found ? 1 : 0;
      }
      done = true;
      break;
    }
    cur ^= 1;
    parity ^= 1;
    long long launches = ph.launches + late_levels;
    long long after = ph.after;
    bool retried = false;
    if (ph.found && after <= before) {
      PhaseOut rt = run_phase<WR, IMP, BU>(p, sm, cur, parity, true, isolated, false);
      cur ^= 1;
      parity ^= 1;
      launches += rt.launches;
      after = rt.after;
      ph.found = rt.found;
      retried = true;
    }
    if (is_leader()) {
      if (recs < p.rec_cap) {
        PhaseRec r;
        r.launches = launches;
        r.before = before;
        r.after = after;
        r.found = ph.found ? 1 : 0;
        r.retry = retried ? 1 : 0;
        p.recs[recs] = r;
      }
      sm.cnt[kStLevels] += (unsigned long long)launches;
      if (retried) sm.cnt[kStRetries]++;
    }
    ++recs;
    card = after;
    if (!ph.found) {
      done = true;
      break;
    }
#if !BM_MG
    late_ok = late_on;  // the full phase found paths: the next one may be late again
#endif
#if BM_MG
    bool err = false;  // any rank's error stops every rank (they all read it after the same barrier)
    for (int q = 0; q < p.world; ++q) err = err || ld_rlx((const unsigned*)&p.peer[q].ctl->error) != 0u;
    if (err) break;
#else
    if (ld_rlx((const unsigned*)&ctl->error) != 0u) break;
#endif
    if (recs >= p.max_phases || recs >= p.rec_cap) break;
  }

  // ---- flush counters and run state ----
  tl_mark(p, kTlEnd, 0);
  __syncthreads();
  if (threadIdx.x < kNumStats && sm.cnt[threadIdx.x]) atomicAdd(&ctl->stats[threadIdx.x], sm.cnt[threadIdx.x]);
  if (is_leader()) {
    ctl->cur = cur;
    ctl->card = card;
    ctl->outer = outer;
    ctl->done = done ? 1 : 0;
    ctl->n_recs = recs < p.rec_cap ? recs : p.rec_cap;
    ctl->phase_parity = parity;
  }
}

// ---------------------------------------------------------------------------
// Upload-time validation (check_csr, csr_graph.cpp:45-64) and offset narrowing.
__global__ void convert_offsets_kernel(const long long* in, unsigned* out, int nc, long long E,
                                       unsigned long long* bad, unsigned long long* empty) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i <= nc;
       i += (long long)gridDim.x * blockDim.x) {
    const long long v = in[i];
    bool ok = v >= 0 && v <= E;
    if (i == 0 && v != 0) ok = false;
    if (i == nc && v != E) ok = false;
    if (i > 0 && in[i - 1] > v) ok = false;
    if (!ok) atomicAdd(bad, 1ull);
    const unsigned e = __ballot_sync(__activemask(), i > 0 && in[i - 1] == v);  // column i-1 is empty
    if (e && (threadIdx.x & 31) == __ffs(__activemask()) - 1) atomicAdd(empty, (unsigned long long)__popc(e));
    out[i] = (unsigned)v;
  }
}

// Flat adjacency check over [j0, j1) (one pass, vector loads): rows out of
// range, and descending neighbour pairs (j-1, j) anywhere — pairs that straddle
// a column start are subtracted by col_start_pairs_kernel. Runs per uploaded
// chunk, overlapped with the copy of the next chunk.
__global__ void check_adj_flat_kernel(const int* adj, long long j0, long long j1, int nr,
                                      unsigned long long* bad_range, unsigned long long* desc) {
  unsigned long long br = 0, ds = 0;
  const long long tot = (long long)gridDim.x * blockDim.x;
  for (long long j = j0 + blockIdx.x * (long long)blockDim.x + threadIdx.x; j < j1; j += tot) {
    const int r = adj[j];
    if (r < 0 || r >= nr) br++;
    if (j > 0 && adj[j - 1] >= r) ds++;
  }
  br = warp_sum(br);
  ds = warp_sum(ds);
  if (lane_id() == 0) {
    if (br) atomicAdd(bad_range, br);
    if (ds) atomicAdd(desc, ds);
  }
}
__global__ void col_start_pairs_kernel(const unsigned* offs, const int* adj, int nc, unsigned long long* desc_fix) {
  unsigned long long f = 0;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < nc; c += (long long)gridDim.x * blockDim.x) {
    const unsigned b = offs[c];
    if (b > 0 && offs[c + 1] > b && adj[b - 1] >= adj[b]) f++;
  }
  f = warp_sum(f);
  if (lane_id() == 0 && f) atomicAdd(desc_fix, f);
}

// Validity half of the Berge certificate (validate, matching.cpp:70-104).
__global__ void validate_kernel(const unsigned* offs, const int* adj, int nc, int nr, int sorted,
                                const int* rmatch, const int* cmatch,
                                unsigned long long* violations, unsigned long long* matched) {
  const long long tot = (long long)gridDim.x * blockDim.x;
  unsigned long long bad = 0, m = 0;
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < nr; r += tot) {
    const int c = rmatch[r];
    if (c == -1) continue;
    if (c < 0 || c >= nc) { bad++; continue; }  // -2 pending flag or out of range
    if (cmatch[c] != (int)r) { bad++; continue; }
    const unsigned b = offs[c], e = offs[c + 1];
    bool has = false;
    if (sorted) {
      unsigned lo = b, hi = e;
      while (lo < hi) {
        const unsigned mid = lo + ((hi - lo) >> 1);
        const int v = adj[mid];
        if (v == (int)r) { has = true; break; }
        if (v < (int)r) lo = mid + 1; else hi = mid;
      }
    } else {
      for (unsigned j = b; j < e && !has; ++j) has = adj[j] == (int)r;
    }
    if (!has) bad++; else m++;
  }
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < nc; c += tot) {
    const int r = cmatch[c];
    if (r == -1) continue;
    if (r < 0 || r >= nr) { bad++; continue; }
    if (rmatch[r] != (int)c) bad++;
  }
  bad = warp_sum(bad);
  m = warp_sum(m);
  if ((threadIdx.x & 31) == 0) {
    if (bad) atomicAdd(violations, bad);
    if (m) atomicAdd(matched, m);
  }
}

// Maximality half of the certificate (is_maximum, matching.cpp:106-131) as a
// plain queue BFS that shares nothing with driver_kernel: alternating levels
// from every free non-isolated column over the plain rmatch, a visited bitmap
// of its own, one warp per frontier column, one launch per level. A free row
// reached from a free column is an augmenting path.
__global__ void verify_roots_kernel(const unsigned* offs, const int* cmatch, int nc, unsigned* vis, int* q,
                                    unsigned* qn) {
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < nc; c += (long long)gridDim.x * blockDim.x) {
    if (cmatch[c] != -1 || offs[c + 1] == offs[c]) continue;
    atomicOr(vis + (c >> 5), 1u << (c & 31));
    q[atomicAdd(qn, 1u)] = (int)c;
  }
}
__global__ void verify_level_kernel(const unsigned* offs, const int* adj, const int* rmatch, const int* q,
                                    unsigned n, unsigned* vis, int* qnext, unsigned* qn, unsigned* found) {
  const long long warps = (long long)gridDim.x * blockDim.x / 32;
  for (long long i = (blockIdx.x * (long long)blockDim.x + threadIdx.x) / 32; i < n; i += warps) {
    if (*(volatile unsigned*)found) return;
    const int c = q[i];
    for (unsigned j = offs[c] + lane_id(); j < offs[c + 1]; j += 32) {
      const int m = rmatch[adj[j]];
      if (m == -1) {
        *found = 1u;
      } else if (m >= 0) {
        const unsigned bit = 1u << (m & 31);
        if (!(atomicOr(vis + (m >> 5), bit) & bit)) qnext[atomicAdd(qn, 1u)] = m;
      }
    }
  }
}

// Row-state (de)interleaving between the caller's plain rmatch / predecessor
// arrays and the device layout (see RM / PR).
__global__ void rows_pack_kernel(const int* plain, int* rm, int nr, int rs) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < nr; r += (long long)gridDim.x * blockDim.x)
    rm[rs * r] = plain[r];
}
__global__ void rows_unpack_kernel(const int* a, int* out, int nr, int rs) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < nr; r += (long long)gridDim.x * blockDim.x)
    out[r] = a[rs * r];
}
__global__ void rows_fill_kernel(int* a, int nr, int rs, int v) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < nr; r += (long long)gridDim.x * blockDim.x)
    a[rs * r] = v;
}

// permute_random on the device (csr_graph.cpp:80-90): column c becomes
// cperm[c], row r becomes rperm[r], each column's rows re-sorted.
__global__ void perm_degrees_kernel(const unsigned* offs, const int* cperm, unsigned* deg, int nc) {
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < nc; c += (long long)gridDim.x * blockDim.x)
    deg[cperm[c]] = offs[c + 1] - offs[c];
}
__global__ void perm_scatter_kernel(const unsigned* offs, const int* adj, const int* cperm, const int* rperm,
                                    const unsigned* noffs, int* nadj, int nc) {
  const long long warps = (long long)gridDim.x * blockDim.x / 32;
  for (long long c = (blockIdx.x * (long long)blockDim.x + threadIdx.x) / 32; c < nc; c += warps) {
    const unsigned b = offs[c], e = offs[c + 1], d = noffs[cperm[c]];
    for (unsigned j = b + lane_id(); j < e; j += 32) nadj[d + (j - b)] = rperm[adj[j]];
  }
}

// Validity of a resident initial matching (plain arrays), checked once at load.
__global__ void init_check_kernel(const unsigned* offs, const int* adj, int sorted, const int* rmatch,
                                  const int* cmatch, int nc, int nr, unsigned long long* bad) {
  unsigned long long b = 0;
  const long long tot = (long long)gridDim.x * blockDim.x;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < nc; c += tot) {
    const int r = cmatch[c];
    if (r < -1 || r >= nr) b++;
    else if (r >= 0 && rmatch[r] != (int)c) b++;
    else if (r >= 0 && !has_edge(adj, offs[c], offs[c + 1], r, sorted != 0)) b++;  // a pair must be an edge
  }
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < nr; r += tot) {
    const int v = rmatch[r];
    if (v < -1 || v >= nc) b++;
    else if (v >= 0 && cmatch[v] != (int)r) b++;
  }
  b = warp_sum(b);
  if (lane_id() == 0 && b) atomicAdd(bad, b);
}

// Transposed adjacency (rows -> columns) for bottom-up levels: count,
// exclusive scan (CUB), scatter. Row lists come out unsorted (not needed).
// Row index (transpose) for the pulled levels. A one-pass scatter (an atomic
// cursor bump and a 4-byte store per edge at a random place of the 4E-byte
// index, after an atomic degree count into nr counters) turns every access
// into a partial-sector DRAM read-modify-write once the arrays outgrow L2:
// 9.6 ms at C2, ~300 ms at C5. Instead the edges are first bucketed by row
// range, so that everything after that works inside one L2-sized window:
//   bucket_hist   bucket sizes (NB <= 512 counters, CTA-aggregated)
//   bucket_partition  streams the CSC once and appends every edge as a
//                 (row, col) pair to its bucket (CTA-staged runs)
//   pair_count    row degrees, streaming the pairs bucket by bucket
//   (CUB scan)    row offsets
//   pair_scatter  the row index, streaming the pairs bucket by bucket
// The last two hand out chunks in order from a global counter, so the whole
// grid stays within one or two buckets: each bucket's counters (<= 2 MB) and
// slice of the index (<= 32 MB) stay in L2 and leave it as full sectors.
constexpr int kTpChunk = 2048;   // edges per CTA step of bucket_partition (8 per thread)
constexpr int kPairChunk = 4096; // pairs per CTA step of the ordered passes (16 per thread)
constexpr int kMaxBuckets = 512;

// Edges [0, E) of adj; rows outside [0, nr) are left out (the partition below
// skips them too), so a chunk whose range check has not been read yet is safe.
__global__ void __launch_bounds__(256) bucket_hist_kernel(const int* adj, unsigned E, int shift, int nb, int nr,
                                                          unsigned* bcount) {
  __shared__ unsigned hist[kMaxBuckets];
  for (int b = threadIdx.x; b < nb; b += blockDim.x) hist[b] = 0;
  __syncthreads();
  for (unsigned long long j = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; j < E;
       j += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned r = (unsigned)ld_ro(adj + j);
    if (r < (unsigned)nr) atomicAdd(&hist[r >> shift], 1u);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < nb; b += blockDim.x)
    if (hist[b]) atomicAdd(bcount + b, hist[b]);
}

// pcur[b] = first pair slot of bucket b (base + exclusive scan of nb <= 512
// counts); start, when given, keeps a copy (the run table of a chunked build).
__global__ void bucket_base_kernel(const unsigned* bcount, int nb, unsigned* pcur, unsigned base = 0,
                                   unsigned* start = nullptr) {
  if (threadIdx.x == 0) {
    unsigned run = base;
    for (int b = 0; b < nb; ++b) {
      pcur[b] = run;
      if (start) start[b] = run;
      run += bcount[b];
    }
  }
}

// First column whose range [offs[c], offs[c+1]) holds edge j (offs ascending, offs[0] = 0).
__device__ __forceinline__ int column_of(const unsigned* offs, int lo, int hi, unsigned j) {
  while (hi - lo > 1) {  // invariant: offs[lo] <= j < offs[hi]
    const int mid = (lo + hi) >> 1;
    if (ld_ro(offs + mid) <= j) lo = mid; else hi = mid;
  }
  return lo;
}

// Edges [jbase, jbase + E) (global adjacency positions; offs must be valid).
__global__ void __launch_bounds__(256) bucket_partition_kernel(const unsigned* offs, const int* adj, int col_base, int nc,
                                                                unsigned E, int shift, int nb, unsigned* pcur,
                                                                int2* pairs, unsigned jbase = 0, int nr = INT_MAX) {
  __shared__ unsigned hist[kMaxBuckets];
  __shared__ unsigned base[kMaxBuckets];   // global slot of this chunk's run of each bucket
  __shared__ unsigned lbase[kMaxBuckets];  // its slot in the stage
  __shared__ unsigned wsum[8];
  __shared__ int2 stage[kTpChunk];
  __shared__ unsigned short sbk[kTpChunk];
  __shared__ int span[2];
  constexpr int kPer = kTpChunk / 256;
  const unsigned nchunks = (unsigned)(((unsigned long long)E + kTpChunk - 1) / kTpChunk);
  for (unsigned ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
    // (64-bit end: E may be within one chunk of 2^32)
    const unsigned j0 = jbase + ch * kTpChunk;
    const unsigned j1 = (unsigned)min((unsigned long long)jbase + E, (unsigned long long)j0 + kTpChunk);
    for (int b = threadIdx.x; b < nb; b += blockDim.x) hist[b] = 0;
    if (threadIdx.x < 2) span[threadIdx.x] = column_of(offs, 0, nc, threadIdx.x ? j1 - 1 : j0) + threadIdx.x;
    __syncthreads();
    // this thread's kPer consecutive edges [jb, je)
    const unsigned jb = j0 + threadIdx.x * kPer, je = min(j1, jb + kPer);
    int row[kPer];
    unsigned short rank[kPer];
    int col = jb < je ? column_of(offs, span[0], span[1], jb) : 0;
    unsigned next = jb < je ? ld_ro(offs + col + 1) : 0;
    int cols[kPer];
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const unsigned j = jb + k;
      row[k] = -1;
      if (j < je) {
        while (j >= next) next = ld_ro(offs + (++col) + 1);  // empty columns are skipped
        row[k] = ld_ro(adj + j);
        cols[k] = col_base + col;  // (global id: a rank's slice starts at col_base)
        if ((unsigned)row[k] < (unsigned)nr) rank[k] = (unsigned short)atomicAdd(&hist[row[k] >> shift], 1u);
        else row[k] = -1;  // out of range: the upload fails on it; leave it out here
      }
    }
    __syncthreads();
    // CTA-local bucket-major order: exclusive scan of the (<= 512) bucket counts,
    // two per thread; then one global reservation per non-empty bucket
    {
      const int b0 = 2 * threadIdx.x;
      const unsigned c0 = b0 < nb ? hist[b0] : 0u, c1 = b0 + 1 < nb ? hist[b0 + 1] : 0u;
      const unsigned incl = warp_incl_scan(c0 + c1);
      if (lane_id() == 31) wsum[threadIdx.x >> 5] = incl;
      __syncthreads();
      unsigned wb = 0;
      for (int w = 0; w < (int)(threadIdx.x >> 5); ++w) wb += wsum[w];
      const unsigned ex = wb + incl - (c0 + c1);
      if (b0 < nb) {
        lbase[b0] = ex;
        if (c0) base[b0] = atomicAdd(pcur + b0, c0);
      }
      if (b0 + 1 < nb) {
        lbase[b0 + 1] = ex + c0;
        if (c1) base[b0 + 1] = atomicAdd(pcur + b0 + 1, c1);
      }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kPer; ++k)
      if (row[k] >= 0) {
        const unsigned b = (unsigned)row[k] >> shift;
        const unsigned slot = lbase[b] + rank[k];
        stage[slot] = make_int2(row[k], cols[k]);
        sbk[slot] = (unsigned short)b;
      }
    __syncthreads();
    // runs of one bucket are contiguous in the stage and in the output: coalesced stores
    const unsigned nstage = lbase[nb - 1] + hist[nb - 1];  // edges kept (all of them on a valid graph)
    for (unsigned i = threadIdx.x; i < nstage; i += blockDim.x) {
      const unsigned b = sbk[i];
      pairs[base[b] + (i - lbase[b])] = stage[i];
    }
    __syncthreads();
  }
}

// Ordered passes over the bucketed pairs: chunks are handed out in order, so
// the grid's working set is one or two buckets wide.
template <bool kScatter>
__global__ void __launch_bounds__(256) pair_pass_kernel(const int2* pairs, unsigned E, unsigned* ticket,
                                                        unsigned* cursor, int* radj, int row_lo, int row_hi) {
  // rows outside [row_lo, row_hi) belong to another rank (multi-GPU inbox); cursor is indexed from row_lo
  __shared__ unsigned chunk;
  constexpr int kPer = kPairChunk / 256;
  for (;;) {
    if (threadIdx.x == 0) chunk = atomicAdd(ticket, 1u);
    __syncthreads();
    const unsigned long long j0 = (unsigned long long)chunk * kPairChunk;
    __syncthreads();
    if (j0 >= E) break;
    int2 rc[kPer];
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const unsigned long long j = j0 + k * 256 + threadIdx.x;
      rc[k] = j < E ? pairs[j] : make_int2(-1, 0);
    }
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      if (rc[k].x < row_lo || rc[k].x >= row_hi) continue;
      if (kScatter) radj[atomicAdd(cursor + (rc[k].x - row_lo), 1u)] = rc[k].y;
      else atomicAdd(cursor + (rc[k].x - row_lo), 1u);
    }
  }
}

// Chunked build (bm_upload_csc overlaps it with the copy): chunk k of the
// upload partitions its own edges into its own slice of the pairs, bucket by
// bucket, so that bucket b of chunk k is the run [start[k nb + b], + cnt[..]).
// The scatter then takes the runs bucket-major (every chunk's run of bucket 0,
// then of bucket 1, ...) so that, as in the one-pass build, the grid works
// inside one bucket's L2-sized slice of the index at a time.
// tpre = exclusive prefix of the runs' tile counts in bucket-major order.
__global__ void __launch_bounds__(1024) run_tiles_kernel(const unsigned* cnt, int K, int nb, unsigned* tpre) {
  __shared__ unsigned wsum[32];
  const int n = K * nb;
  const int per = (n + blockDim.x - 1) / blockDim.x;
  const int i0 = threadIdx.x * per, i1 = min(n, i0 + per);
  unsigned t = 0;
  for (int i = i0; i < i1; ++i) {  // i = b K + k (bucket-major)
    const int b = i / K, k = i % K;
    t += (cnt[k * nb + b] + kPairChunk - 1) / kPairChunk;
  }
  const unsigned incl = warp_incl_scan(t);
  if (lane_id() == 31) wsum[threadIdx.x >> 5] = incl;
  __syncthreads();
  unsigned run = incl - t;
  for (int w = 0; w < (int)(threadIdx.x >> 5); ++w) run += wsum[w];
  for (int i = i0; i < i1; ++i) {
    tpre[i] = run;
    const int b = i / K, k = i % K;
    run += (cnt[k * nb + b] + kPairChunk - 1) / kPairChunk;
  }
  if (i1 == n && i0 < i1) tpre[n] = run;
  if (n == 0 && threadIdx.x == 0) tpre[0] = 0;
}

__global__ void __launch_bounds__(256) pair_scatter_runs_kernel(const int2* pairs, const unsigned* start,
                                                                const unsigned* cnt, const unsigned* tpre, int K,
                                                                int nb, unsigned* ticket, unsigned* cursor, int* radj,
                                                                int nr) {
  __shared__ unsigned chunk;
  constexpr int kPer = kPairChunk / 256;
  const int n = K * nb;
  const unsigned total = ld_ro(tpre + n);
  for (;;) {
    if (threadIdx.x == 0) chunk = atomicAdd(ticket, 1u);
    __syncthreads();
    const unsigned t = chunk;
    __syncthreads();
    if (t >= total) break;
    int lo = 0, hi = n;  // the run holding tile t: tpre[lo] <= t < tpre[lo + 1]
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (ld_ro(tpre + mid) <= t) lo = mid; else hi = mid;
    }
    const int b = lo / K, k = lo % K;
    const unsigned s0 = ld_ro(start + k * nb + b), c0 = ld_ro(cnt + k * nb + b);
    const unsigned j0 = (t - ld_ro(tpre + lo)) * kPairChunk;
    int2 rc[kPer];
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      const unsigned j = j0 + q * 256 + threadIdx.x;
      rc[q] = j < c0 ? pairs[(unsigned long long)s0 + j] : make_int2(-1, 0);
    }
#pragma unroll
    for (int q = 0; q < kPer; ++q)
      if ((unsigned)rc[q].x < (unsigned)nr) radj[atomicAdd(cursor + rc[q].x, 1u)] = rc[q].y;
  }
}

