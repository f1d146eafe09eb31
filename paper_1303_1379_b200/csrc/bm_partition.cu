// bm_partition.cu — 1-D column partition of the matching driver over several
// GPUs: one bm_part per rank, BFS levels expanded by the
// owner of each frontier column, frontier/endpoint records exchanged by the
// caller (NCCL all-gather over NVLink, or any transport), every replica kept
// identical by applying the same concatenated records in the same order.
//
// Reference correspondence (paths relative to /root/reference/proj):
//   part_roots_kernel      init_bfs_array / init_root        src/gpu_match.cpp:8-21
//   part_expand_kernel     gpubfs / gpubfs_wr (one level)    src/gpu_match.cpp:42-70, 99-133
//   part_merge_*           the level's claims made global: the reference's
//                          last-writer-wins stores (kernel_grid.hpp:20-27)
//                          become a deterministic lowest-record-wins rule
//   part_alternate_kernel  alternate / alternate_walk        src/gpu_match.cpp:144-186
//   part_fix_*             fix_matching (three rules)        src/gpu_match.cpp:220-245
//
// Layout per rank: the CSC slice of its columns [col_lo, col_hi) (offsets
// rebased to 0), replicated rmatch/cmatch (caller-owned device buffers so the
// caller can broadcast them in place), replicated pred, a replicated dead-root
// bitmap and the local frontier {col, root}.
#include <algorithm>
#include <climits>
#include <cstdint>
#include <string>

#include <cuda_runtime.h>

#include "bm_device.cuh"
#include "bmatch_b200.h"

void bm_internal_set_error(const std::string& msg);  // bm_engine.cu

namespace bmp {

using namespace bm;

constexpr int kVis = 1 << 30;  // visited flag in the mate's rmatch entry (as bm_engine.cu)
constexpr int kMaxWorld = 8;   // ranks of one NVLink domain (P2P exchange)
constexpr int kThr = 256;

struct PartDev {
  int nc, nr, col_lo, col_hi;
  const unsigned long long* offs;  // local, col_hi - col_lo + 1
  const int* adj;
  int* rmatch;
  int* cmatch;
  int* pred;
  unsigned* dead;
  // per-level winner keys, ((~stamp) << 32) | record index: a lower key wins,
  // keys of earlier levels are larger, so the arrays never need a reset pass
  unsigned long long* winC;  // nc
  unsigned long long* winR;  // nc (roots)
  unsigned long long* winE;  // nr
  unsigned stamp;            // merge counter of this handle
  int ep_one, wr;
  // P2P exchange: records go straight into every rank's receive slabs (peer
  // memory over NVLink, CUDA IPC); record k of sender s at [s * cap + k]
  int p2p, rank, world;
  long long ccap, ecap;
  int4* peer_claims[kMaxWorld];
  int4* peer_eps[kMaxWorld];
};

__device__ __forceinline__ unsigned long long win_key(const PartDev& d, long long i) {
  return ((unsigned long long)(0xffffffffu - d.stamp) << 32) | (unsigned long long)(unsigned)i;
}

__device__ __forceinline__ bool dead_root(const PartDev& d, int root) {
  return (ld_rlx(d.dead + (root >> 5)) >> (root & 31)) & 1u;
}

// Warp-aggregated append of one int4 record.
__device__ __forceinline__ void append(int4* out, int* count, int4 rec) {
  const unsigned m = __activemask();
  const int leader = __ffs(m) - 1;
  const int rank = __popc(m & ((1u << lane_id()) - 1));
  int base = 0;
  if ((int)lane_id() == leader) base = atomicAdd(count, __popc(m));
  base = __shfl_sync(m, base, leader);
  out[base + rank] = rec;
}

__global__ void part_roots_kernel(PartDev d, int2* F, int* nF) {
  for (int c = d.col_lo + blockIdx.x * blockDim.x + threadIdx.x; c < d.col_hi; c += gridDim.x * blockDim.x) {
    const unsigned long long b = d.offs[c - d.col_lo], e = d.offs[c - d.col_lo + 1];
    if (d.cmatch[c] < 0 && e > b) {
      const unsigned m = __activemask();
      const int leader = __ffs(m) - 1;
      const int rank = __popc(m & ((1u << lane_id()) - 1));
      int base = 0;
      if ((int)lane_id() == leader) base = atomicAdd(nF, __popc(m));
      base = __shfl_sync(m, base, leader);
      F[base + rank] = make_int2(c, c);
    }
  }
}

// One level over the local frontier. Each 8-lane group of a warp takes one
// entry and strides over its rows; entries of degree >= kBig are done by the
// whole warp afterwards (degree skew, e.g. R-MAT hubs). Local claims are
// deduplicated with the rmatch visited bit and the -1 -> -2 CAS; the merge
// decides the global winners.
constexpr int kGroup = 8;
constexpr unsigned long long kBig = 256;     // whole warp per entry
constexpr unsigned long long kHuge = 16384;  // whole grid per entry (part_expand_huge_kernel)

// Records are staged in shared memory and reserved with one global atomic per
// CTA batch (a warp-level atomic per record batch on a single counter
// serialises in L2); a full stage falls back to a warp-aggregated global append.
constexpr int kStageC = 1024, kStageE = 256;
struct PartSmem {
  int4 c[kStageC];
  int4 e[kStageE];
  int nc, ne, bc, be;
};

__device__ __forceinline__ void stage(const PartDev& d, bool is_claim, int4* buf, int* n, int cap, int4* out,
                                      int* count, int4 rec) {
  const unsigned m = __activemask();
  const int leader = __ffs(m) - 1;
  const int rank = __popc(m & ((1u << lane_id()) - 1));
  int base = 0;
  if ((int)lane_id() == leader) base = atomicAdd(n, __popc(m));
  base = __shfl_sync(m, base, leader) + rank;
  if (base < cap) {
    buf[base] = rec;
  } else if (!d.p2p) {
    append(out, count, rec);
  } else {  // stage full: reserve in the rank's record list and write every rank's slab directly
    const unsigned m2 = __activemask();
    const int l2 = __ffs(m2) - 1;
    const int r2 = __popc(m2 & ((1u << lane_id()) - 1));
    int b2 = 0;
    if ((int)lane_id() == l2) b2 = atomicAdd(count, __popc(m2));
    b2 = __shfl_sync(m2, b2, l2) + r2;
    for (int r = 0; r < d.world; ++r) {
      if (is_claim) d.peer_claims[r][(long long)d.rank * d.ccap + b2] = rec;
      else d.peer_eps[r][(long long)d.rank * d.ecap + b2] = rec;
    }
  }
}

__device__ __forceinline__ void part_edge(const PartDev& d, PartSmem& sm, int row, int c, int root, int4* claims,
                                          int* n_claims, int4* eps, int* n_eps) {
  const int cm = ld_rlx(d.rmatch + row);
  if (cm >= 0) {
    if (!(cm & kVis) && !(atomicOr(d.rmatch + row, kVis) & kVis))
      stage(d, true, sm.c, &sm.nc, kStageC, claims, n_claims, make_int4(cm, c, root, row));
  } else if (cm == -1) {
    if (d.ep_one && dead_root(d, root)) return;
    if (atomicCAS(d.rmatch + row, -1, -2) == -1)
      stage(d, false, sm.e, &sm.ne, kStageE, eps, n_eps, make_int4(row, c, root, 0));
  }
}

// Copies the CTA's staged records to the global record arrays (CTA-uniform call).
__device__ __forceinline__ void flush_stage(const PartDev& d, PartSmem& sm, int4* claims, int* n_claims, int4* eps,
                                            int* n_eps) {
  __syncthreads();
  const int nc = min(sm.nc, kStageC), ne = min(sm.ne, kStageE);
  if (threadIdx.x == 0) {
    sm.bc = nc ? atomicAdd(n_claims, nc) : 0;
    sm.be = ne ? atomicAdd(n_eps, ne) : 0;
  }
  __syncthreads();
  if (d.p2p) {  // the fused exchange: every rank's slab for this sender, over NVLink
    for (int r = 0; r < d.world; ++r) {
      int4* pc = d.peer_claims[r] + (long long)d.rank * d.ccap + sm.bc;
      int4* pe = d.peer_eps[r] + (long long)d.rank * d.ecap + sm.be;
      for (int i = threadIdx.x; i < nc; i += blockDim.x) pc[i] = sm.c[i];
      for (int i = threadIdx.x; i < ne; i += blockDim.x) pe[i] = sm.e[i];
    }
  } else {
    for (int i = threadIdx.x; i < nc; i += blockDim.x) claims[sm.bc + i] = sm.c[i];
    for (int i = threadIdx.x; i < ne; i += blockDim.x) eps[sm.be + i] = sm.e[i];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    sm.nc = 0;
    sm.ne = 0;
  }
}

__global__ void __launch_bounds__(kThr) part_expand_kernel(PartDev d, const int2* F, int n, int4* claims,
                                                           int* n_claims, int4* eps, int* n_eps,
                                                           unsigned long long* stats, int2* huge, int* n_huge) {
  __shared__ PartSmem sm;
  if (threadIdx.x == 0) {
    sm.nc = 0;
    sm.ne = 0;
  }
  __syncthreads();
  const int lane = lane_id();
  const int grp = lane / kGroup, g = lane % kGroup;
  constexpr int kPerCta = kThr / kGroup;  // entries per CTA batch
  unsigned long long trav = 0, cexp = 0;
  for (long long cbase = (long long)blockIdx.x * kPerCta; cbase < n; cbase += (long long)gridDim.x * kPerCta) {
    const long long w = cbase + threadIdx.x / kGroup;
    int c = 0, root = 0;
    unsigned long long b = 0, e = 0;
    if (w < n) {
      const int2 ent = F[w];
      c = ent.x;
      root = ent.y;
      if (!(d.wr && dead_root(d, root))) {  // gpu_match.cpp:106-108
        b = d.offs[c - d.col_lo];
        e = d.offs[c - d.col_lo + 1];
      }
    }
    if (e - b >= kHuge) {  // hubs (R-MAT): deferred to the grid-wide pass
      if (g == 0) huge[atomicAdd(n_huge, 1)] = make_int2((int)w, 0);
      b = e = 0;
    }
    const bool big = e - b >= kBig;
    if (g == 0 && e > b) {
      cexp++;
      trav += e - b;
    }
    if (!big)
      for (unsigned long long j = b + g; j < e; j += kGroup)
        part_edge(d, sm, d.adj[j], c, root, claims, n_claims, eps, n_eps);
    unsigned bigm = __ballot_sync(kFull, big && g == 0);
    while (bigm) {  // whole warp on each high-degree entry of this batch
      const int src = __ffs(bigm) - 1;
      bigm &= bigm - 1;
      const int bc = __shfl_sync(kFull, c, src), br = __shfl_sync(kFull, root, src);
      const unsigned long long bb = __shfl_sync(kFull, b, src), be = __shfl_sync(kFull, e, src);
      for (unsigned long long j = bb + lane; j < be; j += 32)
        part_edge(d, sm, d.adj[j], bc, br, claims, n_claims, eps, n_eps);
    }
    (void)grp;
    flush_stage(d, sm, claims, n_claims, eps, n_eps);
  }
  trav = warp_sum(trav);
  cexp = warp_sum(cexp);
  if (lane == 0 && (trav | cexp)) {
    atomicAdd(stats + 0, trav);
    atomicAdd(stats + 1, cexp);
  }
}

// The hub entries of this level: every warp of the grid strides over each
// hub's rows in turn (a hub can hold a sizeable share of the level's edges).
__global__ void __launch_bounds__(kThr) part_expand_huge_kernel(PartDev d, const int2* F, const int2* huge,
                                                                const int* n_huge, int4* claims, int* n_claims,
                                                                int4* eps, int* n_eps, unsigned long long* stats) {
  __shared__ PartSmem sm;
  if (threadIdx.x == 0) {
    sm.nc = 0;
    sm.ne = 0;
  }
  __syncthreads();
  const int nh = *n_huge;
  unsigned long long trav = 0, cexp = 0;
  const long long gt = (long long)gridDim.x * blockDim.x;
  for (int h = 0; h < nh; ++h) {
    const int2 ent = F[huge[h].x];
    const int c = ent.x, root = ent.y;
    const unsigned long long b = d.offs[c - d.col_lo], e = d.offs[c - d.col_lo + 1];
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      cexp++;
      trav += e - b;
    }
    // CTA-uniform trip count so flush_stage's barriers line up
    for (unsigned long long base = b + (unsigned long long)blockIdx.x * blockDim.x; base < e; base += gt) {
      const unsigned long long j = base + threadIdx.x;
      if (j < e) part_edge(d, sm, d.adj[j], c, root, claims, n_claims, eps, n_eps);
      flush_stage(d, sm, claims, n_claims, eps, n_eps);
    }
  }
  trav = warp_sum(trav);
  cexp = warp_sum(cexp);
  if (lane_id() == 0 && (trav | cexp)) {
    atomicAdd(stats + 0, trav);
    atomicAdd(stats + 1, cexp);
  }
}

// Records of all ranks, rank-major: record k of rank r sits at r*stride + k
// and has the global key r*stride + k (its order). Lower key wins.
struct Gathered {
  const int4* rec;
  const int* counts;  // device per-rank counts
  long long stride;
  int world;
};

// The t-th valid record (ranks in order, k < counts[rank]) -> its global key
// i = rank * stride + k and the record; false past the last one.
__device__ __forceinline__ bool rec_at(const Gathered& g, long long t, long long& i, int4& r) {
  for (int rank = 0; rank < g.world; ++rank) {
    const long long c = g.counts[rank];
    if (t < c) {
      i = (long long)rank * g.stride + t;
      r = g.rec[i];
      return true;
    }
    t -= c;
  }
  return false;
}
__device__ __forceinline__ long long rec_total(const Gathered& g) {
  long long s = 0;
  for (int rank = 0; rank < g.world; ++rank) s += g.counts[rank];
  return s;
}

// Endpoints, step 1 (ONE_PER_TREE): lowest record per live root.
__global__ void part_ep_root_kernel(PartDev d, Gathered g) {
  const long long tot = rec_total(g);
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < tot; t += (long long)gridDim.x * blockDim.x) {
    int4 r;
    long long i;
    if (!rec_at(g, t, i, r)) continue;
    if (d.ep_one && !dead_root(d, r.z)) atomicMin(d.winR + r.z, win_key(d, i));
  }
}
// Step 2: lowest surviving record per row.
__global__ void part_ep_row_kernel(PartDev d, Gathered g) {
  const long long tot = rec_total(g);
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < tot; t += (long long)gridDim.x * blockDim.x) {
    int4 r;
    long long i;
    if (!rec_at(g, t, i, r)) continue;
    if (d.ep_one ? (d.winR[r.z] == win_key(d, i)) : true) atomicMin(d.winE + r.x, win_key(d, i));
  }
}
// Step 3: winners become endpoints everywhere; a row no record won goes back to -1.
__global__ void part_ep_apply_kernel(PartDev d, Gathered g, int* ep_list, int* n_ep, int keep_list, int* found) {
  const long long tot = rec_total(g);
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < tot; t += (long long)gridDim.x * blockDim.x) {
    int4 r;
    long long i;
    if (!rec_at(g, t, i, r)) continue;
    const unsigned long long w = d.winE[r.x];
    if (w == win_key(d, i)) {
      d.rmatch[r.x] = -2;
      d.pred[r.x] = r.y;
      if (d.wr) atomicOr(d.dead + (r.z >> 5), 1u << (r.z & 31));
      if (keep_list) ep_list[atomicAdd(n_ep, 1)] = r.x;
      *found = 1;
    } else if ((w >> 32) != (0xffffffffu - d.stamp)) {
      d.rmatch[r.x] = -1;  // flagged by a rank, won by nobody this level: free again
    }
  }
}
// Claims: lowest record per column wins; the winner's discoverer becomes
// pred[row] on every rank, and the owner of the column queues it (unless its
// tree found a path at this level).
__global__ void part_claim_min_kernel(PartDev d, Gathered g) {
  const long long tot = rec_total(g);
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < tot; t += (long long)gridDim.x * blockDim.x) {
    int4 r;
    long long i;
    if (!rec_at(g, t, i, r)) continue;
    atomicMin(d.winC + r.x, win_key(d, i));
  }
}
__global__ void part_claim_apply_kernel(PartDev d, Gathered g, int2* Fn, int* nFn, unsigned long long* n_live) {
  const long long tot = rec_total(g);
  unsigned long long live = 0;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < tot; t += (long long)gridDim.x * blockDim.x) {
    int4 r;
    long long i;
    if (!rec_at(g, t, i, r)) continue;
    if (d.winC[r.x] != win_key(d, i)) continue;
    d.rmatch[r.w] = r.x | kVis;
    d.pred[r.w] = r.y;
    if (d.wr && dead_root(d, r.z)) continue;
    live++;
    if (r.x >= d.col_lo && r.x < d.col_hi) Fn[atomicAdd(nFn, 1)] = make_int2(r.x, r.z);
  }
  live = warp_sum(live);
  if (lane_id() == 0 && live) atomicAdd(n_live, live);
}
// P2P exchange: after this rank's expand, publish its record counts in every
// rank's count table and bump every rank's arrival counter (system-scope
// release: the records and counts are visible before the arrival).
__global__ void part_signal_kernel(const int* n_claims, const int* n_eps, int* const* peer_counts,
                                   unsigned* const* peer_flags, int rank, int world, int parity) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const int c = *n_claims, e = *n_eps;
  for (int r = 0; r < world; ++r) {
    peer_counts[r][parity * 2 * kMaxWorld + rank] = c;
    peer_counts[r][parity * 2 * kMaxWorld + kMaxWorld + rank] = e;
  }
  __threadfence_system();
  for (int r = 0; r < world; ++r) atomicAdd_system(peer_flags[r], 1u);
}
// Waits until every rank has signalled this level (arrivals >= target).
__global__ void part_wait_kernel(const unsigned* flag, unsigned target, int* timeout) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const long long t0 = clock64();
  for (;;) {
    unsigned v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
    if ((int)(v - target) >= 0) break;
    __nanosleep(256);
    if (clock64() - t0 > (1ll << 38)) {  // ~140 s: a peer is gone
      *timeout = 1;
      break;
    }
  }
  __threadfence_system();
}

__global__ void part_sweep_kernel(int* rmatch, int nr) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < nr; r += (long long)gridDim.x * blockDim.x) {
    const int v = rmatch[r];
    if (v >= 0 && (v & kVis)) rmatch[r] = v & ~kVis;
  }
}

// ALTERNATE (gpu_match.cpp:144-154) from the endpoint list; serial = one thread.
__global__ void part_alternate_kernel(PartDev d, const int* ep_list, int n_ep, int serial, unsigned long long* stats) {
  unsigned long long walks = 0, steps = 0;
  const long long start = serial ? (blockIdx.x == 0 && threadIdx.x == 0 ? 0 : n_ep)
                                 : blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long stride = serial ? 1 : (long long)gridDim.x * blockDim.x;
  for (long long k = start; k < n_ep; k += stride) {
    int row = ep_list[k];
    walks++;
    long long guard = 0;
    while (row != -1) {
      const int col = ld_rlx(d.pred + row);
      if (col < 0) break;
      const int mr = ld_rlx(d.cmatch + col);
      if (mr >= 0 && ld_rlx(d.pred + mr) == col) break;  // claimed by another walk this phase
      st_rlx(d.cmatch + col, row);
      st_rlx(d.rmatch + row, col);
      row = mr;
      steps++;
      if (++guard > d.nc) break;
    }
  }
  walks = warp_sum(walks);
  steps = warp_sum(steps);
  if (lane_id() == 0 && (walks | steps)) {
    atomicAdd(stats + 2, walks);
    atomicAdd(stats + 3, steps);
  }
}

// FIX rules 1+2 (rows), then rule 3 (columns) + cardinality (gpu_match.cpp:220-245).
__global__ void part_fix_rows_kernel(PartDev d, unsigned long long* stats) {
  unsigned long long resets = 0;
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < d.nr; r += (long long)gridDim.x * blockDim.x) {
    const int v = d.rmatch[r];
    if (v == -2 || (v >= 0 && d.cmatch[v] != (int)r)) {
      d.rmatch[r] = -1;
      resets++;
    }
  }
  resets = warp_sum(resets);
  if (lane_id() == 0 && resets) atomicAdd(stats + 4, resets);
}
__global__ void part_fix_cols_kernel(PartDev d, unsigned long long* stats, unsigned long long* matched) {
  unsigned long long resets = 0, m = 0;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < d.nc; c += (long long)gridDim.x * blockDim.x) {
    const int r = d.cmatch[c];
    if (r >= 0 && d.rmatch[r] != (int)c) {
      d.cmatch[c] = -1;
      resets++;
    } else if (r >= 0) {
      m++;
    }
  }
  resets = warp_sum(resets);
  m = warp_sum(m);
  if (lane_id() == 0) {
    if (resets) atomicAdd(stats + 4, resets);
    if (m) atomicAdd(matched, m);
  }
}
__global__ void part_count_kernel(const int* rmatch, int nr, unsigned long long* matched) {
  unsigned long long m = 0;
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < nr; r += (long long)gridDim.x * blockDim.x)
    m += rmatch[r] >= 0;
  m = warp_sum(m);
  if (lane_id() == 0 && m) atomicAdd(matched, m);
}
__global__ void fill_kernel(int* p, long long n, int v) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    p[i] = v;
}

}  // namespace bmp

using namespace bmp;

struct bm_part {
  int device = 0, rank = 0, world = 1, sms = 148;
  cudaStream_t own = nullptr, stream = nullptr;
  int nc = -1, nr = -1, col_lo = 0, col_hi = 0;
  long long E = 0;
  unsigned long long* offs = nullptr;
  int* adj = nullptr;
  int* rmatch = nullptr;  // caller-owned (bm_part_bind_state)
  int* cmatch = nullptr;
  int *pred = nullptr, *ep_list = nullptr;
  unsigned long long *winC = nullptr, *winR = nullptr, *winE = nullptr;
  unsigned stamp = 0;
  unsigned* dead = nullptr;
  int2* F[2] = {nullptr, nullptr};
  int2* huge = nullptr;  // hub entries of the current level
  int cur = 0;
  int* cnt = nullptr;                     // [0] nF cur, [1] nF next, [2] claims, [3] eps, [4] n_ep list, [5] found, [6..] gathered counts
  unsigned long long* stats = nullptr;    // trav, cexp, walks, steps, resets, live, matched
  int ep_one = 1, wr = 1;
  int n_cur = 0;
  long long launches = 0;  // kernels launched since the last bm_part_reset_stats
  long long cap_claims = 0;
  // P2P exchange (bm_part_p2p_*): receive slabs by level parity, count table, arrival counter
  bool p2p = false;
  long long ccap = 0, ecap = 0;
  int4* recv_claims = nullptr;  // 2 parities x world x ccap
  int4* recv_eps = nullptr;     // 2 parities x world x ecap
  int* recv_counts = nullptr;   // [parity][claims | eps][kMaxWorld]
  unsigned* flag = nullptr;     // arrivals of every rank's signal
  int* timeout = nullptr;
  int4* peer_claims[kMaxWorld] = {};
  int4* peer_eps[kMaxWorld] = {};
  int** dpeer_counts = nullptr;       // device copies of the peers' count tables / counters
  unsigned** dpeer_flags = nullptr;
  void* opened[kMaxWorld][4] = {};    // IPC mappings to close
};

namespace {

bm_status pfail(bm_status s, const std::string& m) {
  bm_internal_set_error(m);
  return s;
}
#define PCUDA(call)                                                                          \
  do {                                                                                       \
    cudaError_t e_ = (call);                                                                 \
    if (e_ != cudaSuccess)                                                                   \
      return pfail(e_ == cudaErrorMemoryAllocation ? BM_ERR_OOM : BM_ERR_CUDA,               \
                   std::string(#call) + ": " + cudaGetErrorString(e_));                      \
  } while (0)

template <typename T>
void pfree(T*& p) {
  if (p) cudaFree(p);
  p = nullptr;
}

PartDev dev_of(const bm_part* pt, int parity = -1) {
  PartDev d{};
  if (parity >= 0 && pt->p2p) {
    d.p2p = 1;
    d.rank = pt->rank;
    d.world = pt->world;
    d.ccap = pt->ccap;
    d.ecap = pt->ecap;
    for (int r = 0; r < pt->world; ++r) {
      d.peer_claims[r] = pt->peer_claims[r] + (long long)parity * pt->world * pt->ccap;
      d.peer_eps[r] = pt->peer_eps[r] + (long long)parity * pt->world * pt->ecap;
    }
  }
  d.nc = pt->nc;
  d.nr = pt->nr;
  d.col_lo = pt->col_lo;
  d.col_hi = pt->col_hi;
  d.offs = pt->offs;
  d.adj = pt->adj;
  d.rmatch = pt->rmatch;
  d.cmatch = pt->cmatch;
  d.pred = pt->pred;
  d.dead = pt->dead;
  d.winC = pt->winC;
  d.winR = pt->winR;
  d.winE = pt->winE;
  d.stamp = pt->stamp;
  d.ep_one = pt->ep_one;
  d.wr = pt->wr;
  return d;
}

int blocks_for(const bm_part* pt, long long n) {
  return (int)std::max<long long>(1, std::min<long long>((long long)pt->sms * 8, (n + kThr - 1) / kThr));
}

bm_status ready(bm_part* pt, bool need_state) {
  if (!pt) return pfail(BM_ERR_INVALID_ARG, "null partition handle");
  if (pt->nc < 0) return pfail(BM_ERR_INVALID_ARG, "no graph slice uploaded (bm_part_upload)");
  if (need_state && (!pt->rmatch || !pt->cmatch))
    return pfail(BM_ERR_INVALID_ARG, "no matching state bound (bm_part_bind_state)");
  return BM_OK;
}

}  // namespace

extern "C" {

bm_status bm_part_create(int32_t device, int32_t rank, int32_t world, bm_part** out) {
  if (!out) return pfail(BM_ERR_INVALID_ARG, "null output pointer");
  *out = nullptr;
  if (world < 1 || rank < 0 || rank >= world) return pfail(BM_ERR_INVALID_ARG, "rank/world out of range");
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) return pfail(BM_ERR_CUDA, "no CUDA device available (the engine has no CPU fallback)");
  if (device < 0 || device >= n) return pfail(BM_ERR_INVALID_ARG, "device index out of range");
  PCUDA(cudaSetDevice(device));
  cudaDeviceProp prop{};
  PCUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10) return pfail(BM_ERR_CUDA, "this build targets sm_100a (B200)");
  auto* pt = new bm_part();
  pt->device = device;
  pt->rank = rank;
  pt->world = world;
  pt->sms = prop.multiProcessorCount;
  e = cudaStreamCreateWithFlags(&pt->own, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaMalloc(&pt->cnt, sizeof(int) * 64);
  if (e == cudaSuccess) e = cudaMalloc(&pt->stats, sizeof(unsigned long long) * 8);
  if (e != cudaSuccess) {
    bm_part_destroy(pt);
    return pfail(BM_ERR_CUDA, std::string("bm_part_create: ") + cudaGetErrorString(e));
  }
  pt->stream = pt->own;
  cudaMemset(pt->stats, 0, sizeof(unsigned long long) * 8);
  *out = pt;
  return BM_OK;
}

bm_status bm_part_destroy(bm_part* pt) {
  if (!pt) return BM_OK;
  cudaSetDevice(pt->device);
  if (pt->stream) cudaStreamSynchronize(pt->stream);
  pfree(pt->offs);
  pfree(pt->adj);
  pfree(pt->pred);
  pfree(pt->winC);
  pfree(pt->winR);
  pfree(pt->winE);
  pfree(pt->ep_list);
  pfree(pt->dead);
  pfree(pt->F[0]);
  pfree(pt->F[1]);
  pfree(pt->huge);
  pfree(pt->cnt);
  pfree(pt->stats);
  for (int r = 0; r < kMaxWorld; ++r)
    for (int k = 0; k < 4; ++k)
      if (pt->opened[r][k]) cudaIpcCloseMemHandle(pt->opened[r][k]);
  pfree(pt->recv_claims);
  pfree(pt->recv_eps);
  pfree(pt->recv_counts);
  pfree(pt->flag);
  pfree(pt->timeout);
  pfree(pt->dpeer_counts);
  pfree(pt->dpeer_flags);
  if (pt->own) cudaStreamDestroy(pt->own);
  delete pt;
  return BM_OK;
}

bm_status bm_part_set_stream(bm_part* pt, void* stream) {
  if (!pt) return pfail(BM_ERR_INVALID_ARG, "null partition handle");
  pt->stream = stream ? static_cast<cudaStream_t>(stream) : pt->own;
  return BM_OK;
}

bm_status bm_part_upload(bm_part* pt, int32_t nc, int32_t nr, int32_t col_lo, int32_t col_hi,
                         const int64_t* cxadj_slice, const int32_t* cadj_slice) {
  if (!pt) return pfail(BM_ERR_INVALID_ARG, "null partition handle");
  if (nc < 0 || nr < 0 || col_lo < 0 || col_hi < col_lo || col_hi > nc)
    return pfail(BM_ERR_INVALID_ARG, "bad partition bounds");
  if (nc >= kVis) return pfail(BM_ERR_INVALID_ARG, "nc must be < 2^30");
  if (!cxadj_slice || cxadj_slice[0] != 0) return pfail(BM_ERR_INVALID_ARG, "cxadj slice must start at 0");
  const int ncl = col_hi - col_lo;
  const long long E = cxadj_slice[ncl];
  if (E < 0) return pfail(BM_ERR_INVALID_ARG, "negative edge count");
  for (int i = 0; i < ncl; ++i)
    if (cxadj_slice[i + 1] < cxadj_slice[i]) return pfail(BM_ERR_INVALID_ARG, "cxadj slice must be non-decreasing");
  if (E > 0 && !cadj_slice) return pfail(BM_ERR_INVALID_ARG, "null cadj slice");
  PCUDA(cudaSetDevice(pt->device));
  PCUDA(cudaStreamSynchronize(pt->stream));
  pfree(pt->offs);
  pfree(pt->adj);
  pfree(pt->pred);
  pfree(pt->winC);
  pfree(pt->winR);
  pfree(pt->winE);
  pfree(pt->ep_list);
  pfree(pt->dead);
  pfree(pt->F[0]);
  pfree(pt->F[1]);
  pfree(pt->huge);
  pt->nc = -1;
  PCUDA(cudaMalloc(&pt->offs, sizeof(unsigned long long) * (ncl + 1)));
  PCUDA(cudaMalloc(&pt->adj, sizeof(int) * std::max<long long>(E, 1)));
  PCUDA(cudaMalloc(&pt->pred, sizeof(int) * std::max(nr, 1)));
  PCUDA(cudaMalloc(&pt->winC, sizeof(unsigned long long) * std::max(nc, 1)));
  PCUDA(cudaMalloc(&pt->winR, sizeof(unsigned long long) * std::max(nc, 1)));
  PCUDA(cudaMalloc(&pt->winE, sizeof(unsigned long long) * std::max(nr, 1)));
  PCUDA(cudaMalloc(&pt->ep_list, sizeof(int) * std::max(nr, 1)));
  PCUDA(cudaMalloc(&pt->dead, sizeof(unsigned) * ((nc + 31) / 32 + 1)));
  PCUDA(cudaMalloc(&pt->F[0], sizeof(int2) * std::max(ncl, 1)));
  PCUDA(cudaMalloc(&pt->F[1], sizeof(int2) * std::max(ncl, 1)));
  PCUDA(cudaMalloc(&pt->huge, sizeof(int2) * std::max(ncl, 1)));
  PCUDA(cudaMemcpyAsync(pt->offs, cxadj_slice, sizeof(long long) * (ncl + 1), cudaMemcpyHostToDevice, pt->stream));
  if (E > 0) PCUDA(cudaMemcpyAsync(pt->adj, cadj_slice, sizeof(int) * E, cudaMemcpyHostToDevice, pt->stream));
  PCUDA(cudaMemsetAsync(pt->winC, 0xff, sizeof(unsigned long long) * std::max(nc, 1), pt->stream));
  PCUDA(cudaMemsetAsync(pt->winR, 0xff, sizeof(unsigned long long) * std::max(nc, 1), pt->stream));
  PCUDA(cudaMemsetAsync(pt->winE, 0xff, sizeof(unsigned long long) * std::max(nr, 1), pt->stream));
  pt->stamp = 0;
  fill_kernel<<<64, kThr, 0, pt->stream>>>(pt->pred, std::max(nr, 1), -1);
  PCUDA(cudaGetLastError());
  PCUDA(cudaStreamSynchronize(pt->stream));
  pt->nc = nc;
  pt->nr = nr;
  pt->col_lo = col_lo;
  pt->col_hi = col_hi;
  pt->E = E;
  pt->cap_claims = std::max<long long>(1, std::min<long long>((long long)nc, E));
  return BM_OK;
}

bm_status bm_part_bind_state(bm_part* pt, void* rmatch_dev, void* cmatch_dev) {
  bm_status s = ready(pt, false);
  if (s != BM_OK) return s;
  if ((!rmatch_dev && pt->nr > 0) || (!cmatch_dev && pt->nc > 0)) return pfail(BM_ERR_INVALID_ARG, "null state buffer");
  pt->rmatch = static_cast<int*>(rmatch_dev);
  pt->cmatch = static_cast<int*>(cmatch_dev);
  return BM_OK;
}

bm_status bm_part_record_capacity(bm_part* pt, int64_t* claims_cap, int64_t* endpoints_cap) {
  bm_status s = ready(pt, false);
  if (s != BM_OK) return s;
  if (claims_cap) *claims_cap = pt->cap_claims;
  if (endpoints_cap) *endpoints_cap = std::max<long long>(1, std::min<long long>((long long)pt->nr, pt->E));
  return BM_OK;
}

bm_status bm_part_begin_phase(bm_part* pt, int32_t bfs_kernel, int32_t endpoint_policy, int64_t* n_roots_local) {
  bm_status s = ready(pt, true);
  if (s != BM_OK) return s;
  if (bfs_kernel != BM_BFS_GPUBFS && bfs_kernel != BM_BFS_WR) return pfail(BM_ERR_INVALID_ARG, "unknown bfs kernel");
  if (endpoint_policy < BM_EP_AUTO || endpoint_policy > BM_EP_ONE_PER_TREE)
    return pfail(BM_ERR_INVALID_ARG, "unknown endpoint policy");
  PCUDA(cudaSetDevice(pt->device));
  pt->wr = bfs_kernel == BM_BFS_WR;
  pt->ep_one = pt->wr && endpoint_policy != BM_EP_EVERY;
  pt->cur = 0;
  PCUDA(cudaMemsetAsync(pt->cnt, 0, sizeof(int) * 64, pt->stream));
  PCUDA(cudaMemsetAsync(pt->dead, 0, sizeof(unsigned) * ((pt->nc + 31) / 32 + 1), pt->stream));
  const int ncl = pt->col_hi - pt->col_lo;
  if (ncl > 0) {
    part_roots_kernel<<<blocks_for(pt, ncl), kThr, 0, pt->stream>>>(dev_of(pt), pt->F[0], pt->cnt);
    pt->launches++;
  }
  PCUDA(cudaGetLastError());
  int n = 0;
  PCUDA(cudaMemcpyAsync(&n, pt->cnt, sizeof(int), cudaMemcpyDeviceToHost, pt->stream));
  PCUDA(cudaStreamSynchronize(pt->stream));
  pt->n_cur = n;
  if (n_roots_local) *n_roots_local = n;
  return BM_OK;
}

bm_status bm_part_expand(bm_part* pt, void* claims_out, void* endpoints_out, int32_t* n_claims, int32_t* n_endpoints) {
  bm_status s = ready(pt, true);
  if (s != BM_OK) return s;
  if (!claims_out || !endpoints_out) return pfail(BM_ERR_INVALID_ARG, "null record buffer");
  PCUDA(cudaSetDevice(pt->device));
  PCUDA(cudaMemsetAsync(pt->cnt + 2, 0, sizeof(int) * 2, pt->stream));
  PCUDA(cudaMemsetAsync(pt->cnt + 63, 0, sizeof(int), pt->stream));  // hub count
  if (pt->n_cur > 0) {
    part_expand_kernel<<<blocks_for(pt, (long long)pt->n_cur * kGroup), kThr, 0, pt->stream>>>(
        dev_of(pt), pt->F[pt->cur], pt->n_cur, static_cast<int4*>(claims_out), pt->cnt + 2,
        static_cast<int4*>(endpoints_out), pt->cnt + 3, pt->stats, pt->huge, pt->cnt + 63);
    pt->launches++;
    part_expand_huge_kernel<<<pt->sms * 4, kThr, 0, pt->stream>>>(
        dev_of(pt), pt->F[pt->cur], pt->huge, pt->cnt + 63, static_cast<int4*>(claims_out), pt->cnt + 2,
        static_cast<int4*>(endpoints_out), pt->cnt + 3, pt->stats);
    pt->launches++;
  }
  PCUDA(cudaGetLastError());
  int c[2] = {0, 0};
  PCUDA(cudaMemcpyAsync(c, pt->cnt + 2, sizeof(c), cudaMemcpyDeviceToHost, pt->stream));
  PCUDA(cudaStreamSynchronize(pt->stream));
  if (n_claims) *n_claims = c[0];
  if (n_endpoints) *n_endpoints = c[1];
  return BM_OK;
}

bm_status bm_part_merge(bm_part* pt, const void* claims_all, const int32_t* claim_counts, int64_t claim_stride,
                        const void* endpoints_all, const int32_t* endpoint_counts, int64_t endpoint_stride,
                        int64_t* n_next_total, int32_t* found) {
  bm_status s = ready(pt, true);
  if (s != BM_OK) return s;
  if (!claim_counts || !endpoint_counts || claim_stride < 0 || endpoint_stride < 0)
    return pfail(BM_ERR_INVALID_ARG, "bad record counts");
  for (int r = 0; r < pt->world; ++r)
    if (claim_counts[r] < 0 || claim_counts[r] > claim_stride || endpoint_counts[r] < 0 ||
        endpoint_counts[r] > endpoint_stride)
      return pfail(BM_ERR_INVALID_ARG, "record count exceeds its stride");
  PCUDA(cudaSetDevice(pt->device));
  // counts to the device: [6, 6+world) claims, [6+world, 6+2*world) endpoints
  if (2 * pt->world + 6 > 63) return pfail(BM_ERR_INVALID_ARG, "world too large");  // cnt[63]: hub count
  PCUDA(cudaMemcpyAsync(pt->cnt + 6, claim_counts, sizeof(int) * pt->world, cudaMemcpyHostToDevice, pt->stream));
  PCUDA(cudaMemcpyAsync(pt->cnt + 6 + pt->world, endpoint_counts, sizeof(int) * pt->world, cudaMemcpyHostToDevice,
                        pt->stream));
  PCUDA(cudaMemsetAsync(pt->stats + 5, 0, sizeof(unsigned long long), pt->stream));
  PCUDA(cudaMemsetAsync(pt->cnt + 1, 0, sizeof(int), pt->stream));
  pt->stamp++;  // a fresh key space: every earlier level's winner key loses
  const PartDev d = dev_of(pt);
  const Gathered ge{static_cast<const int4*>(endpoints_all), pt->cnt + 6 + pt->world, endpoint_stride, pt->world};
  const Gathered gc{static_cast<const int4*>(claims_all), pt->cnt + 6, claim_stride, pt->world};
  const long long te = (long long)pt->world * endpoint_stride, tc = (long long)pt->world * claim_stride;
  if (te > 0) {
    const int b = blocks_for(pt, te);
    part_ep_root_kernel<<<b, kThr, 0, pt->stream>>>(d, ge);
    pt->launches++;
    part_ep_row_kernel<<<b, kThr, 0, pt->stream>>>(d, ge);
    pt->launches++;
    part_ep_apply_kernel<<<b, kThr, 0, pt->stream>>>(d, ge, pt->ep_list, pt->cnt + 4, pt->rank == 0, pt->cnt + 5);
    pt->launches++;
  }
  if (tc > 0) {
    const int b = blocks_for(pt, tc);
    part_claim_min_kernel<<<b, kThr, 0, pt->stream>>>(d, gc);
    pt->launches++;
    part_claim_apply_kernel<<<b, kThr, 0, pt->stream>>>(d, gc, pt->F[pt->cur ^ 1], pt->cnt + 1, pt->stats + 5);
    pt->launches++;
  }
  PCUDA(cudaGetLastError());
  int nxt[5] = {0, 0, 0, 0, 0};
  unsigned long long live = 0;
  PCUDA(cudaMemcpyAsync(nxt, pt->cnt + 1, sizeof(nxt), cudaMemcpyDeviceToHost, pt->stream));
  PCUDA(cudaMemcpyAsync(&live, pt->stats + 5, sizeof(live), cudaMemcpyDeviceToHost, pt->stream));
  PCUDA(cudaStreamSynchronize(pt->stream));
  pt->cur ^= 1;
  pt->n_cur = nxt[0];
  if (n_next_total) *n_next_total = (int64_t)live;
  if (found) *found = nxt[4] != 0;
  return BM_OK;
}

bm_status bm_part_end_bfs(bm_part* pt) {
  bm_status s = ready(pt, true);
  if (s != BM_OK) return s;
  PCUDA(cudaSetDevice(pt->device));
  part_sweep_kernel<<<blocks_for(pt, pt->nr), kThr, 0, pt->stream>>>(pt->rmatch, pt->nr);
  pt->launches++;
  PCUDA(cudaGetLastError());
  PCUDA(cudaStreamSynchronize(pt->stream));
  return BM_OK;
}

bm_status bm_part_augment(bm_part* pt, int32_t serial, int64_t* cardinality) {
  bm_status s = ready(pt, true);
  if (s != BM_OK) return s;
  if (pt->rank != 0) return pfail(BM_ERR_LOGIC, "ALTERNATE runs on rank 0 (it holds the endpoint list)");
  PCUDA(cudaSetDevice(pt->device));
  int n_ep = 0;
  PCUDA(cudaMemcpyAsync(&n_ep, pt->cnt + 4, sizeof(int), cudaMemcpyDeviceToHost, pt->stream));
  PCUDA(cudaStreamSynchronize(pt->stream));
  const PartDev d = dev_of(pt);
  if (n_ep > 0)
    part_alternate_kernel<<<serial ? 1 : blocks_for(pt, n_ep), serial ? 32 : kThr, 0, pt->stream>>>(
        d, pt->ep_list, n_ep, serial, pt->stats);
    pt->launches++;
  part_fix_rows_kernel<<<blocks_for(pt, pt->nr), kThr, 0, pt->stream>>>(d, pt->stats);
  pt->launches++;
  PCUDA(cudaMemsetAsync(pt->stats + 6, 0, sizeof(unsigned long long), pt->stream));
  part_fix_cols_kernel<<<blocks_for(pt, pt->nc), kThr, 0, pt->stream>>>(d, pt->stats, pt->stats + 6);
  pt->launches++;
  PCUDA(cudaGetLastError());
  unsigned long long m = 0;
  PCUDA(cudaMemcpyAsync(&m, pt->stats + 6, sizeof(m), cudaMemcpyDeviceToHost, pt->stream));
  PCUDA(cudaStreamSynchronize(pt->stream));
  if (cardinality) *cardinality = (int64_t)m;
  return BM_OK;
}

bm_status bm_part_cardinality(bm_part* pt, int64_t* cardinality) {
  bm_status s = ready(pt, true);
  if (s != BM_OK) return s;
  PCUDA(cudaSetDevice(pt->device));
  PCUDA(cudaMemsetAsync(pt->stats + 7, 0, sizeof(unsigned long long), pt->stream));
  part_count_kernel<<<blocks_for(pt, pt->nr), kThr, 0, pt->stream>>>(pt->rmatch, pt->nr, pt->stats + 7);
  pt->launches++;
  PCUDA(cudaGetLastError());
  unsigned long long m = 0;
  PCUDA(cudaMemcpyAsync(&m, pt->stats + 7, sizeof(m), cudaMemcpyDeviceToHost, pt->stream));
  PCUDA(cudaStreamSynchronize(pt->stream));
  if (cardinality) *cardinality = (int64_t)m;
  return BM_OK;
}

bm_status bm_part_stats(bm_part* pt, int64_t* edges_traversed, int64_t* columns_scanned, int64_t* walks,
                        int64_t* walk_steps, int64_t* fix_resets) {
  if (!pt) return pfail(BM_ERR_INVALID_ARG, "null partition handle");
  PCUDA(cudaSetDevice(pt->device));
  unsigned long long st[8];
  PCUDA(cudaMemcpyAsync(st, pt->stats, sizeof(st), cudaMemcpyDeviceToHost, pt->stream));
  PCUDA(cudaStreamSynchronize(pt->stream));
  if (edges_traversed) *edges_traversed = (int64_t)st[0];
  if (columns_scanned) *columns_scanned = (int64_t)st[1];
  if (walks) *walks = (int64_t)st[2];
  if (walk_steps) *walk_steps = (int64_t)st[3];
  if (fix_resets) *fix_resets = (int64_t)st[4];
  return BM_OK;
}

bm_status bm_part_p2p_export(bm_part* pt, int64_t ccap, int64_t ecap, void* handles) {
  bm_status s = ready(pt, true);
  if (s != BM_OK) return s;
  if (pt->world > kMaxWorld) return pfail(BM_ERR_INVALID_ARG, "P2P exchange supports up to 8 ranks");
  if (ccap < 1 || ecap < 1 || !handles) return pfail(BM_ERR_INVALID_ARG, "bad P2P capacities");
  PCUDA(cudaSetDevice(pt->device));
  for (int r = 0; r < kMaxWorld; ++r)
    for (int k = 0; k < 4; ++k)
      if (pt->opened[r][k]) {
        cudaIpcCloseMemHandle(pt->opened[r][k]);
        pt->opened[r][k] = nullptr;
      }
  pt->p2p = false;
  pfree(pt->recv_claims);
  pfree(pt->recv_eps);
  pfree(pt->recv_counts);
  pfree(pt->flag);
  pfree(pt->timeout);
  pt->ccap = ccap;
  pt->ecap = ecap;
  PCUDA(cudaMalloc(&pt->recv_claims, sizeof(int4) * 2 * pt->world * ccap));
  PCUDA(cudaMalloc(&pt->recv_eps, sizeof(int4) * 2 * pt->world * ecap));
  PCUDA(cudaMalloc(&pt->recv_counts, sizeof(int) * 4 * kMaxWorld));
  PCUDA(cudaMalloc(&pt->flag, sizeof(unsigned)));
  PCUDA(cudaMalloc(&pt->timeout, sizeof(int)));
  PCUDA(cudaMemset(pt->recv_counts, 0, sizeof(int) * 4 * kMaxWorld));
  PCUDA(cudaMemset(pt->flag, 0, sizeof(unsigned)));
  PCUDA(cudaMemset(pt->timeout, 0, sizeof(int)));
  cudaIpcMemHandle_t* h = static_cast<cudaIpcMemHandle_t*>(handles);
  PCUDA(cudaIpcGetMemHandle(&h[0], pt->recv_claims));
  PCUDA(cudaIpcGetMemHandle(&h[1], pt->recv_eps));
  PCUDA(cudaIpcGetMemHandle(&h[2], pt->recv_counts));
  PCUDA(cudaIpcGetMemHandle(&h[3], pt->flag));
  return BM_OK;
}

bm_status bm_part_p2p_import(bm_part* pt, const void* all_handles) {
  bm_status s = ready(pt, true);
  if (s != BM_OK) return s;
  if (!pt->recv_claims || !all_handles) return pfail(BM_ERR_INVALID_ARG, "call bm_part_p2p_export first");
  PCUDA(cudaSetDevice(pt->device));
  for (int r = 0; r < kMaxWorld; ++r)  // mappings of an earlier setup (e.g. a previous graph)
    for (int k = 0; k < 4; ++k)
      if (pt->opened[r][k]) {
        cudaIpcCloseMemHandle(pt->opened[r][k]);
        pt->opened[r][k] = nullptr;
      }
  const cudaIpcMemHandle_t* h = static_cast<const cudaIpcMemHandle_t*>(all_handles);
  int* counts[kMaxWorld] = {};
  unsigned* flags[kMaxWorld] = {};
  for (int r = 0; r < pt->world; ++r) {
    if (r == pt->rank) {
      pt->peer_claims[r] = pt->recv_claims;
      pt->peer_eps[r] = pt->recv_eps;
      counts[r] = pt->recv_counts;
      flags[r] = pt->flag;
      continue;
    }
    void* ptrs[4];
    for (int k = 0; k < 4; ++k) {
      PCUDA(cudaIpcOpenMemHandle(&ptrs[k], h[4 * r + k], cudaIpcMemLazyEnablePeerAccess));
      pt->opened[r][k] = ptrs[k];
    }
    pt->peer_claims[r] = static_cast<int4*>(ptrs[0]);
    pt->peer_eps[r] = static_cast<int4*>(ptrs[1]);
    counts[r] = static_cast<int*>(ptrs[2]);
    flags[r] = static_cast<unsigned*>(ptrs[3]);
  }
  pfree(pt->dpeer_counts);
  pfree(pt->dpeer_flags);
  PCUDA(cudaMalloc(&pt->dpeer_counts, sizeof(int*) * kMaxWorld));
  PCUDA(cudaMalloc(&pt->dpeer_flags, sizeof(unsigned*) * kMaxWorld));
  PCUDA(cudaMemcpy(pt->dpeer_counts, counts, sizeof(int*) * kMaxWorld, cudaMemcpyHostToDevice));
  PCUDA(cudaMemcpy(pt->dpeer_flags, flags, sizeof(unsigned*) * kMaxWorld, cudaMemcpyHostToDevice));
  pt->p2p = true;
  return BM_OK;
}

bm_status bm_part_expand_p2p(bm_part* pt, int32_t parity) {
  bm_status s = ready(pt, true);
  if (s != BM_OK) return s;
  if (!pt->p2p) return pfail(BM_ERR_INVALID_ARG, "P2P exchange not set up (bm_part_p2p_import)");
  PCUDA(cudaSetDevice(pt->device));
  parity &= 1;
  PCUDA(cudaMemsetAsync(pt->cnt + 2, 0, sizeof(int) * 2, pt->stream));
  PCUDA(cudaMemsetAsync(pt->cnt + 63, 0, sizeof(int), pt->stream));
  const PartDev d = dev_of(pt, parity);
  if (pt->n_cur > 0) {
    part_expand_kernel<<<blocks_for(pt, (long long)pt->n_cur * kGroup), kThr, 0, pt->stream>>>(
        d, pt->F[pt->cur], pt->n_cur, nullptr, pt->cnt + 2, nullptr, pt->cnt + 3, pt->stats, pt->huge, pt->cnt + 63);
    part_expand_huge_kernel<<<pt->sms * 4, kThr, 0, pt->stream>>>(d, pt->F[pt->cur], pt->huge, pt->cnt + 63, nullptr,
                                                                  pt->cnt + 2, nullptr, pt->cnt + 3, pt->stats);
    pt->launches += 2;
  }
  part_signal_kernel<<<1, 32, 0, pt->stream>>>(pt->cnt + 2, pt->cnt + 3, pt->dpeer_counts, pt->dpeer_flags, pt->rank,
                                               pt->world, parity);
  pt->launches++;
  PCUDA(cudaGetLastError());
  return BM_OK;
}

bm_status bm_part_merge_p2p(bm_part* pt, int32_t parity, uint32_t arrivals, int64_t* n_next_total, int32_t* found) {
  bm_status s = ready(pt, true);
  if (s != BM_OK) return s;
  if (!pt->p2p) return pfail(BM_ERR_INVALID_ARG, "P2P exchange not set up (bm_part_p2p_import)");
  PCUDA(cudaSetDevice(pt->device));
  parity &= 1;
  part_wait_kernel<<<1, 32, 0, pt->stream>>>(pt->flag, arrivals, pt->timeout);
  PCUDA(cudaMemsetAsync(pt->stats + 5, 0, sizeof(unsigned long long), pt->stream));
  PCUDA(cudaMemsetAsync(pt->cnt + 1, 0, sizeof(int), pt->stream));
  pt->stamp++;
  const PartDev d = dev_of(pt);
  const int* counts = pt->recv_counts + parity * 2 * kMaxWorld;
  const Gathered gc{pt->recv_claims + (long long)parity * pt->world * pt->ccap, counts, pt->ccap, pt->world};
  const Gathered ge{pt->recv_eps + (long long)parity * pt->world * pt->ecap, counts + kMaxWorld, pt->ecap, pt->world};
  const int b = pt->sms * 8;
  part_ep_root_kernel<<<b, kThr, 0, pt->stream>>>(d, ge);
  part_ep_row_kernel<<<b, kThr, 0, pt->stream>>>(d, ge);
  part_ep_apply_kernel<<<b, kThr, 0, pt->stream>>>(d, ge, pt->ep_list, pt->cnt + 4, pt->rank == 0, pt->cnt + 5);
  part_claim_min_kernel<<<b, kThr, 0, pt->stream>>>(d, gc);
  part_claim_apply_kernel<<<b, kThr, 0, pt->stream>>>(d, gc, pt->F[pt->cur ^ 1], pt->cnt + 1, pt->stats + 5);
  pt->launches += 6;
  PCUDA(cudaGetLastError());
  int nxt[5] = {0, 0, 0, 0, 0}, to = 0;
  unsigned long long live = 0;
  PCUDA(cudaMemcpyAsync(nxt, pt->cnt + 1, sizeof(nxt), cudaMemcpyDeviceToHost, pt->stream));
  PCUDA(cudaMemcpyAsync(&live, pt->stats + 5, sizeof(live), cudaMemcpyDeviceToHost, pt->stream));
  PCUDA(cudaMemcpyAsync(&to, pt->timeout, sizeof(int), cudaMemcpyDeviceToHost, pt->stream));
  PCUDA(cudaStreamSynchronize(pt->stream));
  if (to) return pfail(BM_ERR_NCCL, "P2P exchange timed out waiting for a peer");
  pt->cur ^= 1;
  pt->n_cur = nxt[0];
  if (n_next_total) *n_next_total = (int64_t)live;
  if (found) *found = nxt[4] != 0;
  return BM_OK;
}

bm_status bm_part_launch_count(bm_part* pt, int64_t* launches) {
  if (!pt) return pfail(BM_ERR_INVALID_ARG, "null partition handle");
  if (launches) *launches = pt->launches;
  return BM_OK;
}

bm_status bm_part_reset_stats(bm_part* pt) {
  if (!pt) return pfail(BM_ERR_INVALID_ARG, "null partition handle");
  pt->launches = 0;
  PCUDA(cudaSetDevice(pt->device));
  PCUDA(cudaMemsetAsync(pt->stats, 0, sizeof(unsigned long long) * 8, pt->stream));
  return BM_OK;
}

}  // extern "C"
