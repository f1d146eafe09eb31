// bm_engine.cu — B200 (sm_100a) maximum-cardinality bipartite matching engine.
//
// One cooperative, persistent kernel runs the whole augmenting-path driver of
// arXiv 1303.1379 on the device: initial matching (optional), every phase's
// level-synchronous BFS, ALTERNATE, FIXMATCHING and the termination test. The
// host launches it once per bm_run (or once per phase when an observer is
// attached) and reads one small control block back at the end. There is no
// per-level host synchronisation; levels and stages are separated by a
// software grid barrier (one atomic per CTA).
//
// Reference correspondence (paths relative to /root/reference/proj):
//   setup stage            init_bfs_array / init_root                      src/gpu_match.cpp:8-21, 277-282
//   expand_level           gpubfs / gpubfs_wr (Alg. 2 / Alg. 4)            src/gpu_match.cpp:23-135
//   level loop             expand_bfs                                       src/gpu_match.cpp:247-266
//   alternate stage        alternate / alternate_wr / alternate_walk       src/gpu_match.cpp:144-218
//   fix stages             fix_matching (three rules)                       src/gpu_match.cpp:220-245
//   phase loop             run_phase / run_driver / apfb / apsb             src/gpu_match.cpp:268-376
//   greedy init            cheap_matching (first-fit), parallelised        src/matching.cpp:13-26
//
// B200 design (not a translation of the reference's host loops):
//   * Frontier queues instead of an O(nc) level test per launch
//     (gpu_match.cpp:48/105). A level is a run of 16-byte entries
//     {col, root, adj_begin, edge_prefix}; one packed 64-bit atomicAdd per CTA
//     flush ((count<<33)|edges) hands out slots AND the level-local edge
//     prefix, so the next level is cut into equal *edge* tiles whatever the
//     degree skew.
//     While pushing, each entry also records itself in a granule index (one
//     u32 per kGran edges), so a tile finds its first entry with one load.
//   * "Unvisited" is one bit (bit 30) of the column's mate entry in rmatch,
//     claimed with atomicOr: the rmatch[row] gather every traversed edge makes
//     anyway also answers the visited test, instead of a bfs_array gather.
//   * WR: the early-exit test (gpu_match.cpp:106-108) reads a 1-bit-per-root
//     "dead" bitmap (L2-resident) instead of bfs_array[root]; a tree holds at
//     most one free row (bm_endpoint_policy ONE_PER_TREE, CAS on its root
//     mark), which leaves the other free rows to other trees. Correctness
//     never depends on either (ALTERNATE's claim check + FIX do).
//   * Row state: the mate and the visited bit share a word; above 72 MB the
//     predecessor joins them in one 8-byte slot (see RM / PR).
//   * Optional pulled (bottom-up) dense levels: bu_prep / bu_sweep, compiled
//     into separate kernel instances (driver_kernel<..., BU=true>).
//   * FIXMATCHING touches only what ALTERNATE wrote. Every walk step writes
//     rmatch[row] = pred[row] and cmatch[pred[row]] = row, and logs the pair;
//     the only other entries that can become inconsistent are the pending
//     endpoints (-2) and the row a walk leaves dangling when it breaks. Those
//     sets are exactly the inconsistent set of the reference's three full
//     passes, so the restricted FIX is the reference FIX.
//   * Predecessors are never reset: a walk only reads pred[] of rows whose
//     column was claimed in the current phase (the endpoint, the original
//     mate of a claimed column, or a row a walk wrote this phase), all of which
//     were written in this phase's BFS.
//   * The next phase's roots come from this phase's roots plus columns FIX
//     unmatched; nothing is O(nc) per phase except the dead-root bitmap clear
//     and the visited-bit sweep over rmatch.
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cstdint>
#include <condition_variable>
#include <deque>
#include <mutex>
#include <thread>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include <cooperative_groups.h>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_sort.cuh>
#include <cuda_runtime.h>

#include "bm_device.cuh"
#include "bm_host_util.hpp"
#include "bmatch_b200.h"

namespace cg = cooperative_groups;

namespace bm {
#include "bm_kernels.cuh"
}  // namespace bm

// ===========================================================================
// Host side: the C ABI.
// ===========================================================================
using namespace bm;

namespace {

thread_local std::string g_err;

bm_status fail(bm_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

bm_status cuda_fail(cudaError_t e, const char* what) {
  const bm_status s = (e == cudaErrorMemoryAllocation) ? BM_ERR_OOM : BM_ERR_CUDA;
  return fail(s, std::string(what) + ": " + cudaGetErrorString(e));
}

#define BM_CUDA(call)                                 \
  do {                                                \
    cudaError_t e_ = (call);                          \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
  } while (0)

template <typename T>
void dfree(T*& p) {
  if (p) cudaFree(p);
  p = nullptr;
}

// Graph-sized buffers only grow: re-uploading a graph of the same or smaller
// size reuses them (cudaMalloc/cudaFree of GB buffers costs milliseconds).
struct CapMap {
  std::vector<std::pair<const void*, size_t>> caps;
  size_t& operator[](const void* k) {
    for (auto& kv : caps)
      if (kv.first == k) return kv.second;
    caps.emplace_back(k, 0);
    return caps.back().second;
  }
};

template <typename T>
cudaError_t dalloc(CapMap& cm, T*& p, size_t count) {
  count = std::max<size_t>(count, 1);
  size_t& cap = cm[&p];
  if (p && cap >= count) return cudaSuccess;
  dfree(p);
  cap = 0;
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&p), count * sizeof(T));
  if (e == cudaSuccess) cap = count;
  return e;
}

}  // namespace

void bm_internal_set_error(const std::string& msg) { g_err = msg; }

struct bm_handle {
  int device = 0;
  cudaStream_t own = nullptr;
  cudaStream_t stream = nullptr;
  int sms = 0;
  int bps[6] = {0, 0, 0, 0, 0, 0};  // co-resident CTAs per SM, per kernel variant
  // graph
  int nc = -1, nr = -1;
  long long E = 0;
  int sorted = 1;
  unsigned* offs = nullptr;
  int* adj = nullptr;
  // state
  int *rm = nullptr, *cmatch = nullptr, *pred = nullptr, *bfs = nullptr;  // rm: row state (see RM / PR)
  int* pred_plain = nullptr;  // separate predecessors for the plain layout (pred aliases rm + 1 otherwise)
  int rs = 1;                 // row stride of rm / pred
  int pending_launches = 0;   // helper kernels launched for the next run (counted in last_launches)
  // bottom-up levels: transposed adjacency, frontier bitmaps, frontier roots
  bool bu_enabled = false;    // the row index exists for the resident graph
  bool bu_built = false;
  bool bu_auto = false;       // BM_BU_AUTO: the graph is of the kind whose dense levels pay to pull (upload)
  bool bu_huge = false;       // ... and so large that one run repays building the row index
  unsigned* tp_pcur = nullptr;  // row-index build scratch (bucket cursors, bucketed pairs)
  int2* tp_pairs = nullptr;
  unsigned* tp_runs = nullptr;  // chunked build (with the upload): run starts, cursors, counts, tile prefix, tickets
  cudaEvent_t ev_ri = nullptr;  // the row index built with the upload is complete (aux stream)
  // pageable host buffers: copied through pinned staging buffers (xfer_h2d / xfer_d2h)
  void* stg_buf[3] = {nullptr, nullptr, nullptr};
  cudaEvent_t stg_ev[3] = {nullptr, nullptr, nullptr};
  int stg_next = 0;
  unsigned char* tp_tmp = nullptr;  // CUB scan scratch
  double bu_frac = 0.45;      // BM_BU_FRAC (bu_rule 0): a level goes bottom-up when its frontier edges >= bu_frac * E
  int bu_rule = 1;            // 1: want_pull's direction-optimising test (default); 0: the bu_frac threshold
  float bu_alpha = 14.f;      // want_pull: pull when alpha * frontier edges >= edges of the unvisited rows
  double bu_beta = 24.0;      // ... and the frontier holds >= nc / beta columns
  long long nonempty = 0;     // columns with at least one edge (upload)
  int2* P = nullptr;          // lazy-frontier pairs (nc), pulled-capable runs only
  int4* tb = nullptr;         // bucketed pushed levels: (row, col, root) triples (ensure_pb)
  int2* left = nullptr;       // pulled levels' leftover lists: 3 x nr (row, row state)
  // late phases (ensure_late): stamps of the meet-in-the-middle search
  int2* lt_col = nullptr;
  int* lt_croot = nullptr;
  int* lt_row = nullptr;
  int* lt_epoch = nullptr;
  bool lt_ready = false;
  int lt_nc = -1, lt_nr = -1;  // the sizes the stamps were last cleared for
  unsigned long long pb_max = 0;
  int pb_shift = 0, pb_nb = 0;
  unsigned pb_cap = 0;
  int pp_shift = 0, pp_nb = 0;  // bucketed bu_prep (column buckets in tb)
  unsigned pp_cap = 0;
  unsigned* roffs = nullptr;
  int* radj = nullptr;
  unsigned* rcursor = nullptr;
  unsigned* fbit = nullptr;   // kNumFbit * nfbit_words
  int nfbit_words = 0;
  int* croot = nullptr;
  int* rtmp = nullptr;  // plain nr-int staging for host <-> device row arrays
  int *rmatch0 = nullptr, *cmatch0 = nullptr, *EP = nullptr;
  unsigned* dead = nullptr;
  int ndead_words = 0;
  int4* F[2] = {nullptr, nullptr};
  unsigned* gidx[2] = {nullptr, nullptr};
  int2* wlog = nullptr;
  unsigned log_cap = 0;
  Ctrl* ctl = nullptr;
  PhaseRec* recs = nullptr;
  int rec_cap = 4096;
  bool has_init = false;
  bool init_valid = false;  // the loaded initial matching passed init_check_kernel
  bool resumable = false;
  bm_match_opts run_opts{};
  std::vector<long long> phase_launches;  // per outer iteration, current run
  unsigned long long *scratch = nullptr;  // small device counters
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev_up = nullptr;
  cudaStream_t aux = nullptr;  // upload-time checks overlapped with the copies
  double last_ms = 0.0;
  int last_launches = 0;
  CapMap caps;
  unsigned long long* tl = nullptr;
  unsigned tl_cap = 1u << 16;
  std::vector<unsigned long long> timeline;  // host copy for the last run
  // fault injection for the failure-path tests (bm_debug_set)
  long long dbg_phase_bound = 0;
  int dbg_skip_alt_phase = 0;
};

namespace {

bm_status check_handle(bm_handle* h, bool need_graph) {
  if (!h) return fail(BM_ERR_INVALID_ARG, "null handle");
  if (need_graph && h->nc < 0) return fail(BM_ERR_INVALID_ARG, "no graph uploaded (call bm_upload_csc first)");
  return BM_OK;
}

int row_blocks(bm_handle* h) { return std::max(1, std::min(h->sms * 8, (h->nr + 255) / 256)); }

// ---- host <-> device copies ------------------------------------------------
// A pageable host buffer (the C++ shim's std::vectors, plain numpy arrays) is
// copied through a ring of pinned staging buffers: host threads fill (or drain)
// one buffer while the copy engine moves the previous one, so the copy runs
// near the pinned PCIe rate instead of the driver's single-threaded bounce
// path. Pinned (or registered) buffers go straight to cudaMemcpyAsync.
constexpr int kStgBufs = 3;
constexpr size_t kStgBytes = 64ull << 20;
constexpr size_t kStgMin = 8ull << 20;  // smaller copies go direct

bool host_pageable(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return a.type == cudaMemoryTypeUnregistered;
}

bm_status stage_init(bm_handle* h) {
  for (int i = 0; i < kStgBufs; ++i) {
    if (h->stg_buf[i]) continue;
    BM_CUDA(cudaHostAlloc(&h->stg_buf[i], kStgBytes, cudaHostAllocDefault));
    BM_CUDA(cudaEventCreateWithFlags(&h->stg_ev[i], cudaEventDisableTiming));
  }
  return BM_OK;
}

// Host copy threads for the staging ring: a persistent pool (a thread spawn per
// 64 MB piece cost ~10 % of the copy). Process-wide, created on first use and
// never torn down (its threads sleep on a condition variable).
class CopyPool {
 public:
  static CopyPool& get() {
    static CopyPool* pool = new CopyPool();  // (leaked on purpose: no join at exit)
    return *pool;
  }
  // dst <- src, n bytes, split over the pool (the caller takes one part too)
  void copy(void* dst, const void* src, size_t n) {
    const int parts = (int)std::max<size_t>(1, std::min<size_t>((size_t)nthreads_ + 1, n >> 22));  // >= 4 MB each
    if (parts == 1) {
      std::memcpy(dst, src, n);
      return;
    }
    std::lock_guard<std::mutex> one_job(job_mu_);  // (callers on other threads take turns)
    std::unique_lock<std::mutex> lk(mu_);
    dst_ = static_cast<char*>(dst);
    src_ = static_cast<const char*>(src);
    n_ = n;
    parts_ = parts;
    next_ = 1;
    pending_ = parts - 1;
    ++gen_;
    cv_.notify_all();
    lk.unlock();
    part(0);
    lk.lock();
    for (;;) {  // help with parts no worker has taken yet, then wait for the rest
      if (next_ < parts_) {
        const int w = next_++;
        lk.unlock();
        part(w);
        lk.lock();
        if (--pending_ == 0) break;
        continue;
      }
      if (pending_ == 0) break;
      done_.wait(lk);
    }
  }

 private:
  CopyPool() {
    nthreads_ = std::max(0, std::min(15, bm_host::resolve_threads(0) - 1));
    for (int i = 0; i < nthreads_; ++i) std::thread([this] { loop(); }).detach();
  }
  void part(int w) {
    const size_t lo = n_ * (size_t)w / (size_t)parts_, hi = n_ * (size_t)(w + 1) / (size_t)parts_;
    std::memcpy(dst_ + lo, src_ + lo, hi - lo);
  }
  void loop() {
    std::unique_lock<std::mutex> lk(mu_);
    unsigned long long seen = gen_;
    for (;;) {
      cv_.wait(lk, [&] { return gen_ != seen && next_ < parts_; });
      while (next_ < parts_) {
        const int w = next_++;
        lk.unlock();
        part(w);
        lk.lock();
        if (--pending_ == 0) done_.notify_all();
      }
      seen = gen_;
    }
  }
  std::mutex job_mu_, mu_;
  std::condition_variable cv_, done_;
  char* dst_ = nullptr;
  const char* src_ = nullptr;
  size_t n_ = 0;
  int parts_ = 0, next_ = 0, pending_ = 0, nthreads_ = 0;
  unsigned long long gen_ = 0;
};

void par_copy(void* dst, const void* src, size_t n) { CopyPool::get().copy(dst, src, n); }

// Enqueues a host -> device copy on st (returns once the host buffer may be reused).
bm_status xfer_h2d(bm_handle* h, void* dst, const void* src, size_t n, cudaStream_t st) {
  if (n == 0) return BM_OK;
  if (n < kStgMin || !host_pageable(src)) {
    BM_CUDA(cudaMemcpyAsync(dst, src, n, cudaMemcpyHostToDevice, st));
    return BM_OK;
  }
  bm_status s = stage_init(h);
  if (s != BM_OK) return s;
  for (size_t off = 0; off < n; off += kStgBytes) {
    const size_t len = std::min(kStgBytes, n - off);
    const int i = h->stg_next;
    h->stg_next = (i + 1) % kStgBufs;
    BM_CUDA(cudaEventSynchronize(h->stg_ev[i]));  // the buffer's previous copy is done
    par_copy(h->stg_buf[i], static_cast<const char*>(src) + off, len);
    BM_CUDA(cudaMemcpyAsync(static_cast<char*>(dst) + off, h->stg_buf[i], len, cudaMemcpyHostToDevice, st));
    BM_CUDA(cudaEventRecord(h->stg_ev[i], st));
  }
  return BM_OK;
}

// Device -> host copy, complete on return (stream-ordered after earlier work on st).
bm_status xfer_d2h(bm_handle* h, void* dst, const void* src, size_t n, cudaStream_t st) {
  if (n == 0) return BM_OK;
  if (n < kStgMin || !host_pageable(dst)) {
    BM_CUDA(cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToHost, st));
    BM_CUDA(cudaStreamSynchronize(st));
    return BM_OK;
  }
  bm_status s = stage_init(h);
  if (s != BM_OK) return s;
  struct Piece {
    int buf;
    size_t off, len;
  };
  std::deque<Piece> q;
  auto drain = [&]() -> bm_status {
    const Piece pc = q.front();
    q.pop_front();
    BM_CUDA(cudaEventSynchronize(h->stg_ev[pc.buf]));
    par_copy(static_cast<char*>(dst) + pc.off, h->stg_buf[pc.buf], pc.len);
    return BM_OK;
  };
  for (size_t off = 0; off < n; off += kStgBytes) {
    const size_t len = std::min(kStgBytes, n - off);
    if ((int)q.size() == kStgBufs) {  // the oldest piece holds the buffer this one takes
      s = drain();
      if (s != BM_OK) return s;
    }
    const int i = h->stg_next;
    h->stg_next = (i + 1) % kStgBufs;
    BM_CUDA(cudaEventSynchronize(h->stg_ev[i]));
    BM_CUDA(cudaMemcpyAsync(h->stg_buf[i], static_cast<const char*>(src) + off, len, cudaMemcpyDeviceToHost, st));
    BM_CUDA(cudaEventRecord(h->stg_ev[i], st));
    q.push_back({i, off, len});
  }
  while (!q.empty()) {
    s = drain();
    if (s != BM_OK) return s;
  }
  return BM_OK;
}

// plain device array (nr ints) -> row-state mates
bm_status rows_from_plain(bm_handle* h, const int* plain) {
  if (h->nr <= 0) return BM_OK;
  rows_pack_kernel<<<row_blocks(h), 256, 0, h->stream>>>(plain, h->rm, h->nr, h->rs);
  h->pending_launches++;
  BM_CUDA(cudaGetLastError());
  return BM_OK;
}
// row-state mates (off 0) or predecessors (off 1) -> plain device array
bm_status rows_to_plain(bm_handle* h, int* out, int off) {
  if (h->nr <= 0) return BM_OK;
  rows_unpack_kernel<<<row_blocks(h), 256, 0, h->stream>>>(off ? h->pred : h->rm, out, h->nr, h->rs);
  BM_CUDA(cudaGetLastError());
  return BM_OK;
}
bm_status rows_fill(bm_handle* h, int off, int v) {
  if (h->nr <= 0) return BM_OK;
  rows_fill_kernel<<<row_blocks(h), 256, 0, h->stream>>>(off ? h->pred : h->rm, h->nr, h->rs, v);
  h->pending_launches++;
  BM_CUDA(cudaGetLastError());
  return BM_OK;
}
// host rmatch -> row-state mates (through the staging buffer)
bm_status rows_from_host(bm_handle* h, const int32_t* rmatch) {
  if (h->nr <= 0) return BM_OK;
  bm_status s = xfer_h2d(h, h->rtmp, rmatch, sizeof(int) * h->nr, h->stream);
  if (s != BM_OK) return s;
  return rows_from_plain(h, h->rtmp);
}
bm_status rows_to_host(bm_handle* h, int32_t* out, int off) {
  if (h->nr <= 0 || !out) return BM_OK;
  bm_status s = rows_to_plain(h, h->rtmp, off);
  if (s != BM_OK) return s;
  return xfer_d2h(h, out, h->rtmp, sizeof(int) * h->nr, h->stream);
}

// Transposed adjacency (the row index) for pulled levels: allocations and the
// bucket geometry shared by the one-pass build (build_transpose) and the build
// that runs chunk by chunk with the upload (chunked_*). Rows are bucketed so
// that one bucket's slice of radj is at most 32 MB (kernels: bm_kernels.cuh).
bm_status transpose_alloc(bm_handle* h, int nc, int nr, long long E, int* shift_out, int* nb_out) {
  h->bu_enabled = nr > 0 && nc > 0 && E > 0;
  if (!h->bu_enabled) return BM_OK;
  BM_CUDA(dalloc(h->caps, h->roffs, (size_t)nr + 1));
  BM_CUDA(dalloc(h->caps, h->rcursor, (size_t)nr + 1));
  BM_CUDA(dalloc(h->caps, h->radj, (size_t)E + 4));  // (+4: the pulled probes read aligned groups of 4)
  h->nfbit_words = (nc + 31) / 32;
  BM_CUDA(dalloc(h->caps, h->fbit, (size_t)kNumFbit * h->nfbit_words));
  BM_CUDA(dalloc(h->caps, h->croot, (size_t)nc));
  BM_CUDA(dalloc(h->caps, h->P, (size_t)nc + kFSlack(nc)));
  if (dalloc(h->caps, h->left, (size_t)3 * nr) != cudaSuccess) {  // optional (leftover lists): screen instead
    cudaGetLastError();
    h->left = nullptr;
  }
  int shift = 0;
  {
    const long long nb_min = std::max<long long>(1, (E * (long long)sizeof(int) + (32ll << 20) - 1) >> 25);
    while (shift < 31 && ((long long)nr + (1ll << shift) - 1) >> shift > nb_min) ++shift;
  }
  const int nb = (int)(((long long)nr + (1ll << shift) - 1) >> shift);
  if (nb > kMaxBuckets) return fail(BM_ERR_INVALID_ARG, "row index: too many buckets");
  // scratch kept with the handle (a fresh 8E-byte allocation per build costs more than the build):
  // [0, nb) bucket cursors, [kMaxBuckets, +nb) bucket counts, [2 kMaxBuckets, +2) tickets
  BM_CUDA(dalloc(h->caps, h->tp_pcur, (size_t)2 * kMaxBuckets + 2));
  BM_CUDA(dalloc(h->caps, h->tp_pairs, (size_t)E));
  size_t tmp_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, h->rcursor, h->roffs, nr + 1, h->stream);
  // kept with the handle too: a stream-ordered allocation here cost 3-115 ms per build
  // (the default pool hands its memory back at every synchronisation)
  BM_CUDA(dalloc(h->caps, h->tp_tmp, tmp_bytes));
  *shift_out = shift;
  *nb_out = nb;
  return BM_OK;
}

// One-pass build over the resident CSC (bm_prepare_row_index, or the first
// pulling run after an upload that did not build it).
bm_status build_transpose(bm_handle* h, int nc, int nr, long long E) {
  BM_CUDA(cudaStreamWaitEvent(h->stream, h->ev_ri, 0));  // (an earlier chunked build's scatter)
  int shift = 0, nb = 0;
  bm_status s = transpose_alloc(h, nc, nr, E, &shift, &nb);
  if (s != BM_OK) return s;
  if (h->bu_enabled) {
    unsigned* pcur = h->tp_pcur;
    unsigned* bcount = h->tp_pcur + kMaxBuckets;
    unsigned* tickets = h->tp_pcur + 2 * kMaxBuckets;
    int2* pairs = h->tp_pairs;
    BM_CUDA(cudaMemsetAsync(h->tp_pcur, 0, sizeof(unsigned) * (2 * kMaxBuckets + 2), h->stream));
    BM_CUDA(cudaMemsetAsync(h->rcursor, 0, sizeof(unsigned) * ((size_t)nr + 1), h->stream));
    BM_CUDA(cudaMemsetAsync(h->fbit, 0, sizeof(unsigned) * kNumFbit * h->nfbit_words, h->stream));
    const int grid = h->sms * 8;
    bucket_hist_kernel<<<grid, 256, 0, h->stream>>>(h->adj, (unsigned)E, shift, nb, nr, bcount);
    bucket_base_kernel<<<1, 32, 0, h->stream>>>(bcount, nb, pcur);
    const int pa = (int)std::max<long long>(1, std::min<long long>((long long)grid, (E + kTpChunk - 1) / kTpChunk));
    bucket_partition_kernel<<<pa, 256, 0, h->stream>>>(h->offs, h->adj, 0, nc, (unsigned)E, shift, nb, pcur, pairs);
    pair_pass_kernel<false><<<grid, 256, 0, h->stream>>>(pairs, (unsigned)E, tickets, h->rcursor, nullptr, 0, nr);
    size_t tmp_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, h->rcursor, h->roffs, nr + 1, h->stream);
    cub::DeviceScan::ExclusiveSum(h->tp_tmp, tmp_bytes, h->rcursor, h->roffs, nr + 1, h->stream);
    BM_CUDA(cudaMemcpyAsync(h->rcursor, h->roffs, sizeof(unsigned) * ((size_t)nr + 1), cudaMemcpyDeviceToDevice,
                            h->stream));
    pair_pass_kernel<true><<<grid, 256, 0, h->stream>>>(pairs, (unsigned)E, tickets + 1, h->rcursor, h->radj, 0, nr);
    BM_CUDA(cudaGetLastError());
  }
  h->bu_built = true;
  return BM_OK;
}

// The build overlapped with the upload (bm_upload_csc, graphs where AUTO pulls
// from the first run): every adjacency chunk, as soon as its copy lands, is
// bucketed into its own slice of the pairs and its rows counted (aux stream);
// after the last chunk only the scan and the bucket-major scatter remain.
struct ChunkBuild {
  bool on = false;
  int shift = 0, nb = 0, K = 0;
  unsigned *start = nullptr, *cur = nullptr, *cnt = nullptr, *tpre = nullptr, *tickets = nullptr;
};

bm_status chunked_begin(bm_handle* h, int nc, int nr, long long E, long long chunk, ChunkBuild& cb) {
  bm_status s = transpose_alloc(h, nc, nr, E, &cb.shift, &cb.nb);
  if (s != BM_OK || !h->bu_enabled) return s;
  cb.K = (int)((E + chunk - 1) / chunk);
  const size_t kn = (size_t)cb.K * cb.nb;
  BM_CUDA(dalloc(h->caps, h->tp_runs, 4 * kn + 1 + (size_t)cb.K + 1));
  cb.start = h->tp_runs;
  cb.cur = cb.start + kn;
  cb.cnt = cb.cur + kn;
  cb.tpre = cb.cnt + kn;
  cb.tickets = cb.tpre + kn + 1;
  BM_CUDA(cudaMemsetAsync(cb.cnt, 0, sizeof(unsigned) * kn, h->aux));
  BM_CUDA(cudaMemsetAsync(cb.tickets, 0, sizeof(unsigned) * ((size_t)cb.K + 1), h->aux));
  BM_CUDA(cudaMemsetAsync(h->rcursor, 0, sizeof(unsigned) * ((size_t)nr + 1), h->aux));
  BM_CUDA(cudaMemsetAsync(h->fbit, 0, sizeof(unsigned) * kNumFbit * h->nfbit_words, h->aux));
  cb.on = true;
  return BM_OK;
}

// Chunk k = adjacency [j0, j1), enqueued on aux after its copy.
void chunked_chunk(bm_handle* h, const ChunkBuild& cb, int k, int nc, int nr, long long j0, long long j1) {
  const unsigned n = (unsigned)(j1 - j0);
  const size_t o = (size_t)k * cb.nb;
  const int grid = (int)std::max<long long>(1, std::min<long long>((long long)h->sms * 8, (n + 255) / 256));
  bucket_hist_kernel<<<grid, 256, 0, h->aux>>>(h->adj + j0, n, cb.shift, cb.nb, nr, cb.cnt + o);
  bucket_base_kernel<<<1, 32, 0, h->aux>>>(cb.cnt + o, cb.nb, cb.cur + o, (unsigned)j0, cb.start + o);
  const int pa = (int)std::max<long long>(1, std::min<long long>((long long)h->sms * 8, (n + kTpChunk - 1) / kTpChunk));
  bucket_partition_kernel<<<pa, 256, 0, h->aux>>>(h->offs, h->adj, 0, nc, n, cb.shift, cb.nb, cb.cur + o, h->tp_pairs,
                                                   (unsigned)j0, nr);
  pair_pass_kernel<false><<<grid, 256, 0, h->aux>>>(h->tp_pairs + j0, n, cb.tickets + k, h->rcursor, nullptr, 0, nr);
}

// After the last chunk (and the upload's checks): row offsets, then the scatter.
bm_status chunked_end(bm_handle* h, const ChunkBuild& cb, int nr) {
  size_t tmp_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, h->rcursor, h->roffs, nr + 1, h->aux);
  cub::DeviceScan::ExclusiveSum(h->tp_tmp, tmp_bytes, h->rcursor, h->roffs, nr + 1, h->aux);
  BM_CUDA(cudaMemcpyAsync(h->rcursor, h->roffs, sizeof(unsigned) * ((size_t)nr + 1), cudaMemcpyDeviceToDevice, h->aux));
  run_tiles_kernel<<<1, 1024, 0, h->aux>>>(cb.cnt, cb.K, cb.nb, cb.tpre);
  pair_scatter_runs_kernel<<<h->sms * 8, 256, 0, h->aux>>>(h->tp_pairs, cb.start, cb.cnt, cb.tpre, cb.K, cb.nb,
                                                          cb.tickets + cb.K, h->rcursor, h->radj, nr);
  BM_CUDA(cudaGetLastError());
  BM_CUDA(cudaEventRecord(h->ev_ri, h->aux));  // every run waits for it (launch)
  h->bu_built = true;
  return BM_OK;
}

bm_status check_opts(const bm_match_opts* o) {
  if (!o) return fail(BM_ERR_INVALID_ARG, "null options");
  if (o->driver != BM_DRIVER_APFB && o->driver != BM_DRIVER_APSB)
    return fail(BM_ERR_INVALID_ARG, "unknown driver");
  if (o->bfs_kernel != BM_BFS_GPUBFS && o->bfs_kernel != BM_BFS_WR)
    return fail(BM_ERR_INVALID_ARG, "unknown bfs kernel");
  if (o->init < BM_INIT_GIVEN || o->init > BM_INIT_GPU_KS)
    return fail(BM_ERR_INVALID_ARG, "unknown init mode");
  if (o->max_phases < 0) return fail(BM_ERR_INVALID_ARG, "max_phases must be >= 0");
  if (o->claim_policy < BM_CLAIM_REFERENCE || o->claim_policy > BM_CLAIM_AT_DISCOVERY)
    return fail(BM_ERR_INVALID_ARG, "unknown claim policy");
  if (o->endpoint_policy < BM_EP_AUTO || o->endpoint_policy > BM_EP_ONE_PER_TREE)
    return fail(BM_ERR_INVALID_ARG, "unknown endpoint policy");
  if (o->bottom_up < BM_BU_OFF || o->bottom_up > BM_BU_AUTO) return fail(BM_ERR_INVALID_ARG, "unknown bottom_up mode");
  // gpu_match.cpp:272-274
  if (o->improved && o->bfs_kernel != BM_BFS_WR)
    return fail(BM_ERR_LOGIC, "the endpoint-encoded alternation requires the with-root kernel");
  return BM_OK;
}

int variant_of(int wr, int imp, int bu = 0) { return (wr ? (imp ? 2 : 1) : 0) + (bu ? 3 : 0); }

const void* kernel_ptr(int v) {
  switch (v) {
    case 0: return reinterpret_cast<const void*>(&driver_kernel<false, false, false>);
    case 1: return reinterpret_cast<const void*>(&driver_kernel<true, false, false>);
    case 2: return reinterpret_cast<const void*>(&driver_kernel<true, true, false>);
    case 3: return reinterpret_cast<const void*>(&driver_kernel<false, false, true>);
    case 4: return reinterpret_cast<const void*>(&driver_kernel<true, false, true>);
    default: return reinterpret_cast<const void*>(&driver_kernel<true, true, true>);
  }
}

int grid_for(bm_handle* h, int v) {
  long long maxg = (long long)h->sms * std::max(1, h->bps[v]);
  // sanitizer runs: BM_GRID_CTAS=1 makes every grid barrier a no-op (no cross-CTA spinning)
  if (const char* gc = getenv("BM_GRID_CTAS")) maxg = std::max(1ll, std::min(maxg, atoll(gc)));
  const long long work = std::max<long long>({(long long)h->nc, (long long)h->nr, h->E / 8, 1});
  const long long want = (work + kThreads - 1) / kThreads;
  return (int)std::max<long long>(1, std::min(maxg, want));
}

// Clears the visited bitmap when a previous call left it dirty, optionally
// resets predecessors (only for parity probes that report them), and zeroes
// the control block.
bm_status prepare_fresh(bm_handle* h, bool reset_pred = false) {
  if (reset_pred) {
    bm_status s = rows_fill(h, 1, -1);
    if (s != BM_OK) return s;
  }
  BM_CUDA(cudaMemsetAsync(h->ctl, 0, sizeof(Ctrl), h->stream));
  BM_CUDA(cudaMemsetAsync(h->dead, 0, sizeof(unsigned) * std::max(h->ndead_words, 1), h->stream));
  if (h->fbit) BM_CUDA(cudaMemsetAsync(h->fbit, 0, sizeof(unsigned) * kNumFbit * std::max(h->nfbit_words, 1), h->stream));
  return BM_OK;
}

// Tuning hook: BM_PERSIST_MB=<n> marks the first n MB of rmatch as a
// persisting L2 access-policy window on the handle's stream.
void apply_persist(bm_handle* h) {
  const char* e = getenv("BM_PERSIST_MB");
  if (!e || !h->rm) return;
  const size_t want = (size_t)atol(e) << 20;
  if (!want) return;
  cudaDeviceProp prop{};
  cudaGetDeviceProperties(&prop, h->device);
  const size_t lim = std::min<size_t>(want, (size_t)prop.persistingL2CacheMaxSize);
  cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, lim);
  cudaStreamAttrValue a{};
  a.accessPolicyWindow.base_ptr = h->rm;
  a.accessPolicyWindow.num_bytes = std::min<size_t>(std::min<size_t>(want, sizeof(int) * h->rs * (size_t)h->nr),
                                                    (size_t)prop.accessPolicyMaxWindowSize);
  a.accessPolicyWindow.hitRatio = 1.0f;
  a.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
  a.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  cudaStreamSetAttribute(h->stream, cudaStreamAttributeAccessPolicyWindow, &a);
  static bool said = false;
  if (!said) {
    said = true;
    fprintf(stderr, "[bm] persisting L2 window: %zu MB (max persisting %d MB, max window %d MB)\n",
            (size_t)a.accessPolicyWindow.num_bytes >> 20, prop.persistingL2CacheMaxSize >> 20,
            prop.accessPolicyMaxWindowSize >> 20);
  }
}

bm_status launch(bm_handle* h, int v, Params& p, float* ms) {
  apply_persist(h);
  BM_CUDA(cudaStreamWaitEvent(h->stream, h->ev_ri, 0));  // a row index still being built with the upload
  const int G = grid_for(h, v);
  void* args[] = {&p};
  BM_CUDA(cudaEventRecord(h->ev0, h->stream));
  BM_CUDA(cudaLaunchCooperativeKernel(kernel_ptr(v), dim3(G), dim3(kThreads), args, sizeof(Smem), h->stream));
  BM_CUDA(cudaEventRecord(h->ev1, h->stream));
  BM_CUDA(cudaStreamSynchronize(h->stream));
  BM_CUDA(cudaEventElapsedTime(ms, h->ev0, h->ev1));
  return BM_OK;
}

// Whether this run pulls dense levels (bm_bottom_up).
// AUTO pulls on a qualifying graph once its row index exists (bm_prepare_row_index,
// or an earlier ON run), or right away when the graph is so large that the
// first run already repays the build.
bool pulls(const bm_handle* h, const bm_match_opts& o) {
  return o.bottom_up == BM_BU_ON || (o.bottom_up == BM_BU_AUTO && h->bu_auto && (h->bu_built || h->bu_huge));
}

// Bucketed pushed levels (push_bucketed, bm_kernels.cuh): on a row state far
// beyond L2 (interleaved layout), wide pushed levels of pulling runs first
// group their edges by row range. Buckets hold <= 16-24 MB of row state;
// every bucket region has room for 1.25x its share of the widest such level,
// and an overflow region can take a whole level, so any degree skew fits.
// BM_PB=0 disables; BM_PB_MIN / BM_PB_MAX bound the levels (edges).
bm_status ensure_pb(bm_handle* h) {
  const char* e = getenv("BM_PB");
  if ((e && atoi(e) == 0) || h->rs != 2 || h->nr <= 0 || h->E <= 0) {
    h->pb_max = 0;
    return BM_OK;
  }
  unsigned long long tmax = std::min<unsigned long long>((unsigned long long)h->E, 1ull << 28);
  if (const char* m = getenv("BM_PB_MAX")) tmax = std::min<unsigned long long>(tmax, (unsigned long long)atoll(m));
  const unsigned long long rows_target = (24ull << 20) / (4ull * h->rs);
  int shift = 0;
  while ((2ull << shift) <= rows_target) ++shift;
  while ((((unsigned long long)h->nr - 1) >> shift) + 1 > (unsigned long long)kPbMax) ++shift;
  const int nb = (int)((((unsigned long long)h->nr - 1) >> shift) + 1);
  unsigned long long slack = 4096;
  if (const char* sl = getenv("BM_PB_SLACK")) slack = (unsigned long long)atoll(sl);  // tests: 0 forces overflow
  const unsigned cap = (unsigned)std::min<unsigned long long>(0xffff0000ull, (tmax * 5 / 4) / nb + slack);
  const size_t need = (size_t)nb * cap + tmax;
  if (need * sizeof(int4) >= (1ull << 36)) {  // (> 64 GB: do not)
    h->pb_max = 0;
    return BM_OK;
  }
  if (dalloc(h->caps, h->tb, need) != cudaSuccess) {  // an optimisation: without the memory, push unbucketed
    cudaGetLastError();
    h->pb_max = 0;
    return BM_OK;
  }
  h->pb_max = tmax;
  h->pb_shift = shift;
  h->pb_nb = nb;
  h->pb_cap = cap;
  // column buckets of the bucketed bu_prep: <= 16-24 MB of croot each, pairs (int2) in the same buffer
  h->pp_nb = 0;
  const char* pe = getenv("BM_PP");
  if (!(pe && atoi(pe) == 0)) {
    const unsigned long long fcap = (unsigned long long)h->nc + kFSlack(h->nc);
    int cshift = 0;
    while ((2ull << cshift) <= (24ull << 20) / 4) ++cshift;
    while ((((unsigned long long)h->nc - 1) >> cshift) + 1 > (unsigned long long)kPbMax) ++cshift;
    const int cnb = (int)((((unsigned long long)std::max(h->nc, 1) - 1) >> cshift) + 1);
    const unsigned long long ccap = (fcap * 5 / 4) / cnb + slack;
    if ((unsigned long long)cnb * ccap + fcap <= 2ull * need && ccap < 0xffff0000ull) {
      h->pp_nb = cnb;
      h->pp_shift = cshift;
      h->pp_cap = (unsigned)ccap;
    }
  }
  return BM_OK;
}

// Late phases (late_phase, bm_kernels.cuh): phases with few roots first try a
// bounded meet-in-the-middle search. Needs the row index (pulled-capable runs)
// and per-column / per-row stamps, allocated here once per graph size. The
// stamps are epochs that only grow, so they are cleared only when the sizes
// change. BM_LATE=1|0 forces the late phases on|off (default: graphs with at
// least 2^22 columns); an allocation failure leaves them off.
bool late_wanted(const bm_handle* h) {
  const char* e = getenv("BM_LATE");
  if (e && *e) return atoi(e) != 0;
  return h->nc >= (1 << 22);
}

bm_status ensure_late(bm_handle* h) {
  h->lt_ready = false;
  if (!late_wanted(h) || h->nc <= 0 || h->nr <= 0) return BM_OK;
  const void* was[3] = {h->lt_col, h->lt_row, h->lt_epoch};
  if (dalloc(h->caps, h->lt_col, (size_t)h->nc) != cudaSuccess ||
      dalloc(h->caps, h->lt_croot, (size_t)h->nc) != cudaSuccess ||
      dalloc(h->caps, h->lt_row, (size_t)h->nr) != cudaSuccess || dalloc(h->caps, h->lt_epoch, 1) != cudaSuccess) {
    cudaGetLastError();
    h->lt_nc = h->lt_nr = -1;
    return BM_OK;
  }
  if (h->lt_nc != h->nc || h->lt_nr != h->nr || was[0] != h->lt_col || was[1] != h->lt_row ||
      was[2] != h->lt_epoch) {
    BM_CUDA(cudaMemsetAsync(h->lt_col, 0, sizeof(int2) * (size_t)h->nc, h->stream));
    BM_CUDA(cudaMemsetAsync(h->lt_row, 0, sizeof(int) * (size_t)h->nr, h->stream));
    BM_CUDA(cudaMemsetAsync(h->lt_epoch, 0, sizeof(int), h->stream));
    h->lt_nc = h->nc;
    h->lt_nr = h->nr;
  }
  h->lt_ready = true;
  return BM_OK;
}

Params make_params(bm_handle* h, const bm_match_opts& o) {
  Params p{};
  p.nc = h->nc;
  p.nr = h->nr;
  p.offs = h->offs;
  p.adj = h->adj;
  p.rm = h->rm;
  p.rs = h->rs;
  p.cmatch = h->cmatch;
  p.pred = h->pred;
  p.bfs = h->bfs;
  p.dead = h->dead;
  p.roffs = (pulls(h, o) && h->bu_enabled && h->bu_built) ? h->roffs : nullptr;
  p.radj = h->radj;
  for (int b = 0; b < kNumFbit; ++b) p.fbit[b] = h->fbit ? h->fbit + (size_t)b * h->nfbit_words : nullptr;
  p.croot = h->croot;
  p.nfbit_words = h->nfbit_words;
  // pull rule (tuning knobs read per run): BM_BU_FRAC selects the plain edge-share
  // threshold; otherwise want_pull's test with BM_BU_ALPHA / BM_BU_BETA
  h->bu_frac = h->rs == 2 ? 0.2 : 0.45;
  h->bu_rule = 1;
  if (const char* fr = getenv("BM_BU_FRAC")) {
    h->bu_frac = atof(fr);
    h->bu_rule = 0;
  }
  h->bu_alpha = h->rs == 2 ? 8.f : 4.f;  // (C5 sweep with bucketed pushed levels: 6-10 flat, 14 +7 % per phase)
  if (const char* a = getenv("BM_BU_ALPHA")) h->bu_alpha = (float)atof(a);
  h->bu_beta = 24.0;
  if (const char* b = getenv("BM_BU_BETA")) h->bu_beta = atof(b);
  p.bu_min_edges = (unsigned long long)std::max(1.0, h->bu_frac * (double)h->E);
  p.bu_rule = h->bu_rule;
  p.bu_alpha = h->bu_alpha;
  p.bu_min_n = (unsigned)std::min<double>(4e9, (double)h->nc / std::max(1e-9, h->bu_beta));
  p.deg_col = (double)h->E / (double)std::max<long long>(1, h->nonempty);
  p.deg_row = (double)h->E / (double)std::max(1, h->nr);
  p.P = h->P;
  p.pairs_min_edges = std::max<unsigned long long>(1ull << 20, (unsigned long long)h->E / 128);
  if (const char* pm = getenv("BM_PAIRS_MIN_EDGES")) p.pairs_min_edges = (unsigned long long)atoll(pm);
  p.ndead_words = h->ndead_words;
  p.F0 = h->F[0];
  p.F1 = h->F[1];
  p.gidx0 = h->gidx[0];
  p.gidx1 = h->gidx[1];
  p.EP = h->EP;
  p.wlog = h->wlog;
  p.log_cap = h->log_cap;
  p.trace = 0;
  p.claim_mode = o.claim_policy;
  if (const char* cm = getenv("BM_CLAIM_MODE")) p.claim_mode = atoi(cm);  // tuning override
  p.ep_one = (o.bfs_kernel == BM_BFS_WR && o.endpoint_policy != BM_EP_EVERY) ? 1 : 0;
  p.solo_edges = kSoloEdges;
  if (const char* se = getenv("BM_SOLO_EDGES")) p.solo_edges = (unsigned)atol(se);  // tuning / tests
  p.tl = h->tl;
  p.tl_cap = h->tl_cap;
  p.ctl = h->ctl;
  p.recs = h->recs;
  p.rec_cap = h->rec_cap;
  p.apsb = o.driver == BM_DRIVER_APSB;
  p.init_mode = o.init;
  p.fresh = 1;
  p.max_phases = h->rec_cap;
  p.stop_after_bfs = 0;
  p.phase_bound = (long long)h->nc + 1;
  p.fcap = (unsigned long long)h->nc + kFSlack(h->nc);
  p.claim_store = 1;
  if (const char* cs = getenv("BM_CLAIM_STORE")) p.claim_store = atoi(cs);
  p.tb = (h->pb_max && p.roffs) ? h->tb : nullptr;
  {
    // Leftover lists pay where screening every row means streaming a row state
    // far beyond L2 (interleaved layout): C5 -2 % per phase; on C2, whose row
    // state stays in L2, the lists' scattered offset reads cost more (+6 %).
    // BM_BU_LEFT=1|0 forces them on|off.
    const char* lf = getenv("BM_BU_LEFT");
    const bool want = lf && *lf ? atoi(lf) != 0 : h->rs == 2;
    const bool use = p.roffs && h->left && want;
    for (int k = 0; k < 3; ++k) p.left[k] = use ? h->left + (size_t)k * h->nr : nullptr;
  }
  p.pb_min_edges = 1ull << 22;
  if (const char* pm = getenv("BM_PB_MIN")) p.pb_min_edges = (unsigned long long)atoll(pm);
  p.pb_max_edges = h->pb_max;
  p.pb_shift = h->pb_shift;
  p.pb_nb = h->pb_nb;
  p.pb_cap = h->pb_cap;
  p.pp_nb = h->pb_max ? h->pp_nb : 0;
  p.pp_shift = h->pp_shift;
  p.pp_cap = h->pp_cap;
  p.pp_min = 1ull << 22;
  if (const char* pm = getenv("BM_PP_MIN")) p.pp_min = (unsigned long long)atoll(pm);
  {
    const bool late = h->lt_ready && p.roffs && h->P;
    p.lt_col = late ? h->lt_col : nullptr;
    p.lt_croot = h->lt_croot;
    p.lt_row = h->lt_row;
    p.lt_epoch = h->lt_epoch;
    p.lt_qcap = (unsigned)std::min<size_t>(((size_t)h->nc + kFSlack(h->nc)) / 2, 0x7fffffff);
    auto env_u = [](const char* k, unsigned long long d) {
      const char* v = getenv(k);
      return v && *v ? (unsigned long long)atoll(v) : d;
    };
    // (C5 A/B: roots <= nc / 200 with a 16 M forward bound -8 % against 65536 and 4 M;
    //  C2 keeps 65536: its phase 0 late costs +6 %)
    p.lt_max_roots = (unsigned)env_u("BM_LATE_ROOTS", std::max(65536, h->nc / 200));
    // backward bound nc / 10 within [256 K, 2 M] (A/B: C2 0.5-1 M -26 % against 2 M; C5 1 M +7 %,
    // 1.5-2 M even); forward 2048 entries per live root (C5 -1.4 % against 1024)
    p.lt_bcap = (unsigned)env_u("BM_LATE_BCAP", std::min(1 << 21, std::max(1 << 18, h->nc / 10)));
    p.lt_fcap = (unsigned)env_u("BM_LATE_FCAP", 1u << 24);
    p.lt_fper = (unsigned)env_u("BM_LATE_FPER", 2048);
    p.lt_blv = (int)env_u("BM_LATE_BLV", 16);
    p.lt_flv = (int)env_u("BM_LATE_FLV", 64);
  }
  if (h->dbg_phase_bound > 0) p.phase_bound = h->dbg_phase_bound;
  p.sorted = h->sorted;
  p.check = getenv("BM_CHECK") ? atoi(getenv("BM_CHECK")) : 0;
  p.dbg_skip_alt_phase = h->dbg_skip_alt_phase;
  return p;
}

bm_status ctl_error_status(int err) {
  switch (err) {
    case kErrNone: return BM_OK;
    case kErrBound:
      return fail(BM_ERR_BOUND_EXCEEDED, "termination bound exceeded: more than nc + 1 phases");
    case kErrInvalidInit:
      return fail(BM_ERR_INVALID_ARG,
                  "initial matching is not a clean valid matching (pending -2, out of range or asymmetric)");
    case kErrBarrier: return fail(BM_ERR_CUDA, "grid barrier watchdog fired");
    case kErrWalk: return fail(BM_ERR_CUDA, "ALTERNATE walk exceeded nc steps");
    case kErrLevels: return fail(BM_ERR_CUDA, "BFS exceeded nc + 2 levels");
    case kErrWindow: return fail(BM_ERR_CUDA, "inconsistent frontier entries (push window wider than its tile)");
    default: return fail(BM_ERR_CUDA, "unknown device error " + std::to_string(err));
  }
}

// Shared by bm_run/bm_resume/bm_match: runs launches until done, the phase
// budget is spent, or the observer aborts.
bm_status drive(bm_handle* h, const bm_match_opts& o, bool fresh, int64_t* cardinality,
                bm_counters* counters, int64_t* per_iter, int64_t cap, bm_phase_cb cb, void* user,
                int32_t* done_out, bool init_checked = false) {
  const bool bu = pulls(h, o);
  const int v = variant_of(o.bfs_kernel == BM_BFS_WR, o.improved, bu);
  if (bu && !h->bu_built) {  // one-time per resident graph
    bm_status ts = build_transpose(h, h->nc, h->nr, h->E);
    if (ts != BM_OK) return ts;
    BM_CUDA(cudaStreamSynchronize(h->stream));
  }
  if (bu) {
    bm_status ps = ensure_pb(h);
    if (ps != BM_OK) return ps;
    ps = ensure_late(h);
    if (ps != BM_OK) return ps;
  }
  Params p = make_params(h, o);
  p.fresh = fresh ? 1 : 0;
  p.init_checked = init_checked ? 1 : 0;
  if (fresh) {
    h->timeline.clear();
    h->phase_launches.clear();
    h->last_ms = 0.0;
    h->last_launches = h->pending_launches;  // the initial-state kernels of this run
  }
  h->pending_launches = 0;
  long long budget = o.max_phases > 0 ? o.max_phases : -1;
  std::vector<PhaseRec> recs;
  std::vector<int> snap_r, snap_c;
  Ctrl ctl{};
  bool done = false;
  for (;;) {
    int this_launch = cb ? 1 : h->rec_cap;
    if (budget >= 0) this_launch = (int)std::min<long long>(this_launch, budget);
    if (this_launch <= 0) break;
    p.max_phases = this_launch;
    float ms = 0.f;
    bm_status s = launch(h, v, p, &ms);
    if (s != BM_OK) return s;
    h->last_ms += ms;
    h->last_launches += 1;
    BM_CUDA(cudaMemcpy(&ctl, h->ctl, sizeof(Ctrl), cudaMemcpyDeviceToHost));
    {
      const unsigned nt = std::min(ctl.n_tl, h->tl_cap);
      const size_t old = h->timeline.size();
      h->timeline.resize(old + 2 * (size_t)nt);
      if (nt) BM_CUDA(cudaMemcpy(h->timeline.data() + old, h->tl, sizeof(unsigned long long) * 2 * nt,
                                 cudaMemcpyDeviceToHost));
      BM_CUDA(cudaMemsetAsync(&h->ctl->n_tl, 0, sizeof(unsigned), h->stream));
    }
    if (ctl.error) {
      h->resumable = false;
      if (ctl.error == kErrWindow || ctl.error == kErrCheck) {
        std::string d;
        for (int i = 0; i < 8; ++i) d += (i ? "," : "") + std::to_string(ctl.dbg[i]);
        return fail(BM_ERR_CUDA, "inconsistent frontier entries (push window wider than its tile): ls,n,T,i,e,wend,live,level=" + d);
      }
      return ctl_error_status(ctl.error);
    }
    recs.resize(ctl.n_recs);
    if (ctl.n_recs > 0)
      BM_CUDA(cudaMemcpy(recs.data(), h->recs, sizeof(PhaseRec) * ctl.n_recs, cudaMemcpyDeviceToHost));
    for (int i = 0; i < ctl.n_recs; ++i) {
      h->phase_launches.push_back(recs[i].launches);
      if (cb) {
        snap_r.resize(h->nr);
        snap_c.resize(h->nc);
        {
          bm_status rs = rows_to_host(h, snap_r.data(), 0);
          if (rs != BM_OK) return rs;
        }
        BM_CUDA(cudaMemcpy(snap_c.data(), h->cmatch, sizeof(int) * h->nc, cudaMemcpyDeviceToHost));
        bm_phase_event ev{};
        ev.iteration = (int64_t)h->phase_launches.size();
        ev.augmenting_path_found = recs[i].found;
        ev.serial_retry = recs[i].retry;
        ev.cardinality_before = recs[i].before;
        ev.cardinality_after = recs[i].after;
        ev.bfs_launches = recs[i].launches;
        ev.rmatch = snap_r.data();
        ev.nr = h->nr;
        ev.cmatch = snap_c.data();
        ev.nc = h->nc;
        if (cb(&ev, user) != 0) {
          h->resumable = false;
          return fail(BM_ERR_INVALID_ARG, "aborted by observer");
        }
      }
    }
    if (budget >= 0) budget -= ctl.n_recs;
    if (ctl.done) {
      done = true;
      break;
    }
    p.fresh = 0;
    // Each relaunch resets the per-launch record counter; stats accumulate.
    BM_CUDA(cudaMemsetAsync(&h->ctl->n_recs, 0, sizeof(int), h->stream));
  }
  h->resumable = !done;
  h->run_opts = o;
  if (cardinality) *cardinality = ctl.card;
  if (done_out) *done_out = done ? 1 : 0;
  if (counters) {
    std::memset(counters, 0, sizeof(*counters));
    counters->outer_iterations = (int64_t)h->phase_launches.size();
    long long lt = 0;
    for (long long x : h->phase_launches) lt += x;
    counters->bfs_launches_total = lt;
    counters->columns_scanned = (int64_t)ctl.stats[kStCexp];
    counters->alternations_attempted = (int64_t)ctl.stats[kStWalks];
    counters->fix_resets = (int64_t)ctl.stats[kStResets];
    counters->serial_retries = (int64_t)ctl.stats[kStRetries];
    counters->edges_traversed = (int64_t)ctl.stats[kStTrav];
    counters->columns_visited = (int64_t)ctl.stats[kStNvis];
    counters->walk_steps = (int64_t)ctl.stats[kStSteps];
    counters->frontier_entries = (int64_t)ctl.stats[kStEntries];
    counters->cardinality = ctl.card;
    counters->initial_cardinality = ctl.init_card;
    counters->n_phase_records = (int64_t)std::min<size_t>(h->phase_launches.size(), cap > 0 ? (size_t)cap : 0);
  }
  if (per_iter && cap > 0) {
    const size_t k = std::min<size_t>(h->phase_launches.size(), (size_t)cap);
    for (size_t i = 0; i < k; ++i) per_iter[i] = h->phase_launches[i];
  }
  return BM_OK;
}

}  // namespace

extern "C" {

int32_t bm_abi_version(void) { return BM_ABI_VERSION; }

const char* bm_last_error(void) { return g_err.c_str(); }

const char* bm_status_string(int32_t s) {
  switch (s) {
    case BM_OK: return "ok";
    case BM_ERR_INVALID_ARG: return "invalid argument";
    case BM_ERR_LOGIC: return "logic error";
    case BM_ERR_BOUND_EXCEEDED: return "termination bound exceeded";
    case BM_ERR_CUDA: return "cuda error";
    case BM_ERR_OOM: return "out of device memory";
    case BM_ERR_NCCL: return "nccl error";
    case BM_ERR_PARSE: return "parse error";
    case BM_ERR_IO: return "i/o error";
    default: return "unknown status";
  }
}

int32_t bm_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

bm_status bm_create(int32_t device, bm_handle** out) {
  if (!out) return fail(BM_ERR_INVALID_ARG, "null output pointer");
  *out = nullptr;
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0)
    return fail(BM_ERR_CUDA, std::string("no CUDA device available (the engine has no CPU fallback): ") +
                                 (e != cudaSuccess ? cudaGetErrorString(e) : "0 devices"));
  if (device < 0 || device >= n) return fail(BM_ERR_INVALID_ARG, "device index out of range");
  BM_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop{};
  BM_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10)
    return fail(BM_ERR_CUDA, std::string("device ") + prop.name + " is sm_" + std::to_string(prop.major) +
                                 std::to_string(prop.minor) + "; this build targets sm_100a (B200)");
  if (!prop.cooperativeLaunch) return fail(BM_ERR_CUDA, "device does not support cooperative launch");
  auto* h = new bm_handle();
  h->device = device;
  h->sms = prop.multiProcessorCount;
  for (int v = 0; v < 6; ++v) {
    e = cudaFuncSetAttribute(kernel_ptr(v), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Smem));
    if (e == cudaSuccess)
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&h->bps[v], kernel_ptr(v), kThreads, sizeof(Smem));
    if (e != cudaSuccess || h->bps[v] < 1) {
      delete h;
      return fail(BM_ERR_CUDA, std::string("occupancy query failed: ") + cudaGetErrorString(e));
    }
  }
  e = cudaStreamCreateWithFlags(&h->own, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreate(&h->ev0);
  if (e == cudaSuccess) e = cudaEventCreate(&h->ev1);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev_up, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev_ri, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&h->aux, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void**>(&h->ctl), sizeof(Ctrl));
  if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void**>(&h->recs), sizeof(PhaseRec) * h->rec_cap);
  if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void**>(&h->scratch), sizeof(unsigned long long) * 8);
  if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void**>(&h->tl), sizeof(unsigned long long) * 2 * h->tl_cap);
  if (e != cudaSuccess) {
    bm_destroy(h);
    return cuda_fail(e, "bm_create");
  }
  h->stream = h->own;
  *out = h;
  return BM_OK;
}

bm_status bm_destroy(bm_handle* h) {
  if (!h) return BM_OK;
  cudaSetDevice(h->device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  if (h->aux) cudaStreamSynchronize(h->aux);
  dfree(h->offs);
  dfree(h->adj);
  dfree(h->rm);
  dfree(h->rtmp);
  dfree(h->cmatch);
  dfree(h->pred_plain);
  h->pred = nullptr;
  dfree(h->bfs);
  dfree(h->rmatch0);
  dfree(h->cmatch0);
  dfree(h->EP);
  dfree(h->dead);
  dfree(h->roffs);
  dfree(h->radj);
  dfree(h->tp_pcur);
  dfree(h->tp_pairs);
  dfree(h->tp_tmp);
  dfree(h->tp_runs);
  dfree(h->rcursor);
  dfree(h->fbit);
  dfree(h->croot);
  dfree(h->P);
  dfree(h->tb);
  dfree(h->left);
  dfree(h->lt_col);
  dfree(h->lt_croot);
  dfree(h->lt_row);
  dfree(h->lt_epoch);
  dfree(h->gidx[0]);
  dfree(h->gidx[1]);
  dfree(h->wlog);
  dfree(h->F[0]);
  dfree(h->F[1]);
  dfree(h->ctl);
  dfree(h->recs);
  dfree(h->tl);
  dfree(h->scratch);
  if (h->ev0) cudaEventDestroy(h->ev0);
  if (h->ev1) cudaEventDestroy(h->ev1);
  if (h->ev_up) cudaEventDestroy(h->ev_up);
  if (h->ev_ri) cudaEventDestroy(h->ev_ri);
  for (int i = 0; i < kStgBufs; ++i) {
    if (h->stg_buf[i]) cudaFreeHost(h->stg_buf[i]);
    if (h->stg_ev[i]) cudaEventDestroy(h->stg_ev[i]);
  }
  if (h->aux) cudaStreamDestroy(h->aux);
  if (h->own) cudaStreamDestroy(h->own);
  delete h;
  return BM_OK;
}

bm_status bm_set_stream(bm_handle* h, void* stream) {
  bm_status s = check_handle(h, false);
  if (s != BM_OK) return s;
  BM_CUDA(cudaSetDevice(h->device));
  h->stream = stream ? static_cast<cudaStream_t>(stream) : h->own;
  return BM_OK;
}

bm_status bm_upload_csc(bm_handle* h, int32_t nc, int32_t nr, const int64_t* cxadj, const int32_t* cadj) {
  bm_status s = check_handle(h, false);
  if (s != BM_OK) return s;
  if (nc < 0 || nr < 0) return fail(BM_ERR_INVALID_ARG, "negative vertex count");
  if (nc >= kVisBit) return fail(BM_ERR_INVALID_ARG, "nc must be < 2^30 in this build (visited flag in rmatch bit 30)");
  if (!cxadj) return fail(BM_ERR_INVALID_ARG, "null cxadj");
  const long long E = cxadj[nc];
  if (E < 0) return fail(BM_ERR_INVALID_ARG, "cxadj[nc] is negative");
  if (E >= (1ll << 32) - 1) return fail(BM_ERR_INVALID_ARG, "edge count must be < 2^32 - 1 in this build");
  if (E > 0 && !cadj) return fail(BM_ERR_INVALID_ARG, "null cadj");
  BM_CUDA(cudaSetDevice(h->device));
  BM_CUDA(cudaStreamSynchronize(h->stream));
  BM_CUDA(cudaStreamSynchronize(h->aux));  // (a row index build of the previous graph)
  h->nc = -1;
  h->has_init = false;
  h->bu_built = false;
  h->resumable = false;
  // graph
  BM_CUDA(dalloc(h->caps, h->offs, (size_t)nc + 1));
  BM_CUDA(dalloc(h->caps, h->adj, (size_t)E));
  // state (sized by the graph)
  // row layout: interleave {mate, pred} once rmatch alone is far larger than L2
  {
    const char* lay = getenv("BM_ROW_LAYOUT");  // tuning override: "plain" | "interleave"
    bool il = (size_t)nr * sizeof(int) > ((size_t)BM_INTERLEAVE_MB << 20);
    if (lay && !strcmp(lay, "plain")) il = false;
    if (lay && !strcmp(lay, "interleave")) il = true;
    h->rs = il ? 2 : 1;
  }
  BM_CUDA(dalloc(h->caps, h->rm, (size_t)2 * std::max(nr, 1)));
  BM_CUDA(dalloc(h->caps, h->rtmp, nr));
  BM_CUDA(dalloc(h->caps, h->cmatch, nc));
  BM_CUDA(dalloc(h->caps, h->pred_plain, nr));
  h->pred = h->rs == 2 ? h->rm + 1 : h->pred_plain;
  BM_CUDA(dalloc(h->caps, h->bfs, nc));
  BM_CUDA(dalloc(h->caps, h->rmatch0, nr));
  BM_CUDA(dalloc(h->caps, h->cmatch0, nc));
  BM_CUDA(dalloc(h->caps, h->EP, nr));
  h->ndead_words = (nc + 31) / 32;
  BM_CUDA(dalloc(h->caps, h->dead, h->ndead_words));
  const size_t ngran = (size_t)(E / kGran) + 2;
  BM_CUDA(dalloc(h->caps, h->gidx[0], ngran));
  BM_CUDA(dalloc(h->caps, h->gidx[1], ngran));
  h->log_cap = (unsigned)std::min<long long>((long long)nr + nc + 1024, 0xffffffffll);
  BM_CUDA(dalloc(h->caps, h->wlog, h->log_cap));
  BM_CUDA(dalloc(h->caps, h->F[0], (size_t)nc + kFSlack(nc)));
  BM_CUDA(dalloc(h->caps, h->F[1], (size_t)nc + kFSlack(nc)));
  // offsets: int64 staged in F[1] (16 B per column >= 8 B per offset), narrowed to u32
  long long* staged = reinterpret_cast<long long*>(h->F[1]);
  bm_status xs = xfer_h2d(h, staged, cxadj, sizeof(long long) * ((size_t)nc + 1), h->stream);
  if (xs != BM_OK) return xs;
  BM_CUDA(cudaMemsetAsync(h->scratch, 0, sizeof(unsigned long long) * 5, h->stream));
  const int blocks = std::max(1, std::min(h->sms * 8, (nc + 256) / 256));
  convert_offsets_kernel<<<blocks, 256, 0, h->stream>>>(staged, h->offs, nc, E, h->scratch, h->scratch + 4);
  BM_CUDA(cudaGetLastError());
  BM_CUDA(cudaEventRecord(h->ev_up, h->stream));
  BM_CUDA(cudaStreamWaitEvent(h->aux, h->ev_up, 0));
  const char* spb = getenv("BM_PREBUILD");  // build the row index with the upload: 1 always, 0 never
  // default: graphs on which AUTO pulls from the first run (bu_huge; E >= 6 nc is implied by bu_auto),
  // and graphs large enough for late phases (>= 2^22 rows) that look like AUTO will pull
  // them (bu_auto's test on 4096 evenly spaced columns; the upload then decides exactly). C2 e2e:
  // 27.7 -> 22.5 ms, as the first run pulls and takes late phases.
  bool prebuild = nr >= (1 << 26) && E >= 6ll * nc && E > 0;
  if (!prebuild && nr >= (1 << 22) && E >= 6ll * nc && E > 0 && nc > 0) {
    const int S = 4096;
    long long ne = 0;
    for (int i = 0; i < S; ++i) {
      const long long c = (long long)i * nc / S;
      ne += cxadj[c + 1] > cxadj[c] ? 1 : 0;
    }
    const double frac = (double)ne / S;
    prebuild = frac >= 0.8 && (double)E >= 8.0 * frac * (double)nc;
  }
  if (spb && *spb) prebuild = atoi(spb) != 0;
  long long chunk = 32ll << 20;  // adjacency elements per chunk (128 MB)
  if (const char* ch = getenv("BM_UPLOAD_CHUNK")) chunk = std::max(4096ll, atoll(ch));  // tests: many chunks
  ChunkBuild cbuild;
  if (prebuild && E > 0) {
    // the chunk partition walks the offsets: they must be valid before the first chunk
    unsigned long long bad0 = 0;
    BM_CUDA(cudaMemcpyAsync(&bad0, h->scratch, sizeof(bad0), cudaMemcpyDeviceToHost, h->stream));
    BM_CUDA(cudaStreamSynchronize(h->stream));
    if (bad0)
      return fail(BM_ERR_INVALID_ARG, "cxadj is not a valid offset array (cxadj[0]=0, non-decreasing, cxadj[nc]=E)");
    bm_status bs = chunked_begin(h, nc, nr, E, chunk, cbuild);
    if (bs != BM_OK) return bs;
  }
  // adjacency in chunks: the check of chunk k (and its share of the row index)
  // runs on the aux stream while chunk k+1 is still being copied
  for (long long j0 = 0; j0 < E; j0 += chunk) {
    const long long j1 = std::min(E, j0 + chunk);
    xs = xfer_h2d(h, h->adj + j0, cadj + j0, sizeof(int) * (size_t)(j1 - j0), h->stream);
    if (xs != BM_OK) return xs;
    BM_CUDA(cudaEventRecord(h->ev_up, h->stream));
    BM_CUDA(cudaStreamWaitEvent(h->aux, h->ev_up, 0));
    const int cb = (int)std::max<long long>(1, std::min<long long>((long long)h->sms * 8, (j1 - j0 + 255) / 256));
    check_adj_flat_kernel<<<cb, 256, 0, h->aux>>>(h->adj, j0, j1, nr, h->scratch + 1, h->scratch + 2);
    if (cbuild.on) chunked_chunk(h, cbuild, (int)(j0 / chunk), nc, nr, j0, j1);
  }
  if (nc > 0) col_start_pairs_kernel<<<blocks, 256, 0, h->aux>>>(h->offs, h->adj, nc, h->scratch + 3);
  BM_CUDA(cudaGetLastError());
  BM_CUDA(cudaEventRecord(h->ev_up, h->aux));
  BM_CUDA(cudaStreamWaitEvent(h->stream, h->ev_up, 0));
  unsigned long long bad[5] = {0, 0, 0, 0, 0};
  BM_CUDA(cudaMemcpyAsync(bad, h->scratch, sizeof(bad), cudaMemcpyDeviceToHost, h->stream));
  BM_CUDA(cudaStreamSynchronize(h->stream));
  {  // BM_BU_AUTO (bmatch_b200.h): large, few empty columns, average degree >= 8 over the rest
    const long long nonempty = (long long)nc - (long long)bad[4];
    h->nonempty = nonempty;
    h->bu_auto = nr >= (1 << 21) && nonempty * 4 >= 3ll * nc && E >= 8 * nonempty;
    h->bu_huge = nr >= (1 << 26);  // rmatch >= 256 MB: pushed dense levels pay DRAM sectors per gather
    const char* fa = getenv("BM_BU_AUTO");
    if (fa && *fa) h->bu_auto = h->bu_huge = atoi(fa) != 0;
  }
  if (bad[0]) return fail(BM_ERR_INVALID_ARG, "cxadj is not a valid offset array (cxadj[0]=0, non-decreasing, cxadj[nc]=E)");
  if (bad[1]) return fail(BM_ERR_INVALID_ARG, "row index out of range in cadj");
  bad[2] -= bad[3];  // descending pairs inside columns
  h->sorted = bad[2] == 0;
  h->bu_built = false;  // the row index is built on the first bottom-up run ...
  if (cbuild.on) {      // ... or now, finishing the share the chunks did (the runs wait for it)
    bm_status bs = chunked_end(h, cbuild, nr);
    if (bs != BM_OK) return bs;
  }
  h->nr = nr;
  {
    bm_status fs = rows_fill(h, 1, -1);
    if (fs != BM_OK) return fs;
  }
  BM_CUDA(cudaStreamSynchronize(h->stream));
  h->nc = nc;
  h->nr = nr;
  h->E = E;
  return BM_OK;
}

bm_status bm_prepare_row_index(bm_handle* h) {
  bm_status s = check_handle(h, true);
  if (s != BM_OK) return s;
  BM_CUDA(cudaSetDevice(h->device));
  if (!h->bu_built) {
    s = build_transpose(h, h->nc, h->nr, h->E);
    if (s != BM_OK) return s;
  }
  BM_CUDA(cudaStreamSynchronize(h->stream));
  return BM_OK;
}

bm_status bm_download_row_index(bm_handle* h, uint32_t* roffs, int32_t* radj) {
  bm_status s = check_handle(h, true);
  if (s != BM_OK) return s;
  if (!h->bu_built || !h->bu_enabled) return fail(BM_ERR_INVALID_ARG, "the row index has not been built");
  BM_CUDA(cudaSetDevice(h->device));
  BM_CUDA(cudaStreamWaitEvent(h->stream, h->ev_ri, 0));
  if (roffs) {
    s = xfer_d2h(h, roffs, h->roffs, sizeof(unsigned) * ((size_t)h->nr + 1), h->stream);
    if (s != BM_OK) return s;
  }
  if (radj) {
    s = xfer_d2h(h, radj, h->radj, sizeof(int) * (size_t)h->E, h->stream);
    if (s != BM_OK) return s;
  }
  BM_CUDA(cudaStreamSynchronize(h->stream));
  return BM_OK;
}

bm_status bm_bottom_up_auto(bm_handle* h, int32_t* enabled) {
  bm_status s = check_handle(h, true);
  if (s != BM_OK) return s;
  if (enabled) *enabled = h->bu_auto ? (h->bu_huge ? 2 : 1) : 0;
  return BM_OK;
}

bm_status bm_graph_info(bm_handle* h, int32_t* nc, int32_t* nr, int64_t* nedges) {
  bm_status s = check_handle(h, true);
  if (s != BM_OK) return s;
  if (nc) *nc = h->nc;
  if (nr) *nr = h->nr;
  if (nedges) *nedges = h->E;
  return BM_OK;
}

bm_status bm_load_matching(bm_handle* h, const int32_t* rmatch, const int32_t* cmatch) {
  bm_status s = check_handle(h, true);
  if (s != BM_OK) return s;
  if ((!rmatch && h->nr > 0) || (!cmatch && h->nc > 0)) return fail(BM_ERR_INVALID_ARG, "null matching array");
  BM_CUDA(cudaSetDevice(h->device));
  if (h->nr > 0) {
    s = xfer_h2d(h, h->rmatch0, rmatch, sizeof(int) * h->nr, h->stream);
    if (s != BM_OK) return s;
  }
  if (h->nc > 0) {
    s = xfer_h2d(h, h->cmatch0, cmatch, sizeof(int) * h->nc, h->stream);
    if (s != BM_OK) return s;
  }
  BM_CUDA(cudaMemsetAsync(h->scratch, 0, sizeof(unsigned long long), h->stream));
  const int blocks = std::max(1, std::min(h->sms * 8, (std::max(h->nc, h->nr) + 255) / 256));
  init_check_kernel<<<blocks, 256, 0, h->stream>>>(h->offs, h->adj, h->sorted, h->rmatch0, h->cmatch0, h->nc,
                                                   h->nr, h->scratch);
  BM_CUDA(cudaGetLastError());
  unsigned long long bad = 0;
  BM_CUDA(cudaMemcpyAsync(&bad, h->scratch, sizeof(bad), cudaMemcpyDeviceToHost, h->stream));
  BM_CUDA(cudaStreamSynchronize(h->stream));
  h->has_init = true;
  h->init_valid = bad == 0;
  return BM_OK;
}

bm_status bm_run(bm_handle* h, const bm_match_opts* opts, int64_t* cardinality, bm_counters* counters,
                 int64_t* per_iter, int64_t cap, bm_phase_cb cb, void* user, int32_t* done) {
  bm_status s = check_handle(h, true);
  if (s != BM_OK) return s;
  s = check_opts(opts);
  if (s != BM_OK) return s;
  BM_CUDA(cudaSetDevice(h->device));
  if (opts->init == BM_INIT_GIVEN) {
    if (!h->has_init) return fail(BM_ERR_INVALID_ARG, "no initial matching loaded (bm_load_matching)");
    if (!h->init_valid)
      return fail(BM_ERR_INVALID_ARG,
                  "initial matching is not a clean valid matching (pending -2, out of range or asymmetric)");
    s = rows_from_plain(h, h->rmatch0);
    if (s != BM_OK) return s;
    BM_CUDA(cudaMemcpyAsync(h->cmatch, h->cmatch0, sizeof(int) * std::max(h->nc, 1), cudaMemcpyDeviceToDevice, h->stream));
  } else {
    s = rows_fill(h, 0, -1);
    if (s != BM_OK) return s;
    BM_CUDA(cudaMemsetAsync(h->cmatch, 0xff, sizeof(int) * std::max(h->nc, 1), h->stream));
  }
  s = prepare_fresh(h);
  if (s != BM_OK) return s;
  // (given: validated by bm_load_matching; GPU-built: valid by construction)
  return drive(h, *opts, true, cardinality, counters, per_iter, cap, cb, user, done, true);
}

bm_status bm_resume(bm_handle* h, const bm_match_opts* opts, int64_t* cardinality, bm_counters* counters,
                    int64_t* per_iter, int64_t cap, bm_phase_cb cb, void* user, int32_t* done) {
  bm_status s = check_handle(h, true);
  if (s != BM_OK) return s;
  s = check_opts(opts);
  if (s != BM_OK) return s;
  if (!h->resumable) return fail(BM_ERR_INVALID_ARG, "nothing to resume");
  if (opts->driver != h->run_opts.driver || opts->bfs_kernel != h->run_opts.bfs_kernel ||
      opts->improved != h->run_opts.improved)
    return fail(BM_ERR_INVALID_ARG, "resume must use the same driver/kernel as the stopped run");
  BM_CUDA(cudaSetDevice(h->device));
  BM_CUDA(cudaMemsetAsync(&h->ctl->n_recs, 0, sizeof(int), h->stream));
  return drive(h, *opts, false, cardinality, counters, per_iter, cap, cb, user, done);
}

bm_status bm_download_matching(bm_handle* h, int32_t* rmatch, int32_t* cmatch) {
  bm_status s = check_handle(h, true);
  if (s != BM_OK) return s;
  BM_CUDA(cudaSetDevice(h->device));
  s = rows_to_host(h, rmatch, 0);
  if (s != BM_OK) return s;
  if (cmatch && h->nc > 0) {
    s = xfer_d2h(h, cmatch, h->cmatch, sizeof(int) * h->nc, h->stream);
    if (s != BM_OK) return s;
  }
  BM_CUDA(cudaStreamSynchronize(h->stream));
  return BM_OK;
}

bm_status bm_debug_set(bm_handle* h, int32_t key, int64_t value) {
  bm_status s = check_handle(h, false);
  if (s != BM_OK) return s;
  switch (key) {
    case BM_DEBUG_PHASE_BOUND: h->dbg_phase_bound = value; return BM_OK;
    case BM_DEBUG_SKIP_ALTERNATE_PHASE: h->dbg_skip_alt_phase = (int)value; return BM_OK;
    default: return fail(BM_ERR_INVALID_ARG, "unknown debug key");
  }
}

bm_status bm_last_kernel_time(bm_handle* h, double* ms, int32_t* launches) {
  bm_status s = check_handle(h, false);
  if (s != BM_OK) return s;
  if (ms) *ms = h->last_ms;
  if (launches) *launches = h->last_launches;
  return BM_OK;
}

bm_status bm_last_phase_launches(bm_handle* h, int64_t* out, int64_t cap, int64_t* n) {
  bm_status s = check_handle(h, false);
  if (s != BM_OK) return s;
  if (n) *n = (int64_t)h->phase_launches.size();
  if (out && cap > 0) {
    const size_t k = std::min<size_t>(h->phase_launches.size(), (size_t)cap);
    for (size_t i = 0; i < k; ++i) out[i] = h->phase_launches[i];
  }
  return BM_OK;
}

bm_status bm_debug_stats(bm_handle* h, uint64_t* out, int64_t cap, int64_t* n) {
  bm_status s = check_handle(h, false);
  if (s != BM_OK) return s;
  Ctrl ctl{};
  BM_CUDA(cudaMemcpy(&ctl, h->ctl, sizeof(Ctrl), cudaMemcpyDeviceToHost));
  if (n) *n = kNumStats;
  for (int64_t i = 0; i < std::min<int64_t>(cap, kNumStats); ++i) out[i] = ctl.stats[i];
  return BM_OK;
}

bm_status bm_timeline(bm_handle* h, uint64_t* out, int64_t cap, int64_t* n) {
  bm_status s = check_handle(h, false);
  if (s != BM_OK) return s;
  const int64_t total = (int64_t)h->timeline.size() / 2;
  if (n) *n = total;
  if (out && cap > 0)
    std::memcpy(out, h->timeline.data(), sizeof(uint64_t) * 2 * (size_t)std::min<int64_t>(cap, total));
  return BM_OK;
}

bm_status bm_match(bm_handle* h, const bm_match_opts* opts, int32_t* rmatch, int32_t* cmatch,
                   int64_t* cardinality, bm_counters* counters, int64_t* per_iter, int64_t cap,
                   bm_phase_cb cb, void* user) {
  bm_status s = check_handle(h, true);
  if (s != BM_OK) return s;
  s = check_opts(opts);
  if (s != BM_OK) return s;
  if ((!rmatch && h->nr > 0) || (!cmatch && h->nc > 0)) return fail(BM_ERR_INVALID_ARG, "null matching array");
  BM_CUDA(cudaSetDevice(h->device));
  if (opts->init == BM_INIT_GIVEN) {
    s = rows_from_host(h, rmatch);
    if (s != BM_OK) return s;
    if (h->nc > 0) {
      s = xfer_h2d(h, h->cmatch, cmatch, sizeof(int) * h->nc, h->stream);
      if (s != BM_OK) return s;
    }
  } else {
    s = rows_fill(h, 0, -1);
    if (s != BM_OK) return s;
    BM_CUDA(cudaMemsetAsync(h->cmatch, 0xff, sizeof(int) * std::max(h->nc, 1), h->stream));
  }
  s = prepare_fresh(h);
  if (s != BM_OK) return s;
  int32_t done = 0;
  bm_match_opts o = *opts;
  o.max_phases = 0;  // the one-call entry always runs to the maximum
  // a given initial matching is validated in the kernel's setup; the GPU-built one needs no check
  s = drive(h, o, true, cardinality, counters, per_iter, cap, cb, user, &done, opts->init != BM_INIT_GIVEN);
  if (s != BM_OK) return s;
  return bm_download_matching(h, rmatch, cmatch);
}

bm_status bm_bfs_phase(bm_handle* h, int32_t driver, int32_t bfs_kernel, int32_t improved,
                       const int32_t* rmatch_in, const int32_t* cmatch_in, int32_t* bfs_array,
                       int32_t* predecessor, int32_t* rmatch_out, int64_t* launches, int32_t* path_found) {
  bm_status s = check_handle(h, true);
  if (s != BM_OK) return s;
  bm_match_opts o{};
  o.driver = driver;
  o.bfs_kernel = bfs_kernel;
  o.improved = improved;
  o.init = BM_INIT_GIVEN;
  o.endpoint_policy = BM_EP_EVERY;  // the probe reports the reference's -2 flags
  s = check_opts(&o);
  if (s != BM_OK) return s;
  if ((!rmatch_in && h->nr > 0) || (!cmatch_in && h->nc > 0)) return fail(BM_ERR_INVALID_ARG, "null matching array");
  BM_CUDA(cudaSetDevice(h->device));
  s = rows_from_host(h, rmatch_in);
  if (s != BM_OK) return s;
  if (h->nc > 0) BM_CUDA(cudaMemcpyAsync(h->cmatch, cmatch_in, sizeof(int) * h->nc, cudaMemcpyHostToDevice, h->stream));
  s = prepare_fresh(h, true);
  if (s != BM_OK) return s;
  const int v = variant_of(bfs_kernel == BM_BFS_WR, improved);
  Params p = make_params(h, o);
  p.stop_after_bfs = 1;
  p.trace = 1;
  p.max_phases = 1;
  float ms = 0.f;
  s = launch(h, v, p, &ms);
  if (s != BM_OK) return s;
  h->resumable = false;
  Ctrl ctl{};
  BM_CUDA(cudaMemcpy(&ctl, h->ctl, sizeof(Ctrl), cudaMemcpyDeviceToHost));
  if (ctl.error) return ctl_error_status(ctl.error);
  if (bfs_array && h->nc > 0) BM_CUDA(cudaMemcpy(bfs_array, h->bfs, sizeof(int) * h->nc, cudaMemcpyDeviceToHost));
  s = rows_to_host(h, predecessor, 1);
  if (s != BM_OK) return s;
  s = rows_to_host(h, rmatch_out, 0);
  if (s != BM_OK) return s;
  if (launches) *launches = ctl.bfs_levels_last;
  if (path_found) *path_found = ctl.path_found_last;
  return BM_OK;
}

bm_status bm_permute_random(bm_handle* h, const int32_t* cperm, const int32_t* rperm) {
  bm_status s = check_handle(h, true);
  if (s != BM_OK) return s;
  if ((h->nc > 0 && !cperm) || (h->nr > 0 && !rperm)) return fail(BM_ERR_INVALID_ARG, "null permutation");
  if (h->E > 0x7fffffffll) return fail(BM_ERR_INVALID_ARG, "bm_permute_random supports E < 2^31 (segmented sort)");
  {  // a permutation, not just any map (the device scatter relies on it)
    std::vector<char> seen((size_t)std::max(h->nc, h->nr), 0);
    for (int i = 0; i < h->nc; ++i) {
      if (cperm[i] < 0 || cperm[i] >= h->nc || seen[cperm[i]]) return fail(BM_ERR_INVALID_ARG, "cperm is not a permutation");
      seen[cperm[i]] = 1;
    }
    std::fill(seen.begin(), seen.end(), 0);
    for (int i = 0; i < h->nr; ++i) {
      if (rperm[i] < 0 || rperm[i] >= h->nr || seen[rperm[i]]) return fail(BM_ERR_INVALID_ARG, "rperm is not a permutation");
      seen[rperm[i]] = 1;
    }
  }
  BM_CUDA(cudaSetDevice(h->device));
  BM_CUDA(cudaStreamSynchronize(h->aux));  // (a row index still being built with the upload)
  const int nc = h->nc, nr = h->nr;
  const long long E = h->E;
  int *dcp = nullptr, *drp = nullptr, *nadj = nullptr, *sadj = nullptr;
  unsigned *deg = nullptr, *noffs = nullptr;
  void* tmp = nullptr;
  size_t tmp_scan = 0, tmp_sort = 0;
  auto cleanup = [&]() {
    cudaFree(dcp); cudaFree(drp); cudaFree(nadj); cudaFree(sadj); cudaFree(deg); cudaFree(tmp);
  };
  cudaError_t e = cudaMalloc(&dcp, sizeof(int) * std::max(nc, 1));
  if (e == cudaSuccess) e = cudaMalloc(&drp, sizeof(int) * std::max(nr, 1));
  if (e == cudaSuccess) e = cudaMalloc(&deg, sizeof(unsigned) * ((size_t)nc + 1));
  if (e == cudaSuccess) e = cudaMalloc(&nadj, sizeof(int) * std::max<long long>(E, 1));
  if (e == cudaSuccess) e = cudaMalloc(&sadj, sizeof(int) * std::max<long long>(E, 1));
  if (e != cudaSuccess) {
    cleanup();
    return cuda_fail(e, "bm_permute_random");
  }
  noffs = deg;  // scanned in place: deg[nc] = 0 -> offsets
  const int blocks = std::max(1, std::min(h->sms * 8, (nc + 255) / 256));
  cudaMemcpyAsync(dcp, cperm, sizeof(int) * nc, cudaMemcpyHostToDevice, h->stream);
  cudaMemcpyAsync(drp, rperm, sizeof(int) * nr, cudaMemcpyHostToDevice, h->stream);
  cudaMemsetAsync(deg, 0, sizeof(unsigned) * ((size_t)nc + 1), h->stream);
  if (nc > 0) perm_degrees_kernel<<<blocks, 256, 0, h->stream>>>(h->offs, dcp, deg, nc);
  cub::DeviceScan::ExclusiveSum(nullptr, tmp_scan, deg, noffs, nc + 1, h->stream);
  cub::DeviceSegmentedSort::SortKeys(nullptr, tmp_sort, nadj, sadj, (int64_t)E, nc, noffs, noffs + 1, h->stream);
  e = cudaMalloc(&tmp, std::max<size_t>(std::max(tmp_scan, tmp_sort), 1));
  if (e != cudaSuccess) {
    cleanup();
    return cuda_fail(e, "bm_permute_random temp");
  }
  cub::DeviceScan::ExclusiveSum(tmp, tmp_scan, deg, noffs, nc + 1, h->stream);
  if (nc > 0) {
    const int wb = std::max(1, std::min(h->sms * 16, (int)(((long long)nc * 32 + 255) / 256)));
    perm_scatter_kernel<<<wb, 256, 0, h->stream>>>(h->offs, h->adj, dcp, drp, noffs, nadj, nc);
    cub::DeviceSegmentedSort::SortKeys(tmp, tmp_sort, nadj, sadj, (int64_t)E, nc, noffs, noffs + 1, h->stream);
  }
  e = cudaGetLastError();
  if (e == cudaSuccess && E > 0) e = cudaMemcpyAsync(h->adj, sadj, sizeof(int) * E, cudaMemcpyDeviceToDevice, h->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(h->offs, noffs, sizeof(unsigned) * ((size_t)nc + 1), cudaMemcpyDeviceToDevice, h->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
  cleanup();
  if (e != cudaSuccess) return cuda_fail(e, "bm_permute_random");
  h->sorted = 1;
  h->bu_built = false;
  h->has_init = false;  // an initial matching of the old labelling no longer applies
  h->resumable = false;
  return BM_OK;
}

bm_status bm_download_csc(bm_handle* h, int64_t* cxadj, int32_t* cadj) {
  bm_status s = check_handle(h, true);
  if (s != BM_OK) return s;
  BM_CUDA(cudaSetDevice(h->device));
  if (cxadj) {
    std::vector<unsigned> o((size_t)h->nc + 1);
    BM_CUDA(cudaMemcpy(o.data(), h->offs, sizeof(unsigned) * o.size(), cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < o.size(); ++i) cxadj[i] = o[i];
  }
  if (cadj && h->E > 0) BM_CUDA(cudaMemcpy(cadj, h->adj, sizeof(int) * h->E, cudaMemcpyDeviceToHost));
  return BM_OK;
}

bm_status bm_verify(bm_handle* h, const int32_t* rmatch, const int32_t* cmatch, int64_t* violations,
                    int32_t* is_max, int64_t* cardinality) {
  bm_status s = check_handle(h, true);
  if (s != BM_OK) return s;
  if ((!rmatch && h->nr > 0) || (!cmatch && h->nc > 0)) return fail(BM_ERR_INVALID_ARG, "null matching array");
  BM_CUDA(cudaSetDevice(h->device));
  s = rows_from_host(h, rmatch);  // leaves the plain copy in rtmp for validate_kernel
  if (s != BM_OK) return s;
  if (h->nc > 0) {
    s = xfer_h2d(h, h->cmatch, cmatch, sizeof(int) * h->nc, h->stream);
    if (s != BM_OK) return s;
  }
  BM_CUDA(cudaMemsetAsync(h->scratch, 0, sizeof(unsigned long long) * 4, h->stream));
  const int blocks = std::max(1, std::min(h->sms * 8, (std::max(h->nc, h->nr) + 255) / 256));
  validate_kernel<<<blocks, 256, 0, h->stream>>>(h->offs, h->adj, h->nc, h->nr, h->sorted, h->rtmp,
                                                 h->cmatch, h->scratch, h->scratch + 1);
  BM_CUDA(cudaGetLastError());
  unsigned long long res[2] = {0, 0};
  BM_CUDA(cudaMemcpyAsync(res, h->scratch, sizeof(res), cudaMemcpyDeviceToHost, h->stream));
  BM_CUDA(cudaStreamSynchronize(h->stream));
  h->resumable = false;
  if (violations) *violations = (int64_t)res[0];
  if (cardinality) *cardinality = (int64_t)res[1];
  if (is_max) *is_max = 0;
  if (res[0] != 0) return BM_OK;
  // Maximality half (is_maximum, matching.cpp:106-131): a queue BFS of its own
  // (verify_*_kernel), not the engine's driver kernel, so a BFS bug in the
  // engine cannot both stop a run early and certify its result.
  unsigned* vis = h->dead;  // nc bits; free outside a run
  int* qa = reinterpret_cast<int*>(h->F[0]);
  int* qb = reinterpret_cast<int*>(h->F[1]);
  unsigned* cnt = reinterpret_cast<unsigned*>(h->scratch + 4);  // [0] queue length, [1] found
  BM_CUDA(cudaMemsetAsync(vis, 0, sizeof(unsigned) * std::max(h->ndead_words, 1), h->stream));
  BM_CUDA(cudaMemsetAsync(cnt, 0, sizeof(unsigned) * 2, h->stream));
  const int cblocks = std::max(1, std::min(h->sms * 8, (h->nc + 255) / 256));
  if (h->nc > 0) verify_roots_kernel<<<cblocks, 256, 0, h->stream>>>(h->offs, h->cmatch, h->nc, vis, qa, cnt);
  BM_CUDA(cudaGetLastError());
  unsigned st[2] = {0, 0};
  BM_CUDA(cudaMemcpyAsync(st, cnt, sizeof(st), cudaMemcpyDeviceToHost, h->stream));
  BM_CUDA(cudaStreamSynchronize(h->stream));
  for (long long lv = 0; st[0] > 0 && !st[1]; ++lv) {
    if (lv > (long long)h->nc + 1) return fail(BM_ERR_CUDA, "verify BFS exceeded nc + 1 levels");
    const unsigned n = st[0];
    BM_CUDA(cudaMemsetAsync(cnt, 0, sizeof(unsigned), h->stream));
    const int vb = (int)std::max<long long>(1, std::min<long long>((long long)h->sms * 16, ((long long)n * 32 + 255) / 256));
    verify_level_kernel<<<vb, 256, 0, h->stream>>>(h->offs, h->adj, h->rtmp, qa, n, vis, qb, cnt, cnt + 1);
    BM_CUDA(cudaGetLastError());
    BM_CUDA(cudaMemcpyAsync(st, cnt, sizeof(st), cudaMemcpyDeviceToHost, h->stream));
    BM_CUDA(cudaStreamSynchronize(h->stream));
    std::swap(qa, qb);
  }
  if (is_max) *is_max = st[1] ? 0 : 1;
  return BM_OK;
}

}  // extern "C"
