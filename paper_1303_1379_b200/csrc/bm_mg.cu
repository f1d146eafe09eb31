// bm_mg.cu — multi-GPU engine: the persistent driver kernel of bm_engine.cu,
// compiled with BM_MG = 1, over a 1-D column partition.
//
// One rank per GPU (one process per GPU under torchrun; or several ranks on
// one device in one process, each on its own stream, for testing). Rank q owns
//   * columns [cb[q], cb[q+1]): their CSC slice, cmatch, root marks, frontier
//     roots and the pair inbox its columns are routed to;
//   * rows [rb[q], rb[q+1]): their row state {mate, pred} and, for pulled
//     levels, their slice of the row index (the distributed transpose below).
// Every other rank's state is addressed through peer pointers (CUDA IPC over
// NVLink, or plain pointers for ranks of the same process): a claim is a
// system-scope atomic at the row's owner, a winner column is stored straight
// into its owner's inbox, and the level barrier spans the team (MgTeam in rank
// 0's memory). There is no host round trip per level and no collective call on
// the data path: the whole APFB/APsB run is one launch per rank, as on one GPU.
// The dead-root bitmap and the pulled levels' frontier bitmap are replicated;
// each rank copies its own words into the peers' replicas.
#include <algorithm>
#include <climits>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include <unistd.h>

#include <cooperative_groups.h>
#include <cub/device/device_scan.cuh>
#include <cuda_runtime.h>

#include "bm_device.cuh"
#include "bmatch_b200.h"

namespace cg = cooperative_groups;

#define BM_MG 1
namespace bmg {
using namespace bm;
#include "bm_kernels.cuh"
}  // namespace bmg

void bm_internal_set_error(const std::string& msg);

namespace {

using bmg::Ctrl;
using bmg::MgTeam;
using bmg::Params;
using bmg::PhaseRec;
using bmg::Smem;
using bmg::kMaxRanks;
using bmg::kNumFbit;

bm_status fail(bm_status s, const std::string& msg) {
  bm_internal_set_error(msg);
  return s;
}
bm_status cuda_fail(cudaError_t e, const char* what) {
  const bm_status s = (e == cudaErrorMemoryAllocation) ? BM_ERR_OOM : BM_ERR_CUDA;
  return fail(s, std::string(what) + ": " + cudaGetErrorString(e));
}
#define BM_CUDA(call)                                   \
  do {                                                  \
    cudaError_t e_ = (call);                            \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
  } while (0)

template <typename T>
void dfree(T*& p) {
  if (p) cudaFree(p);
  p = nullptr;
}
template <typename T>
cudaError_t dnew(T*& p, size_t count) {
  dfree(p);
  return cudaMalloc(reinterpret_cast<void**>(&p), std::max<size_t>(count, 1) * sizeof(T));
}
// Grows a buffer only when it is too small, so that re-uploading a graph of the
// same size reuses the allocations (a free + malloc of GB-sized buffers per
// upload cost more than the copy).
using CapMap = std::map<const void*, size_t>;
template <typename T>
cudaError_t dgrow(CapMap& caps, T*& p, size_t count) {
  count = std::max<size_t>(count, 1);
  size_t& cap = caps[&p];
  if (p && cap >= count) return cudaSuccess;
  dfree(p);
  cap = 0;
  const cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&p), count * sizeof(T));
  if (e == cudaSuccess) cap = count;
  return e;
}

// The buffers a rank shares, in blob order.
enum Shared { kShRm, kShPred, kShCm, kShBfs, kShCroot, kShDead, kShFbit, kShP, kShEP, kShF0, kShF1, kShCtl,
              kShTeam, kShOut, kShOutIdx, kNumShared };

struct Blob {
  int32_t pid;
  int32_t rank;
  int32_t device;
  int32_t pad;
  uint64_t ptr[kNumShared];
  cudaIpcMemHandle_t ipc[kNumShared];
};

}  // namespace

struct bm_mg {
  int device = 0, rank = 0, world = 1, share = 1;
  cudaStream_t own = nullptr, stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  int sms = 0, bps[3] = {0, 0, 0};
  // partition
  int nc = -1, nr = -1;
  long long E = 0, E_total = 0;
  std::vector<int> cb, rb;  // world + 1 bounds each
  int clo = 0, chi = 0, rlo = 0, rhi = 0;
  int rs = 1;
  int sorted = 1;
  long long fcap = 0;
  // own buffers (allocation bases)
  unsigned* offs = nullptr;
  int* adj = nullptr;
  int *rm = nullptr, *pred_plain = nullptr, *cmatch = nullptr, *bfs = nullptr, *croot = nullptr;
  unsigned *dead = nullptr, *fbit = nullptr;
  int nfbit_words = 0, ndead_words = 0;
  int2* P = nullptr;
  int* EP = nullptr;
  int4* F[2] = {nullptr, nullptr};
  unsigned* gidx[2] = {nullptr, nullptr};
  int2* wlog = nullptr;
  unsigned log_cap = 0;
  Ctrl* ctl = nullptr;
  PhaseRec* recs = nullptr;
  int rec_cap = 4096;
  MgTeam* team = nullptr;  // rank 0 allocates it; shared
  int* rtmp = nullptr;     // staging for plain row arrays
  // row index (pulled levels): outbox = this rank's edges bucketed by global row range
  int2* outbox = nullptr;
  unsigned* out_idx = nullptr;  // [0, nb) bucket bases, [kMaxBuckets, +nb) bucket counts, then tickets
  int shift = 0, nb = 0;
  int2* inbox = nullptr;
  long long inbox_n = 0;
  unsigned *roffs = nullptr, *rcursor = nullptr;
  int* radj = nullptr;
  unsigned char* scan_tmp = nullptr;
  size_t scan_bytes = 0;
  bool row_index = false;
  double deg_col = 0, deg_row = 0;
  long long nonempty = 0;
  // peers
  bmg::PeerPtrs peer[kMaxRanks];
  void* opened[kMaxRanks][kNumShared] = {};
  CapMap caps;                            // capacities of the dgrow buffers
  long long* stage64 = nullptr;           // the slice's int64 offsets, before narrowing on the device
  unsigned long long* scratch = nullptr;  // upload check counters
  int2* peer_outbox[kMaxRanks] = {};
  unsigned* peer_out_idx[kMaxRanks] = {};
  MgTeam* team_ptr = nullptr;
  bool imported = false;
  double last_ms = 0;
  bm_match_opts last_opts{};
};

namespace {

// Even 32-aligned split of n into world ranges.
void split(int n, int world, std::vector<int>& b) {
  b.assign(world + 1, 0);
  for (int q = 1; q < world; ++q) {
    long long x = (long long)n * q / world;
    x = (x + 31) / 32 * 32;
    b[q] = (int)std::min<long long>(x, n);
  }
  b[world] = n;
}

void close_peers(bm_mg* h) {
  for (int q = 0; q < kMaxRanks; ++q)
    for (int k = 0; k < kNumShared; ++k)
      if (h->opened[q][k]) {
        cudaIpcCloseMemHandle(h->opened[q][k]);
        h->opened[q][k] = nullptr;
      }
  h->imported = false;
}

const void* mg_kernel(int wr, int imp) {
  if (!wr) return reinterpret_cast<const void*>(&bmg::driver_kernel<false, false, true>);
  if (!imp) return reinterpret_cast<const void*>(&bmg::driver_kernel<true, false, true>);
  return reinterpret_cast<const void*>(&bmg::driver_kernel<true, true, true>);
}

}  // namespace

extern "C" {

bm_status bm_mg_partition(int32_t n, int32_t world, int32_t* bounds) {
  if (world < 1 || world > kMaxRanks) return fail(BM_ERR_INVALID_ARG, "world must be in [1, 8]");
  if (n < 0 || !bounds) return fail(BM_ERR_INVALID_ARG, "bad partition arguments");
  std::vector<int> b;
  split(n, world, b);
  for (int q = 0; q <= world; ++q) bounds[q] = b[q];
  return BM_OK;
}

bm_status bm_mg_create(int32_t device, int32_t rank, int32_t world, int32_t share, bm_mg** out) {
  if (!out) return fail(BM_ERR_INVALID_ARG, "null output pointer");
  *out = nullptr;
  if (world < 1 || world > kMaxRanks || rank < 0 || rank >= world)
    return fail(BM_ERR_INVALID_ARG, "rank/world out of range (world <= 8)");
  if (share < 1 || share > world) return fail(BM_ERR_INVALID_ARG, "share must be in [1, world]");
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0)
    return fail(BM_ERR_CUDA, "no CUDA device available (the engine has no CPU fallback)");
  if (device < 0 || device >= n) return fail(BM_ERR_INVALID_ARG, "device index out of range");
  BM_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop{};
  BM_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10) return fail(BM_ERR_CUDA, "this build targets sm_100a (B200)");
  auto* h = new bm_mg();
  h->device = device;
  h->rank = rank;
  h->world = world;
  h->share = share;
  h->sms = prop.multiProcessorCount;
  for (int v = 0; v < 3; ++v) {
    const void* k = mg_kernel(v >= 1, v == 2);
    e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Smem));
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&h->bps[v], k, bmg::kThreads, sizeof(Smem));
    if (e != cudaSuccess || h->bps[v] < 1) {
      delete h;
      return fail(BM_ERR_CUDA, "occupancy query failed");
    }
  }
  e = cudaStreamCreateWithFlags(&h->own, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreate(&h->ev0);
  if (e == cudaSuccess) e = cudaEventCreate(&h->ev1);
  if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void**>(&h->ctl), sizeof(Ctrl));
  if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void**>(&h->recs), sizeof(PhaseRec) * h->rec_cap);
  if (e == cudaSuccess && rank == 0) e = cudaMalloc(reinterpret_cast<void**>(&h->team), sizeof(MgTeam));
  if (e == cudaSuccess && rank == 0) e = cudaMemset(h->team, 0, sizeof(MgTeam));
  if (e == cudaSuccess) e = cudaMemset(h->ctl, 0, sizeof(Ctrl));
  if (e != cudaSuccess) {
    bm_mg_destroy(h);
    return cuda_fail(e, "bm_mg_create");
  }
  h->stream = h->own;
  *out = h;
  return BM_OK;
}

bm_status bm_mg_destroy(bm_mg* h) {
  if (!h) return BM_OK;
  cudaSetDevice(h->device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  close_peers(h);
  dfree(h->offs);
  dfree(h->stage64);
  dfree(h->scratch);
  dfree(h->adj);
  dfree(h->rm);
  dfree(h->pred_plain);
  dfree(h->cmatch);
  dfree(h->bfs);
  dfree(h->croot);
  dfree(h->dead);
  dfree(h->fbit);
  dfree(h->P);
  dfree(h->EP);
  dfree(h->F[0]);
  dfree(h->F[1]);
  dfree(h->gidx[0]);
  dfree(h->gidx[1]);
  dfree(h->wlog);
  dfree(h->ctl);
  dfree(h->recs);
  dfree(h->team);
  dfree(h->rtmp);
  dfree(h->outbox);
  dfree(h->out_idx);
  dfree(h->inbox);
  dfree(h->roffs);
  dfree(h->rcursor);
  dfree(h->radj);
  dfree(h->scan_tmp);
  if (h->ev0) cudaEventDestroy(h->ev0);
  if (h->ev1) cudaEventDestroy(h->ev1);
  if (h->own) cudaStreamDestroy(h->own);
  delete h;
  return BM_OK;
}

bm_status bm_mg_set_stream(bm_mg* h, void* stream) {
  if (!h) return fail(BM_ERR_INVALID_ARG, "null handle");
  h->stream = stream ? static_cast<cudaStream_t>(stream) : h->own;
  return BM_OK;
}

// This rank's slice: columns [cb[rank], cb[rank+1]) (cxadj rebased to 0) and
// the row ownership rb (both world + 1 bounds, 32-aligned inner bounds, the
// same on every rank). e_total: edges of the whole graph.
bm_status bm_mg_upload(bm_mg* h, int32_t nc, int32_t nr, int64_t e_total, const int32_t* cb, const int32_t* rb,
                       const int64_t* cxadj, const int32_t* cadj) {
  if (!h || !cb || !rb || !cxadj) return fail(BM_ERR_INVALID_ARG, "null argument");
  if (nc < 0 || nr < 0 || nc >= (1 << 30)) return fail(BM_ERR_INVALID_ARG, "vertex counts out of range");
  for (int q = 0; q < h->world; ++q) {
    if (cb[q] > cb[q + 1] || rb[q] > rb[q + 1]) return fail(BM_ERR_INVALID_ARG, "bounds must ascend");
    if (q > 0 && ((cb[q] % 32 && cb[q] != nc) || (rb[q] % 32 && rb[q] != nr)))
      return fail(BM_ERR_INVALID_ARG, "inner bounds must be 32-aligned (or the end)");
  }
  if (cb[0] != 0 || cb[h->world] != nc || rb[0] != 0 || rb[h->world] != nr)
    return fail(BM_ERR_INVALID_ARG, "bounds must cover [0, nc) and [0, nr)");
  BM_CUDA(cudaSetDevice(h->device));
  BM_CUDA(cudaStreamSynchronize(h->stream));
  close_peers(h);
  h->nc = nc;
  h->nr = nr;
  h->cb.assign(cb, cb + h->world + 1);
  h->rb.assign(rb, rb + h->world + 1);
  h->clo = cb[h->rank];
  h->chi = cb[h->rank + 1];
  h->rlo = rb[h->rank];
  h->rhi = rb[h->rank + 1];
  const int ncl = h->chi - h->clo, nrl = h->rhi - h->rlo;
  const long long E = cxadj[ncl];
  if (cxadj[0] != 0 || E < 0 || E >= (1ll << 32) - 1) return fail(BM_ERR_INVALID_ARG, "bad slice offsets");
  h->E = E;
  h->E_total = e_total;
  // The slice is checked on the device while it lands (check_csr, csr_graph.cpp:45-64):
  // offsets non-decreasing and narrowed to u32, rows in range, per-column order.
  BM_CUDA(dgrow(h->caps, h->stage64, (size_t)ncl + 1));
  BM_CUDA(dgrow(h->caps, h->scratch, 8));
  BM_CUDA(dgrow(h->caps, h->offs, (size_t)ncl + 1));
  BM_CUDA(dgrow(h->caps, h->adj, (size_t)E));
  BM_CUDA(cudaMemsetAsync(h->scratch, 0, sizeof(unsigned long long) * 8, h->stream));
  BM_CUDA(cudaMemcpyAsync(h->stage64, cxadj, sizeof(long long) * ((size_t)ncl + 1), cudaMemcpyHostToDevice, h->stream));
  const int cblocks = std::max(1, std::min(h->sms * 8, (ncl + 256) / 256));
  bmg::convert_offsets_kernel<<<cblocks, 256, 0, h->stream>>>(h->stage64, h->offs, ncl, E, h->scratch, h->scratch + 4);
  if (E) BM_CUDA(cudaMemcpyAsync(h->adj, cadj, sizeof(int) * (size_t)E, cudaMemcpyHostToDevice, h->stream));
  const int ablocks = (int)std::max<long long>(1, std::min<long long>((long long)h->sms * 8, (E + 255) / 256));
  if (E) bmg::check_adj_flat_kernel<<<ablocks, 256, 0, h->stream>>>(h->adj, 0, E, nr, h->scratch + 1, h->scratch + 2);
  if (ncl) bmg::col_start_pairs_kernel<<<cblocks, 256, 0, h->stream>>>(h->offs, h->adj, ncl, h->scratch + 3);
  BM_CUDA(cudaGetLastError());
  unsigned long long chk[5] = {0, 0, 0, 0, 0};
  BM_CUDA(cudaMemcpyAsync(chk, h->scratch, sizeof(chk), cudaMemcpyDeviceToHost, h->stream));
  BM_CUDA(cudaStreamSynchronize(h->stream));
  if (chk[0]) return fail(BM_ERR_INVALID_ARG, "cxadj slice must be non-decreasing");
  if (chk[1]) return fail(BM_ERR_INVALID_ARG, "row index out of range in cadj");
  h->sorted = (chk[2] - chk[3]) == 0 ? 1 : 0;
  h->nonempty = (long long)ncl - (long long)chk[4];
  h->rs = ((size_t)nr * sizeof(int) > ((size_t)72 << 20)) ? 2 : 1;
  if (const char* lay = getenv("BM_ROW_LAYOUT")) h->rs = strcmp(lay, "plain") ? 2 : 1;
  // frontier capacity: the same on every rank (the store-claim rule compares against it)
  int maxc = 0;
  for (int q = 0; q < h->world; ++q) maxc = std::max(maxc, cb[q + 1] - cb[q]);
  h->fcap = (long long)maxc + (long long)bmg::kFSlack(maxc);
  BM_CUDA(dgrow(h->caps, h->rm, (size_t)2 * std::max(nrl, 1)));
  BM_CUDA(dgrow(h->caps, h->pred_plain, nrl));
  BM_CUDA(dgrow(h->caps, h->rtmp, nrl));
  BM_CUDA(dgrow(h->caps, h->cmatch, ncl));
  BM_CUDA(dgrow(h->caps, h->bfs, ncl));
  BM_CUDA(dgrow(h->caps, h->croot, ncl));
  h->ndead_words = h->nfbit_words = (nc + 31) / 32;
  BM_CUDA(dgrow(h->caps, h->dead, h->ndead_words));
  BM_CUDA(dgrow(h->caps, h->fbit, (size_t)kNumFbit * h->nfbit_words));
  BM_CUDA(dgrow(h->caps, h->P, h->fcap));
  BM_CUDA(dgrow(h->caps, h->F[0], h->fcap));
  BM_CUDA(dgrow(h->caps, h->F[1], h->fcap));
  BM_CUDA(dgrow(h->caps, h->EP, std::max(nr, 1)));
  const size_t ngran = (size_t)(E / bmg::kGran) + 2;
  BM_CUDA(dgrow(h->caps, h->gidx[0], ngran));
  BM_CUDA(dgrow(h->caps, h->gidx[1], ngran));
  h->log_cap = (unsigned)std::min<long long>((long long)nr + nc + 1024, 0xffffffffll);
  BM_CUDA(dgrow(h->caps, h->wlog, h->log_cap));
  BM_CUDA(cudaMemset(h->pred_plain, 0xff, sizeof(int) * std::max(nrl, 1)));
  BM_CUDA(cudaMemset(h->rm, 0xff, sizeof(int) * 2 * std::max(nrl, 1)));  // mates -1, interleaved preds -1
  BM_CUDA(cudaMemset(h->fbit, 0, sizeof(unsigned) * kNumFbit * h->nfbit_words));
  // row index: bucket the rows so that one bucket's slice of an index is <= 32 MB
  {
    const long long nb_min = std::max<long long>(1, (e_total * 4 + (32ll << 20) - 1) >> 25);
    int shift = 0;
    while (shift < 31 && ((long long)nr + (1ll << shift) - 1) >> shift > nb_min) ++shift;
    h->shift = shift;
    h->nb = (int)(((long long)nr + (1ll << shift) - 1) >> shift);
    if (h->nb > bmg::kMaxBuckets) return fail(BM_ERR_INVALID_ARG, "row index: too many buckets");
  }
  BM_CUDA(dgrow(h->caps, h->outbox, E));
  BM_CUDA(dgrow(h->caps, h->out_idx, 2 * bmg::kMaxBuckets + 4));
  h->deg_col = (double)e_total / (double)std::max(1ll, (long long)nc);  // refined below by the team
  h->deg_row = (double)e_total / (double)std::max(1, nr);
  h->row_index = false;
  BM_CUDA(cudaDeviceSynchronize());
  return BM_OK;
}

// Shared buffers of this rank: raw pointers (ranks of the same process) and
// CUDA IPC handles (other processes). blob: sizeof(Blob) bytes.
bm_status bm_mg_blob_size(int64_t* bytes) {
  if (!bytes) return fail(BM_ERR_INVALID_ARG, "null pointer");
  *bytes = sizeof(Blob);
  return BM_OK;
}

bm_status bm_mg_export(bm_mg* h, void* blob_out) {
  if (!h || !blob_out) return fail(BM_ERR_INVALID_ARG, "null argument");
  if (h->nc < 0) return fail(BM_ERR_INVALID_ARG, "upload the slice first");
  BM_CUDA(cudaSetDevice(h->device));
  Blob b{};
  b.pid = (int32_t)getpid();
  b.rank = h->rank;
  b.device = h->device;
  void* ptrs[kNumShared] = {h->rm, h->pred_plain, h->cmatch, h->bfs, h->croot, h->dead, h->fbit, h->P, h->EP,
                            h->F[0], h->F[1], h->ctl, h->team, h->outbox, h->out_idx};
  for (int k = 0; k < kNumShared; ++k) {
    b.ptr[k] = reinterpret_cast<uint64_t>(ptrs[k]);
    if (ptrs[k]) BM_CUDA(cudaIpcGetMemHandle(&b.ipc[k], ptrs[k]));
  }
  std::memcpy(blob_out, &b, sizeof(b));
  return BM_OK;
}

// blobs: world Blob records in rank order.
bm_status bm_mg_import(bm_mg* h, const void* blobs) {
  if (!h || !blobs) return fail(BM_ERR_INVALID_ARG, "null argument");
  BM_CUDA(cudaSetDevice(h->device));
  close_peers(h);
  const Blob* bl = static_cast<const Blob*>(blobs);
  const int mypid = (int)getpid();
  for (int q = 0; q < h->world; ++q) {
    if (bl[q].rank != q) return fail(BM_ERR_INVALID_ARG, "blobs must be in rank order");
    void* p[kNumShared] = {};
    for (int k = 0; k < kNumShared; ++k) {
      if (!bl[q].ptr[k]) continue;
      if (bl[q].pid == mypid) {
        p[k] = reinterpret_cast<void*>(bl[q].ptr[k]);
        if (bl[q].device != h->device && k == 0) {  // ranks of this process on two devices
          cudaError_t pe = cudaDeviceEnablePeerAccess(bl[q].device, 0);
          if (pe == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
          else if (pe != cudaSuccess) return cuda_fail(pe, "cudaDeviceEnablePeerAccess");
        }
      } else {
        if (bl[q].device != h->device) {
          int can = 0;
          cudaDeviceCanAccessPeer(&can, h->device, bl[q].device);
          if (!can) return fail(BM_ERR_CUDA, "no peer access between the ranks' devices (NVLink/P2P required)");
        }
        cudaIpcMemHandle_t hd = bl[q].ipc[k];
        BM_CUDA(cudaIpcOpenMemHandle(&p[k], hd, cudaIpcMemLazyEnablePeerAccess));
        h->opened[q][k] = p[k];
      }
    }
    const long long rlo = h->rb[q], clo = h->cb[q];
    bmg::PeerPtrs& pp = h->peer[q];
    int* rmq = static_cast<int*>(p[kShRm]);
    pp.rm = rmq - h->rs * rlo;
    pp.pred = (h->rs == 2 ? rmq + 1 : static_cast<int*>(p[kShPred])) - h->rs * rlo;
    pp.cmatch = static_cast<int*>(p[kShCm]) - clo;
    pp.bfs = static_cast<int*>(p[kShBfs]) - clo;
    pp.croot = static_cast<int*>(p[kShCroot]) - clo;
    pp.dead = static_cast<unsigned*>(p[kShDead]);
    pp.fbit = static_cast<unsigned*>(p[kShFbit]);
    pp.P = static_cast<int2*>(p[kShP]);
    pp.EP = static_cast<int*>(p[kShEP]);
    pp.F0 = static_cast<int4*>(p[kShF0]);
    pp.F1 = static_cast<int4*>(p[kShF1]);
    pp.ctl = static_cast<Ctrl*>(p[kShCtl]);
    h->peer_outbox[q] = static_cast<int2*>(p[kShOut]);
    h->peer_out_idx[q] = static_cast<unsigned*>(p[kShOutIdx]);
    if (q == 0) h->team_ptr = static_cast<MgTeam*>(p[kShTeam]);
  }
  if (!h->team_ptr) return fail(BM_ERR_INVALID_ARG, "rank 0 exported no team block");
  h->imported = true;
  return BM_OK;
}

// The initial matching of this rank's rows and columns (plain arrays).
bm_status bm_mg_load_matching(bm_mg* h, const int32_t* rmatch_slice, const int32_t* cmatch_slice) {
  if (!h || !rmatch_slice || !cmatch_slice) return fail(BM_ERR_INVALID_ARG, "null argument");
  BM_CUDA(cudaSetDevice(h->device));
  const int ncl = h->chi - h->clo, nrl = h->rhi - h->rlo;
  if (ncl) BM_CUDA(cudaMemcpyAsync(h->cmatch, cmatch_slice, sizeof(int) * ncl, cudaMemcpyHostToDevice, h->stream));
  if (nrl) {
    BM_CUDA(cudaMemcpyAsync(h->rtmp, rmatch_slice, sizeof(int) * nrl, cudaMemcpyHostToDevice, h->stream));
    bmg::rows_pack_kernel<<<std::max(1, std::min(h->sms * 8, (nrl + 255) / 256)), 256, 0, h->stream>>>(
        h->rtmp, h->rm, nrl, h->rs);
    BM_CUDA(cudaGetLastError());
  }
  BM_CUDA(cudaStreamSynchronize(h->stream));
  return BM_OK;
}

// Row index for pulled levels, step 1 (every rank): bucket this rank's edges
// by global row range into its outbox. A host barrier must separate it from
// step 2 on every rank.
bm_status bm_mg_row_index_begin(bm_mg* h) {
  if (!h || h->nc < 0) return fail(BM_ERR_INVALID_ARG, "upload the slice first");
  BM_CUDA(cudaSetDevice(h->device));
  const int ncl = h->chi - h->clo;
  unsigned* pcur = h->out_idx;
  unsigned* bcount = h->out_idx + bmg::kMaxBuckets;
  BM_CUDA(cudaMemsetAsync(h->out_idx, 0, sizeof(unsigned) * (2 * bmg::kMaxBuckets + 4), h->stream));
  if (h->E > 0) {
    const int grid = h->sms * 8;
    bmg::bucket_hist_kernel<<<grid, 256, 0, h->stream>>>(h->adj, (unsigned)h->E, h->shift, h->nb, INT_MAX, bcount);
    bmg::bucket_base_kernel<<<1, 32, 0, h->stream>>>(bcount, h->nb, pcur);
    const int pa = (int)std::max<long long>(1, std::min<long long>(grid, (h->E + bmg::kTpChunk - 1) / bmg::kTpChunk));
    bmg::bucket_partition_kernel<<<pa, 256, 0, h->stream>>>(h->offs, h->adj, h->clo, ncl, (unsigned)h->E, h->shift, h->nb,
                                                            pcur, h->outbox);
    // pcur now holds each bucket's end; the start is end - count
  }
  BM_CUDA(cudaGetLastError());
  BM_CUDA(cudaStreamSynchronize(h->stream));
  return BM_OK;
}

// Step 2: gather the buckets that hold this rank's rows from every rank's
// outbox (peer memory), then count, scan and scatter them into the row index
// of this rank's rows (the ordered passes of the single-GPU build).
bm_status bm_mg_row_index_end(bm_mg* h) {
  if (!h || !h->imported) return fail(BM_ERR_INVALID_ARG, "import the team's blobs first");
  BM_CUDA(cudaSetDevice(h->device));
  const int nrl = h->rhi - h->rlo;
  const int b0 = h->rlo >> h->shift;
  const int b1 = nrl ? ((h->rhi - 1) >> h->shift) : b0 - 1;  // buckets overlapping [rlo, rhi)
  std::vector<long long> seg_lo(h->world), seg_n(h->world);
  long long total = 0;
  for (int q = 0; q < h->world; ++q) {
    std::vector<unsigned> idx(2 * bmg::kMaxBuckets);
    BM_CUDA(cudaMemcpy(idx.data(), h->peer_out_idx[q], sizeof(unsigned) * 2 * bmg::kMaxBuckets, cudaMemcpyDefault));
    long long lo = 0, n = 0;
    if (b1 >= b0) {
      lo = (long long)idx[b0] - idx[bmg::kMaxBuckets + b0];  // end - count = start of bucket b0
      const long long hi = idx[b1];                          // end of bucket b1
      n = hi - lo;
    }
    seg_lo[q] = lo;
    seg_n[q] = n;
    total += n;
  }
  BM_CUDA(dgrow(h->caps, h->inbox, total));
  long long at = 0;
  for (int q = 0; q < h->world; ++q) {
    if (seg_n[q]) BM_CUDA(cudaMemcpyAsync(h->inbox + at, h->peer_outbox[q] + seg_lo[q], sizeof(int2) * seg_n[q],
                                          cudaMemcpyDefault, h->stream));
    at += seg_n[q];
  }
  h->inbox_n = total;
  long long mine = 0;  // edges of this rank's rows (straddling buckets also carry other ranks' rows)
  BM_CUDA(dgrow(h->caps, h->roffs, (size_t)nrl + 1));
  BM_CUDA(dgrow(h->caps, h->rcursor, (size_t)nrl + 1));
  BM_CUDA(cudaMemsetAsync(h->rcursor, 0, sizeof(unsigned) * ((size_t)nrl + 1), h->stream));
  unsigned* tickets = h->out_idx + 2 * bmg::kMaxBuckets;
  BM_CUDA(cudaMemsetAsync(tickets, 0, sizeof(unsigned) * 2, h->stream));
  const int grid = h->sms * 8;
  if (total) bmg::pair_pass_kernel<false><<<grid, 256, 0, h->stream>>>(h->inbox, (unsigned)total, tickets, h->rcursor,
                                                                       nullptr, h->rlo, h->rhi);
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, h->rcursor, h->roffs, nrl + 1, h->stream);
  if (tb > h->scan_bytes) {
    BM_CUDA(dgrow(h->caps, h->scan_tmp, tb));
    h->scan_bytes = tb;
  }
  cub::DeviceScan::ExclusiveSum(h->scan_tmp, tb, h->rcursor, h->roffs, nrl + 1, h->stream);
  unsigned last = 0;
  BM_CUDA(cudaMemcpyAsync(&last, h->roffs + nrl, sizeof(unsigned), cudaMemcpyDeviceToHost, h->stream));
  BM_CUDA(cudaStreamSynchronize(h->stream));
  mine = last;
  BM_CUDA(dgrow(h->caps, h->radj, mine + 4));  // (+4: the pulled probes read aligned groups of 4)
  BM_CUDA(cudaMemcpyAsync(h->rcursor, h->roffs, sizeof(unsigned) * ((size_t)nrl + 1), cudaMemcpyDeviceToDevice,
                          h->stream));
  if (total) bmg::pair_pass_kernel<true><<<grid, 256, 0, h->stream>>>(h->inbox, (unsigned)total, tickets + 1,
                                                                      h->rcursor, h->radj, h->rlo, h->rhi);
  BM_CUDA(cudaGetLastError());
  BM_CUDA(cudaStreamSynchronize(h->stream));
  h->row_index = true;
  return BM_OK;
}

// Enqueues this rank's persistent driver kernel. Every rank of the team must
// launch before any can finish (the level barrier spans the team): ranks of
// one process launch on their own streams first, then call bm_mg_finish.
bm_status bm_mg_launch(bm_mg* h, const bm_match_opts* o) {
  if (!h || !o) return fail(BM_ERR_INVALID_ARG, "null argument");
  if (!h->imported) return fail(BM_ERR_INVALID_ARG, "import the team's blobs first");
  if (o->driver != BM_DRIVER_APFB && o->driver != BM_DRIVER_APSB) return fail(BM_ERR_INVALID_ARG, "unknown driver");
  if (o->bfs_kernel != BM_BFS_GPUBFS && o->bfs_kernel != BM_BFS_WR) return fail(BM_ERR_INVALID_ARG, "unknown kernel");
  if (o->improved && o->bfs_kernel != BM_BFS_WR)
    return fail(BM_ERR_LOGIC, "the endpoint-encoded alternation requires the with-root kernel");
  if (o->init != BM_INIT_GIVEN && o->init != BM_INIT_GPU_GREEDY && o->init != BM_INIT_GPU_KS)
    return fail(BM_ERR_INVALID_ARG, "unknown init mode");
  BM_CUDA(cudaSetDevice(h->device));
  const int ncl = h->chi - h->clo, nrl = h->rhi - h->rlo;
  BM_CUDA(cudaMemsetAsync(h->ctl, 0, sizeof(Ctrl), h->stream));
  BM_CUDA(cudaMemsetAsync(h->dead, 0, sizeof(unsigned) * h->ndead_words, h->stream));
  BM_CUDA(cudaMemsetAsync(h->fbit, 0, sizeof(unsigned) * kNumFbit * h->nfbit_words, h->stream));
  // (the team block is zeroed once, at creation: another rank's kernel may already be
  // arriving at its barrier; a run leaves its count at 0 and its path flags clear)
  const bool pull = h->row_index && o->bottom_up != BM_BU_OFF;
  Params p{};
  p.nc = h->nc;
  p.nr = h->nr;
  // local bases, pre-offset so that global ids index them
  p.offs = h->offs - h->clo;
  p.adj = h->adj;
  p.rm = h->rm - (long long)h->rs * h->rlo;
  p.rs = h->rs;
  p.pred = (h->rs == 2 ? h->rm + 1 : h->pred_plain) - (long long)h->rs * h->rlo;
  p.cmatch = h->cmatch - h->clo;
  p.bfs = h->bfs - h->clo;
  p.croot = h->croot - h->clo;
  p.dead = h->dead;
  p.ndead_words = h->ndead_words;
  p.F0 = h->F[0];
  p.F1 = h->F[1];
  p.gidx0 = h->gidx[0];
  p.gidx1 = h->gidx[1];
  p.EP = h->EP;
  p.wlog = h->wlog;
  p.log_cap = h->log_cap;
  p.ctl = h->ctl;
  p.recs = h->recs;
  p.rec_cap = h->rec_cap;
  p.apsb = o->driver == BM_DRIVER_APSB;
  p.init_mode = o->init;
  p.fresh = 1;
  p.init_checked = 0;
  p.sorted = h->sorted;
  p.dbg_skip_alt_phase = 0;
  p.check = 0;
  p.max_phases = h->rec_cap;
  p.stop_after_bfs = 0;
  p.trace = 0;
  p.claim_mode = o->claim_policy;
  p.ep_one = (o->bfs_kernel == BM_BFS_WR && o->endpoint_policy != BM_EP_EVERY) ? 1 : 0;
  // A team of one runs the single-GPU level loop (narrow levels on block 0 alone,
  // winners as entries unless the level is wide); a larger team routes every
  // winner as a pair and has no solo hand-over.
  p.solo_edges = h->world == 1 ? bmg::kSoloEdges : 0;
  if (const char* se = getenv("BM_SOLO_EDGES")) p.solo_edges = h->world == 1 ? (unsigned)atol(se) : 0;
  p.roffs = pull ? h->roffs - h->rlo : nullptr;
  p.radj = h->radj;
  for (int b = 0; b < kNumFbit; ++b) p.fbit[b] = h->fbit + (size_t)b * h->nfbit_words;
  p.nfbit_words = h->nfbit_words;
  p.bu_rule = 1;
  p.bu_alpha = h->rs == 2 ? 14.f : 4.f;
  if (const char* a = getenv("BM_BU_ALPHA")) p.bu_alpha = (float)atof(a);
  p.bu_min_n = (unsigned)std::min<double>(4e9, (double)h->nc / 24.0);
  p.bu_min_edges = 0;
  if (const char* fr = getenv("BM_BU_FRAC")) {  // the plain edge-share rule (tests: 0 pulls every level)
    p.bu_rule = 0;
    p.bu_min_edges = (unsigned long long)std::max(0.0, atof(fr) * (double)h->E_total);
  }
  p.deg_col = h->deg_col;
  p.deg_row = h->deg_row;
  p.P = h->P;
  p.pairs_min_edges = h->world == 1 ? std::max<unsigned long long>(1ull << 20, (unsigned long long)h->E_total / 128) : 0;
  p.phase_bound = (long long)h->nc + 1;
  p.fcap = (unsigned long long)h->fcap;
  p.claim_store = 1;
  if (const char* cs = getenv("BM_CLAIM_STORE")) p.claim_store = atoi(cs);
  p.tl = nullptr;
  p.tl_cap = 0;
  p.world = h->world;
  p.rank = h->rank;
  p.col_lo = h->clo;
  p.col_hi = h->chi;
  p.row_lo = h->rlo;
  p.row_hi = h->rhi;
  for (int i = 0; i < kMaxRanks - 1; ++i) {
    p.cb[i] = i + 1 < h->world ? h->cb[i + 1] : INT_MAX;
    p.rb[i] = i + 1 < h->world ? h->rb[i + 1] : INT_MAX;
  }
  p.world_solo = 0;
  p.team = h->team_ptr;
  for (int q = 0; q < h->world; ++q) p.peer[q] = h->peer[q];
  (void)ncl;
  (void)nrl;
  const int v = o->bfs_kernel == BM_BFS_WR ? (o->improved ? 2 : 1) : 0;
  const long long cap = (long long)h->sms * h->bps[v] / h->share;
  const int G = (int)std::max<long long>(1, cap);
  void* args[] = {&p};
  BM_CUDA(cudaEventRecord(h->ev0, h->stream));
  BM_CUDA(cudaLaunchCooperativeKernel(mg_kernel(o->bfs_kernel == BM_BFS_WR, o->improved), dim3(G),
                                      dim3(bmg::kThreads), args, sizeof(Smem), h->stream));
  BM_CUDA(cudaEventRecord(h->ev1, h->stream));
  h->last_opts = *o;
  return BM_OK;
}

// Waits for this rank's kernel and reads the result. counters: this rank's
// work counters; outer_iterations, bfs_launches_total, cardinality and the
// per-phase records are the team's (identical on every rank).
bm_status bm_mg_finish(bm_mg* h, int64_t* cardinality, bm_counters* counters) {
  if (!h) return fail(BM_ERR_INVALID_ARG, "null handle");
  BM_CUDA(cudaSetDevice(h->device));
  BM_CUDA(cudaStreamSynchronize(h->stream));
  float ms = 0.f;
  BM_CUDA(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
  h->last_ms = ms;
  Ctrl ctl{};
  BM_CUDA(cudaMemcpy(&ctl, h->ctl, sizeof(Ctrl), cudaMemcpyDeviceToHost));
  if (ctl.error) {
    switch (ctl.error) {
      case bmg::kErrBound: return fail(BM_ERR_BOUND_EXCEEDED, "termination bound exceeded: more than nc + 1 phases");
      case bmg::kErrInvalidInit:
        return fail(BM_ERR_INVALID_ARG, "initial matching is not a clean valid matching");
      default: return fail(BM_ERR_CUDA, "device error " + std::to_string(ctl.error));
    }
  }
  std::vector<PhaseRec> recs(std::max(ctl.n_recs, 0));
  if (ctl.n_recs > 0)
    BM_CUDA(cudaMemcpy(recs.data(), h->recs, sizeof(PhaseRec) * ctl.n_recs, cudaMemcpyDeviceToHost));
  if (cardinality) *cardinality = ctl.card;
  if (counters) {
    std::memset(counters, 0, sizeof(*counters));
    counters->outer_iterations = (int64_t)recs.size();
    long long lt = 0, retries = 0;
    for (auto& r : recs) {
      lt += r.launches;
      retries += r.retry;
    }
    counters->bfs_launches_total = lt;
    counters->serial_retries = retries;
    counters->columns_scanned = (int64_t)ctl.stats[bmg::kStCexp];
    counters->alternations_attempted = (int64_t)ctl.stats[bmg::kStWalks];
    counters->fix_resets = (int64_t)ctl.stats[bmg::kStResets];
    counters->edges_traversed = (int64_t)ctl.stats[bmg::kStTrav];
    counters->columns_visited = (int64_t)ctl.stats[bmg::kStNvis];
    counters->walk_steps = (int64_t)ctl.stats[bmg::kStSteps];
    counters->frontier_entries = (int64_t)ctl.stats[bmg::kStEntries];
    counters->cardinality = ctl.card;
    counters->initial_cardinality = ctl.init_card;
    counters->n_phase_records = (int64_t)recs.size();
  }
  if (!ctl.done) return fail(BM_ERR_CUDA, "the run stopped before the maximum (phase records exhausted)");
  return BM_OK;
}

bm_status bm_mg_run(bm_mg* h, const bm_match_opts* o, int64_t* cardinality, bm_counters* counters) {
  bm_status s = bm_mg_launch(h, o);
  if (s != BM_OK) return s;
  return bm_mg_finish(h, cardinality, counters);
}

bm_status bm_mg_download(bm_mg* h, int32_t* rmatch_slice, int32_t* cmatch_slice) {
  if (!h) return fail(BM_ERR_INVALID_ARG, "null handle");
  BM_CUDA(cudaSetDevice(h->device));
  const int ncl = h->chi - h->clo, nrl = h->rhi - h->rlo;
  if (cmatch_slice && ncl)
    BM_CUDA(cudaMemcpyAsync(cmatch_slice, h->cmatch, sizeof(int) * ncl, cudaMemcpyDeviceToHost, h->stream));
  if (rmatch_slice && nrl) {
    bmg::rows_unpack_kernel<<<std::max(1, std::min(h->sms * 8, (nrl + 255) / 256)), 256, 0, h->stream>>>(
        h->rm, h->rtmp, nrl, h->rs);
    BM_CUDA(cudaGetLastError());
    BM_CUDA(cudaMemcpyAsync(rmatch_slice, h->rtmp, sizeof(int) * nrl, cudaMemcpyDeviceToHost, h->stream));
  }
  BM_CUDA(cudaStreamSynchronize(h->stream));
  return BM_OK;
}

bm_status bm_mg_kernel_time(bm_mg* h, double* ms) {
  if (!h || !ms) return fail(BM_ERR_INVALID_ARG, "null argument");
  *ms = h->last_ms;
  return BM_OK;
}

bm_status bm_mg_info(bm_mg* h, int64_t* local_edges, int64_t* row_index_edges, int32_t* pulled_capable) {
  if (!h) return fail(BM_ERR_INVALID_ARG, "null handle");
  if (local_edges) *local_edges = h->E;
  if (row_index_edges) *row_index_edges = h->inbox_n;
  if (pulled_capable) *pulled_capable = h->row_index ? 1 : 0;
  return BM_OK;
}

}  // extern "C"
