// bm_host_util.hpp — internal helpers shared by the host-side translation
// units (bm_host.cpp: generators; bm_io.cpp: file ingest): a thread pool-free
// parallel loop, and the one sorted + de-duplicated CSC builder every host
// producer funnels into (the result of the reference's from_edge_list,
// csr_graph.cpp:10-43). Not part of the C ABI.
#pragma once

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "bmatch_b200.h"

void bm_internal_set_error(const std::string& msg);  // bm_engine.cu

namespace bm_host {

inline bm_status hfail(bm_status s, const std::string& m) {
  bm_internal_set_error(m);
  return s;
}

inline int resolve_threads(int t) {
  if (t > 0) return t;
  const unsigned hc = std::thread::hardware_concurrency();
  return hc ? (int)hc : 1;
}

template <typename F>
void parallel_for(long long n, int threads, F&& fn) {  // fn(begin, end, worker)
  if (n <= 0) return;
  threads = (int)std::max<long long>(1, std::min<long long>(threads, n));
  if (threads == 1) {
    fn(0LL, n, 0);
    return;
  }
  std::vector<std::thread> pool;
  pool.reserve(threads);
  for (int w = 0; w < threads; ++w) {
    const long long b = n * w / threads, e = n * (w + 1) / threads;
    pool.emplace_back([&, b, e, w] { fn(b, e, w); });
  }
  for (auto& t : pool) t.join();
}

// Dynamic-chunk parallel loop over [0, chunks).
template <typename F>
void parallel_chunks(long long chunks, int threads, F&& fn) {
  std::atomic<long long> next{0};
  parallel_for(threads, threads, [&](long long, long long, int) {
    for (;;) {
      const long long c = next.fetch_add(1);
      if (c >= chunks) break;
      fn(c);
    }
  });
}

// Builds a sorted, de-duplicated CSC from a chunked edge producer.
// produce(chunk, emit) must call emit(c, r) for the same edges every time it
// is called with the same chunk.
template <typename Produce>
bm_status build_csc(int nc, int nr, long long chunks, int threads, long long capacity, Produce&& produce,
                    int64_t* cxadj, int32_t* cadj, int64_t* nedges) {
  (void)nr;
  std::memset(cxadj, 0, sizeof(int64_t) * ((size_t)nc + 1));
  // Pass 1: degrees into cxadj[c + 1].
  std::atomic<long long> total{0};
  parallel_chunks(chunks, threads, [&](long long ch) {
    long long local = 0;
    produce(ch, [&](int c, int) {
      __atomic_fetch_add(&cxadj[c + 1], 1, __ATOMIC_RELAXED);
      ++local;
    });
    total.fetch_add(local);
  });
  if (total.load() > capacity) return hfail(BM_ERR_INVALID_ARG, "generator exceeded its capacity");
  // Exclusive prefix shifted by one: cxadj[c+1] = start of column c.
  {
    int64_t run = 0;
    for (long long c = 0; c < nc; ++c) {
      const int64_t d = cxadj[c + 1];
      cxadj[c + 1] = run;
      run += d;
    }
  }
  // Pass 2: scatter; afterwards cxadj[c+1] = end of column c.
  parallel_chunks(chunks, threads, [&](long long ch) {
    produce(ch, [&](int c, int r) {
      const int64_t pos = __atomic_fetch_add(&cxadj[c + 1], 1, __ATOMIC_RELAXED);
      cadj[pos] = r;
    });
  });
  // Per-column sort + unique; new degrees into a temporary.
  std::vector<int32_t> ndeg((size_t)std::max(nc, 1));
  parallel_chunks((nc + 4095) / 4096, threads, [&](long long ch) {
    const long long c0 = ch * 4096, c1 = std::min<long long>(nc, c0 + 4096);
    for (long long c = c0; c < c1; ++c) {
      int32_t* b = cadj + cxadj[c];
      int32_t* e = cadj + cxadj[c + 1];
      std::sort(b, e);
      ndeg[c] = (int32_t)(std::unique(b, e) - b);
    }
  });
  // Compaction (left moves only, so a sequential sweep is safe). On entry to
  // iteration c, cxadj[c] still holds the raw end of column c-1 = the raw
  // start of column c; it is then overwritten with the compacted start.
  int64_t w = 0;
  for (long long c = 0; c < nc; ++c) {
    const int64_t b = cxadj[c];  // start of column c in the raw layout
    const int32_t d = ndeg[c];
    if (w != b && d > 0) std::memmove(cadj + w, cadj + b, sizeof(int32_t) * (size_t)d);
    cxadj[c] = w;
    w += d;
  }
  cxadj[nc] = w;
  *nedges = w;
  return BM_OK;
}

}  // namespace bm_host

namespace bm_host {

// The CSC invariants of check_csr (csr_graph.cpp:45-64) on every host core,
// reporting the first failing column in column order with bm_check_csc's
// messages. Offsets are checked first so a malformed array never drives an
// out-of-bounds read of cadj.
inline bm_status check_csc_mt(int32_t nc, int32_t nr, const int64_t* cxadj, const int32_t* cadj, int threads) {
  if (nc < 0 || nr < 0) return hfail(BM_ERR_INVALID_ARG, "negative vertex count");
  if (!cxadj) return hfail(BM_ERR_INVALID_ARG, "null cxadj");
  if (cxadj[0] != 0) return hfail(BM_ERR_INVALID_ARG, "cxadj[0] is not 0");
  threads = resolve_threads(threads);
  const long long blk = 1 << 16, nblk = ((long long)nc + blk - 1) / blk;
  std::atomic<long long> first{nc};
  auto lower = [&](long long c) {
    long long cur = first.load(std::memory_order_relaxed);
    while (c < cur && !first.compare_exchange_weak(cur, c)) {
    }
  };
  parallel_chunks(nblk, threads, [&](long long b) {
    const long long c0 = b * blk, c1 = std::min<long long>(nc, c0 + blk);
    for (long long c = c0; c < c1 && c < first.load(std::memory_order_relaxed); ++c)
      if (cxadj[c] > cxadj[c + 1]) {
        lower(c);
        break;
      }
  });
  if (first.load() < nc) return hfail(BM_ERR_INVALID_ARG, "cxadj decreases at column " + std::to_string(first.load()));
  if (nc > 0 && cxadj[nc] > 0 && !cadj) return hfail(BM_ERR_INVALID_ARG, "null cadj");
  parallel_chunks(nblk, threads, [&](long long b) {
    const long long c0 = b * blk, c1 = std::min<long long>(nc, c0 + blk);
    for (long long c = c0; c < c1 && c < first.load(std::memory_order_relaxed); ++c) {
      bool bad = false;
      for (int64_t j = cxadj[c]; j < cxadj[c + 1] && !bad; ++j)
        bad = cadj[j] < 0 || cadj[j] >= nr || (j > cxadj[c] && cadj[j - 1] >= cadj[j]);
      if (bad) {
        lower(c);
        break;
      }
    }
  });
  const long long c = first.load();
  if (c < nc) {
    for (int64_t j = cxadj[c]; j < cxadj[c + 1]; ++j) {  // the serial check's message for column c
      if (cadj[j] < 0 || cadj[j] >= nr)
        return hfail(BM_ERR_INVALID_ARG, "row index out of range in column " + std::to_string(c));
      if (j > cxadj[c] && cadj[j - 1] >= cadj[j])
        return hfail(BM_ERR_INVALID_ARG, "column " + std::to_string(c) + " slice is not strictly ascending");
    }
  }
  return BM_OK;
}

}  // namespace bm_host
