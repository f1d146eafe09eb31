// bm_host.cpp — parallel host-side CSC builders, synthetic generators and
// small host utilities. Not on the matching hot path.
//
// Every generator funnels into one builder: edges are produced chunk by
// chunk (twice: once to count column degrees, once to scatter rows), then
// each column is sorted and de-duplicated, which is exactly the result of the
// reference's from_edge_list (csr_graph.cpp:10-43: sort pairs, unique, CSC).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "bmatch_b200.h"
#include "bmatch_b200_gen.h"
#include "bm_host_util.hpp"

namespace {

using namespace bm_host;

inline uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

// Counter-based stream: value k of stream s under seed.
struct Stream {
  uint64_t key;
  Stream(uint64_t seed, uint64_t s) : key(splitmix64(seed * 0x2545f4914f6cdd1dULL + s)) {}
  uint64_t operator()(uint64_t k) const { return splitmix64(key ^ splitmix64(k)); }
  static uint32_t below(uint64_t v, uint32_t n) { return (uint32_t)(((v >> 32) * (uint64_t)n) >> 32); }
  static double unit(uint64_t v) { return (double)(v >> 11) * (1.0 / 9007199254740992.0); }
};

// Keyed bijection on [0, n): a 4-round Feistel network on 2*hb bits with
// cycle walking (the domain is at most 4n, so ~<4 rounds of walking).
struct Perm {
  uint64_t n = 0;
  int hb = 0;
  uint64_t mask = 0;
  uint64_t keys[4] = {0, 0, 0, 0};
  Perm(uint64_t n_, uint64_t seed) : n(n_) {
    int bits = 1;
    while ((1ULL << bits) < n) ++bits;
    hb = (bits + 1) / 2;
    mask = (1ULL << hb) - 1;
    for (int i = 0; i < 4; ++i) keys[i] = splitmix64(seed * 0x9e3779b97f4a7c15ULL + 0x1234567ULL * (i + 1));
  }
  uint64_t round(uint64_t x) const {
    uint64_t L = x >> hb, R = x & mask;
    for (int i = 0; i < 4; ++i) {
      const uint64_t F = splitmix64(R ^ keys[i]) & mask;
      const uint64_t nl = R;
      R = L ^ F;
      L = nl;
    }
    return (L << hb) | R;
  }
  uint64_t operator()(uint64_t x) const {
    if (n <= 1) return x;
    do {
      x = round(x);
    } while (x >= n);
    return x;
  }
};

}  // namespace

extern "C" {

int64_t bm_gen_uniform_capacity(int32_t nc, double avg_degree) {
  if (nc <= 0 || avg_degree <= 0) return 0;
  return std::llround(nc * avg_degree);
}

bm_status bm_gen_uniform(int32_t nc, int32_t nr, double avg_degree, uint64_t seed, int32_t threads,
                         int64_t* cxadj, int32_t* cadj, int64_t* nedges) {
  if (nc < 0 || nr < 0 || !cxadj || !nedges) return hfail(BM_ERR_INVALID_ARG, "bad arguments");
  *nedges = 0;
  if (nc <= 0 || nr <= 0 || avg_degree <= 0) {  // csr_graph.cpp:96-99
    std::memset(cxadj, 0, sizeof(int64_t) * ((size_t)std::max(nc, 0) + 1));
    return BM_OK;
  }
  const long long K = std::llround(nc * avg_degree);
  const int T = resolve_threads(threads);
  // Replay points of the single mt19937_64 stream (csr_graph.cpp:101-109).
  const long long chunks = std::max<long long>(1, std::min<long long>((long long)T * 8, (K + 65535) / 65536));
  std::vector<std::mt19937_64> snaps;
  snaps.reserve(chunks);
  {
    std::mt19937_64 rng(seed);
    std::uniform_int_distribution<int> col_pick(0, nc - 1);
    std::uniform_int_distribution<int> row_pick(0, nr - 1);
    for (long long ch = 0; ch < chunks; ++ch) {
      snaps.push_back(rng);
      const long long b = K * ch / chunks, e = K * (ch + 1) / chunks;
      for (long long k = b; k < e; ++k) {
        (void)col_pick(rng);
        (void)row_pick(rng);
      }
    }
  }
  auto produce = [&](long long ch, auto&& emit) {
    std::mt19937_64 rng = snaps[ch];
    std::uniform_int_distribution<int> col_pick(0, nc - 1);
    std::uniform_int_distribution<int> row_pick(0, nr - 1);
    const long long b = K * ch / chunks, e = K * (ch + 1) / chunks;
    for (long long k = b; k < e; ++k) {
      const int c = col_pick(rng);
      const int r = row_pick(rng);
      emit(c, r);
    }
  };
  return build_csc(nc, nr, chunks, T, K, produce, cxadj, cadj, nedges);
}

int64_t bm_gen_planted_capacity(int32_t n, double avg_degree) {
  if (n <= 0) return 0;
  return (int64_t)n + std::max<long long>(0, std::llround((avg_degree - 1.0) * n));
}

bm_status bm_gen_planted(int32_t n, double avg_degree, uint64_t seed, int32_t threads, int64_t* cxadj,
                         int32_t* cadj, int64_t* nedges) {
  if (n < 0 || !cxadj || !nedges) return hfail(BM_ERR_INVALID_ARG, "bad arguments");
  *nedges = 0;
  if (n == 0) {
    cxadj[0] = 0;
    return BM_OK;
  }
  const long long K = bm_gen_planted_capacity(n, avg_degree);
  const int T = resolve_threads(threads);
  const Perm pi((uint64_t)n, seed ^ 0x51ed270b27a4c3f1ULL);
  const Stream sc(seed, 1), sr(seed, 2);
  const long long chunk = 1 << 16;
  const long long chunks = (K + chunk - 1) / chunk;
  auto produce = [&](long long ch, auto&& emit) {
    const long long b = ch * chunk, e = std::min<long long>(K, b + chunk);
    for (long long k = b; k < e; ++k) {
      if (k < n) {
        emit((int)k, (int)pi((uint64_t)k));
      } else {
        emit((int)Stream::below(sc((uint64_t)k), (uint32_t)n), (int)Stream::below(sr((uint64_t)k), (uint32_t)n));
      }
    }
  };
  return build_csc(n, n, chunks, T, K, produce, cxadj, cadj, nedges);
}

int64_t bm_gen_rmat_capacity(int32_t scale, double edge_factor) {
  if (scale < 0 || scale > 30) return 0;
  return std::llround(edge_factor * (double)(1LL << scale));
}

bm_status bm_gen_rmat(int32_t scale, double edge_factor, double a, double b, double c, uint64_t seed,
                      int32_t permute, int32_t threads, int64_t* cxadj, int32_t* cadj, int64_t* nedges) {
  if (scale < 0 || scale > 30 || !cxadj || !nedges) return hfail(BM_ERR_INVALID_ARG, "bad arguments");
  if (a < 0 || b < 0 || c < 0 || a + b + c > 1.0) return hfail(BM_ERR_INVALID_ARG, "bad R-MAT probabilities");
  const int n = 1 << scale;
  const long long K = bm_gen_rmat_capacity(scale, edge_factor);
  const int T = resolve_threads(threads);
  const Perm pc((uint64_t)n, seed ^ 0xc0ffee1234567ULL), pr((uint64_t)n, seed ^ 0xbadc0de987654ULL);
  const Stream s(seed, 3);
  const double ab = a + b, abc = a + b + c;
  const long long chunk = 1 << 15;
  const long long chunks = std::max<long long>(1, (K + chunk - 1) / chunk);
  auto produce = [&](long long ch, auto&& emit) {
    const long long b0 = ch * chunk, e0 = std::min<long long>(K, b0 + chunk);
    for (long long k = b0; k < e0; ++k) {
      uint32_t r = 0, cc = 0;
      for (int l = 0; l < scale; ++l) {
        const double u = Stream::unit(s((uint64_t)k * (uint64_t)scale + (uint64_t)l));
        const int q = u < a ? 0 : (u < ab ? 1 : (u < abc ? 2 : 3));
        r = (r << 1) | (uint32_t)(q >> 1);
        cc = (cc << 1) | (uint32_t)(q & 1);
      }
      if (permute) emit((int)pc(cc), (int)pr(r));
      else emit((int)cc, (int)r);
    }
  };
  return build_csc(n, n, chunks, T, K, produce, cxadj, cadj, nedges);
}

int64_t bm_gen_banded_capacity(int32_t n, int32_t band) {
  if (n <= 0 || band <= 0) return 0;
  return (int64_t)n * band;
}

bm_status bm_gen_banded(int32_t n, int32_t band, double delete_frac, uint64_t seed, int32_t permute,
                        int32_t threads, int64_t* cxadj, int32_t* cadj, int64_t* nedges, int64_t* live_rows) {
  if (n < 0 || band <= 0 || !cxadj || !nedges) return hfail(BM_ERR_INVALID_ARG, "bad arguments");
  *nedges = 0;
  const int T = resolve_threads(threads);
  const Stream sd(seed, 4);
  auto dead = [&](long long r) { return Stream::unit(sd((uint64_t)r)) < delete_frac; };
  if (live_rows) {
    std::atomic<long long> live{0};
    parallel_for(n, T, [&](long long b, long long e, int) {
      long long l = 0;
      for (long long r = b; r < e; ++r) l += !dead(r);
      live.fetch_add(l);
    });
    *live_rows = live.load();
  }
  if (n == 0) {
    cxadj[0] = 0;
    return BM_OK;
  }
  const Perm pc((uint64_t)n, seed ^ 0x7777aaaa5555ULL), pr((uint64_t)n, seed ^ 0x3333cccc9999ULL);
  const long long K = (long long)n * band;
  const long long chunk = 1 << 16;
  const long long chunks = (K + chunk - 1) / chunk;
  auto produce = [&](long long ch, auto&& emit) {
    const long long b = ch * chunk, e = std::min<long long>(K, b + chunk);
    for (long long k = b; k < e; ++k) {
      const long long c = k / band, r = c + k % band;
      if (r >= n || dead(r)) continue;
      if (permute) emit((int)pc((uint64_t)c), (int)pr((uint64_t)r));
      else emit((int)c, (int)r);
    }
  };
  return build_csc(n, n, chunks, T, K, produce, cxadj, cadj, nedges);
}

bm_status bm_check_csc(int32_t nc, int32_t nr, const int64_t* cxadj, const int32_t* cadj) {
  return check_csc_mt(nc, nr, cxadj, cadj, 0);
}

uint64_t bm_csc_digest(int32_t nc, int32_t nr, const int64_t* cxadj, const int32_t* cadj) {
  uint64_t h = 1469598103934665603ULL;
  auto mix = [&](uint64_t v) {
    h ^= v;
    h *= 1099511628211ULL;
  };
  mix((uint64_t)(uint32_t)nc);
  mix((uint64_t)(uint32_t)nr);
  if (!cxadj) return h;
  for (long long c = 0; c <= nc; ++c) mix((uint64_t)cxadj[c]);
  const int64_t E = cxadj[nc];
  for (int64_t j = 0; j < E; ++j) mix((uint64_t)(uint32_t)cadj[j]);
  return h;
}

bm_status bm_host_cheap_matching(int32_t nc, int32_t nr, const int64_t* cxadj, const int32_t* cadj,
                                 int32_t* rmatch, int32_t* cmatch) {
  if (nc < 0 || nr < 0 || !cxadj || (!rmatch && nr > 0) || (!cmatch && nc > 0))
    return hfail(BM_ERR_INVALID_ARG, "bad arguments");
  for (int r = 0; r < nr; ++r) rmatch[r] = -1;
  for (int c = 0; c < nc; ++c) {
    cmatch[c] = -1;
    for (int64_t j = cxadj[c]; j < cxadj[c + 1]; ++j) {
      const int r = cadj[j];
      if (rmatch[r] < 0) {
        rmatch[r] = c;
        cmatch[c] = r;
        break;
      }
    }
  }
  return BM_OK;
}

}  // extern "C"

extern "C" bm_status bm_permutation_pair(int32_t nc, int32_t nr, uint64_t seed, int32_t* cperm, int32_t* rperm) {
  // random_permutation + permute_random's draw order (csr_graph.cpp:68-90): columns
  // first, then rows, from one mt19937_64 seeded with `seed`; Fisher-Yates from
  // the top with uniform_int_distribution<int>(0, i) (libstdc++, as the reference).
  if (nc < 0 || nr < 0) return hfail(BM_ERR_INVALID_ARG, "negative size");
  if ((nc > 0 && !cperm) || (nr > 0 && !rperm)) return hfail(BM_ERR_INVALID_ARG, "null permutation buffer");
  std::mt19937_64 rng(seed);
  auto fill = [&rng](int32_t n, int32_t* perm) {
    for (int32_t i = 0; i < n; ++i) perm[i] = i;
    for (int32_t i = n - 1; i > 0; --i) {
      std::uniform_int_distribution<int> pick(0, i);
      std::swap(perm[i], perm[pick(rng)]);
    }
  };
  fill(nc, cperm);
  fill(nr, rperm);
  return BM_OK;
}

