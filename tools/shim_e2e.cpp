// shim_e2e.cpp — end-to-end time of the real drop-in path: the reference's
// C++ types (bmatch::BipartiteCsr / MatchingState, std::vector storage, i.e.
// pageable host memory) handed to bmatch::b200::apfb (include/bmatch_b200.hpp),
// which uploads, matches and downloads through the C ABI on every call — what a
// caller of the reference's registry pays. Wall clock per call, after warm-up.
//
// usage: shim_e2e <C2|C5> [reps]   prints one JSON line
//   C2: planted 10M x 10M, degree 16, seed 2024 (bench.py's C2)
//   C5: uniform 100M x 100M, degree 16, seed 5 (the reference's generator)
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "bmatch/csr_graph.hpp"
#include "bmatch/matching.hpp"
#include "bmatch_b200.hpp"
#include "bmatch_b200_gen.h"

using namespace bmatch;

int main(int argc, char** argv) {
  const std::string cfg = argc > 1 ? argv[1] : "C2";
  const int reps = argc > 2 ? std::max(1, atoi(argv[2])) : 5;
  BipartiteCsr g;
  int64_t ne = 0;
  if (cfg == "C2") {
    const int n = 10000000;
    g.nc = g.nr = n;
    g.cxadj.resize((size_t)n + 1);
    g.cadj.resize((size_t)bm_gen_planted_capacity(n, 16.0));
    if (bm_gen_planted(n, 16.0, 2024, 0, g.cxadj.data(), g.cadj.data(), &ne) != BM_OK) return 2;
  } else if (cfg == "C5") {
    const int n = 100000000;
    g.nc = g.nr = n;
    g.cxadj.resize((size_t)n + 1);
    g.cadj.resize((size_t)bm_gen_uniform_capacity(n, 16.0));
    if (bm_gen_uniform(n, n, 16.0, 5, 0, g.cxadj.data(), g.cadj.data(), &ne) != BM_OK) return 2;
  } else {
    fprintf(stderr, "unknown config %s\n", cfg.c_str());
    return 1;
  }
  g.cadj.resize((size_t)ne);
  g.name = cfg;
  const MatchingState init = cheap_matching(g);  // the reference's first-fit (matching.cpp:13-26)
  std::vector<double> ms;
  long long card = 0;
  for (int i = 0; i < reps + 1; ++i) {
    MatchingState m = init;  // (the copy is outside the timed call, as the caller owns it)
    const auto t0 = std::chrono::steady_clock::now();
    DriverResult r = b200::apfb(g, std::move(m), GridConfig{}, Schedule::parallel(), BfsKernel::GpubfsWr);
    const auto t1 = std::chrono::steady_clock::now();
    card = cardinality(r.matching);
    if (i) ms.push_back(std::chrono::duration<double, std::milli>(t1 - t0).count());
  }
  std::sort(ms.begin(), ms.end());
  double mean = 0;
  for (double x : ms) mean += x;
  mean /= (double)ms.size();
  printf("{\"config\": \"%s\", \"edges\": %lld, \"reps\": %d, \"ms_mean\": %.3f, \"ms_median\": %.3f, "
         "\"ms_min\": %.3f, \"cardinality\": %lld, \"path\": \"bmatch::b200::apfb from std::vector (pageable)\"}\n",
         cfg.c_str(), (long long)ne, reps, mean, ms[ms.size() / 2], ms.front(), card);
  return 0;
}
