// b200_suite.cpp — the paper's evaluation artefacts (Table 1 geomeans, the
// speedup and performance profiles of Figs. 3-4) produced
// by the REFERENCE's own suite runner with the B200 ids registered beside its
// CPU algorithms. Built by `make suite` where the
// reference sources exist; links the reference library and the engine.
//
// usage: b200_suite <out_dir> [reps]
//   writes <out_dir>/{original,rcp}_records.{csv,json}, *_geomean.csv,
//   *_speedup_<algo>.csv (vs the fastest CPU algorithm per instance, as the
//   paper does) and *_performance_profile.csv, and prints a summary.
//
// Instances: synthetic graphs of the BASELINE families at suite-friendly
// sizes (the reference suite reads Matrix Market text, so instances are kept
// to a few million edges), written under <out_dir>/instances. The "rcp" pass
// is the paper's random row/column permutation (run_suite's permute_seed).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <map>
#include <string>
#include <vector>

#include "bmatch/algorithms.hpp"
#include "bmatch/bench.hpp"
#include "bmatch/csr_graph.hpp"
#include "bmatch/matrix_market.hpp"
#include "bmatch_b200.hpp"
#include "bmatch_b200_gen.h"

using namespace bmatch;
namespace fs = std::filesystem;

namespace {

using GenFn = bm_status (*)(int64_t*, int32_t*, int64_t*);

BipartiteCsr from_generator(int nc, int nr, int64_t capacity, const std::string& name,
                            const std::function<bm_status(int64_t*, int32_t*, int64_t*)>& gen) {
  BipartiteCsr g;
  g.nc = nc;
  g.nr = nr;
  g.name = name;
  g.cxadj.assign((size_t)nc + 1, 0);
  g.cadj.assign((size_t)capacity, 0);
  int64_t ne = 0;
  b200::throw_on(gen(g.cxadj.data(), g.cadj.data(), &ne));
  g.cadj.resize((size_t)ne);
  return g;
}

std::vector<BipartiteCsr> instances() {
  std::vector<BipartiteCsr> gs;
  for (auto [n, d, s] : std::vector<std::tuple<int, double, uint64_t>>{{200000, 4.0, 1}, {500000, 8.0, 2}, {1000000, 3.0, 3}})
    gs.push_back(from_generator(n, n, bm_gen_uniform_capacity(n, d), "uniform-" + std::to_string(n) + "-d" + std::to_string((int)d),
                                [=](int64_t* cx, int32_t* a, int64_t* ne) { return bm_gen_uniform(n, n, d, s, 0, cx, a, ne); }));
  for (auto [n, d] : std::vector<std::pair<int, double>>{{300000, 4.0}, {1000000, 8.0}})
    gs.push_back(from_generator(n, n, bm_gen_planted_capacity(n, d), "planted-" + std::to_string(n) + "-d" + std::to_string((int)d),
                                [=](int64_t* cx, int32_t* a, int64_t* ne) { return bm_gen_planted(n, d, 7, 0, cx, a, ne); }));
  for (int sc : {16, 18})
    gs.push_back(from_generator(1 << sc, 1 << sc, bm_gen_rmat_capacity(sc, 8.0), "rmat-" + std::to_string(sc),
                                [=](int64_t* cx, int32_t* a, int64_t* ne) {
                                  return bm_gen_rmat(sc, 8.0, 0.57, 0.19, 0.19, 11, 0, 0, cx, a, ne);
                                }));
  for (int n : {300000, 1000000}) {
    int64_t live = 0;
    gs.push_back(from_generator(n, n, bm_gen_banded_capacity(n, 3), "band3-" + std::to_string(n),
                                [&, n](int64_t* cx, int32_t* a, int64_t* ne) {
                                  return bm_gen_banded(n, 3, 0.05, 13, 0, 0, cx, a, ne, &live);
                                }));
  }
  return gs;
}

template <typename T>
void write_csv(const fs::path& p, const std::string& header, const std::vector<T>& rows) {
  std::ofstream out(p);
  out << header << "\n";
  for (const auto& r : rows) out << r << "\n";
}

void report(const std::string& tag, const SuiteResult& res, const std::vector<std::string>& algos,
            const std::vector<std::string>& cpu, const fs::path& out) {
  {
    std::ofstream f(out / (tag + "_records.csv"));
    write_records_csv(res.records, f);
    std::ofstream j(out / (tag + "_records.json"));
    write_records_json(res.records, j);
  }
  // Table 1 analogue: geometric mean time per algorithm
  std::vector<std::string> geo;
  std::map<std::string, double> gm;
  for (const auto& a : algos) {
    std::vector<double> t;
    for (const auto& r : res.records)
      if (r.algorithm == a) t.push_back(std::max(r.time_s, 1e-9));
    gm[a] = geometric_mean(t);
    char buf[160];
    std::snprintf(buf, sizeof buf, "%s,%.6g", a.c_str(), gm[a]);
    geo.push_back(buf);
  }
  write_csv(out / (tag + "_geomean.csv"), "algorithm,geomean_s", geo);
  // Figs. 3-4 analogue: speedup of each B200 id over the fastest CPU algorithm per instance
  std::vector<BenchRecord> with_best = res.records;
  std::map<std::string, double> best;
  for (const auto& r : res.records)
    if (std::find(cpu.begin(), cpu.end(), r.algorithm) != cpu.end())
      best[r.instance] = best.count(r.instance) ? std::min(best[r.instance], r.time_s) : r.time_s;
  for (const auto& [inst, t] : best) {
    BenchRecord b;
    b.instance = inst;
    b.algorithm = "best-cpu";
    b.time_s = t;
    with_best.push_back(b);
  }
  std::vector<double> grid;
  for (int i = -2; i <= 16; ++i) grid.push_back(i * 0.5);
  std::printf("\n[%s] geometric mean time (s) over %zu instances\n", tag.c_str(), best.size());
  for (const auto& a : algos) std::printf("  %-14s %10.5f\n", a.c_str(), gm[a]);
  for (const auto& a : algos) {
    if (a.find("b200") == std::string::npos) continue;
    const auto prof = speedup_profile(with_best, "best-cpu", a, grid);
    std::vector<std::string> rows;
    for (const auto& pt : prof) {
      char buf[96];
      std::snprintf(buf, sizeof buf, "%.2f,%.4f", pt.x, pt.y);
      rows.push_back(buf);
    }
    write_csv(out / (tag + "_speedup_" + a + ".csv"), "log2_speedup_at_least,fraction_of_instances", rows);
    double lg = 0;
    int n = 0;
    for (const auto& r : res.records)
      if (r.algorithm == a && best.count(r.instance)) {
        lg += std::log(best[r.instance] / std::max(r.time_s, 1e-9));
        ++n;
      }
    std::printf("  %s vs fastest CPU algorithm per instance: geometric-mean speedup %.1fx\n", a.c_str(),
                n ? std::exp(lg / n) : 0.0);
  }
  const auto perf = performance_profile(res.records, algos);
  std::vector<std::string> rows;
  for (const auto& [a, pts] : perf)
    for (const auto& pt : pts) {
      char buf[160];
      std::snprintf(buf, sizeof buf, "%s,%.6g,%.4f", a.c_str(), pt.x, pt.y);
      rows.push_back(buf);
    }
  write_csv(out / (tag + "_performance_profile.csv"), "algorithm,ratio_to_best,fraction_of_instances", rows);
  std::printf("  cardinality mismatches across algorithms: %zu\n", res.mismatches.size());
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: %s <out_dir> [reps]\n", argv[0]);
    return 2;
  }
  const fs::path out = argv[1];
  const int reps = argc > 2 ? std::atoi(argv[2]) : 3;
  fs::create_directories(out / "instances");
  std::vector<std::string> paths;
  for (const BipartiteCsr& g : instances()) {
    const fs::path p = out / "instances" / (g.name + ".mtx");
    std::ofstream f(p);
    write_matrix_market(g, f);
    paths.push_back(p.string());
  }
  b200::register_algorithms();
  const std::vector<std::string> cpu = {"hk", "pfp", "apfb-wr-ct", "apsb-wr-ct"};
  std::vector<std::string> algos = cpu;
  for (const char* a : {"apfb-wr-b200", "apsb-wr-b200", "apfb-gpubfs-b200"}) algos.push_back(a);
  SuiteOptions opt;
  opt.repetitions = reps;
  opt.schedule = Schedule::parallel();  // the reference's own grid algorithms on every host core
  bool ok = true;
  for (int pass = 0; pass < 2; ++pass) {
    if (pass == 1) opt.permute_seed = 2024;  // RCP: random row/column permutation
    const SuiteResult res = run_suite(paths, algos, opt);
    ok = ok && res.ok() && res.load_errors.empty();
    report(pass ? "rcp" : "original", res, algos, cpu, out);
  }
  std::printf("\n%s\n", ok ? "SUITE OK (no cardinality mismatch)" : "SUITE FAILED");
  return ok ? 0 : 1;
}
