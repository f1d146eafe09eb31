// shim_test.cpp — drop-in test of include/bmatch_b200.hpp against the
// REFERENCE's own C++ API (test infrastructure; built by `make shimtest` into
// oracle/_ref/ where /root/reference exists, and run by tests/test_shim.py).
//
// It links the reference library compiled unmodified from its sources
// (oracle/_ref/libbmatch_ref.so) and the B200 engine, registers the B200 ids
// through bmatch::register_algorithm, and then drives them exactly as the
// reference's callers do:
//   * make_algorithm(id)(g, init, schedule)        (algorithms.cpp:64-93)
//   * bmatch::b200::apfb / apsb with an observer   (gpu_match.hpp:133-144)
//   * run_suite over Matrix Market files, whose built-in cardinality-mismatch
//     gate compares every id with hk                (bench.cpp:28-76)
// Every output must pass the reference's validate + is_maximum
// (matching.cpp:70-131) and match hopcroft_karp's cardinality.
//
// usage: shim_test            (GPU present: full run; prints "PASS <n checks>")
//        shim_test --no-gpu   (expects every B200 call to throw: no CPU fallback)
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "bmatch/algorithms.hpp"
#include "bmatch/baselines.hpp"
#include "bmatch/bench.hpp"
#include "bmatch/csr_graph.hpp"
#include "bmatch/matrix_market.hpp"
#include "bmatch_b200.hpp"

using namespace bmatch;

static int g_checks = 0;
#define CHECK(cond)                                                              \
  do {                                                                           \
    ++g_checks;                                                                  \
    if (!(cond)) {                                                               \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);      \
      std::exit(1);                                                              \
    }                                                                            \
  } while (0)

static BipartiteCsr fork_graph() {  // paper Fig. 1 (tests/oracles.hpp:59-61)
  return from_edge_list(2, 3, {{0, 0}, {1, 0}, {1, 1}, {1, 2}}, "fork");
}

static BipartiteCsr complete_graph(int nc, int nr) {
  std::vector<Edge> e;
  for (int c = 0; c < nc; ++c)
    for (int r = 0; r < nr; ++r) e.push_back({c, r});
  return from_edge_list(nc, nr, e, "complete");
}

static std::vector<BipartiteCsr> corpus() {
  std::vector<BipartiteCsr> gs;
  gs.push_back(from_edge_list(0, 0, {}, "empty"));
  gs.push_back(from_edge_list(5, 4, {}, "edgeless"));
  gs.push_back(fork_graph());
  gs.push_back(complete_graph(12, 9));
  const int sizes[][2] = {{1, 1}, {7, 5}, {20, 31}, {64, 64}, {200, 150}, {1000, 1000}, {5000, 4000}};
  const double degs[] = {1.0, 2.0, 4.0, 8.0};
  std::uint64_t seed = 11;
  for (auto& s : sizes)
    for (double d : degs) gs.push_back(generate_random_bipartite(s[0], s[1], d, seed++));
  gs.push_back(permute_random(generate_random_bipartite(100000, 100000, 8.0, 1), 5));
  return gs;
}

static void check_result(const BipartiteCsr& g, const MatchingState& m, long long want) {
  CHECK(validate(g, m).ok());
  CHECK(is_maximum(g, m));
  CHECK(cardinality(m) == want);
}

int main(int argc, char** argv) {
  const bool no_gpu = argc > 1 && std::string(argv[1]) == "--no-gpu";
  b200::register_algorithms();
  for (const char* id : {"apfb-wr-b200", "apfb-gpubfs-b200", "apsb-wr-b200", "apsb-gpubfs-b200"})
    CHECK(make_algorithm(id).has_value());

  // 0. file I/O drop-ins (host only, so they run with or without a GPU):
  //    the parallel reader must rebuild exactly what the reference wrote and
  //    read, and raise the reference's ParseError with its line number.
  {
    namespace fs = std::filesystem;
    const fs::path p = fs::temp_directory_path() / "bmatch_b200_shim_io.mtx";
    const BipartiteCsr g = generate_random_bipartite(5000, 4000, 3.0, 8);
    {
      std::ofstream out(p);
      write_matrix_market(g, out);
    }
    const BipartiteCsr mine = b200::load_matrix_market(p.string(), 4);
    const BipartiteCsr theirs = load_matrix_market(p.string());
    CHECK(mine.nc == theirs.nc && mine.nr == theirs.nr && mine.name == theirs.name);
    CHECK(mine.cxadj == theirs.cxadj && mine.cadj == theirs.cadj);
    b200::write_matrix_market(g, p.string());
    CHECK(load_matrix_market(p.string()).cadj == g.cadj);
    b200::save_csc(g, p.string() + ".bcsc");
    CHECK(b200::load_csc(p.string() + ".bcsc").cadj == g.cadj);
    fs::remove(p);
    fs::remove(p.string() + ".bcsc");
    long long line = 0;
    std::string what;
    try {
      b200::read_matrix_market("%%MatrixMarket matrix coordinate pattern general\n2 2 1\n3 1\n");
    } catch (const ParseError& e) {
      line = e.line;
      what = e.what();
    }
    CHECK(line == 3 && what == "line 3: row index 3 outside [1, 2]");
  }

  if (no_gpu) {  // the product path must fail loudly, never fall back to the CPU
    const BipartiteCsr g = fork_graph();
    bool threw = false;
    try {
      (*make_algorithm("apfb-wr-b200"))(g, cheap_matching(g), Schedule::serial());
    } catch (const std::runtime_error&) {
      threw = true;
    }
    CHECK(threw);
    std::printf("PASS %d (no-gpu)\n", g_checks);
    return 0;
  }

  // 1. registry path, every id, against hopcroft_karp
  for (const BipartiteCsr& g : corpus()) {
    const MatchingState init = cheap_matching(g);
    const long long want = cardinality(hopcroft_karp(g, init));
    for (const char* id : {"apfb-wr-b200", "apfb-gpubfs-b200", "apsb-wr-b200", "apsb-gpubfs-b200"}) {
      AlgorithmResult r = (*make_algorithm(id))(g, init, Schedule::parallel());
      check_result(g, r.matching, want);
      CHECK(r.counters.has_value());
      CHECK((long long)r.counters->bfs_launches_per_iteration.size() == r.counters->outer_iterations);
      CHECK(r.counters->outer_iterations >= 1);
    }
  }

  // 2. driver entry points with an observer (gpu_match.cpp:350-353 contract)
  {
    const BipartiteCsr g = generate_random_bipartite(3000, 3000, 3.0, 77);
    const MatchingState init = cheap_matching(g);
    long long prev = cardinality(init), phases = 0;
    PhaseObserver obs = [&](const PhaseEvent& ev) {
      CHECK(ev.iteration == ++phases);
      CHECK(ev.cardinality_before == prev);
      CHECK(ev.cardinality_after >= ev.cardinality_before);
      CHECK(validate(g, ev.state).ok());
      CHECK(cardinality(ev.state) == ev.cardinality_after);
      prev = ev.cardinality_after;
    };
    DriverResult r = b200::apfb(g, init, GridConfig{}, Schedule::serial(), BfsKernel::GpubfsWr, obs);
    CHECK(phases == r.counters.outer_iterations);
    check_result(g, r.matching, cardinality(hopcroft_karp(g, init)));
    phases = 0;
    prev = cardinality(init);
    r = b200::apsb(g, init, GridConfig{}, Schedule::serial(), BfsKernel::GpubfsWr, true, obs);
    check_result(g, r.matching, cardinality(hopcroft_karp(g, init)));
    // an observer exception reaches the caller
    bool threw = false;
    try {
      b200::apfb(g, init, GridConfig{}, Schedule::serial(), BfsKernel::Gpubfs,
                 [](const PhaseEvent&) { throw std::domain_error("observer"); });
    } catch (const std::domain_error&) {
      threw = true;
    }
    CHECK(threw);
  }

  // 3. error mapping: the reference's exception types
  {
    const BipartiteCsr g = fork_graph();
    bool logic = false;
    try {
      b200::apsb(g, cheap_matching(g), GridConfig{}, Schedule::serial(), BfsKernel::Gpubfs, true);
    } catch (const std::logic_error&) {
      logic = true;
    }
    CHECK(logic);
    MatchingState bad = MatchingState::unmatched(g.nc, g.nr);
    bad.rmatch[0] = 1;  // asymmetric: cmatch[1] != 0
    bool invalid = false;
    try {
      b200::apfb(g, bad, GridConfig{}, Schedule::serial(), BfsKernel::GpubfsWr);
    } catch (const std::invalid_argument&) {
      invalid = true;
    }
    CHECK(invalid);
    // the nc + 1 phase bound (gpu_match.cpp:313-320) -> std::runtime_error; the
    // bound is lowered through the engine's fault-injection hook
    const BipartiteCsr gr = generate_random_bipartite(50000, 50000, 6.0, 9);
    const MatchingState gi = cheap_matching(gr);
    bm_handle* h = b200::thread_engine(0).get();
    CHECK(bm_debug_set(h, BM_DEBUG_PHASE_BOUND, 1) == BM_OK);
    bool bound = false;
    try {
      b200::apfb(gr, gi, GridConfig{}, Schedule::serial(), BfsKernel::GpubfsWr);
    } catch (const std::runtime_error& e) {
      bound = std::string(e.what()).find("bound") != std::string::npos;
    }
    CHECK(bound);
    CHECK(bm_debug_set(h, BM_DEBUG_PHASE_BOUND, 0) == BM_OK);
    // a raced phase with no progress takes the serial retry (gpu_match.cpp:328-343)
    CHECK(bm_debug_set(h, BM_DEBUG_SKIP_ALTERNATE_PHASE, 1) == BM_OK);
    const DriverResult rr = b200::apfb(gr, gi, GridConfig{}, Schedule::serial(), BfsKernel::GpubfsWr);
    CHECK(rr.counters.serial_retries == 1);
    CHECK(bm_debug_set(h, BM_DEBUG_SKIP_ALTERNATE_PHASE, 0) == BM_OK);
    check_result(gr, rr.matching, cardinality(hopcroft_karp(gr, gi)));
  }

  // 4. the reference's suite runner with its cardinality-mismatch gate
  {
    namespace fs = std::filesystem;
    const fs::path dir = fs::temp_directory_path() / "bmatch_b200_shim_suite";
    fs::create_directories(dir);
    std::vector<std::string> paths;
    int k = 0;
    for (const BipartiteCsr& g : {generate_random_bipartite(2000, 2000, 2.0, 5),
                                  generate_random_bipartite(3000, 2500, 4.0, 6), complete_graph(12, 9)}) {
      const fs::path p = dir / ("g" + std::to_string(k++) + ".mtx");
      std::ofstream out(p);
      write_matrix_market(g, out);
      paths.push_back(p.string());
    }
    SuiteOptions opt;
    opt.repetitions = 2;
    opt.permute_seed = 3;
    const SuiteResult res = run_suite(paths, {"hk", "apfb-wr-b200", "apsb-wr-b200", "apfb-gpubfs-b200"}, opt);
    CHECK(res.load_errors.empty());
    CHECK(res.ok());
    CHECK(res.records.size() == 12);
    fs::remove_all(dir);
  }

  std::printf("PASS %d\n", g_checks);
  return 0;
}
