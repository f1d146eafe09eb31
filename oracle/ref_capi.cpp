// ref_capi.cpp — a thin extern "C" wrapper over the UNMODIFIED reference
// library (compiled from /root/reference/proj/src by `make ref` into
// oracle/_ref/libbmatch_ref.so). TEST/BASELINE INFRASTRUCTURE ONLY: it lets
// the Python tests and bench.py's reference arm call the reference's own
// public API (make_algorithm, apfb/apsb, the BFS/ALTERNATE/FIX kernels,
// validate/is_maximum, generate_random_bipartite) through ctypes.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "bmatch/algorithms.hpp"
#include "bmatch/baselines.hpp"
#include "bmatch/csr_graph.hpp"
#include "bmatch/gpu_match.hpp"
#include "bmatch/kernel_grid.hpp"
#include "bmatch/matching.hpp"
#include "bmatch/matrix_market.hpp"

using namespace bmatch;

namespace {
thread_local std::string g_ref_err;

MatchingState to_state(const BipartiteCsr& g, const int32_t* rmatch, const int32_t* cmatch) {
  MatchingState m;
  m.rmatch.assign(rmatch, rmatch + g.nr);
  m.cmatch.assign(cmatch, cmatch + g.nc);
  return m;
}

void from_state(const MatchingState& m, int32_t* rmatch, int32_t* cmatch) {
  if (rmatch) std::memcpy(rmatch, m.rmatch.data(), sizeof(int32_t) * m.rmatch.size());
  if (cmatch) std::memcpy(cmatch, m.cmatch.data(), sizeof(int32_t) * m.cmatch.size());
}

GridConfig grid_of(int32_t tot) { return GridConfig{GridMode::Ct, tot, tot}; }
}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_ref_err.c_str(); }
int32_t ref_hw_threads(void) { return (int32_t)std::thread::hardware_concurrency(); }

void* ref_graph_from_csc(int32_t nc, int32_t nr, const int64_t* cxadj, const int32_t* cadj) {
  auto* g = new BipartiteCsr();
  g->nc = nc;
  g->nr = nr;
  g->cxadj.assign(cxadj, cxadj + nc + 1);
  g->cadj.assign(cadj, cadj + cxadj[nc]);
  return g;
}

void* ref_generate_random_bipartite(int32_t nc, int32_t nr, double deg, uint64_t seed) {
  return new BipartiteCsr(generate_random_bipartite(nc, nr, deg, seed));
}

void* ref_permute_random(void* h, uint64_t seed) {
  return new BipartiteCsr(permute_random(*static_cast<BipartiteCsr*>(h), seed));
}

void ref_graph_info(void* h, int32_t* nc, int32_t* nr, int64_t* ne) {
  auto* g = static_cast<BipartiteCsr*>(h);
  *nc = g->nc;
  *nr = g->nr;
  *ne = g->num_edges();
}

void ref_graph_copy(void* h, int64_t* cxadj, int32_t* cadj) {
  auto* g = static_cast<BipartiteCsr*>(h);
  std::memcpy(cxadj, g->cxadj.data(), sizeof(int64_t) * g->cxadj.size());
  if (!g->cadj.empty()) std::memcpy(cadj, g->cadj.data(), sizeof(int32_t) * g->cadj.size());
}

// read_matrix_market on an in-memory stream (matrix_market.cpp:29-99). Returns
// a graph handle, or null with *err_kind = 1 (ParseError; *err_line set) or 2
// (another exception, e.g. from_edge_list's out_of_range); message in
// ref_last_error().
void* ref_read_matrix_market(const char* text, int64_t len, int32_t* err_kind, int64_t* err_line) {
  *err_kind = 0;
  *err_line = 0;
  try {
    std::istringstream in(std::string(text, (size_t)len));
    return new BipartiteCsr(read_matrix_market(in));
  } catch (const ParseError& e) {
    *err_kind = 1;
    *err_line = e.line;
    g_ref_err = e.what();
  } catch (const std::exception& e) {
    *err_kind = 2;
    g_ref_err = e.what();
  }
  return nullptr;
}

// write_matrix_market (matrix_market.cpp:111-118) into a caller buffer;
// returns the byte length (copies only when cap is large enough).
int64_t ref_write_matrix_market(void* h, char* out, int64_t cap) {
  std::ostringstream os;
  write_matrix_market(*static_cast<BipartiteCsr*>(h), os);
  const std::string s = os.str();
  if (out && cap >= (int64_t)s.size()) std::memcpy(out, s.data(), s.size());
  return (int64_t)s.size();
}

void ref_graph_free(void* h) { delete static_cast<BipartiteCsr*>(h); }

int32_t ref_check_csr(void* h) {
  try {
    check_csr(*static_cast<BipartiteCsr*>(h));
    return 0;
  } catch (const std::exception& e) {
    g_ref_err = e.what();
    return 1;
  }
}

void ref_cheap_matching(void* h, int32_t* rmatch, int32_t* cmatch) {
  from_state(cheap_matching(*static_cast<BipartiteCsr*>(h)), rmatch, cmatch);
}

int64_t ref_brute_force_maximum(void* h) { return brute_force_maximum(*static_cast<BipartiteCsr*>(h)); }

int64_t ref_validate(void* h, const int32_t* rmatch, const int32_t* cmatch) {
  auto* g = static_cast<BipartiteCsr*>(h);
  try {
    return (int64_t)validate(*g, to_state(*g, rmatch, cmatch)).violations.size();
  } catch (const std::exception& e) {
    g_ref_err = e.what();
    return -1;
  }
}

int32_t ref_is_maximum(void* h, const int32_t* rmatch, const int32_t* cmatch) {
  auto* g = static_cast<BipartiteCsr*>(h);
  try {
    return is_maximum(*g, to_state(*g, rmatch, cmatch)) ? 1 : 0;
  } catch (const std::exception& e) {
    g_ref_err = e.what();
    return -1;
  }
}

// Runs a registry algorithm (make_algorithm, algorithms.cpp:64-93) under a
// schedule string (parse_schedule, kernel_grid.cpp:145-163) and times the
// call with steady_clock (bench.cpp:59-63). counters[6] = {outer, scanned,
// walks, resets, retries, launches_total}. Returns 0 ok, 1 unknown id, 2 error.
int32_t ref_run(void* h, const char* id, const char* schedule, int32_t ct_threads, int32_t* rmatch,
                int32_t* cmatch, int64_t* counters, int64_t* launches, int64_t cap, double* seconds) {
  auto* g = static_cast<BipartiteCsr*>(h);
  try {
    AlgorithmOptions opts;
    if (ct_threads > 0) {
      opts.ct_thread_num = ct_threads;
      opts.max_threads = ct_threads;
    }
    auto fn = make_algorithm(id, opts);
    if (!fn) {
      g_ref_err = std::string("unknown algorithm ") + id;
      return 1;
    }
    const MatchingState init = to_state(*g, rmatch, cmatch);
    const Schedule sched = parse_schedule(schedule);
    const auto t0 = std::chrono::steady_clock::now();
    AlgorithmResult res = (*fn)(*g, init, sched);
    const auto t1 = std::chrono::steady_clock::now();
    if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
    from_state(res.matching, rmatch, cmatch);
    if (counters) {
      std::memset(counters, 0, sizeof(int64_t) * 6);
      if (res.counters) {
        counters[0] = res.counters->outer_iterations;
        counters[1] = res.counters->columns_scanned;
        counters[2] = res.counters->alternations_attempted;
        counters[3] = res.counters->fix_resets;
        counters[4] = res.counters->serial_retries;
        counters[5] = res.counters->bfs_launches_total();
        if (launches)
          for (size_t i = 0; i < res.counters->bfs_launches_per_iteration.size() && (int64_t)i < cap; ++i)
            launches[i] = res.counters->bfs_launches_per_iteration[i];
      }
    }
    return 0;
  } catch (const std::exception& e) {
    g_ref_err = e.what();
    return 2;
  }
}

// Single kernels under the Serial schedule on a CT grid of `tot` threads.
int64_t ref_gpubfs(void* h, int32_t tot, int32_t wr, int32_t improved, int32_t bfs_level, int32_t* bfs,
                   int32_t* pred, int32_t* root, int32_t* rmatch, int32_t* cmatch, int32_t* flags) {
  auto* g = static_cast<BipartiteCsr*>(h);
  try {
    BfsPhaseState phase;
    phase.start_level = 2;
    phase.bfs_level = bfs_level;
    phase.bfs_array.assign(bfs, bfs + g->nc);
    phase.predecessor.assign(pred, pred + g->nr);
    if (wr) phase.root.assign(root, root + g->nc);
    phase.vertex_inserted = flags[0];
    phase.augmenting_path_found = flags[1];
    MatchingState m = to_state(*g, rmatch, cmatch);
    PhaseCounters pc;
    if (wr) gpubfs_wr(phase, *g, m, grid_of(tot), Schedule::serial(), improved != 0, &pc);
    else gpubfs(phase, *g, m, grid_of(tot), Schedule::serial(), &pc);
    std::memcpy(bfs, phase.bfs_array.data(), sizeof(int32_t) * g->nc);
    std::memcpy(pred, phase.predecessor.data(), sizeof(int32_t) * g->nr);
    if (wr) std::memcpy(root, phase.root.data(), sizeof(int32_t) * g->nc);
    from_state(m, rmatch, cmatch);
    flags[0] = phase.vertex_inserted;
    flags[1] = phase.augmenting_path_found;
    return pc.columns_scanned;
  } catch (const std::exception& e) {
    g_ref_err = e.what();
    return -1;
  }
}

int64_t ref_alternate(void* h, int32_t tot, int32_t wr_encoded, const int32_t* bfs, const int32_t* pred,
                      int32_t* rmatch, int32_t* cmatch) {
  auto* g = static_cast<BipartiteCsr*>(h);
  MatchingState m = to_state(*g, rmatch, cmatch);
  PhaseCounters pc;
  if (wr_encoded) {
    BfsPhaseState phase;
    phase.bfs_array.assign(bfs, bfs + g->nc);
    phase.predecessor.assign(pred, pred + g->nr);
    alternate_wr(*g, m, phase, grid_of(tot), Schedule::serial(), &pc);
  } else {
    std::vector<int> p(pred, pred + g->nr);
    alternate(*g, m, p, grid_of(tot), Schedule::serial(), &pc);
  }
  from_state(m, rmatch, cmatch);
  return pc.alternations_attempted;
}

int64_t ref_fix_matching(int32_t nc, int32_t nr, int32_t* rmatch, int32_t* cmatch) {
  MatchingState m;
  m.rmatch.assign(rmatch, rmatch + nr);
  m.cmatch.assign(cmatch, cmatch + nc);
  PhaseCounters pc;
  fix_matching(m, &pc);
  std::memcpy(rmatch, m.rmatch.data(), sizeof(int32_t) * nr);
  std::memcpy(cmatch, m.cmatch.data(), sizeof(int32_t) * nc);
  return pc.fix_resets;
}

}  // extern "C"
