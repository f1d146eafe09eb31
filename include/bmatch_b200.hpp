// bmatch_b200.hpp — header-only C++ shim that puts the B200 engine behind the
// reference's own C++ entry points. A maintainer adds this header (and links
// libbmatch_b200.so) to the reference tree; nothing in the reference changes.
//
// Include it after the reference headers are on the include path
// (-I <reference>/proj/include). It provides, in namespace bmatch::b200:
//
//   apfb(g, init, grid, schedule, kernel, observer)            replaces bmatch::apfb
//        (include/bmatch/gpu_match.hpp:133-135)
//   apsb(g, init, grid, schedule, kernel, improved, observer)  replaces bmatch::apsb
//        (include/bmatch/gpu_match.hpp:141-144)
//   register_algorithms()                                     registers the ids
//        apfb-wr-b200, apfb-gpubfs-b200, apsb-wr-b200, apsb-gpubfs-b200 through
//        bmatch::register_algorithm (include/bmatch/algorithms.hpp:42,
//        src/algorithms.cpp:95-97), so run_suite (src/bench.cpp:31-36, 61) and
//        the CLI's `match --algo` (src/cli.cpp:59-76) reach the B200 engine
//        with no other change. With shadow_reference_ids = true it also
//        replaces the reference's own ids apfb-wr-ct, apsb-wr-ct, ... .
//   load_matrix_market(path), read_matrix_market(text), write_matrix_market(g, path)
//        replace the reference's Matrix Market I/O (include/bmatch/matrix_market.hpp:
//        14-24) with the parallel reader/writer of bmatch_b200_io.h; same graph,
//        same bytes, same ParseError{line}
//   load_csc(path), save_csc(g, path)                         binary CSC files
//
// Behaviour the reference's callers rely on is kept:
//   * same parameter lists; GridConfig and Schedule are accepted and ignored
//     (the GPU grid is sized internally);
//   * DriverResult{matching, counters} with PhaseCounters filled as the
//     reference fills them (outer_iterations, bfs_launches_per_iteration,
//     columns_scanned, alternations_attempted, fix_resets, serial_retries);
//   * the observer fires after every phase with the state after FIX
//     (gpu_match.cpp:350-353); exceptions it throws propagate to the caller;
//   * errors surface as the reference's exception types: std::logic_error for
//     the improved alternation without the with-root kernel
//     (gpu_match.cpp:272-274), std::runtime_error when the nc + 1 phase bound
//     is exceeded (gpu_match.cpp:317-320), std::invalid_argument for an invalid
//     initial matching; device failures are std::runtime_error.
//
// Threading: one engine handle per (thread, device), created on first use;
// a handle is not reentrant, different threads get different handles.
#pragma once

#include <exception>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "bmatch/algorithms.hpp"
#include "bmatch/csr_graph.hpp"
#include "bmatch/gpu_match.hpp"
#include "bmatch/kernel_grid.hpp"
#include "bmatch/matching.hpp"
#include "bmatch/parse_error.hpp"
#include "bmatch_b200.h"
#include "bmatch_b200_io.h"

namespace bmatch::b200 {

// Maps a C status to the reference's exception types.
inline void throw_on(bm_status s) {
  if (s == BM_OK) return;
  std::string msg = std::string("bmatch_b200: ") + bm_last_error();
  switch (s) {
    case BM_ERR_INVALID_ARG: throw std::invalid_argument(msg);
    case BM_ERR_LOGIC: throw std::logic_error(msg);
    case BM_ERR_BOUND_EXCEEDED: throw std::runtime_error(msg);
    default: throw std::runtime_error(msg + " (" + bm_status_string(s) + ")");
  }
}

// RAII owner of one engine handle (device buffers + stream).
class Engine {
 public:
  explicit Engine(int device = 0) { throw_on(bm_create(device, &h_)); }
  ~Engine() { bm_destroy(h_); }
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;
  bm_handle* get() const { return h_; }

  // Copies g to HBM (device buffers are reused when they are large enough).
  // Every call uploads: the reference's AlgorithmFn receives the graph by
  // reference with no identity guarantee, so caching by address is unsafe.
  void upload(const BipartiteCsr& g) {
    throw_on(bm_upload_csc(h_, g.nc, g.nr, g.cxadj.data(), g.cadj.data()));
  }

 private:
  bm_handle* h_ = nullptr;
};

inline Engine& thread_engine(int device = 0) {
  thread_local std::vector<std::unique_ptr<Engine>> engines;
  if ((int)engines.size() <= device) engines.resize(device + 1);
  if (!engines[device]) engines[device] = std::make_unique<Engine>(device);
  return *engines[device];
}

namespace detail {

struct ObserverCtx {
  const PhaseObserver* observer;
  std::exception_ptr error;
};

// bm_phase_cb -> PhaseObserver (gpu_match.hpp:115-124); exceptions are parked
// and rethrown after the C call returns, never thrown across the C ABI.
inline int observer_trampoline(const bm_phase_event* ev, void* user) {
  auto* ctx = static_cast<ObserverCtx*>(user);
  try {
    MatchingState state;
    state.rmatch.assign(ev->rmatch, ev->rmatch + ev->nr);
    state.cmatch.assign(ev->cmatch, ev->cmatch + ev->nc);
    PhaseEvent pe{ev->iteration, ev->augmenting_path_found != 0, ev->cardinality_before,
                  ev->cardinality_after, ev->serial_retry != 0, ev->bfs_launches, state};
    (*ctx->observer)(pe);
    return 0;
  } catch (...) {
    ctx->error = std::current_exception();
    return 1;
  }
}

inline DriverResult run(const BipartiteCsr& g, MatchingState init, bool shortest, BfsKernel kernel,
                        bool improved, const PhaseObserver& observer, int device) {
  if ((int)init.rmatch.size() != g.nr || (int)init.cmatch.size() != g.nc)
    throw std::invalid_argument("bmatch_b200: initial matching does not fit the graph");
  Engine& eng = thread_engine(device);
  eng.upload(g);
  bm_match_opts o{};
  o.driver = shortest ? BM_DRIVER_APSB : BM_DRIVER_APFB;
  o.bfs_kernel = kernel == BfsKernel::GpubfsWr ? BM_BFS_WR : BM_BFS_GPUBFS;
  o.improved = improved ? 1 : 0;
  o.init = BM_INIT_GIVEN;
  o.bottom_up = BM_BU_AUTO;  // pull dense levels where the engine judges it pays
  bm_counters ct{};
  // A small per-phase buffer (a buffer of nc + 2 entries, zeroed on every call,
  // cost 160 ms of page faults at 1e8 columns); longer runs fetch the rest after.
  std::vector<int64_t> launches((size_t)std::min<int64_t>((int64_t)g.nc + 2, 1024));
  int64_t card = 0;
  ObserverCtx ctx{&observer, nullptr};
  const bm_status s =
      bm_match(eng.get(), &o, init.rmatch.data(), init.cmatch.data(), &card, &ct, launches.data(),
               (int64_t)launches.size(), observer ? &observer_trampoline : nullptr, observer ? &ctx : nullptr);
  if (ctx.error) std::rethrow_exception(ctx.error);
  throw_on(s);
  if (ct.outer_iterations > (int64_t)launches.size()) {
    launches.resize((size_t)ct.outer_iterations);
    int64_t n = 0;
    throw_on(bm_last_phase_launches(eng.get(), launches.data(), (int64_t)launches.size(), &n));
    ct.n_phase_records = n;
  }
  DriverResult res;
  res.matching = std::move(init);
  res.counters.outer_iterations = ct.outer_iterations;
  res.counters.bfs_launches_per_iteration.assign(launches.begin(), launches.begin() + ct.n_phase_records);
  res.counters.columns_scanned = ct.columns_scanned;
  res.counters.alternations_attempted = ct.alternations_attempted;
  res.counters.fix_resets = ct.fix_resets;
  res.counters.serial_retries = ct.serial_retries;
  return res;
}

}  // namespace detail

// bmatch::apfb (gpu_match.hpp:133-135) on the B200.
inline DriverResult apfb(const BipartiteCsr& g, MatchingState init, const GridConfig& /*grid*/,
                         const Schedule& /*schedule*/, BfsKernel kernel, const PhaseObserver& observer = {},
                         int device = 0) {
  return detail::run(g, std::move(init), false, kernel, false, observer, device);
}

// bmatch::apsb (gpu_match.hpp:141-144) on the B200.
inline DriverResult apsb(const BipartiteCsr& g, MatchingState init, const GridConfig& /*grid*/,
                         const Schedule& /*schedule*/, BfsKernel kernel, bool improved_alternate,
                         const PhaseObserver& observer = {}, int device = 0) {
  if (improved_alternate && kernel != BfsKernel::GpubfsWr)  // gpu_match.cpp:272-274
    throw std::logic_error("improved alternation requires the GPUBFS-WR kernel");
  return detail::run(g, std::move(init), true, kernel, improved_alternate, observer, device);
}

// Registers the B200 runners with the reference registry
// (algorithms.hpp:42). Ids mirror grid_algos() (algorithms.cpp:19-27): the
// endpoint-encoded alternation is used by apsb-wr only.
inline void register_algorithms(int device = 0, bool shadow_reference_ids = false) {
  struct Algo {
    const char* base;
    bool shortest;
    BfsKernel kernel;
    bool improved;
  };
  static const Algo algos[] = {
      {"apfb-gpubfs", false, BfsKernel::Gpubfs, false},
      {"apfb-wr", false, BfsKernel::GpubfsWr, false},
      {"apsb-gpubfs", true, BfsKernel::Gpubfs, false},
      {"apsb-wr", true, BfsKernel::GpubfsWr, true},
  };
  for (const Algo& a : algos) {
    AlgorithmFn fn = [a, device](const BipartiteCsr& g, const MatchingState& init, const Schedule&) {
      DriverResult r = detail::run(g, init, a.shortest, a.kernel, a.improved, PhaseObserver{}, device);
      return AlgorithmResult{std::move(r.matching), std::move(r.counters)};
    };
    register_algorithm(std::string(a.base) + "-b200", fn);
    if (shadow_reference_ids) {
      register_algorithm(std::string(a.base) + "-ct", fn);
      register_algorithm(std::string(a.base) + "-mt", fn);
      register_algorithm(a.base, fn);
    }
  }
}

namespace detail {

// Runs a bm_mm_* reader; rethrows BM_ERR_PARSE as the reference's ParseError.
template <typename Info, typename Load>
BipartiteCsr read_mm(Info&& info, Load&& load) {
  auto check = [](bm_status s, int64_t line) {
    if (s != BM_ERR_PARSE) return throw_on(s);
    std::string msg = bm_last_error();  // "line N: message", as ParseError::what()
    const std::string head = "line " + std::to_string(line) + ": ";
    if (msg.compare(0, head.size(), head) == 0) msg = msg.substr(head.size());
    throw ParseError(line, msg);
  };
  bm_mm_header h{};
  int64_t line = 0;
  bm_status s = info(&h, &line);  // (the status must be taken before `line` is read)
  check(s, line);
  BipartiteCsr g;
  g.nc = h.ncols;
  g.nr = h.nrows;
  g.cxadj.assign((size_t)h.ncols + 1, 0);
  g.cadj.assign((size_t)h.capacity, 0);
  int64_t ne = 0;
  s = load(h.capacity, g.cxadj.data(), g.cadj.data(), &ne, &line);
  check(s, line);
  g.cadj.resize((size_t)ne);
  g.cadj.shrink_to_fit();
  return g;
}

inline std::string stem(const std::string& path) {
  const size_t slash = path.find_last_of('/');
  std::string base = slash == std::string::npos ? path : path.substr(slash + 1);
  const size_t dot = base.find_last_of('.');
  return dot == std::string::npos || dot == 0 ? base : base.substr(0, dot);
}

}  // namespace detail

// read_matrix_market on an in-memory text (matrix_market.cpp:29-99).
inline BipartiteCsr read_matrix_market(const std::string& text, int threads = 0) {
  return detail::read_mm(
      [&](bm_mm_header* h, int64_t* line) { return bm_mm_parse_info(text.data(), (int64_t)text.size(), h, line); },
      [&](int64_t cap, int64_t* cx, int32_t* adj, int64_t* ne, int64_t* line) {
        return bm_mm_parse(text.data(), (int64_t)text.size(), threads, cap, cx, adj, ne, line);
      });
}

// load_matrix_market (matrix_market.cpp:101-108): memory-mapped, parsed on every core.
inline BipartiteCsr load_matrix_market(const std::string& path, int threads = 0) {
  BipartiteCsr g = detail::read_mm(
      [&](bm_mm_header* h, int64_t* line) { return bm_mm_info(path.c_str(), h, line); },
      [&](int64_t cap, int64_t* cx, int32_t* adj, int64_t* ne, int64_t* line) {
        return bm_mm_load(path.c_str(), threads, cap, cx, adj, ne, line);
      });
  g.name = detail::stem(path);
  return g;
}

// write_matrix_market (matrix_market.cpp:111-118) to a file, byte for byte.
inline void write_matrix_market(const BipartiteCsr& g, const std::string& path, int threads = 0) {
  throw_on(bm_mm_write(path.c_str(), g.nc, g.nr, g.cxadj.data(), g.cadj.data(), threads));
}

inline void save_csc(const BipartiteCsr& g, const std::string& path, int threads = 0) {
  throw_on(bm_csc_write(path.c_str(), g.nc, g.nr, g.cxadj.data(), g.cadj.data(), threads));
}

inline BipartiteCsr load_csc(const std::string& path, int threads = 0) {
  BipartiteCsr g;
  int64_t ne = 0;
  throw_on(bm_csc_info(path.c_str(), &g.nc, &g.nr, &ne));
  g.cxadj.assign((size_t)g.nc + 1, 0);
  g.cadj.assign((size_t)ne, 0);
  throw_on(bm_csc_read(path.c_str(), threads, ne, g.cxadj.data(), g.cadj.data()));
  g.name = detail::stem(path);
  return g;
}

}  // namespace bmatch::b200
