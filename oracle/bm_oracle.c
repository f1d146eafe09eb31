/*
 * bm_oracle.c — CPU restatement of the reference matching path (see
 * bm_oracle.h). TEST INFRASTRUCTURE ONLY: the checker for the B200 engine,
 * never part of the product path.
 *
 * Parity is pinned by tests/test_oracle.py against fixtures produced by the
 * reference itself (oracle/_ref, compiled from /root/reference sources by
 * `make ref`; generator script tests/golden/make_golden.py).
 */
#include "bm_oracle.h"

#include <limits.h>
#include <stdlib.h>
#include <string.h>

/* ---- matching.cpp ---------------------------------------------------- */

void or_cheap_matching(const or_graph* g, int32_t* rmatch, int32_t* cmatch) {
  for (int32_t r = 0; r < g->nr; ++r) rmatch[r] = -1;
  for (int32_t c = 0; c < g->nc; ++c) {
    cmatch[c] = -1;
    for (int64_t j = g->cxadj[c]; j < g->cxadj[c + 1]; ++j) {
      const int32_t r = g->cadj[j];
      if (rmatch[r] < 0) { /* first free row wins, matching.cpp:17-23 */
        rmatch[r] = c;
        cmatch[c] = r;
        break;
      }
    }
  }
}

int64_t or_cardinality(int32_t nr, const int32_t* rmatch) {
  int64_t k = 0;
  for (int32_t r = 0; r < nr; ++r) k += rmatch[r] >= 0;
  return k;
}

static int has_edge(const or_graph* g, int32_t c, int32_t r) {
  int64_t lo = g->cxadj[c], hi = g->cxadj[c + 1];
  while (lo < hi) { /* slices are strictly ascending (csr_graph.hpp:14-17) */
    const int64_t mid = lo + (hi - lo) / 2;
    if (g->cadj[mid] == r) return 1;
    if (g->cadj[mid] < r) lo = mid + 1; else hi = mid;
  }
  return 0;
}

int64_t or_validate(const or_graph* g, const int32_t* rmatch, const int32_t* cmatch) {
  int64_t bad = 0;
  for (int32_t r = 0; r < g->nr; ++r) {
    const int32_t c = rmatch[r];
    if (c == -1) continue;
    if (c == -2 || c < 0 || c >= g->nc) { bad++; continue; } /* PendingFlag / OutOfRange */
    if (cmatch[c] != r) { bad++; continue; }                 /* Asymmetry */
    if (!has_edge(g, c, r)) bad++;                           /* NonEdge */
  }
  for (int32_t c = 0; c < g->nc; ++c) {
    const int32_t r = cmatch[c];
    if (r == -1) continue;
    if (r < 0 || r >= g->nr) { bad++; continue; }
    if (rmatch[r] != c) bad++;
  }
  return bad;
}

int32_t or_is_maximum(const or_graph* g, const int32_t* rmatch, const int32_t* cmatch) {
  if (or_validate(g, rmatch, cmatch) != 0) return -1;
  char* seen = (char*)calloc((size_t)g->nc + 1, 1);
  int32_t* queue = (int32_t*)malloc(sizeof(int32_t) * ((size_t)g->nc + 1));
  int64_t head = 0, tail = 0;
  int32_t result = 1;
  for (int32_t c = 0; c < g->nc; ++c)
    if (cmatch[c] < 0) {
      seen[c] = 1;
      queue[tail++] = c;
    }
  while (head < tail && result) {
    const int32_t c = queue[head++];
    for (int64_t j = g->cxadj[c]; j < g->cxadj[c + 1]; ++j) {
      const int32_t next = rmatch[g->cadj[j]];
      if (next < 0) { result = 0; break; } /* reached a free row: augmenting path */
      if (!seen[next]) {
        seen[next] = 1;
        queue[tail++] = next;
      }
    }
  }
  free(seen);
  free(queue);
  return result;
}

static int bf_augment(const or_graph* g, int32_t c, int32_t* rmatch, int32_t* cmatch, char* seen) {
  seen[c] = 1;
  for (int64_t j = g->cxadj[c]; j < g->cxadj[c + 1]; ++j) {
    const int32_t r = g->cadj[j];
    if (rmatch[r] < 0) {
      rmatch[r] = c;
      cmatch[c] = r;
      return 1;
    }
  }
  for (int64_t j = g->cxadj[c]; j < g->cxadj[c + 1]; ++j) {
    const int32_t r = g->cadj[j];
    const int32_t holder = rmatch[r];
    if (!seen[holder] && bf_augment(g, holder, rmatch, cmatch, seen)) {
      rmatch[r] = c;
      cmatch[c] = r;
      return 1;
    }
  }
  return 0;
}

int64_t or_brute_force_maximum(const or_graph* g) {
  int32_t* rmatch = (int32_t*)malloc(sizeof(int32_t) * ((size_t)g->nr + 1));
  int32_t* cmatch = (int32_t*)malloc(sizeof(int32_t) * ((size_t)g->nc + 1));
  char* seen = (char*)malloc((size_t)g->nc + 1);
  int64_t matched = 0;
  for (int32_t r = 0; r < g->nr; ++r) rmatch[r] = -1;
  for (int32_t c = 0; c < g->nc; ++c) cmatch[c] = -1;
  for (int32_t c = 0; c < g->nc; ++c) {
    if (cmatch[c] >= 0) continue;
    memset(seen, 0, (size_t)g->nc + 1);
    matched += bf_augment(g, c, rmatch, cmatch, seen);
  }
  free(rmatch);
  free(cmatch);
  free(seen);
  return matched;
}

/* ---- baselines.cpp: Hopcroft-Karp ------------------------------------ */

static int hk_dfs(const or_graph* g, int32_t c0, int32_t* rmatch, int32_t* cmatch, int32_t* dist,
                  int64_t* iter, int32_t* stack, int32_t* rows) {
  int64_t sp = 0, rp = 0;
  stack[sp++] = c0;
  while (sp > 0) {
    const int32_t c = stack[sp - 1];
    int advanced = 0;
    while (iter[c] < g->cxadj[c + 1]) {
      const int32_t r = g->cadj[iter[c]++];
      const int32_t next = rmatch[r];
      if (next < 0) { /* free row: flip the whole stack (baselines.cpp:30-37) */
        rows[rp++] = r;
        for (int64_t k = 0; k < sp; ++k) {
          cmatch[stack[k]] = rows[k];
          rmatch[rows[k]] = stack[k];
        }
        return 1;
      }
      if (dist[next] == dist[c] + 1) {
        rows[rp++] = r;
        stack[sp++] = next;
        advanced = 1;
        break;
      }
    }
    if (!advanced) { /* dead end: retire the column for this phase */
      dist[c] = INT_MAX;
      sp--;
      if (rp > 0) rp--;
    }
  }
  return 0;
}

void or_hopcroft_karp(const or_graph* g, int32_t* rmatch, int32_t* cmatch) {
  const size_t n = (size_t)g->nc + 1;
  int32_t* dist = (int32_t*)malloc(sizeof(int32_t) * n);
  int64_t* iter = (int64_t*)malloc(sizeof(int64_t) * n);
  int32_t* queue = (int32_t*)malloc(sizeof(int32_t) * n);
  int32_t* stack = (int32_t*)malloc(sizeof(int32_t) * n);
  int32_t* rows = (int32_t*)malloc(sizeof(int32_t) * n);
  for (;;) {
    int64_t head = 0, tail = 0;
    int found = 0;
    for (int32_t c = 0; c < g->nc; ++c) {
      dist[c] = INT_MAX;
      if (cmatch[c] < 0) {
        dist[c] = 0;
        queue[tail++] = c;
      }
    }
    while (head < tail) {
      const int32_t c = queue[head++];
      for (int64_t j = g->cxadj[c]; j < g->cxadj[c + 1]; ++j) {
        const int32_t next = rmatch[g->cadj[j]];
        if (next < 0) found = 1;
        else if (dist[next] == INT_MAX) {
          dist[next] = dist[c] + 1;
          queue[tail++] = next;
        }
      }
    }
    if (!found) break;
    for (int32_t c = 0; c < g->nc; ++c) iter[c] = g->cxadj[c];
    for (int32_t c = 0; c < g->nc; ++c)
      if (cmatch[c] < 0 && dist[c] == 0) hk_dfs(g, c, rmatch, cmatch, dist, iter, stack, rows);
  }
  free(dist);
  free(iter);
  free(queue);
  free(stack);
  free(rows);
}

void or_alternating_bfs_depths(const or_graph* g, const int32_t* rmatch, const int32_t* cmatch,
                               int32_t* depth) {
  int32_t* queue = (int32_t*)malloc(sizeof(int32_t) * ((size_t)g->nc + 1));
  int64_t head = 0, tail = 0;
  for (int32_t c = 0; c < g->nc; ++c) {
    depth[c] = -1;
    if (cmatch[c] < 0) {
      depth[c] = 0;
      queue[tail++] = c;
    }
  }
  while (head < tail) {
    const int32_t c = queue[head++];
    for (int64_t j = g->cxadj[c]; j < g->cxadj[c + 1]; ++j) {
      const int32_t next = rmatch[g->cadj[j]];
      if (next >= 0 && depth[next] < 0) {
        depth[next] = depth[c] + 1;
        queue[tail++] = next;
      }
    }
  }
  free(queue);
}

/* ---- gpu_match.cpp --------------------------------------------------- */

void or_init_bfs_array(int32_t nc, const int32_t* cmatch, int32_t start_level, int32_t* bfs) {
  for (int32_t c = 0; c < nc; ++c) bfs[c] = cmatch[c] > -1 ? start_level - 1 : start_level;
}

void or_init_root(int32_t nc, const int32_t* cmatch, int32_t* root) {
  for (int32_t c = 0; c < nc; ++c) root[c] = cmatch[c] > -1 ? 0 : c;
}

/* Serial schedule: virtual thread tid visits vertices i*tot + tid for
 * i < get_process_count(n, tid, tot) (kernel_grid.hpp:117-126). */
#define FOR_SERIAL_GRID(n, tot, v)                                              \
  for (int64_t tid_ = 0; tid_ < (tot); ++tid_)                                  \
    for (int64_t i_ = 0, cnt_ = (n) / (tot) + (tid_ < (n) % (tot) ? 1 : 0);     \
         i_ < cnt_; ++i_)                                                       \
      for (int64_t v = i_ * (tot) + tid_, once_ = 1; once_; once_ = 0)

int64_t or_gpubfs(const or_graph* g, int32_t tot, int32_t bfs_level, int32_t start_level,
                  int32_t* bfs, int32_t* pred, int32_t* rmatch, int32_t* flags) {
  const int32_t unvisited = start_level - 1;
  int64_t scans = 0;
  if (tot < 1) tot = 1;
  FOR_SERIAL_GRID((int64_t)g->nc, (int64_t)tot, col) {
    if (bfs[col] != bfs_level) continue;
    scans++;
    for (int64_t j = g->cxadj[col]; j < g->cxadj[col + 1]; ++j) {
      const int32_t row = g->cadj[j];
      const int32_t cm = rmatch[row];
      if (cm > -1) {
        if (bfs[cm] == unvisited) {
          flags[0] = 1;
          bfs[cm] = bfs_level + 1;
          pred[row] = (int32_t)col;
        }
      } else if (cm == -1) {
        rmatch[row] = -2;
        pred[row] = (int32_t)col;
        flags[1] = 1;
      }
    }
  }
  return scans;
}

int64_t or_gpubfs_wr(const or_graph* g, int32_t tot, int32_t bfs_level, int32_t start_level,
                     int32_t improved, int32_t* bfs, int32_t* pred, int32_t* root, int32_t* rmatch,
                     int32_t* flags) {
  if (improved && start_level != 2) return -1; /* gpu_match.cpp:77-80 */
  const int32_t unvisited = start_level - 1;
  const int32_t found_mark = start_level - 2;
  int64_t scans = 0;
  if (tot < 1) tot = 1;
  FOR_SERIAL_GRID((int64_t)g->nc, (int64_t)tot, col) {
    if (bfs[col] != bfs_level) continue;
    const int32_t my_root = root[col];
    if (bfs[my_root] < unvisited) continue; /* the tree already found a path */
    scans++;
    for (int64_t j = g->cxadj[col]; j < g->cxadj[col + 1]; ++j) {
      const int32_t row = g->cadj[j];
      const int32_t cm = rmatch[row];
      if (cm > -1) {
        if (bfs[cm] == unvisited) {
          flags[0] = 1;
          bfs[cm] = bfs_level + 1;
          root[cm] = my_root;
          pred[row] = (int32_t)col;
        }
      } else if (cm == -1) {
        bfs[my_root] = improved ? -row : found_mark;
        rmatch[row] = -2;
        pred[row] = (int32_t)col;
        flags[1] = 1;
      }
    }
  }
  return scans;
}

static void walk(int32_t row, const int32_t* pred, int32_t* rmatch, int32_t* cmatch) {
  while (row != -1) {
    const int32_t col = pred[row];
    const int32_t mr = cmatch[col];
    if (mr >= 0 && pred[mr] == col) break; /* column already claimed this phase */
    cmatch[col] = row;
    rmatch[row] = col;
    row = mr;
  }
}

int64_t or_alternate(const or_graph* g, int32_t tot, const int32_t* pred, int32_t* rmatch, int32_t* cmatch) {
  int64_t walks = 0;
  if (tot < 1) tot = 1;
  FOR_SERIAL_GRID((int64_t)g->nr, (int64_t)tot, row) {
    if (rmatch[row] != -2) continue;
    walks++;
    walk((int32_t)row, pred, rmatch, cmatch);
  }
  return walks;
}

int64_t or_alternate_wr(const or_graph* g, int32_t tot, const int32_t* bfs, const int32_t* pred,
                        int32_t* rmatch, int32_t* cmatch) {
  int64_t walks = 0;
  if (tot < 1) tot = 1;
  FOR_SERIAL_GRID((int64_t)g->nc, (int64_t)tot, col) {
    const int32_t mark = bfs[col];
    if (mark > 0) continue;
    walks++;
    walk(-mark, pred, rmatch, cmatch);
  }
  return walks;
}

int64_t or_fix_matching(int32_t nc, int32_t nr, int32_t* rmatch, int32_t* cmatch) {
  int64_t resets = 0;
  for (int32_t r = 0; r < nr; ++r)
    if (rmatch[r] == -2) {
      rmatch[r] = -1;
      resets++;
    }
  for (int32_t r = 0; r < nr; ++r) {
    const int32_t c = rmatch[r];
    if (c >= 0 && cmatch[c] != r) {
      rmatch[r] = -1;
      resets++;
    }
  }
  for (int32_t c = 0; c < nc; ++c) {
    const int32_t r = cmatch[c];
    if (r >= 0 && rmatch[r] != c) {
      cmatch[c] = -1;
      resets++;
    }
  }
  return resets;
}

typedef struct phase_result {
  int found;
  int64_t launches, scans, walks, resets;
} phase_result;

static phase_result or_run_phase(const or_graph* g, int32_t tot, int32_t shortest, int32_t kernel,
                                 int32_t improved, int32_t* rmatch, int32_t* cmatch, int32_t* bfs,
                                 int32_t* pred, int32_t* root) {
  const int32_t L0 = 2; /* gpu_match.cpp:275 */
  phase_result res = {0, 0, 0, 0, 0};
  int32_t flags[2] = {1, 0};
  int32_t level = L0;
  or_init_bfs_array(g->nc, cmatch, L0, bfs);
  for (int32_t r = 0; r < g->nr; ++r) pred[r] = -1;
  if (kernel == 1) or_init_root(g->nc, cmatch, root);
  while (flags[0]) { /* expand_bfs, gpu_match.cpp:253-264 */
    flags[0] = 0;
    if (kernel == 0) res.scans += or_gpubfs(g, tot, level, L0, bfs, pred, rmatch, flags);
    else res.scans += or_gpubfs_wr(g, tot, level, L0, improved, bfs, pred, root, rmatch, flags);
    res.launches++;
    if (shortest && flags[1]) break;
    level++;
  }
  if (improved) res.walks = or_alternate_wr(g, tot, bfs, pred, rmatch, cmatch);
  else res.walks = or_alternate(g, tot, pred, rmatch, cmatch);
  res.resets = or_fix_matching(g->nc, g->nr, rmatch, cmatch);
  res.found = flags[1];
  return res;
}

int32_t or_driver(const or_graph* g, int32_t tot, int32_t shortest, int32_t kernel, int32_t improved,
                  int32_t* rmatch, int32_t* cmatch, or_counters* ct) {
  if (improved && kernel != 1) return 2; /* gpu_match.cpp:272-274 */
  const size_t nc1 = (size_t)g->nc + 1, nr1 = (size_t)g->nr + 1;
  int32_t* bfs = (int32_t*)malloc(sizeof(int32_t) * nc1);
  int32_t* root = (int32_t*)malloc(sizeof(int32_t) * nc1);
  int32_t* pred = (int32_t*)malloc(sizeof(int32_t) * nr1);
  or_counters local;
  memset(&local, 0, sizeof(local));
  if (!ct) ct = &local;
  int64_t* launches = ct->launches;
  const int64_t cap = ct->launches_cap;
  memset(ct, 0, sizeof(*ct));
  ct->launches = launches;
  ct->launches_cap = cap;
  const int64_t bound = (int64_t)g->nc + 1;
  int64_t before = or_cardinality(g->nr, rmatch);
  int32_t status = 0;
  for (;;) {
    ct->outer_iterations++;
    if (ct->outer_iterations > bound) { status = 3; break; }
    phase_result ph = or_run_phase(g, tot, shortest, kernel, improved, rmatch, cmatch, bfs, pred, root);
    int64_t it_launches = ph.launches;
    int64_t after = or_cardinality(g->nr, rmatch);
    if (ph.found && after <= before) { /* serial retry, gpu_match.cpp:328-343 */
      phase_result rt = or_run_phase(g, tot, shortest, kernel, improved, rmatch, cmatch, bfs, pred, root);
      it_launches += rt.launches;
      ct->columns_scanned += rt.scans;
      ct->alternations_attempted += rt.walks;
      ct->fix_resets += rt.resets;
      ct->serial_retries++;
      ph.found = rt.found;
      after = or_cardinality(g->nr, rmatch);
    }
    if (ct->launches && ct->outer_iterations - 1 < ct->launches_cap)
      ct->launches[ct->outer_iterations - 1] = it_launches;
    ct->bfs_launches_total += it_launches;
    ct->columns_scanned += ph.scans;
    ct->alternations_attempted += ph.walks;
    ct->fix_resets += ph.resets;
    if (!ph.found) break;
    before = after;
  }
  free(bfs);
  free(root);
  free(pred);
  return status;
}
