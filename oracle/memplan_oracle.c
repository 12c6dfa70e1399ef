/* TEST INFRASTRUCTURE ONLY — see memplan_oracle.h. Plain-C restatement of
 * the reference planner's hot path; every function cites the reference
 * file:line it restates. Compiled by oracle/Makefile into
 * oracle/_build/liboracle.so. Deliberately scalar and literal: it mirrors
 * the reference loops (including their complexity) rather than the GPU
 * algorithms, so an agreement between the two is evidence, not tautology.
 */
#include "memplan_oracle.h"

#include <stdlib.h>
#include <string.h>

/* graph.cpp:239-254: length n, each node once and in range, every sink of
 * every edge (data and control) strictly after its source. */
int or_is_topological_order(const or_graph* g, const int32_t* order, int64_t len) {
  if (len != g->n) return 0;
  int32_t* pos = (int32_t*)malloc(sizeof(int32_t) * (size_t)(g->n > 0 ? g->n : 1));
  for (int32_t v = 0; v < g->n; ++v) pos[v] = -1;
  int ok = 1;
  for (int64_t i = 0; i < len && ok; ++i) {
    int32_t v = order[i];
    if (v < 0 || v >= g->n || pos[v] != -1) ok = 0;
    else pos[v] = (int32_t)i;
  }
  for (int32_t e = 0; e < g->num_edges && ok; ++e) {
    int32_t s0 = pos[g->edge_src[e]];
    for (int64_t k = g->sink_off[e]; k < g->sink_off[e + 1]; ++k)
      if (pos[g->sinks[k]] <= s0) { ok = 0; break; }
  }
  free(pos);
  return ok;
}

/* schedule.cpp:23-31 */
int or_positions_of(const or_graph* g, const int32_t* order, int64_t len, int32_t* pos) {
  if (!or_is_topological_order(g, order, len)) return 1; /* InvalidOrder */
  for (int32_t v = 0; v < g->n; ++v) pos[v] = 0;
  for (int64_t i = 0; i < len; ++i) pos[order[i]] = (int32_t)i + 1;
  return 0;
}

/* schedule.cpp:33-50 */
int or_lifetimes_from_order(const or_graph* g, const int32_t* order, int64_t len,
                            int32_t* lo, int32_t* hi) {
  int32_t* pos = (int32_t*)malloc(sizeof(int32_t) * (size_t)(g->n > 0 ? g->n : 1));
  if (or_positions_of(g, order, len, pos)) { free(pos); return 1; }
  for (int32_t e = 0; e < g->num_edges; ++e) {
    lo[e] = pos[g->edge_src[e]];
    hi[e] = lo[e];
    if (g->sink_off[e] == g->sink_off[e + 1]) {
      hi[e] = g->n;
    } else {
      for (int64_t k = g->sink_off[e]; k < g->sink_off[e + 1]; ++k)
        if (pos[g->sinks[k]] > hi[e]) hi[e] = pos[g->sinks[k]];
    }
  }
  free(pos);
  return 0;
}

/* schedule.cpp:69-79 — the literal per-timestep accumulation. */
int or_resident_bytes_per_step(const or_graph* g, const int32_t* order, int64_t len,
                               uint64_t* out) {
  int32_t E = g->num_edges;
  int32_t* lo = (int32_t*)malloc(sizeof(int32_t) * (size_t)(E > 0 ? E : 1));
  int32_t* hi = (int32_t*)malloc(sizeof(int32_t) * (size_t)(E > 0 ? E : 1));
  if (or_lifetimes_from_order(g, order, len, lo, hi)) { free(lo); free(hi); return 1; }
  for (int32_t t = 0; t < g->n; ++t) out[t] = 0;
  for (int32_t e = 0; e < E; ++e)
    for (int32_t t = lo[e]; t <= hi[e]; ++t) out[t - 1] += g->edge_size[e];
  free(lo);
  free(hi);
  return 0;
}

/* schedule.cpp:81-88 */
int or_peak_resident_bytes(const or_graph* g, const int32_t* order, int64_t len,
                           uint64_t* peak) {
  uint64_t* rs = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(g->n > 0 ? g->n : 1));
  if (or_resident_bytes_per_step(g, order, len, rs)) { free(rs); return 1; }
  uint64_t best = 0;
  for (int32_t t = 0; t < g->n; ++t) if (rs[t] > best) best = rs[t];
  *peak = best;
  free(rs);
  return 0;
}

/* plan.cpp:122-143 (bytes, peak_rs, peak_step; the per-step live id lists
 * are not restated). contains(t) is lo <= t <= hi (analysis.hpp:31-32). */
void or_timeline_from_lifetimes(const or_graph* g, const int32_t* lo, const int32_t* hi,
                                int32_t horizon, uint64_t* bytes, uint64_t* peak_rs,
                                int32_t* peak_step) {
  uint64_t best = 0;
  int32_t best_t = 0;
  for (int32_t t = 1; t <= horizon; ++t) {
    uint64_t b = 0;
    for (int32_t e = 0; e < g->num_edges; ++e)
      if (lo[e] <= t && t <= hi[e]) b += g->edge_size[e];
    if (bytes) bytes[t - 1] = b;
    if (b > best) { best = b; best_t = t; }
  }
  if (horizon > 0 && best_t == 0) best_t = 1;
  *peak_rs = best;
  *peak_step = best_t;
}

/* plan.cpp:101-120: source first, then sinks in declaration order; the
 * first node without a timestep raises InvalidOrder. */
int or_realized_lifetimes(const or_graph* g, const int32_t* timestep_of, int32_t horizon,
                          int32_t* lo, int32_t* hi, int32_t* missing) {
  for (int32_t e = 0; e < g->num_edges; ++e) {
    int32_t s = g->edge_src[e];
    if (timestep_of[s] == 0) { *missing = s; return 1; }
    int32_t l = timestep_of[s];
    int32_t h = g->sink_off[e] == g->sink_off[e + 1] ? horizon : l;
    for (int64_t k = g->sink_off[e]; k < g->sink_off[e + 1]; ++k) {
      int32_t w = g->sinks[k];
      if (timestep_of[w] == 0) { *missing = w; return 1; }
      if (timestep_of[w] > h) h = timestep_of[w];
    }
    lo[e] = l;
    hi[e] = h;
  }
  return 0;
}

/* analysis.hpp:28-37 */
static int disjoint(int32_t alo, int32_t ahi, int32_t blo, int32_t bhi) {
  return alo > ahi || blo > bhi || ahi < blo || bhi < alo;
}

static int pair_live(const int32_t* lo, const int32_t* hi, const uint64_t* size,
                     const uint8_t* pinned, int32_t i, int32_t j) {
  if (size[i] == 0 || size[j] == 0) return 0;             /* encode.cpp:329-331 */
  if (pinned && pinned[i] && pinned[j]) return 0;          /* encode.cpp:351 */
  return !disjoint(lo[i], hi[i], lo[j], hi[j]);            /* encode.cpp:354 */
}

/* encode.cpp:347-367 pair enumeration order: data edges a<b in edge-index
 * order. */
int64_t or_overlap_pairs(int32_t num_edges, const int32_t* lo, const int32_t* hi,
                         const uint64_t* size, const uint8_t* pinned,
                         int32_t* pairs, int64_t cap) {
  int64_t count = 0;
  for (int32_t i = 0; i < num_edges; ++i)
    for (int32_t j = i + 1; j < num_edges; ++j) {
      if (!pair_live(lo, hi, size, pinned, i, j)) continue;
      if (pairs && count < cap) {
        pairs[2 * count] = i;
        pairs[2 * count + 1] = j;
      }
      ++count;
    }
  return count;
}

void or_overlap_row_stats(int32_t num_edges, const int32_t* lo, const int32_t* hi,
                          const uint64_t* size, const uint8_t* pinned,
                          int64_t row_begin, int64_t row_end,
                          int64_t* row_count, uint64_t* row_hash) {
  for (int64_t i = row_begin; i < row_end; ++i) {
    int64_t c = 0;
    uint64_t h = 1469598103934665603ull;
    for (int32_t j = (int32_t)i + 1; j < num_edges; ++j) {
      if (!pair_live(lo, hi, size, pinned, (int32_t)i, j)) continue;
      ++c;
      h = (h ^ (uint64_t)(uint32_t)j) * 1099511628211ull;
    }
    row_count[i - row_begin] = c;
    row_hash[i - row_begin] = h;
  }
}

/* plan.cpp:390-404 */
int64_t or_validate_pairs(int32_t num_edges, const int32_t* lo, const int32_t* hi,
                          const uint64_t* size, const uint8_t* has_addr,
                          const uint64_t* addr, int32_t* viol, int64_t cap) {
  int64_t count = 0;
  for (int32_t i = 0; i < num_edges; ++i) {
    if (size[i] == 0 || !has_addr[i]) continue;
    for (int32_t j = i + 1; j < num_edges; ++j) {
      if (size[j] == 0 || !has_addr[j]) continue;
      if (disjoint(lo[i], hi[i], lo[j], hi[j])) continue;
      uint64_t a_lo = addr[i], b_lo = addr[j];
      if (a_lo < b_lo + size[j] && b_lo < a_lo + size[i]) {
        if (viol && count < cap) {
          viol[2 * count] = i;
          viol[2 * count + 1] = j;
        }
        ++count;
      }
    }
  }
  return count;
}

/* pipeline.cpp:146-160 (iterates the address map, i.e. edges with an
 * address in index order). */
int or_addresses_feasible(int32_t num_edges, const int32_t* lo, const int32_t* hi,
                          const uint64_t* size, const uint8_t* has_addr,
                          const uint64_t* addr) {
  for (int32_t i = 0; i < num_edges; ++i) {
    if (!has_addr[i]) continue;
    for (int32_t j = i + 1; j < num_edges; ++j) {
      if (!has_addr[j]) continue;
      if (disjoint(lo[i], hi[i], lo[j], hi[j])) continue;
      if (addr[i] < addr[j] + size[j] && addr[j] < addr[i] + size[i]) return 0;
    }
  }
  return 1;
}

/* placement.cpp:64-67 */
double or_fragmentation(uint64_t mr, uint64_t rs) {
  if (mr == 0) return 0.0;
  return (double)(mr - rs) / (double)mr;
}

/* pipeline.cpp:270-275 */
uint64_t or_peak_mem(int32_t num_edges, const uint64_t* size, const uint8_t* has_addr,
                     const uint64_t* addr) {
  uint64_t peak = 0;
  for (int32_t e = 0; e < num_edges; ++e)
    if (has_addr[e] && addr[e] + size[e] > peak) peak = addr[e] + size[e];
  return peak;
}

/* placement.cpp:25-62, literally: repeatedly the longest-lived data edge whose
 * lifetime fits strictly inside the window (ties: larger size, then smaller id),
 * stacked at the next base; the window shrinks to its lifetime. */
uint64_t or_preallocate_pyramid(int32_t num_edges, const int32_t* lo, const int32_t* hi,
                                const uint64_t* size, const int32_t* id_rank, uint8_t* taken,
                                uint64_t* addr) {
  uint64_t base = 0;
  int64_t min_start = 0, max_end = INT64_MAX;
  for (int32_t e = 0; e < num_edges; ++e) taken[e] = 0;
  while (max_end > min_start) {
    int32_t pick = -1;
    for (int32_t e = 0; e < num_edges; ++e) {
      if (taken[e] || size[e] == 0) continue;
      if (lo[e] <= min_start || hi[e] >= max_end) continue;
      if (pick < 0) {
        pick = e;
        continue;
      }
      const int d_new = hi[e] - lo[e], d_old = hi[pick] - lo[pick];
      if (d_new != d_old) {
        if (d_new > d_old) pick = e;
      } else if (size[e] != size[pick]) {
        if (size[e] > size[pick]) pick = e;
      } else if (id_rank[e] < id_rank[pick]) {
        pick = e;
      }
    }
    if (pick < 0) break;
    taken[pick] = 1;
    addr[pick] = base;
    base += size[pick];
    min_start = lo[pick];
    max_end = hi[pick];
  }
  return base;
}

/* analysis.hpp:28-37 */
static int or_disjoint(int32_t alo, int32_t ahi, int32_t blo, int32_t bhi) {
  return alo > ahi || blo > bhi || ahi < blo || bhi < alo;
}

/* placement.cpp:182-204, literally: for each data edge not preplaced, in edge
 * order, start at 0 and bump past every placed, lifetime-overlapping tensor
 * whose range intersects, until a full pass moves nothing. `placed` is a
 * std::map, iterated in edge-index order. */
void or_greedy_pack(int32_t num_edges, const int32_t* lo, const int32_t* hi, const uint64_t* size,
                    const uint8_t* fixed, uint64_t* addr, uint8_t* has) {
  for (int32_t e = 0; e < num_edges; ++e) has[e] = fixed && fixed[e] ? 1 : 0;
  for (int32_t e = 0; e < num_edges; ++e) {
    if (size[e] == 0 || has[e]) continue;
    uint64_t at = 0;
    int moved = 1;
    while (moved) {
      moved = 0;
      for (int32_t w = 0; w < num_edges; ++w) {
        if (!has[w]) continue;
        if (or_disjoint(lo[e], hi[e], lo[w], hi[w])) continue;
        const uint64_t w_top = addr[w] + size[w];
        if (at < w_top && addr[w] < at + size[e]) {
          at = w_top;
          moved = 1;
        }
      }
    }
    addr[e] = at;
    has[e] = 1;
  }
}

/* ---- run_baseline (placement.cpp:69-180) ------------------------------------ */
typedef struct {
  uint64_t addr, size;
  int free_;
  int32_t edge;
} or_block;

typedef struct {
  or_block* b;
  int64_t n, cap;
} or_arena;

static void or_arena_insert(or_arena* a, int64_t at, or_block blk) {
  if (a->n == a->cap) {
    a->cap = a->cap ? 2 * a->cap : 16;
    a->b = (or_block*)realloc(a->b, (size_t)a->cap * sizeof(or_block));
  }
  memmove(a->b + at + 1, a->b + at, (size_t)(a->n - at) * sizeof(or_block));
  a->b[at] = blk;
  ++a->n;
}

static void or_arena_erase(or_arena* a, int64_t at) {
  memmove(a->b + at, a->b + at + 1, (size_t)(a->n - at - 1) * sizeof(or_block));
  --a->n;
}

static uint64_t or_arena_top(const or_arena* a) {
  return a->n ? a->b[a->n - 1].addr + a->b[a->n - 1].size : 0;
}

/* Arena::allocate (placement.cpp:80-101) and grow (:117-128) */
static void or_arena_allocate(or_arena* a, int32_t edge, uint64_t size, int best_fit) {
  int64_t pick = -1;
  for (int64_t i = 0; i < a->n; ++i) {
    if (!a->b[i].free_ || a->b[i].size < size) continue;
    if (!best_fit) {
      pick = i;
      break;
    }
    if (pick < 0 || a->b[i].size < a->b[pick].size) pick = i;
  }
  if (pick < 0) {
    if (a->n && a->b[a->n - 1].free_) {
      or_block* last = &a->b[a->n - 1];
      last->size = size;
      last->free_ = 0;
      last->edge = edge;
      return;
    }
    or_block nb = {or_arena_top(a), size, 0, edge};
    or_arena_insert(a, a->n, nb);
    return;
  }
  const uint64_t addr = a->b[pick].addr;
  if (a->b[pick].size > size) {
    or_block rest = {addr + size, a->b[pick].size - size, 1, -1};
    a->b[pick].size = size;
    or_arena_insert(a, pick + 1, rest);
  }
  a->b[pick].free_ = 0;
  a->b[pick].edge = edge;
}

/* Arena::release (:103-111) + coalesce (:130-139) */
static void or_arena_release(or_arena* a, int32_t edge) {
  for (int64_t i = 0; i < a->n; ++i) {
    if (a->b[i].free_ || a->b[i].edge != edge) continue;
    a->b[i].free_ = 1;
    a->b[i].edge = -1;
    if (i + 1 < a->n && a->b[i + 1].free_) {
      a->b[i].size += a->b[i + 1].size;
      or_arena_erase(a, i + 1);
    }
    if (i > 0 && a->b[i - 1].free_) {
      a->b[i - 1].size += a->b[i].size;
      or_arena_erase(a, i);
    }
    return;
  }
}

int or_run_baseline(const or_graph* g, const int32_t* order, int64_t len, int best_fit,
                    uint64_t* mr_peak, uint64_t* rs_at_peak, double* frag) {
  const int32_t n = g->n, E = g->num_edges;
  int32_t* lo = (int32_t*)malloc(sizeof(int32_t) * (E ? E : 1));
  int32_t* hi = (int32_t*)malloc(sizeof(int32_t) * (E ? E : 1));
  if (or_lifetimes_from_order(g, order, len, lo, hi)) {
    free(lo);
    free(hi);
    return 1;
  }
  /* frees[t]: data edges whose hi + 1 == t, in edge order (placement.cpp:155-158) */
  int64_t* off = (int64_t*)calloc((size_t)n + 3, sizeof(int64_t));
  int32_t* lst = (int32_t*)malloc(sizeof(int32_t) * (E ? E : 1));
  for (int32_t e = 0; e < E; ++e)
    if (g->edge_size[e] > 0) ++off[hi[e] + 1 + 1];
  for (int32_t t = 0; t <= n + 1; ++t) off[t + 1] += off[t];
  {
    int64_t* cur = (int64_t*)malloc(sizeof(int64_t) * ((size_t)n + 2));
    memcpy(cur, off, sizeof(int64_t) * ((size_t)n + 2));
    for (int32_t e = 0; e < E; ++e)
      if (g->edge_size[e] > 0) lst[cur[hi[e] + 1]++] = e;
    free(cur);
  }
  or_arena a = {0, 0, 0};
  uint64_t live = 0, mr = 0, rs = 0;
  for (int32_t t = 1; t <= n; ++t) {
    for (int64_t q = off[t]; q < off[t + 1]; ++q) {
      or_arena_release(&a, lst[q]);
      live -= g->edge_size[lst[q]];
    }
    const int32_t v = order[t - 1];
    for (int32_t e = 0; e < E; ++e) {  /* fanout(v) in edge order */
      if (g->edge_src[e] != v || g->edge_size[e] == 0) continue;
      or_arena_allocate(&a, e, g->edge_size[e], best_fit);
      live += g->edge_size[e];
      if (or_arena_top(&a) > mr) {
        mr = or_arena_top(&a);
        rs = live;
      }
    }
  }
  *mr_peak = mr;
  *rs_at_peak = rs;
  *frag = or_fragmentation(mr, rs);
  free(a.b);
  free(off);
  free(lst);
  free(lo);
  free(hi);
  return 0;
}

/* ---- encode_joint's pair set (encode.cpp:401-408, analysis.cpp:11-113) ---------- */
typedef struct {
  const or_graph* g;
  int32_t* fanin_off; /* per node: edges whose sink list holds it */
  int32_t* fanin;
  int8_t* memo;       /* [n*n]: 0 unknown, 1 reaches, 2 does not */
} or_reach;

/* ReachabilityCache::reaches (analysis.cpp:79-92): ancestor is a proper ancestor of v */
static int or_reaches(or_reach* r, int32_t ancestor, int32_t v) {
  if (ancestor == v) return 0;
  int8_t* m = &r->memo[(size_t)ancestor * r->g->n + v];
  if (*m) return *m == 1;
  int found = 0;
  for (int32_t q = r->fanin_off[v]; q < r->fanin_off[v + 1] && !found; ++q) {
    const int32_t src = r->g->edge_src[r->fanin[q]];
    if (src == ancestor || or_reaches(r, ancestor, src)) found = 1;
  }
  *m = found ? 1 : 2;
  return found;
}

/* edge_precedes (analysis.cpp:94-113), literally */
static int or_edge_precedes(const or_graph* g, const int32_t* mul_lo, const int32_t* mul_hi,
                            or_reach* r, int32_t e1, int32_t e2) {
  if (or_disjoint(mul_lo[e1], mul_hi[e1], mul_lo[e2], mul_hi[e2])) return 1;
  const int64_t a = g->sink_off[e1], b = g->sink_off[e1 + 1];
  if (a == b) return 0;
  const int32_t src2 = g->edge_src[e2];
  for (int64_t k = a; k < b; ++k)
    if (!or_reaches(r, g->sinks[k], src2)) return 0;
  /* ends1 = sinks(e1) + src(e1) */
  if (src2 == g->edge_src[e1]) return 0;
  for (int64_t k = a; k < b; ++k)
    if (g->sinks[k] == src2) return 0;
  for (int64_t q = g->sink_off[e2]; q < g->sink_off[e2 + 1]; ++q) {
    const int32_t s = g->sinks[q];
    if (s == g->edge_src[e1]) return 0;
    for (int64_t k = a; k < b; ++k)
      if (g->sinks[k] == s) return 0;
  }
  return 1;
}

int64_t or_joint_pairs(const or_graph* g, int filter, int32_t* pairs, int64_t cap) {
  const int32_t n = g->n, E = g->num_edges;
  int32_t* mul_lo = (int32_t*)malloc(sizeof(int32_t) * (E ? E : 1));
  int32_t* mul_hi = (int32_t*)malloc(sizeof(int32_t) * (E ? E : 1));
  or_reach r = {g, (int32_t*)calloc((size_t)n + 1, sizeof(int32_t)), NULL,
                (int8_t*)calloc((size_t)n * (n ? n : 1), 1)};
  /* compute_levels / compute_bounds (analysis.cpp:11-62) over a Kahn order */
  int32_t* order = (int32_t*)malloc(sizeof(int32_t) * (n ? n : 1));
  int32_t* indeg = (int32_t*)calloc((size_t)n + 1, sizeof(int32_t));
  int32_t* fwd = (int32_t*)calloc((size_t)n + 1, sizeof(int32_t));
  int32_t* bwd = (int32_t*)calloc((size_t)n + 1, sizeof(int32_t));
  for (int64_t k = 0; k < g->sink_off[E]; ++k) ++indeg[g->sinks[k]];
  for (int32_t e = 0; e < E; ++e)
    for (int64_t k = g->sink_off[e]; k < g->sink_off[e + 1]; ++k) ++r.fanin_off[g->sinks[k] + 1];
  for (int32_t v = 0; v < n; ++v) r.fanin_off[v + 1] += r.fanin_off[v];
  r.fanin = (int32_t*)malloc(sizeof(int32_t) * (size_t)(r.fanin_off[n] ? r.fanin_off[n] : 1));
  {
    int32_t* cur = (int32_t*)malloc(sizeof(int32_t) * (n ? n : 1));
    for (int32_t v = 0; v < n; ++v) cur[v] = r.fanin_off[v];
    for (int32_t e = 0; e < E; ++e)
      for (int64_t k = g->sink_off[e]; k < g->sink_off[e + 1]; ++k) r.fanin[cur[g->sinks[k]]++] = e;
    free(cur);
  }
  int32_t head = 0, tail = 0;
  for (int32_t v = 0; v < n; ++v)
    if (!indeg[v]) order[tail++] = v;
  while (head < tail) {
    const int32_t v = order[head++];
    for (int32_t e = 0; e < E; ++e) {
      if (g->edge_src[e] != v) continue;
      for (int64_t k = g->sink_off[e]; k < g->sink_off[e + 1]; ++k)
        if (--indeg[g->sinks[k]] == 0) order[tail++] = g->sinks[k];
    }
  }
  int64_t at = -1;
  if (tail == n) {
    for (int32_t i = 0; i < n; ++i) {  /* forward: longest edge count from a source */
      const int32_t v = order[i];
      for (int32_t q = r.fanin_off[v]; q < r.fanin_off[v + 1]; ++q) {
        const int32_t src = g->edge_src[r.fanin[q]];
        if (fwd[src] + 1 > fwd[v]) fwd[v] = fwd[src] + 1;
      }
    }
    for (int32_t i = n - 1; i >= 0; --i) {  /* backward: longest edge count to a terminal */
      const int32_t v = order[i];
      for (int32_t e = 0; e < E; ++e) {
        if (g->edge_src[e] != v) continue;
        for (int64_t k = g->sink_off[e]; k < g->sink_off[e + 1]; ++k)
          if (bwd[g->sinks[k]] + 1 > bwd[v]) bwd[v] = bwd[g->sinks[k]] + 1;
      }
    }
    for (int32_t e = 0; e < E; ++e) {  /* mul = [asap(src), max alap(sinks) or n] */
      int32_t hi = n;
      if (g->sink_off[e + 1] > g->sink_off[e]) {
        hi = 0;
        for (int64_t k = g->sink_off[e]; k < g->sink_off[e + 1]; ++k)
          if (n - bwd[g->sinks[k]] > hi) hi = n - bwd[g->sinks[k]];
      }
      mul_lo[e] = 1 + fwd[g->edge_src[e]];
      mul_hi[e] = hi;
    }
    at = 0;
    for (int32_t i = 0; i < E; ++i) {
      if (g->edge_size[i] == 0) continue;
      for (int32_t j = i + 1; j < E; ++j) {
        if (g->edge_size[j] == 0) continue;
        if (filter && (or_edge_precedes(g, mul_lo, mul_hi, &r, i, j) ||
                       or_edge_precedes(g, mul_lo, mul_hi, &r, j, i)))
          continue;
        if (pairs && at < cap) {
          pairs[2 * at] = i;
          pairs[2 * at + 1] = j;
        }
        ++at;
      }
    }
  }
  free(mul_lo); free(mul_hi); free(order); free(indeg); free(fwd); free(bwd);
  free(r.fanin_off); free(r.fanin); free(r.memo);
  return at;
}
