// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" harness around the UNMODIFIED reference planner (`libmemplan`,
// compiled from /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libmemplan_ref.so). It lets the Python tests, the golden-vector
// generator and bench.py's reference / cpu_baseline arm call the reference's
// own functions on plain arrays:
//
//   ref_lifetimes_from_order     -> memplan::lifetimes_from_order   (proj/src/schedule.cpp:33-50)
//   ref_resident_bytes_per_step  -> memplan::resident_bytes_per_step (proj/src/schedule.cpp:69-79)
//   ref_peak_resident_bytes      -> memplan::peak_resident_bytes    (proj/src/schedule.cpp:81-88)
//   ref_score_orders             -> peak_resident_bytes per candidate + first-minimum argmin
//   ref_timeline_from_lifetimes  -> memplan::timeline_from_lifetimes (proj/src/plan.cpp:122-143)
//   ref_realized_lifetimes       -> memplan::realized_lifetimes     (proj/src/plan.cpp:101-120)
//   ref_encode_address_pairs     -> memplan::encode_addresses pair loop (proj/src/encode.cpp:347-367)
//   ref_validate_plan            -> memplan::validate_plan          (proj/src/plan.cpp:315-419)
//   ref_greedy_pack              -> memplan::greedy_pack            (proj/src/placement.cpp:182-204)
//   ref_fragmentation            -> memplan::fragmentation          (proj/src/placement.cpp:64-67)
//   ref_enumerate_min_peak       -> memplan::enumerate_min_peak     (proj/src/oracle.cpp:98-110)
//   ref_generate_graph / ref_load_graph / ref_save_graph / ref_graph_csr
//
// Every entry point catches memplan::Error and returns a status code plus the
// exception text (ref_last_error), so a Python caller sees the reference's own
// error class and message.

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <map>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "memplan/encode.hpp"
#include "memplan/errors.hpp"
#include "memplan/generate.hpp"
#include "memplan/graph.hpp"
#include "memplan/graph_io.hpp"
#include "memplan/lp_format.hpp"
#include "memplan/milp.hpp"
#include "memplan/oracle.hpp"
#include "memplan/pipeline.hpp"
#include "memplan/placement.hpp"
#include "memplan/plan.hpp"
#include "memplan/schedule.hpp"

using namespace memplan;

namespace {

thread_local std::string g_last_error;

enum RefStatus : int {
  REF_OK = 0,
  REF_INVALID_ORDER = 1,
  REF_ERROR = 2,         // any other memplan::Error
  REF_CAPACITY = 3,      // caller buffer too small
  REF_UNKNOWN = 4,       // non-memplan exception
};

int fail_from_current() {
  try {
    throw;
  } catch (const InvalidOrder& e) {
    g_last_error = e.what();
    return REF_INVALID_ORDER;
  } catch (const Error& e) {
    g_last_error = e.what();
    return REF_ERROR;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return REF_UNKNOWN;
  }
}

std::vector<NodeIndex> to_order(const int32_t* order, int64_t len) {
  return std::vector<NodeIndex>(order, order + len);
}

std::vector<Interval> to_intervals(const int32_t* lo, const int32_t* hi,
                                   int64_t n) {
  std::vector<Interval> out(n);
  for (int64_t i = 0; i < n; ++i) out[i] = Interval{lo[i], hi[i]};
  return out;
}

int copy_text(const std::string& s, char* buf, int64_t cap, int64_t* len) {
  *len = static_cast<int64_t>(s.size());
  if (buf == nullptr) return REF_OK;
  if (static_cast<int64_t>(s.size()) + 1 > cap) return REF_CAPACITY;
  std::memcpy(buf, s.data(), s.size());
  buf[s.size()] = '\0';
  return REF_OK;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_last_error.c_str(); }

// ---- graph construction / io ---------------------------------------------

int ref_load_graph(const char* text, void** out) {
  try {
    *out = new Graph(load_graph(text));
    return REF_OK;
  } catch (...) {
    return fail_from_current();
  }
}

int ref_generate_graph(int kind, int layers, uint64_t size, uint64_t seed,
                       void** out) {
  try {
    GeneratorSpec spec;
    spec.kind = static_cast<GraphKind>(kind);
    spec.layers = layers;
    spec.size = size;
    spec.seed = seed;
    *out = new Graph(generate_graph(spec));
    return REF_OK;
  } catch (...) {
    return fail_from_current();
  }
}

void ref_graph_free(void* g) { delete static_cast<Graph*>(g); }

int ref_save_graph(const void* g, char* buf, int64_t cap, int64_t* len) {
  try {
    return copy_text(save_graph(*static_cast<const Graph*>(g)), buf, cap, len);
  } catch (...) {
    return fail_from_current();
  }
}

void ref_graph_dims(const void* gp, int32_t* n, int32_t* e, int64_t* s) {
  const Graph& g = *static_cast<const Graph*>(gp);
  *n = g.num_nodes();
  *e = g.num_edges();
  int64_t total = 0;
  for (int i = 0; i < g.num_edges(); ++i) total += g.sinks_of(i).size();
  *s = total;
}

// The reference's own indexing as CSR: edge_src[E], sink_off[E+1],
// sinks[S], size[E], is_control[E].
void ref_graph_csr(const void* gp, int32_t* src, int64_t* sink_off,
                   int32_t* sinks, uint64_t* size, uint8_t* is_control) {
  const Graph& g = *static_cast<const Graph*>(gp);
  int64_t at = 0;
  for (int e = 0; e < g.num_edges(); ++e) {
    src[e] = g.source_of(e);
    sink_off[e] = at;
    for (NodeIndex s : g.sinks_of(e)) sinks[at++] = s;
    size[e] = g.edge(e).size;
    is_control[e] = g.edge(e).kind == EdgeKind::kControl ? 1 : 0;
  }
  sink_off[g.num_edges()] = at;
}

int ref_is_topological_order(const void* gp, const int32_t* order,
                             int64_t len) {
  return is_topological_order(*static_cast<const Graph*>(gp),
                              to_order(order, len))
             ? 1
             : 0;
}

int ref_topological_order(const void* gp, int32_t* out) {
  const Graph& g = *static_cast<const Graph*>(gp);
  std::vector<NodeIndex> order = topological_order(g);
  std::copy(order.begin(), order.end(), out);
  return static_cast<int>(order.size());
}

// ---- hot path: lifetimes / resident bytes / peak --------------------------

int ref_lifetimes_from_order(const void* gp, const int32_t* order, int64_t len,
                             int32_t* lo, int32_t* hi) {
  try {
    std::vector<Interval> lt =
        lifetimes_from_order(*static_cast<const Graph*>(gp), to_order(order, len));
    for (size_t e = 0; e < lt.size(); ++e) {
      lo[e] = lt[e].lo;
      hi[e] = lt[e].hi;
    }
    return REF_OK;
  } catch (...) {
    return fail_from_current();
  }
}

int ref_resident_bytes_per_step(const void* gp, const int32_t* order,
                                int64_t len, uint64_t* out) {
  try {
    std::vector<std::uint64_t> rs = resident_bytes_per_step(
        *static_cast<const Graph*>(gp), to_order(order, len));
    std::copy(rs.begin(), rs.end(), out);
    return REF_OK;
  } catch (...) {
    return fail_from_current();
  }
}

int ref_peak_resident_bytes(const void* gp, const int32_t* order, int64_t len,
                            uint64_t* out) {
  try {
    *out = peak_resident_bytes(*static_cast<const Graph*>(gp),
                               to_order(order, len));
    return REF_OK;
  } catch (...) {
    return fail_from_current();
  }
}

// Candidate scoring the only way the reference can: one peak_resident_bytes
// call per order (proj/src/pipeline.cpp:297-302, proj/tools/memplan_main.cpp:192),
// InvalidOrder mapped to valid=0. Candidates are split statically over
// `threads` host threads (the function is pure). Returns the
// first-minimum index among valid candidates in *best (-1 if none).
int ref_score_orders(const void* gp, const int32_t* orders, int64_t num_orders,
                     int64_t n, uint64_t* peak, uint8_t* valid, int threads,
                     int64_t* best) {
  const Graph& g = *static_cast<const Graph*>(gp);
  if (threads < 1) threads = 1;
  std::vector<std::thread> pool;
  std::atomic<int> status{REF_OK};
  auto work = [&](int t) {
    int64_t begin = num_orders * t / threads;
    int64_t end = num_orders * (t + 1) / threads;
    for (int64_t c = begin; c < end; ++c) {
      try {
        peak[c] = peak_resident_bytes(g, to_order(orders + c * n, n));
        valid[c] = 1;
      } catch (const InvalidOrder&) {
        peak[c] = 0;
        valid[c] = 0;
      } catch (...) {
        status = REF_UNKNOWN;
      }
    }
  };
  for (int t = 1; t < threads; ++t) pool.emplace_back(work, t);
  work(0);
  for (auto& th : pool) th.join();
  int64_t b = -1;
  for (int64_t c = 0; c < num_orders; ++c)
    if (valid[c] && (b < 0 || peak[c] < peak[b])) b = c;
  *best = b;
  return status;
}

// Input preparation for bench.py's reference arm (so that arm never loads the
// product library): seeded random topological orders of a reference Graph,
// randomised Kahn over the (edge, sink) multigraph with one splitmix64 stream
// per candidate - the same draws as mp_random_topo_orders, so both arms score
// identical candidates. Not part of the reference; not timed.
int ref_random_topo_orders(const void* gp, int64_t num_orders, uint64_t seed, int threads,
                           int32_t* out) {
  const Graph& g = *static_cast<const Graph*>(gp);
  const int32_t n = g.num_nodes(), E = g.num_edges();
  std::vector<int32_t> indeg(n, 0), off(n + 1, 0), succ;
  for (int32_t e = 0; e < E; ++e) {
    off[g.source_of(e) + 1] += (int32_t)g.sinks_of(e).size();
    for (NodeIndex s : g.sinks_of(e)) ++indeg[s];
  }
  for (int32_t v = 0; v < n; ++v) off[v + 1] += off[v];
  succ.resize(off[n]);
  {
    std::vector<int32_t> fill(off.begin(), off.end() - 1);
    for (int32_t e = 0; e < E; ++e)
      for (NodeIndex s : g.sinks_of(e)) succ[fill[g.source_of(e)]++] = s;
  }
  std::atomic<int> status{REF_OK};
  auto work = [&](int64_t c0, int64_t c1) {
    std::vector<int32_t> deg, ready;
    for (int64_t c = c0; c < c1; ++c) {
      uint64_t st = seed * 0xD1B54A32D192ED03ull + (uint64_t)c * 0x9E3779B97F4A7C15ull + 1;
      deg = indeg;
      ready.clear();
      for (int32_t v = 0; v < n; ++v)
        if (deg[v] == 0) ready.push_back(v);
      int32_t* row = out + c * (int64_t)n;
      int32_t k = 0;
      while (!ready.empty()) {
        uint64_t z = (st += 0x9E3779B97F4A7C15ull);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z ^= z >> 31;
        const size_t pick = (size_t)(z % ready.size());
        const int32_t v = ready[pick];
        ready[pick] = ready.back();
        ready.pop_back();
        row[k++] = v;
        for (int32_t q = off[v]; q < off[v + 1]; ++q)
          if (--deg[succ[q]] == 0) ready.push_back(succ[q]);
      }
      if (k != n) status = REF_UNKNOWN;
    }
  };
  if (threads < 1) threads = 1;
  if (threads > num_orders) threads = (int)std::max<int64_t>(1, num_orders);
  std::vector<std::thread> pool;
  for (int t = 1; t < threads; ++t)
    pool.emplace_back(work, num_orders * t / threads, num_orders * (t + 1) / threads);
  work(0, num_orders / threads);
  for (auto& th : pool) th.join();
  return status;
}

int ref_timeline_from_lifetimes(const void* gp, const int32_t* lo,
                                const int32_t* hi, int32_t horizon,
                                uint64_t* bytes, uint64_t* peak_rs,
                                int32_t* peak_step) {
  try {
    const Graph& g = *static_cast<const Graph*>(gp);
    ResidentTimeline t =
        timeline_from_lifetimes(g, to_intervals(lo, hi, g.num_edges()), horizon);
    if (bytes) std::copy(t.bytes.begin(), t.bytes.end(), bytes);
    *peak_rs = t.peak_rs;
    *peak_step = t.peak_step;
    return REF_OK;
  } catch (...) {
    return fail_from_current();
  }
}

// timestep_of[v] == 0 means node v is absent from the map.
int ref_realized_lifetimes(const void* gp, const int32_t* timestep_of,
                           int32_t horizon, int32_t* lo, int32_t* hi) {
  try {
    const Graph& g = *static_cast<const Graph*>(gp);
    std::map<std::string, int> steps;
    for (int v = 0; v < g.num_nodes(); ++v)
      if (timestep_of[v] != 0) steps[g.node(v).id] = timestep_of[v];
    std::vector<Interval> lt = realized_lifetimes(g, steps, horizon);
    for (size_t e = 0; e < lt.size(); ++e) {
      lo[e] = lt[e].lo;
      hi[e] = lt[e].hi;
    }
    return REF_OK;
  } catch (...) {
    return fail_from_current();
  }
}

// ---- overlap pairs: the encode_addresses pair loop ------------------------
//
// Runs the real encode_addresses (with or without the edge_precedes filter)
// and reads the emitted pair list back out of the model's below(i,j)
// variables, which are created in pair-emission order (encode.cpp:358-359).
// `pinned[e]` != 0 marks a preplaced edge (offset `pinned_addr[e]`).
// With pairs == nullptr only the count (constraint_counts["live_pair"]) is
// returned.
int ref_encode_address_pairs(const void* gp, const int32_t* lo,
                             const int32_t* hi, const uint8_t* pinned,
                             const uint64_t* pinned_addr, int filter,
                             int32_t* pairs, int64_t cap, int64_t* count) {
  try {
    const Graph& g = *static_cast<const Graph*>(gp);
    std::map<EdgeIndex, std::uint64_t> pre;
    if (pinned)
      for (int e = 0; e < g.num_edges(); ++e)
        if (pinned[e]) pre[e] = pinned_addr ? pinned_addr[e] : 0;
    EncodeOptions opts;
    opts.filter_pairs = filter != 0;
    MilpModel model = encode_addresses(
        g, to_intervals(lo, hi, g.num_edges()), pre, opts);
    auto it = model.constraint_counts.find(kTagLivePair);
    *count = it == model.constraint_counts.end() ? 0 : it->second;
    if (pairs == nullptr) return REF_OK;
    if (*count > cap) return REF_CAPACITY;
    std::map<std::string, EdgeIndex> by_id;
    for (int e = 0; e < g.num_edges(); ++e) by_id[g.edge(e).id] = e;
    int64_t at = 0;
    for (const Variable& v : model.vars) {
      if (v.name.rfind("below(", 0) != 0) continue;
      std::string inner = v.name.substr(6, v.name.size() - 7);
      size_t comma = inner.find(',');
      if (comma == std::string::npos || inner.find(',', comma + 1) != std::string::npos) {
        g_last_error = "ref harness: edge ids containing ',' are unsupported";
        return REF_UNKNOWN;
      }
      pairs[2 * at] = by_id.at(inner.substr(0, comma));
      pairs[2 * at + 1] = by_id.at(inner.substr(comma + 1));
      ++at;
    }
    *count = at;
    return REF_OK;
  } catch (...) {
    return fail_from_current();
  }
}

// The pair loop of encode_joint (encode.cpp:401-408) without the model: data edges
// a < b, skipped when filter_pairs and edge_precedes either way (analysis.cpp:94-113),
// with the reference's compute_bounds and ReachabilityCache. Two-phase like the above.
int ref_joint_pairs(const void* gp, int filter, int32_t* pairs, int64_t cap, int64_t* count) {
  try {
    const Graph& g = *static_cast<const Graph*>(gp);
    const LifetimeBounds bounds = compute_bounds(g);
    ReachabilityCache reach(g);
    std::vector<EdgeIndex> data;
    for (int e = 0; e < g.num_edges(); ++e)
      if (g.edge(e).size > 0) data.push_back(e);
    int64_t at = 0;
    for (size_t a = 0; a < data.size(); ++a)
      for (size_t b = a + 1; b < data.size(); ++b) {
        const EdgeIndex i = data[a], j = data[b];
        if (filter && (edge_precedes(g, bounds, i, j, &reach) ||
                       edge_precedes(g, bounds, j, i, &reach)))
          continue;
        if (pairs && at < cap) {
          pairs[2 * at] = i;
          pairs[2 * at + 1] = j;
        }
        ++at;
      }
    *count = at;
    return pairs && at > cap ? REF_CAPACITY : REF_OK;
  } catch (...) {
    return fail_from_current();
  }
}

// write_lp(encode_addresses(...)) (lp_format.cpp:88-121): the model text
int ref_encode_addresses_lp(const void* gp, const int32_t* lo, const int32_t* hi,
                            const uint8_t* pinned, const uint64_t* pinned_addr, int filter,
                            char* buf, int64_t cap, int64_t* len) {
  try {
    const Graph& g = *static_cast<const Graph*>(gp);
    std::map<EdgeIndex, std::uint64_t> pre;
    if (pinned)
      for (int e = 0; e < g.num_edges(); ++e)
        if (pinned[e]) pre[e] = pinned_addr ? pinned_addr[e] : 0;
    EncodeOptions opts;
    opts.filter_pairs = filter != 0;
    const std::string text =
        write_lp(encode_addresses(g, to_intervals(lo, hi, g.num_edges()), pre, opts));
    return copy_text(text, buf, cap, len);
  } catch (...) {
    return fail_from_current();
  }
}

// ---- validation -------------------------------------------------------------
//
// Builds a MemoryPlan from arrays and runs the reference validate_plan.
//   sequence[seq_len]      node indexes (may repeat / be partial, for tamper tests)
//   timestep_of[n]         0 = node has no timestep entry
//   has_addr[E], addr[E]   address map by edge
// Violations come back as "tag\tdetail\n" lines in buf.
int ref_validate_plan(const void* gp, const int32_t* sequence, int64_t seq_len,
                      const int32_t* timestep_of, const uint8_t* has_addr,
                      const uint64_t* addr, uint64_t peak_mem,
                      uint64_t stored_peak_rs, int32_t stored_peak_step,
                      char* buf, int64_t cap, int64_t* len,
                      int32_t* num_violations) {
  try {
    const Graph& g = *static_cast<const Graph*>(gp);
    MemoryPlan plan;
    for (int64_t i = 0; i < seq_len; ++i)
      plan.sequence.steps.push_back(g.node(sequence[i]).id);
    for (int v = 0; v < g.num_nodes(); ++v)
      if (timestep_of[v] != 0) plan.sequence.timestep_of[g.node(v).id] = timestep_of[v];
    for (int e = 0; e < g.num_edges(); ++e)
      if (has_addr[e]) plan.addresses[g.edge(e).id] = addr[e];
    plan.peak_mem = peak_mem;
    plan.timeline.peak_rs = stored_peak_rs;
    plan.timeline.peak_step = stored_peak_step;
    ValidationReport r = validate_plan(plan, g);
    std::string text;
    for (const auto& v : r.violations) text += v.tag + "\t" + v.detail + "\n";
    *num_violations = static_cast<int32_t>(r.violations.size());
    return copy_text(text, buf, cap, len);
  } catch (...) {
    return fail_from_current();
  }
}

// Lowest-feasible-offset packing (placement.cpp:182-204) with nothing
// preplaced; writes addr[e] for data edges (0 for control edges).
int ref_greedy_pack(const void* gp, const int32_t* lo, const int32_t* hi,
                    uint64_t* addr) {
  try {
    const Graph& g = *static_cast<const Graph*>(gp);
    auto placed = greedy_pack(g, to_intervals(lo, hi, g.num_edges()), {});
    for (int e = 0; e < g.num_edges(); ++e) addr[e] = 0;
    for (const auto& [e, a] : placed) addr[e] = a;
    return REF_OK;
  } catch (...) {
    return fail_from_current();
  }
}

// preallocate_pyramid (placement.cpp:25-62): taken/addr per edge, reserved_base
int ref_preallocate_pyramid(const void* gp, const int32_t* lo, const int32_t* hi, uint8_t* taken,
                            uint64_t* addr, uint64_t* reserved_base) {
  try {
    const Graph& g = *static_cast<const Graph*>(gp);
    PrePlacement pre = preallocate_pyramid(g, to_intervals(lo, hi, g.num_edges()));
    for (int e = 0; e < g.num_edges(); ++e) {
      taken[e] = 0;
      addr[e] = 0;
    }
    for (const auto& [e, a] : pre.assigned) {
      taken[e] = 1;
      addr[e] = a;
    }
    *reserved_base = pre.reserved_base;
    return REF_OK;
  } catch (...) {
    return fail_from_current();
  }
}

// greedy_pack with a preplaced map (fixed[e] != 0 -> fixed_addr[e]); has[e] = in the result
int ref_greedy_pack_fixed(const void* gp, const int32_t* lo, const int32_t* hi,
                          const uint8_t* fixed, const uint64_t* fixed_addr, uint64_t* addr,
                          uint8_t* has) {
  try {
    const Graph& g = *static_cast<const Graph*>(gp);
    std::map<EdgeIndex, std::uint64_t> pre;
    for (int e = 0; e < g.num_edges(); ++e)
      if (fixed && fixed[e]) pre[e] = fixed_addr[e];
    auto placed = greedy_pack(g, to_intervals(lo, hi, g.num_edges()), pre);
    for (int e = 0; e < g.num_edges(); ++e) {
      addr[e] = 0;
      has[e] = 0;
    }
    for (const auto& [e, a] : placed) {
      addr[e] = a;
      has[e] = 1;
    }
    return REF_OK;
  } catch (...) {
    return fail_from_current();
  }
}

// run_baseline (placement.cpp:150-180)
int ref_run_baseline(const void* gp, const int32_t* order, int64_t len, int best_fit,
                     uint64_t* mr_peak, uint64_t* rs_at_peak, double* frag) {
  try {
    const Graph& g = *static_cast<const Graph*>(gp);
    BaselineResult r = run_baseline(g, to_order(order, len),
                                    best_fit ? FitPolicy::kBestFit : FitPolicy::kFirstFit);
    *mr_peak = r.mr_peak;
    *rs_at_peak = r.rs_at_peak;
    *frag = r.fragmentation;
    return REF_OK;
  } catch (...) {
    return fail_from_current();
  }
}

double ref_fragmentation(uint64_t mr, uint64_t rs) {
  return fragmentation(mr, rs);
}

int ref_enumerate_min_peak(const void* gp, uint64_t* min_peak, int32_t* order) {
  try {
    PeakWitness w = enumerate_min_peak(*static_cast<const Graph*>(gp));
    *min_peak = w.min_peak;
    std::copy(w.order.begin(), w.order.end(), order);
    return REF_OK;
  } catch (...) {
    return fail_from_current();
  }
}

// Full reference planner on a graph (internal solvers only); returns the
// canonical plan file text (plan.cpp:205-231) for golden fixtures.
int ref_plan_graph(const void* gp, char* buf, int64_t cap, int64_t* len) {
  try {
    PlanResult r = plan_graph(*static_cast<const Graph*>(gp));
    return copy_text(save_plan(r.plan), buf, cap, len);
  } catch (...) {
    return fail_from_current();
  }
}

}  // extern "C"
