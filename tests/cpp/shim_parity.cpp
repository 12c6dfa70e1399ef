// GPU parity of the C++ drop-in shim (include/memplan_b200.hpp) against the
// reference library itself (compiled from /root/reference by oracle/Makefile),
// both called with the reference's own memplan::Graph. Run by
// tests/test_gpu_cpp_shim.py on a B200:
//
//   shim_parity <graph.json>...   (fixture texts written out by the pytest)
//
// Prints "OK <checks>" and exits 0, or the first mismatch and exits 1.
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "memplan/encode.hpp"
#include "memplan/errors.hpp"
#include "memplan/lp_format.hpp"
#include "memplan/generate.hpp"
#include "memplan/graph.hpp"
#include "memplan/graph_io.hpp"
#include "memplan/pipeline.hpp"
#include "memplan/placement.hpp"
#include "memplan/plan.hpp"
#include "memplan/schedule.hpp"
#include "memplan_b200.hpp"

using namespace memplan;

static long g_checks = 0;

#define EXPECT(cond, what)                                         \
  do {                                                             \
    ++g_checks;                                                    \
    if (!(cond)) {                                                 \
      std::printf("MISMATCH %s at %s:%d\n", what, __FILE__, __LINE__); \
      std::exit(1);                                                \
    }                                                              \
  } while (0)

static bool same(const std::vector<Interval>& a, const std::vector<Interval>& b) {
  if (a.size() != b.size()) return false;
  for (size_t i = 0; i < a.size(); ++i)
    if (a[i].lo != b[i].lo || a[i].hi != b[i].hi) return false;
  return true;
}

static std::vector<NodeIndex> random_topo(const Graph& g, std::mt19937_64& rng) {
  std::vector<int> indeg(g.num_nodes(), 0);
  for (int e = 0; e < g.num_edges(); ++e)
    for (int s : g.sinks_of(e)) ++indeg[s];
  std::vector<NodeIndex> ready, out;
  for (int v = 0; v < g.num_nodes(); ++v)
    if (!indeg[v]) ready.push_back(v);
  while (!ready.empty()) {
    size_t i = rng() % ready.size();
    NodeIndex v = ready[i];
    ready[i] = ready.back();
    ready.pop_back();
    out.push_back(v);
    for (EdgeIndex e : g.fanout(v))
      for (int s : g.sinks_of(e))
        if (--indeg[s] == 0) ready.push_back(s);
  }
  return out;
}

// The pair list encode_addresses emits, read back from its below(i,j) vars.
static std::vector<std::pair<int, int>> ref_pairs(const Graph& g, const std::vector<Interval>& lt,
                                                  const std::map<EdgeIndex, std::uint64_t>& pre) {
  MilpModel m = encode_addresses(g, lt, pre);
  std::map<std::string, int> by_id;
  for (int e = 0; e < g.num_edges(); ++e) by_id[g.edge(e).id] = e;
  std::vector<std::pair<int, int>> out;
  for (const Variable& v : m.vars) {
    if (v.name.rfind("below(", 0) != 0) continue;
    const std::string inner = v.name.substr(6, v.name.size() - 7);
    const size_t comma = inner.find(',');
    out.push_back({by_id.at(inner.substr(0, comma)), by_id.at(inner.substr(comma + 1))});
  }
  return out;
}

template <typename F>
static std::string error_of(F&& f) {
  try {
    f();
  } catch (const Error& e) {
    return e.what();
  }
  return "";
}

static void check_graph(memplan_b200::Planner& dev, const Graph& g, std::mt19937_64& rng) {
  std::vector<std::vector<NodeIndex>> orders;
  std::vector<NodeIndex> program(g.num_nodes());
  for (int v = 0; v < g.num_nodes(); ++v) program[v] = v;
  if (is_topological_order(g, program)) orders.push_back(program);
  for (int i = 0; i < 6; ++i) orders.push_back(random_topo(g, rng));
  if (g.num_nodes() >= 2) {  // invalid candidates
    auto bad = orders.back();
    std::swap(bad.front(), bad.back());
    orders.push_back(bad);
    auto dup = orders.front();
    dup[1] = dup[0];
    orders.push_back(dup);
  }
  orders.push_back(std::vector<NodeIndex>(g.num_nodes() + 1, 0));  // wrong length

  int64_t best = -2;
  auto scores = dev.score_orders(g, orders, &best);
  int64_t ref_best = -1;
  std::uint64_t ref_best_peak = 0;
  for (size_t c = 0; c < orders.size(); ++c) {
    const auto& o = orders[c];
    const std::string ref_err = error_of([&] { lifetimes_from_order(g, o); });
    const std::string dev_err = error_of([&] { dev.lifetimes_from_order(g, o); });
    if (ref_err != dev_err)
      std::printf("graph n=%d E=%d candidate %zu: ref='%s' dev='%s'\n", g.num_nodes(),
                  g.num_edges(), c, ref_err.c_str(), dev_err.c_str());
    EXPECT(ref_err == dev_err, "lifetimes_from_order error text");
    EXPECT(scores[c].valid == ref_err.empty(), "score verdict");
    if (!ref_err.empty()) {
      EXPECT(error_of([&] { dev.peak_resident_bytes(g, o); }) == ref_err, "peak error text");
      if ((int)o.size() == g.num_nodes())
        EXPECT(error_of([&] { dev.run_baseline(g, o); }) ==
                   error_of([&] { run_baseline(g, o); }),
               "run_baseline error text");
      continue;
    }
    const auto lt = lifetimes_from_order(g, o);
    EXPECT(same(lt, dev.lifetimes_from_order(g, o)), "lifetimes");
    EXPECT(positions_of(g, o) == dev.positions_of(g, o), "positions");
    EXPECT(resident_bytes_per_step(g, o) == dev.resident_bytes_per_step(g, o), "resident bytes");
    const std::uint64_t pk = peak_resident_bytes(g, o);
    EXPECT(pk == dev.peak_resident_bytes(g, o), "peak");
    EXPECT(scores[c].peak == pk, "batched peak");
    const ResidentTimeline rt = timeline_from_lifetimes(g, lt, g.num_nodes());
    const ResidentTimeline dt = dev.timeline_from_lifetimes(g, lt, g.num_nodes());
    EXPECT(rt.bytes == dt.bytes && rt.peak_rs == dt.peak_rs && rt.peak_step == dt.peak_step,
           "timeline");
    EXPECT(rt.live == dt.live, "timeline live lists");
    EXPECT(scores[c].peak_step == rt.peak_step, "batched peak_step");
    if (ref_best < 0 || pk < ref_best_peak) {
      ref_best = (int64_t)c;
      ref_best_peak = pk;
    }
    // overlap pairs == encode_addresses' pair set (filter on)
    EXPECT(ref_pairs(g, lt, {}) == dev.overlap_pairs(g, lt), "overlap pairs");
    std::map<EdgeIndex, std::uint64_t> pre;
    for (int e = 0; e < g.num_edges(); e += 3)
      if (g.edge(e).size > 0) pre[e] = 0;
    EXPECT(ref_pairs(g, lt, pre) == dev.overlap_pairs(g, lt, pre), "pinned pairs");
    // addresses: greedy_pack is feasible; collapsing two live tensors is not
    auto packed = greedy_pack(g, lt, {});
    EXPECT(dev.addresses_feasible(g, lt, packed), "greedy_pack feasible");
    // placement heuristics, the arena baseline and the LP text vs the reference
    EXPECT(dev.greedy_pack(g, lt, {}) == packed, "greedy_pack");
    const PrePlacement rp = preallocate_pyramid(g, lt);
    const PrePlacement dp = dev.preallocate_pyramid(g, lt);
    EXPECT(rp.assigned == dp.assigned && rp.remaining == dp.remaining &&
               rp.reserved_base == dp.reserved_base,
           "preallocate_pyramid");
    EXPECT(dev.greedy_pack(g, lt, rp.assigned) == greedy_pack(g, lt, rp.assigned),
           "greedy_pack over the pyramid");
    for (FitPolicy pol : {FitPolicy::kFirstFit, FitPolicy::kBestFit}) {
      const BaselineResult rb = run_baseline(g, o, pol);
      const BaselineResult db = dev.run_baseline(g, o, pol);
      EXPECT(rb.mr_peak == db.mr_peak && rb.rs_at_peak == db.rs_at_peak &&
                 rb.fragmentation == db.fragmentation,
             "run_baseline");
    }
    EXPECT(write_lp(encode_addresses(g, lt, {})) == dev.write_address_lp(g, lt), "LP text");
    EXPECT(write_lp(encode_addresses(g, lt, pre)) == dev.write_address_lp(g, lt, pre),
           "LP text, pinned");
    // realized lifetimes from the order's timesteps
    std::map<std::string, int> ts;
    for (size_t i = 0; i < o.size(); ++i) ts[g.node(o[i]).id] = (int)i + 1;
    EXPECT(same(realized_lifetimes(g, ts, g.num_nodes() + 2),
                dev.realized_lifetimes(g, ts, g.num_nodes() + 2)),
           "realized lifetimes");
    if (!ts.empty()) {
      auto ts2 = ts;
      ts2.erase(ts2.begin());
      EXPECT(error_of([&] { realized_lifetimes(g, ts2, g.num_nodes()); }) ==
                 error_of([&] { dev.realized_lifetimes(g, ts2, g.num_nodes()); }),
             "realized lifetimes error text");
    }
  }
  EXPECT(best == ref_best, "first-minimum argmin");

  // encode_joint's pair loop (encode.cpp:401-408) with the reference's edge_precedes
  {
    const LifetimeBounds bounds = compute_bounds(g);
    ReachabilityCache reach(g);
    std::vector<std::pair<EdgeIndex, EdgeIndex>> ref;
    std::vector<EdgeIndex> data;
    for (int e = 0; e < g.num_edges(); ++e)
      if (g.edge(e).size > 0) data.push_back(e);
    for (size_t a = 0; a < data.size(); ++a)
      for (size_t b = a + 1; b < data.size(); ++b)
        if (!edge_precedes(g, bounds, data[a], data[b], &reach) &&
            !edge_precedes(g, bounds, data[b], data[a], &reach))
          ref.push_back({data[a], data[b]});
    EXPECT(dev.joint_pairs(g) == ref, "joint pairs");
  }

  // validate_plan on the reference planner's own plan, plus tampered copies
  if (g.num_nodes() <= 12) {
    MemoryPlan good = plan_graph(g).plan;
    std::vector<MemoryPlan> plans{good};
    if (good.addresses.size() >= 2) {
      MemoryPlan p = good;
      auto it = p.addresses.begin();
      const auto first = it->second;
      (++it)->second = first;
      plans.push_back(p);
    }
    MemoryPlan low = good;
    low.peak_mem = good.peak_mem ? good.peak_mem - 1 : 0;
    plans.push_back(low);
    MemoryPlan stored = good;
    stored.timeline.peak_rs += 7;
    plans.push_back(stored);
    if (good.sequence.steps.size() >= 2) {
      MemoryPlan swapped = good;
      std::swap(swapped.sequence.timestep_of[good.sequence.steps[0]],
                swapped.sequence.timestep_of[good.sequence.steps[1]]);
      plans.push_back(swapped);
      MemoryPlan missing = good;
      missing.sequence.steps.pop_back();
      missing.sequence.timestep_of.erase(good.sequence.steps.back());
      plans.push_back(missing);
    }
    for (const MemoryPlan& p : plans) {
      const ValidationReport r = validate_plan(p, g);
      const ValidationReport d = dev.validate_plan(p, g);
      bool eq = r.violations.size() == d.violations.size();
      for (size_t i = 0; eq && i < r.violations.size(); ++i)
        eq = r.violations[i].tag == d.violations[i].tag &&
             r.violations[i].detail == d.violations[i].detail;
      EXPECT(eq, "validate_plan report");
    }
  }
}

int main(int argc, char** argv) {
  memplan_b200::Planner dev(0);
  std::mt19937_64 rng(2210);
  for (int i = 1; i < argc; ++i) check_graph(dev, load_graph_file(argv[i]), rng);
  for (auto [kind, layers, size, seed] :
       std::vector<std::tuple<GraphKind, int, uint64_t, uint64_t>>{
           {GraphKind::kChain, 4, 3, 0},          {GraphKind::kForkJoin, 2, 6, 1},
           {GraphKind::kForkJoin, 30, 100, 7},    {GraphKind::kTrainingLike, 2, 8, 0},
           {GraphKind::kTrainingLike, 40, 8, 0},  {GraphKind::kTrainingLike, 300, 1000, 0}}) {
    GeneratorSpec spec;
    spec.kind = kind;
    spec.layers = layers;
    spec.size = size;
    spec.seed = seed;
    check_graph(dev, generate_graph(spec), rng);
  }
  std::printf("OK %ld\n", g_checks);
  return 0;
}
