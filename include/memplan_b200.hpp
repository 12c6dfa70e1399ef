// memplan_b200.hpp — C++ drop-in shim for the reference planner's hot path.
//
// Header-only. Compiled INSIDE the reference project (it includes the
// reference's own headers: memplan/graph.hpp, plan.hpp, schedule.hpp,
// pipeline.hpp, errors.hpp) and links libmemplan_b200.so. Each function
// keeps the reference signature and semantics, including the exception type
// and message, and runs the data-parallel work on the B200 through the C ABI
// (include/memplan_b200.h):
//
//   memplan_b200::lifetimes_from_order     <- memplan::lifetimes_from_order (schedule.cpp:33-50)
//   memplan_b200::positions_of             <- memplan::positions_of (schedule.cpp:23-31)
//   memplan_b200::resident_bytes_per_step  <- memplan::resident_bytes_per_step (schedule.cpp:69-79)
//   memplan_b200::peak_resident_bytes      <- memplan::peak_resident_bytes (schedule.cpp:81-88)
//   memplan_b200::realized_lifetimes       <- memplan::realized_lifetimes (plan.cpp:101-120)
//   memplan_b200::timeline_from_lifetimes  <- memplan::timeline_from_lifetimes (plan.cpp:122-143)
//   memplan_b200::overlap_pairs            <- the pair loop of encode_addresses (encode.cpp:347-367)
//   memplan_b200::validate_plan            <- memplan::validate_plan (plan.cpp:315-419)
//   memplan_b200::addresses_feasible       <- addresses_feasible (pipeline.cpp:146-160)
//   memplan_b200::score_orders / best_order   batched peak_resident_bytes + first-min argmin
//   memplan_b200::preallocate_pyramid      <- memplan::preallocate_pyramid (placement.cpp:25-62)
//   memplan_b200::greedy_pack              <- memplan::greedy_pack (placement.cpp:182-204)
//   memplan_b200::run_baseline             <- memplan::run_baseline (placement.cpp:150-180)
//   memplan_b200::write_address_lp         <- write_lp(encode_addresses(...)) (lp_format.cpp:88-121)
//   memplan_b200::joint_pairs              <- the pair loop of encode_joint (encode.cpp:401-408)
//
// One Planner per device; graphs are uploaded once per Planner and cached by
// address (a memplan::Graph is immutable after build, graph.hpp:61).
#pragma once

#include <algorithm>
#include <cstdint>
#include <map>
#include <memory>
#include <string>
#include <unordered_map>
#include <utility>
#include <vector>

#include "memplan/analysis.hpp"
#include "memplan/errors.hpp"
#include "memplan/graph.hpp"
#include "memplan/milp.hpp"
#include "memplan/placement.hpp"
#include "memplan/plan.hpp"
#include "memplan_b200.h"

namespace memplan_b200 {

// CUDA / capacity failures (no reference analogue; there is no CPU fallback).
class DeviceError : public memplan::Error {
 public:
  explicit DeviceError(const std::string& what) : memplan::Error("DeviceError: " + what) {}
};

inline void check(mp_status s) {
  if (s == MP_OK) return;
  const std::string msg = mp_last_error();
  if (s == MP_E_INVALID_ORDER) {
    const std::string prefix = "InvalidOrder: ";
    throw memplan::InvalidOrder(msg.rfind(prefix, 0) == 0 ? msg.substr(prefix.size()) : msg);
  }
  if (s == MP_E_BAD_GRAPH) throw memplan::InvalidStructure(msg);
  throw DeviceError(msg);
}

struct Score {
  std::uint64_t peak = 0;  // peak_resident_bytes, 0 when invalid
  int peak_step = 0;       // first step attaining it, 0 when invalid
  bool valid = false;      // is_topological_order
};

class Planner {
 public:
  explicit Planner(int device = 0) { check(mp_ctx_create(device, &ctx_)); }
  ~Planner() {
    for (auto& kv : graphs_) mp_graph_free(kv.second.handle);
    mp_ctx_destroy(ctx_);
  }
  Planner(const Planner&) = delete;
  Planner& operator=(const Planner&) = delete;

  mp_ctx* ctx() const { return ctx_; }

  // The device copy of `g` (uploaded on first use). Cached by address AND a
  // fingerprint: a destroyed graph's address can be reused by the next one, which
  // must not hit the stale upload. memplan::Graph is immutable once built
  // (SPEC.md:86-87), so a hit compares a cheap fingerprint (dimensions, total
  // bytes and 64 sampled edges); the full O(E + S) one is taken at upload. At
  // most kMaxGraphs uploads stay cached (least recently used evicted first);
  // release() drops one explicitly.
  static constexpr size_t kMaxGraphs = 16;
  mp_graph* device_graph(const memplan::Graph& g) {
    const std::uint64_t quick = quick_fingerprint(g);
    auto it = graphs_.find(&g);
    if (it != graphs_.end()) {
      if (it->second.quick == quick) {
        it->second.last_use = ++clock_;
        return it->second.handle;
      }
      mp_graph_free(it->second.handle);
      graphs_.erase(it);
    }
    if (graphs_.size() >= kMaxGraphs) {
      auto lru = graphs_.begin();
      for (auto j = graphs_.begin(); j != graphs_.end(); ++j)
        if (j->second.last_use < lru->second.last_use) lru = j;
      mp_graph_free(lru->second.handle);
      graphs_.erase(lru);
    }
    const std::uint64_t fp = fingerprint(g);
    Uploaded u;
    u.fp = fp;
    u.quick = quick;
    u.last_use = ++clock_;
    const int E = g.num_edges();
    u.src.resize(E);
    u.off.resize(E + 1, 0);
    u.size.resize(E);
    for (int e = 0; e < E; ++e) {
      u.src[e] = g.source_of(e);
      u.off[e + 1] = u.off[e] + (int64_t)g.sinks_of(e).size();
      for (int s : g.sinks_of(e)) u.sinks.push_back(s);
      u.size[e] = g.edge(e).size;  // control edges carry 0 bytes (graph.cpp:89-93)
    }
    mp_csr csr{g.num_nodes(), E, u.src.data(), u.off.data(), u.sinks.data(), u.size.data()};
    check(mp_graph_upload(ctx_, &csr, &u.handle));
    return graphs_.emplace(&g, std::move(u)).first->second.handle;
  }

  // ---- schedule.hpp ----------------------------------------------------------
  std::vector<memplan::Interval> lifetimes_from_order(const memplan::Graph& g,
                                                      const std::vector<memplan::NodeIndex>& order) {
    std::vector<int32_t> lo(g.num_edges()), hi(g.num_edges());
    check(mp_lifetimes(ctx_, device_graph(g), order.data(), (int64_t)order.size(), lo.data(),
                       hi.data()));
    std::vector<memplan::Interval> out(g.num_edges());
    for (int e = 0; e < g.num_edges(); ++e) out[e] = memplan::Interval{lo[e], hi[e]};
    return out;
  }

  std::vector<int> positions_of(const memplan::Graph& g,
                                const std::vector<memplan::NodeIndex>& order) {
    lifetimes_from_order(g, order);  // device verdict (throws InvalidOrder)
    std::vector<int> pos(g.num_nodes(), 0);
    for (size_t i = 0; i < order.size(); ++i) pos[order[i]] = (int)i + 1;
    return pos;
  }

  std::vector<std::uint64_t> resident_bytes_per_step(const memplan::Graph& g,
                                                     const std::vector<memplan::NodeIndex>& order) {
    std::vector<std::uint64_t> out(g.num_nodes());
    check(mp_resident_bytes(ctx_, device_graph(g), order.data(), (int64_t)order.size(),
                            out.data()));
    return out;
  }

  std::uint64_t peak_resident_bytes(const memplan::Graph& g,
                                    const std::vector<memplan::NodeIndex>& order) {
    std::uint64_t p = 0;
    check(mp_peak_resident_bytes(ctx_, device_graph(g), order.data(), (int64_t)order.size(), &p));
    return p;
  }

  // ---- batched scoring ---------------------------------------------------------
  std::vector<Score> score_orders(const memplan::Graph& g,
                                  const std::vector<std::vector<memplan::NodeIndex>>& orders,
                                  int64_t* best = nullptr) {
    const int n = g.num_nodes();
    std::vector<Score> out(orders.size());
    std::vector<int32_t> flat;
    std::vector<size_t> rows;  // candidates of the right length go to the device
    for (size_t c = 0; c < orders.size(); ++c)
      if ((int)orders[c].size() == n) {
        rows.push_back(c);
        flat.insert(flat.end(), orders[c].begin(), orders[c].end());
      }
    std::vector<uint64_t> peak(rows.size());
    std::vector<int32_t> step(rows.size());
    std::vector<uint8_t> valid(rows.size());
    int64_t b = -1;
    if (!rows.empty())
      check(mp_score_orders_best(ctx_, device_graph(g), flat.data(), (int64_t)rows.size(),
                                 peak.data(), step.data(), valid.data(), &b));
    for (size_t i = 0; i < rows.size(); ++i) out[rows[i]] = Score{peak[i], step[i], valid[i] != 0};
    if (best) *best = b < 0 ? -1 : (int64_t)rows[b];
    return out;
  }

  // ---- plan.hpp ------------------------------------------------------------------
  std::vector<memplan::Interval> realized_lifetimes(const memplan::Graph& g,
                                                    const std::map<std::string, int>& timestep_of,
                                                    int horizon) {
    std::vector<int32_t> ts(g.num_nodes(), 0), lo(g.num_edges()), hi(g.num_edges());
    for (const auto& [id, t] : timestep_of)
      if (g.has_node(id)) ts[g.node_index(id)] = t;
    int32_t missing = -1;
    const mp_status s = mp_realized_lifetimes(ctx_, device_graph(g), ts.data(), horizon,
                                              lo.data(), hi.data(), &missing);
    if (s == MP_E_INVALID_ORDER)  // plan.cpp:107 message, with the node's id
      throw memplan::InvalidOrder("node " + g.node(missing).id + " has no timestep");
    check(s);
    std::vector<memplan::Interval> out(g.num_edges());
    for (int e = 0; e < g.num_edges(); ++e) out[e] = memplan::Interval{lo[e], hi[e]};
    return out;
  }

  // Bytes, peak_rs and peak_step on the device; the per-step id lists are
  // filled on the host from the lifetimes in O(sum of lifetime lengths)
  // when want_live (string output is host work by nature).
  memplan::ResidentTimeline timeline_from_lifetimes(const memplan::Graph& g,
                                                    const std::vector<memplan::Interval>& lt,
                                                    int horizon, bool want_live = true) {
    std::vector<int32_t> lo(lt.size()), hi(lt.size());
    for (size_t e = 0; e < lt.size(); ++e) {
      lo[e] = lt[e].lo;
      hi[e] = lt[e].hi;
    }
    memplan::ResidentTimeline t;
    t.bytes.assign(horizon > 0 ? horizon : 0, 0);
    int32_t step = 0;
    check(mp_timeline(ctx_, device_graph(g), lo.data(), hi.data(), horizon, t.bytes.data(),
                      &t.peak_rs, &step));
    t.peak_step = step;
    t.live.resize(horizon > 0 ? horizon : 0);
    if (want_live)
      for (int e = 0; e < g.num_edges(); ++e)  // edge order within each step (plan.cpp:128-131)
        for (int s = std::max(1, lt[e].lo); s <= std::min(horizon, lt[e].hi); ++s)
          t.live[s - 1].push_back(g.edge(e).id);
    return t;
  }

  // ---- encode.hpp: the pair set encode_addresses emits rows for --------------------
  std::vector<std::pair<memplan::EdgeIndex, memplan::EdgeIndex>> overlap_pairs(
      const memplan::Graph& g, const std::vector<memplan::Interval>& lt,
      const std::map<memplan::EdgeIndex, std::uint64_t>& preplaced = {}) {
    const int E = g.num_edges();
    std::vector<int32_t> lo(E), hi(E);
    std::vector<uint64_t> size(E);
    std::vector<uint8_t> pin(E, 0);
    for (int e = 0; e < E; ++e) {
      lo[e] = lt[e].lo;
      hi[e] = lt[e].hi;
      size[e] = g.edge(e).size;
    }
    for (const auto& kv : preplaced) pin[kv.first] = 1;
    int64_t count = 0;
    const uint8_t* pp = preplaced.empty() ? nullptr : pin.data();
    check(mp_overlap_pairs(ctx_, E, lo.data(), hi.data(), size.data(), pp, nullptr, 0, &count));
    std::vector<int32_t> flat(2 * count);
    check(mp_overlap_pairs(ctx_, E, lo.data(), hi.data(), size.data(), pp, flat.data(), count,
                           &count));
    std::vector<std::pair<memplan::EdgeIndex, memplan::EdgeIndex>> out(count);
    for (int64_t i = 0; i < count; ++i) out[i] = {flat[2 * i], flat[2 * i + 1]};
    return out;
  }

  // ---- placement.hpp: the producers of the plans validate_plan checks -------------
  memplan::PrePlacement preallocate_pyramid(const memplan::Graph& g,
                                            const std::vector<memplan::Interval>& lt) {
    std::vector<uint64_t> addr;
    std::vector<uint8_t> has;
    uint64_t base = 0;
    place(g, lt, {}, MP_PLACE_PYRAMID_ONLY, &addr, &has, &base);
    memplan::PrePlacement out;
    for (int e = 0; e < g.num_edges(); ++e) {
      if (has[e]) out.assigned[e] = addr[e];
      else if (g.edge(e).size > 0) out.remaining.push_back(e);
    }
    out.reserved_base = base;
    return out;
  }

  std::map<memplan::EdgeIndex, std::uint64_t> greedy_pack(
      const memplan::Graph& g, const std::vector<memplan::Interval>& lt,
      const std::map<memplan::EdgeIndex, std::uint64_t>& preplaced) {
    std::vector<uint64_t> addr;
    std::vector<uint8_t> has;
    place(g, lt, preplaced, 0, &addr, &has, nullptr);
    std::map<memplan::EdgeIndex, std::uint64_t> out;
    for (int e = 0; e < g.num_edges(); ++e)
      if (has[e]) out[e] = addr[e];
    return out;
  }

  memplan::BaselineResult run_baseline(const memplan::Graph& g,
                                       const std::vector<memplan::NodeIndex>& order,
                                       memplan::FitPolicy policy = memplan::FitPolicy::kFirstFit) {
    memplan::BaselineResult r;
    uint8_t valid = 0;
    if ((int)order.size() == g.num_nodes()) {
      std::vector<int32_t> o(order.begin(), order.end());
      check(mp_run_baseline(ctx_, device_graph(g), o.data(), 1,
                            policy == memplan::FitPolicy::kBestFit ? 1 : 0, &r.mr_peak,
                            &r.rs_at_peak, &r.fragmentation, &valid));
    }
    if (!valid)
      throw memplan::InvalidOrder("sequence is not a topological order of the graph");
    return r;
  }

  // ---- encode.cpp:401-408: the joint-mode pair set (edge_precedes filter) ----------
  std::vector<std::pair<memplan::EdgeIndex, memplan::EdgeIndex>> joint_pairs(
      const memplan::Graph& g, bool filter_pairs = true) {
    int64_t count = 0;
    check(mp_joint_pairs(ctx_, device_graph(g), filter_pairs ? 1 : 0, nullptr, 0, &count));
    std::vector<int32_t> flat(2 * count);
    check(mp_joint_pairs(ctx_, device_graph(g), filter_pairs ? 1 : 0, flat.data(), count,
                         &count));
    std::vector<std::pair<memplan::EdgeIndex, memplan::EdgeIndex>> out(count);
    for (int64_t i = 0; i < count; ++i) out[i] = {flat[2 * i], flat[2 * i + 1]};
    return out;
  }

  // ---- encode.hpp + lp_format.hpp: the external placement model as LP text ---------
  std::string write_address_lp(const memplan::Graph& g, const std::vector<memplan::Interval>& lt,
                               const std::map<memplan::EdgeIndex, std::uint64_t>& preplaced = {}) {
    const int E = g.num_edges();
    std::vector<int32_t> lo(E), hi(E);
    std::vector<uint64_t> size(E), paddr(E, 0);
    std::vector<uint8_t> pin(E, 0);
    std::string ids;
    std::vector<int64_t> off(E + 1, 0);
    for (int e = 0; e < E; ++e) {
      lo[e] = lt[e].lo;
      hi[e] = lt[e].hi;
      size[e] = g.edge(e).size;
      ids += g.edge(e).id;
      off[e + 1] = (int64_t)ids.size();
    }
    for (const auto& kv : preplaced) {
      pin[kv.first] = 1;
      paddr[kv.first] = kv.second;
    }
    const uint8_t* pp = preplaced.empty() ? nullptr : pin.data();
    const uint64_t* pa = preplaced.empty() ? nullptr : paddr.data();
    int64_t len = 0;
    check(mp_encode_addresses_lp(ctx_, E, lo.data(), hi.data(), size.data(), pp, pa, ids.data(),
                                 off.data(), nullptr, 0, &len, nullptr));
    std::string text((size_t)len + 1, '\0');
    check(mp_encode_addresses_lp(ctx_, E, lo.data(), hi.data(), size.data(), pp, pa, ids.data(),
                                 off.data(), &text[0], len + 1, &len, nullptr));
    text.resize((size_t)len);
    return text;
  }

  // ---- pipeline.cpp ----------------------------------------------------------------
  bool addresses_feasible(const memplan::Graph& g, const std::vector<memplan::Interval>& lt,
                          const std::map<memplan::EdgeIndex, std::uint64_t>& addresses) {
    const int E = g.num_edges();
    std::vector<int32_t> lo(E), hi(E);
    std::vector<uint64_t> size(E), addr(E, 0);
    std::vector<uint8_t> has(E, 0);
    for (int e = 0; e < E; ++e) {
      lo[e] = lt[e].lo;
      hi[e] = lt[e].hi;
      size[e] = g.edge(e).size;
    }
    for (const auto& kv : addresses) {
      has[kv.first] = 1;
      addr[kv.first] = kv.second;
    }
    int32_t ok = 0;
    check(mp_addresses_feasible(ctx_, E, lo.data(), hi.data(), size.data(), has.data(),
                                addr.data(), &ok));
    return ok != 0;
  }

  // validate_plan (plan.cpp:315-419): the same violations, same order, same
  // text. Coverage / ordering / bounds are id bookkeeping on the host; the
  // realized lifetimes, the O(E^2) pairwise check and peak_rs run on the B200.
  memplan::ValidationReport validate_plan(const memplan::MemoryPlan& plan,
                                          const memplan::Graph& graph) {
    using namespace memplan;
    ValidationReport report;
    auto fail = [&](const std::string& tag, const std::string& detail) {
      report.violations.push_back({tag, detail});
    };
    std::map<std::string, int> seen;
    for (const std::string& id : plan.sequence.steps) {
      if (!graph.has_node(id)) {
        fail(kTagCreateOnce, "sequence names unknown node '" + id + "'");
        continue;
      }
      if (++seen[id] == 2) fail(kTagCreateOnce, "node '" + id + "' appears more than once");
    }
    for (const Node& n : graph.nodes())
      if (!seen.count(n.id)) fail(kTagCreateOnce, "node '" + n.id + "' is missing from the sequence");
    int horizon = graph.num_nodes();
    auto step_of = [&](const std::string& id) -> int {
      auto it = plan.sequence.timestep_of.find(id);
      return it == plan.sequence.timestep_of.end() ? 0 : it->second;
    };
    for (const std::string& id : plan.sequence.steps) {
      const int t = step_of(id);
      if (t <= 0) fail(kTagCreateOnce, "node '" + id + "' has no timestep");
      else horizon = std::max(horizon, t);
    }
    bool order_ok = true;
    for (int e = 0; e < graph.num_edges(); ++e) {
      const TensorEdge& edge = graph.edge(e);
      const int t_src = step_of(edge.source);
      for (const std::string& sink : edge.sinks) {
        const int t_sink = step_of(sink);
        if (t_src <= 0 || t_sink <= 0) continue;
        if (t_sink <= t_src) {
          fail(kTagFaninInMemory, "edge '" + edge.id + "': consumer '" + sink +
                                      "' does not run after producer '" + edge.source + "'");
          order_ok = false;
        }
      }
    }
    for (const auto& [id, addr] : plan.addresses) {
      if (!graph.has_edge(id)) {
        fail(kTagPeakAddress, "address for unknown tensor '" + id + "'");
        continue;
      }
      const TensorEdge& edge = graph.edge(graph.edge_index(id));
      if (addr + edge.size > plan.peak_mem)
        fail(kTagPeakAddress, "tensor '" + id + "' ends at " + std::to_string(addr + edge.size) +
                                  ", above peak_mem " + std::to_string(plan.peak_mem));
    }
    for (const TensorEdge& edge : graph.edges())
      if (edge.size > 0 && !plan.addresses.count(edge.id))
        fail(kTagPeakAddress, "tensor '" + edge.id + "' has no address");
    if (!order_ok) return report;
    for (const Node& n : graph.nodes())
      if (step_of(n.id) <= 0) return report;

    const std::vector<Interval> lt = realized_lifetimes(graph, plan.sequence.timestep_of, horizon);
    const int E = graph.num_edges();
    std::vector<int32_t> lo(E), hi(E);
    std::vector<uint64_t> size(E), addr(E, 0);
    std::vector<uint8_t> has(E, 0);
    for (int e = 0; e < E; ++e) {
      lo[e] = lt[e].lo;
      hi[e] = lt[e].hi;
      size[e] = graph.edge(e).size;
      auto it = plan.addresses.find(graph.edge(e).id);
      if (it != plan.addresses.end()) {
        has[e] = 1;
        addr[e] = it->second;
      }
    }
    int64_t nv = 0;
    check(mp_validate_pairs(ctx_, E, lo.data(), hi.data(), size.data(), has.data(), addr.data(),
                            nullptr, 0, &nv));
    std::vector<int32_t> viol(2 * nv);
    if (nv)
      check(mp_validate_pairs(ctx_, E, lo.data(), hi.data(), size.data(), has.data(),
                              addr.data(), viol.data(), nv, &nv));
    for (int64_t i = 0; i < nv; ++i)
      fail("below_above", "tensors '" + graph.edge(viol[2 * i]).id + "' and '" +
                              graph.edge(viol[2 * i + 1]).id +
                              "' are live together and overlap in memory");
    uint64_t peak_rs = 0;
    int32_t peak_step = 0;
    check(mp_timeline(ctx_, device_graph(graph), lo.data(), hi.data(), horizon, nullptr, &peak_rs,
                      &peak_step));
    if (plan.peak_mem < peak_rs)
      fail(kTagPeakMem, "peak_mem " + std::to_string(plan.peak_mem) +
                            " is below the peak resident bytes " + std::to_string(peak_rs));
    if (plan.timeline.peak_rs != peak_rs)
      fail(kTagPeakMem, "stored peak_rs " + std::to_string(plan.timeline.peak_rs) +
                            " differs from the recomputed " + std::to_string(peak_rs));
    return report;
  }

 private:
  void place(const memplan::Graph& g, const std::vector<memplan::Interval>& lt,
             const std::map<memplan::EdgeIndex, std::uint64_t>& preplaced, uint32_t flags,
             std::vector<uint64_t>* addr, std::vector<uint8_t>* has, uint64_t* base) {
    const int E = g.num_edges();
    std::vector<int32_t> lo(E), hi(E), rank(E);
    std::vector<uint64_t> size(E), faddr(E, 0);
    std::vector<uint8_t> fixed(E, 0);
    std::vector<int> by_id(E);
    for (int e = 0; e < E; ++e) {
      lo[e] = lt[e].lo;
      hi[e] = lt[e].hi;
      size[e] = g.edge(e).size;
      by_id[e] = e;
    }
    // the pyramid's last tie-break compares edge ids (placement.cpp:48-50)
    std::sort(by_id.begin(), by_id.end(),
              [&](int a, int b) { return g.edge(a).id < g.edge(b).id; });
    for (int r = 0; r < E; ++r) rank[by_id[r]] = r;
    for (const auto& kv : preplaced) {
      fixed[kv.first] = 1;
      faddr[kv.first] = kv.second;
    }
    addr->assign(E > 0 ? E : 1, 0);
    has->assign(E > 0 ? E : 1, 0);
    uint64_t peak = 0, b = 0;
    check(mp_place(ctx_, E, 1, lo.data(), hi.data(), size.data(), rank.data(),
                   preplaced.empty() ? nullptr : fixed.data(),
                   preplaced.empty() ? nullptr : faddr.data(), flags, addr->data(), has->data(),
                   &peak, &b));
    if (base) *base = b;
  }

  // Drops the cached device copy of `g` (e.g. before destroying the graph).
 public:
  void release(const memplan::Graph& g) {
    auto it = graphs_.find(&g);
    if (it == graphs_.end()) return;
    mp_graph_free(it->second.handle);
    graphs_.erase(it);
  }

 private:
  static std::uint64_t quick_fingerprint(const memplan::Graph& g) {
    std::uint64_t h = 1469598103934665603ull;
    auto mix = [&h](std::uint64_t x) { h = (h ^ x) * 1099511628211ull; };
    const int E = g.num_edges();
    mix((std::uint64_t)g.num_nodes());
    mix((std::uint64_t)E);
    mix(g.total_bytes());
    for (int k = 0; k < 64 && E > 0; ++k) {
      const int e = (int)((int64_t)k * E / 64);
      mix((std::uint64_t)g.source_of(e));
      mix(g.edge(e).size);
      mix((std::uint64_t)g.sinks_of(e).size());
    }
    return h;
  }

  static std::uint64_t fingerprint(const memplan::Graph& g) {
    std::uint64_t h = 1469598103934665603ull;
    auto mix = [&h](std::uint64_t x) { h = (h ^ x) * 1099511628211ull; };
    mix((std::uint64_t)g.num_nodes());
    mix((std::uint64_t)g.num_edges());
    for (int e = 0; e < g.num_edges(); ++e) {
      mix((std::uint64_t)g.source_of(e));
      mix(g.edge(e).size);
      for (int s : g.sinks_of(e)) mix((std::uint64_t)s + 0x9e3779b97f4a7c15ull);
    }
    return h;
  }

  struct Uploaded {
    std::uint64_t fp = 0, quick = 0, last_use = 0;
    mp_graph* handle = nullptr;
    std::vector<int32_t> src, sinks;
    std::vector<int64_t> off;
    std::vector<uint64_t> size;
  };
  mp_ctx* ctx_ = nullptr;
  std::unordered_map<const memplan::Graph*, Uploaded> graphs_;
  std::uint64_t clock_ = 0;
};

}  // namespace memplan_b200
