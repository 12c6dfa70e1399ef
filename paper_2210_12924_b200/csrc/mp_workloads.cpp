// Workload helpers (host C++, never on a measured path): the reference's
// deterministic graph families and seeded random topological orders.
//
// Graph families follow generate_graph's published semantics
// (generate.hpp:41-46, generate.cpp:45-158) so that the same spec yields the
// same node/edge order and, for fork_join, the same draws from
// std::mt19937_64 / std::uniform_int_distribution (libstdc++). The CSR is
// emitted directly; ids are implied (see paper_2210_12924_b200/graph.py).
#include <algorithm>
#include <cstdint>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "memplan_b200.h"

namespace {

enum Role : uint8_t { kCompute = 0, kWeightUpdate = 1, kSource = 2, kSinkOnly = 3 };

struct Csr {
  int32_t n = 0;
  std::vector<uint8_t> role;
  std::vector<int32_t> src;
  std::vector<int64_t> off{0};
  std::vector<int32_t> sinks;
  std::vector<uint64_t> size;

  int32_t node(Role r) {
    role.push_back(r);
    return n++;
  }
  void edge(int32_t s, std::initializer_list<int32_t> ks, uint64_t sz) {
    src.push_back(s);
    for (int32_t k : ks) sinks.push_back(k);
    off.push_back((int64_t)sinks.size());
    size.push_back(sz);
  }
};

// chain: n0 -> n1 -> ... -> nL, edge t_i of exactly `size` bytes.
Csr make_chain(int32_t layers, uint64_t size) {
  Csr g;
  for (int32_t i = 0; i <= layers; ++i)
    g.node(i == 0 ? kSource : (i == layers ? kSinkOnly : kCompute));
  for (int32_t i = 0; i < layers; ++i) g.edge(i, {i + 1}, size);
  return g;
}

// fork_join: per stage a fork, 2..3 branches (drawn), a join; link edges
// chain the stages; one sinkless "out" edge on the last join. Sizes drawn
// uniformly from [max(1, size/2), size + size/2]. Draw order: link size,
// width, then (fork->branch, branch->join) sizes per branch, then out.
Csr make_fork_join(int32_t layers, uint64_t size, uint64_t seed) {
  std::mt19937_64 rng(seed);
  auto draw_size = [&]() {
    std::uniform_int_distribution<uint64_t> dist(std::max<uint64_t>(1, size / 2),
                                                 size + size / 2);
    return dist(rng);
  };
  Csr g;
  int32_t prev_join = -1;
  for (int32_t d = 0; d < layers; ++d) {
    const int32_t fork = g.node(d == 0 ? kSource : kCompute);
    if (d > 0) {
      const uint64_t s = draw_size();
      g.edge(prev_join, {fork}, s);
    }
    std::uniform_int_distribution<int> width_dist(2, 3);
    const int width = width_dist(rng);
    // join is declared after the branches; its index is known in advance.
    const int32_t join = fork + width + 1;
    for (int b = 0; b < width; ++b) {
      const int32_t branch = g.node(kCompute);
      const uint64_t s1 = draw_size();
      g.edge(fork, {branch}, s1);
      const uint64_t s2 = draw_size();
      g.edge(branch, {join}, s2);
    }
    const int32_t j = g.node(kCompute);
    (void)j;
    prev_join = join;
  }
  const uint64_t s = draw_size();
  g.edge(prev_join, {}, s);
  return g;
}

// training_like: x, w1..wL, fwd1..fwdL, loss, bwdL..bwd1, gnrm, updL..upd1,
// gsink; edges act0..actL, wt1..wtL (4x size), lossv, gbL..gb1 (4x), gn.
Csr make_training_like(int32_t L, uint64_t size) {
  const uint64_t act = size, wt = 4 * size;
  Csr g;
  const int32_t x = g.node(kSource);
  for (int32_t i = 1; i <= L; ++i) g.node(kSource);
  for (int32_t i = 1; i <= L; ++i) g.node(kCompute);
  const int32_t loss = g.node(kCompute);
  for (int32_t i = L; i >= 1; --i) g.node(kCompute);
  const int32_t gnrm = g.node(kCompute);
  for (int32_t i = L; i >= 1; --i) g.node(kWeightUpdate);
  const int32_t gsink = g.node(kSinkOnly);
  auto w = [&](int32_t i) { return i; };
  auto fwd = [&](int32_t i) { return L + i; };
  auto bwd = [&](int32_t i) { return 2 * L + 2 + (L - i); };
  auto upd = [&](int32_t i) { return 3 * L + 3 + (L - i); };
  for (int32_t i = 0; i <= L; ++i) {
    const int32_t s = i == 0 ? x : fwd(i);
    if (i < L) g.edge(s, {fwd(i + 1), bwd(i + 1)}, act);
    else g.edge(s, {loss}, act);
  }
  for (int32_t i = 1; i <= L; ++i) g.edge(w(i), {fwd(i), bwd(i), upd(i)}, wt);
  g.edge(loss, {bwd(L)}, act);
  for (int32_t i = L; i >= 1; --i) g.edge(bwd(i), {i > 1 ? bwd(i - 1) : gnrm, upd(i)}, wt);
  g.edge(gnrm, {gsink}, act);
  return g;
}

inline uint64_t splitmix64(uint64_t& s) {
  uint64_t z = (s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

}  // namespace

extern "C" {

mp_status mp_generate_graph(int kind, int32_t layers, uint64_t size, uint64_t seed,
                            int32_t* num_nodes, int32_t* num_edges, int64_t* num_sinks,
                            int32_t* edge_src, int64_t* sink_off, int32_t* sinks,
                            uint64_t* edge_size, uint8_t* node_role) {
  if (!num_nodes || !num_edges || !num_sinks) return MP_E_INVALID_ARG;
  if (layers < 1 || size < 1) return MP_E_INVALID_ARG;  // InvalidSpec (generate.cpp:163-166)
  Csr g;
  switch (kind) {
    case 0: g = make_chain(layers, size); break;
    case 1: g = make_fork_join(layers, size, seed); break;
    case 2: g = make_training_like(layers, size); break;
    default: return MP_E_INVALID_ARG;
  }
  *num_nodes = g.n;
  *num_edges = (int32_t)g.src.size();
  *num_sinks = (int64_t)g.sinks.size();
  if (edge_src) std::copy(g.src.begin(), g.src.end(), edge_src);
  if (sink_off) std::copy(g.off.begin(), g.off.end(), sink_off);
  if (sinks) std::copy(g.sinks.begin(), g.sinks.end(), sinks);
  if (edge_size) std::copy(g.size.begin(), g.size.end(), edge_size);
  if (node_role) std::copy(g.role.begin(), g.role.end(), node_role);
  return MP_OK;
}

// Randomised Kahn: at every step pick uniformly among the ready nodes.
mp_status mp_random_topo_orders(const mp_csr* csr, int64_t num_orders, uint64_t seed,
                                int32_t num_threads, int32_t* out) {
  if (!csr || (num_orders > 0 && !out) || num_orders < 0) return MP_E_INVALID_ARG;
  const int32_t n = csr->num_nodes, E = csr->num_edges;
  // successor multiset per node and in-degree (edges x sinks, Kahn on the multigraph)
  std::vector<int32_t> indeg(n, 0), succ_off(n + 1, 0), succ;
  for (int32_t e = 0; e < E; ++e) {
    succ_off[csr->edge_src[e] + 1] += (int32_t)(csr->sink_off[e + 1] - csr->sink_off[e]);
    for (int64_t k = csr->sink_off[e]; k < csr->sink_off[e + 1]; ++k) ++indeg[csr->sinks[k]];
  }
  for (int32_t v = 0; v < n; ++v) succ_off[v + 1] += succ_off[v];
  succ.resize(succ_off[n]);
  {
    std::vector<int32_t> fill(succ_off.begin(), succ_off.end() - 1);
    for (int32_t e = 0; e < E; ++e)
      for (int64_t k = csr->sink_off[e]; k < csr->sink_off[e + 1]; ++k)
        succ[fill[csr->edge_src[e]]++] = csr->sinks[k];
  }
  bool cyclic = false;
  auto work = [&](int64_t c0, int64_t c1) {
    std::vector<int32_t> deg, ready;
    ready.reserve(n);
    for (int64_t c = c0; c < c1; ++c) {
      uint64_t st = seed * 0xD1B54A32D192ED03ull + (uint64_t)c * 0x9E3779B97F4A7C15ull + 1;
      deg = indeg;
      ready.clear();
      for (int32_t v = 0; v < n; ++v)
        if (deg[v] == 0) ready.push_back(v);
      int32_t* row = out + c * (int64_t)n;
      int32_t k = 0;
      while (!ready.empty()) {
        const size_t pick = (size_t)(splitmix64(st) % ready.size());
        const int32_t v = ready[pick];
        ready[pick] = ready.back();
        ready.pop_back();
        row[k++] = v;
        for (int32_t q = succ_off[v]; q < succ_off[v + 1]; ++q)
          if (--deg[succ[q]] == 0) ready.push_back(succ[q]);
      }
      if (k != n) cyclic = true;
    }
  };
  int32_t T = num_threads > 0 ? num_threads : (int32_t)std::max(1u, std::thread::hardware_concurrency());
  if (T > num_orders) T = (int32_t)std::max<int64_t>(1, num_orders);
  std::vector<std::thread> pool;
  for (int32_t t = 1; t < T; ++t)
    pool.emplace_back(work, num_orders * t / T, num_orders * (t + 1) / T);
  work(0, num_orders / T);
  for (auto& th : pool) th.join();
  return cyclic ? MP_E_BAD_GRAPH : MP_OK;
}

}  // extern "C"
