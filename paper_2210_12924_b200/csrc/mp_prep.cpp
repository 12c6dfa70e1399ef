// Host-side graph analysis behind mp_graph_upload: derives the tables the
// fused scorer needs so that, per candidate order, the device does the
// minimum number of random accesses. Every derivation is exact for VALID
// (topological) orders, which are the only ones whose scores are reported;
// validity itself is decided from an edge set with the same transitive
// closure as the reference's (graph.cpp:239-254 checks every (src, sink)
// pair; a pair implied by a path of other pairs cannot fail alone).
//
//   preds      per consumer node, its producer nodes minus redundant ones
//              (u -> w is dropped when another successor x of u reaches w)
//   alloc      bytes a node creates at its timestep: sum of its data fanout
//              (lo = pos[src], schedule.cpp:37)
//   sfree      bytes freed after a node: data edges whose last consumer is
//              statically this node (one sink, or every other sink reaches it)
//   dyn        data edges with >= 2 "candidate last" sinks (none reaches another);
//              hi = max over those sinks (schedule.cpp:46) depends on the order
//   scale      gcd of all data sizes; 32-bit arithmetic when total/gcd < 2^32
#include "mp_prep.h"

#include <algorithm>
#include <cstring>
#include <numeric>

namespace mpb {

namespace {

uint64_t gcd64(uint64_t a, uint64_t b) {
  while (b) {
    uint64_t t = a % b;
    a = b;
    b = t;
  }
  return a;
}

// Kahn order; returns false on a cycle.
bool topo(int32_t n, const std::vector<std::vector<int32_t>>& succ, std::vector<int32_t>* order) {
  std::vector<int32_t> indeg(n, 0);
  for (int32_t u = 0; u < n; ++u)
    for (int32_t w : succ[u]) ++indeg[w];
  order->clear();
  order->reserve(n);
  for (int32_t v = 0; v < n; ++v)
    if (!indeg[v]) order->push_back(v);
  for (size_t i = 0; i < order->size(); ++i)
    for (int32_t w : succ[(*order)[i]])
      if (--indeg[w] == 0) order->push_back(w);
  return (int32_t)order->size() == n;
}

}  // namespace

void prepare_scoring(int32_t n, int32_t E, const int32_t* src, const int64_t* sink_off,
                     const int32_t* sinks, const uint64_t* size, ScorePrep* P) {
  *P = ScorePrep();
  P->n = n;
  // distinct successor / predecessor sets (data and control edges)
  std::vector<std::vector<int32_t>> succ(n), pred(n);
  for (int32_t e = 0; e < E; ++e)
    for (int64_t k = sink_off[e]; k < sink_off[e + 1]; ++k) {
      succ[src[e]].push_back(sinks[k]);
      pred[sinks[k]].push_back(src[e]);
    }
  for (int32_t v = 0; v < n; ++v) {
    std::sort(succ[v].begin(), succ[v].end());
    succ[v].erase(std::unique(succ[v].begin(), succ[v].end()), succ[v].end());
    std::sort(pred[v].begin(), pred[v].end());
    pred[v].erase(std::unique(pred[v].begin(), pred[v].end()), pred[v].end());
  }
  std::vector<int32_t> order;
  const bool acyclic = topo(n, succ, &order);

  // Reachability: exact bitset closure for moderate n, 2-hop rule above.
  const bool exact = acyclic && n <= kExactReachMaxNodes;
  const size_t words = ((size_t)n + 63) / 64;
  std::vector<uint64_t> reach;  // reach[v*words + w/64] bit: v reaches w (v != w)
  if (exact) {
    reach.assign((size_t)n * words, 0);
    for (int32_t i = n - 1; i >= 0; --i) {
      const int32_t v = order[i];
      uint64_t* rv = &reach[(size_t)v * words];
      for (int32_t w : succ[v]) {
        const uint64_t* rw = &reach[(size_t)w * words];
        for (size_t q = 0; q < words; ++q) rv[q] |= rw[q];
        rv[w >> 6] |= 1ull << (w & 63);
      }
    }
  }
  auto reaches = [&](int32_t a, int32_t b) -> bool {
    if (exact) return (reach[(size_t)a * words + (b >> 6)] >> (b & 63)) & 1;
    // 2-hop: a -> b directly or a -> x -> b
    if (std::binary_search(succ[a].begin(), succ[a].end(), b)) return true;
    for (int32_t x : succ[a])
      if (std::binary_search(succ[x].begin(), succ[x].end(), b)) return true;
    return false;
  };
  P->exact_reach = exact;

  // Validity edges: drop u -> w when another successor of u reaches w. The
  // first surviving producer of each node goes to the node's own record;
  // the rest form a flat, evenly distributable pair list.
  P->pred1.assign(n, -1);
  for (int32_t w = 0; w < n; ++w) {
    for (int32_t u : pred[w]) {
      bool redundant = false;
      if (acyclic && u != w) {
        for (int32_t x : succ[u]) {
          if (x == w) continue;
          if (exact ? reaches(x, w)
                    : std::binary_search(succ[x].begin(), succ[x].end(), w)) {
            redundant = true;
            break;
          }
        }
      }
      if (redundant) continue;
      ++P->num_reduced_preds;
      if (P->pred1[w] < 0) {
        P->pred1[w] = u;
      } else {
        P->extra_u.push_back(u);
        P->extra_w.push_back(w);
      }
    }
  }

  // Byte tables.
  uint64_t g = 0, total = 0;
  for (int32_t e = 0; e < E; ++e)
    if (size[e]) {
      g = gcd64(g, size[e]);
      total += size[e];
    }
  if (g == 0) g = 1;
  P->scale = g;
  P->narrow = total / g < (uint64_t{1} << 32);
  std::vector<uint64_t> alloc(n, 0), sfree(n, 0);
  for (int32_t e = 0; e < E; ++e) {
    if (!size[e]) continue;
    const uint64_t s = size[e] / g;
    alloc[src[e]] += s;
    const int64_t a = sink_off[e], b = sink_off[e + 1];
    if (b == a) continue;  // sinkless: resident through the horizon
    std::vector<int32_t> cand;
    for (int64_t k = a; k < b; ++k) {
      const int32_t x = sinks[k];
      bool dominated = false;
      if (acyclic)
        for (int64_t q = a; q < b && !dominated; ++q)
          if (q != k && reaches(x, sinks[q])) dominated = true;
      if (!dominated) cand.push_back(x);
    }
    if (cand.size() == 1) {
      sfree[cand[0]] += s;
    } else {
      P->dyn_size.push_back(s);
      P->dyn_sinks.insert(P->dyn_sinks.end(), cand.begin(), cand.end());
      P->dyn_off.push_back((int32_t)P->dyn_sinks.size());
    }
  }
  P->node_x.resize(n);
  P->node_f.resize(n);
  for (int32_t v = 0; v < n; ++v) {
    P->node_x[v] = alloc[v] - sfree[v];  // modular; exact after the prefix sum
    P->node_f[v] = sfree[v];
  }
  // byte-sized scan inputs? x in [-128, 127] and f <= 255 whatever the order:
  // the order-dependent frees can only lower x and raise f at a candidate sink
  {
    std::vector<int64_t> xmin(n), fmax(n);
    bool ok = P->narrow;
    for (int32_t v = 0; v < n; ++v) {
      xmin[v] = (int64_t)alloc[v] - (int64_t)sfree[v];
      fmax[v] = (int64_t)sfree[v];
      ok &= xmin[v] <= 127;
    }
    for (size_t d = 0; d + 1 < P->dyn_off.size(); ++d)
      for (int32_t k = P->dyn_off[d]; k < P->dyn_off[d + 1]; ++k) {
        xmin[P->dyn_sinks[k]] -= (int64_t)P->dyn_size[d];
        fmax[P->dyn_sinks[k]] += (int64_t)P->dyn_size[d];
      }
    bool ok4 = ok;
    for (int32_t v = 0; v < n && ok; ++v) {
      ok = xmin[v] >= -128 && fmax[v] <= 255;
      ok4 = ok4 && xmin[v] >= -8 && xmin[v] + (fmax[v] - (int64_t)sfree[v]) <= 7 && fmax[v] <= 15;
    }
    P->tiny8 = ok;
    P->tiny4 = ok && ok4;
  }
  // second producer per node; the rest (3rd+) as a flat packed list
  P->pred2.assign(n, -1);
  {
    std::vector<int32_t> seen(n, 0);
    for (size_t i = 0; i < P->extra_u.size(); ++i) {
      const int32_t u = P->extra_u[i], w = P->extra_w[i];
      if (seen[w]++ == 0) {
        P->pred2[w] = u;
      } else {
        if (n < 65536) P->extra3_packed.push_back((uint32_t)u | ((uint32_t)w << 16));
        P->extra3_u.push_back(u);
        P->extra3_w.push_back(w);
      }
    }
  }
  // fanout lists in edge order (Graph::fanout, graph.cpp:100)
  {
    P->out_off.assign((size_t)n + 1, 0);
    for (int32_t e = 0; e < E; ++e) ++P->out_off[src[e] + 1];
    for (int32_t v = 0; v < n; ++v) P->out_off[v + 1] += P->out_off[v];
    std::vector<int32_t> cur(P->out_off.begin(), P->out_off.end() - 1);
    P->out_edges.assign(E, 0);
    for (int32_t e = 0; e < E; ++e) P->out_edges[cur[src[e]]++] = e;
  }
  P->node_rec32.assign(4 * (size_t)n, 0);
  P->node_u2.assign(2 * (size_t)n, -1);
  for (int32_t v = 0; v < n; ++v) {
    P->node_rec32[4 * v] = (uint32_t)P->node_x[v];
    P->node_rec32[4 * v + 1] = (uint32_t)P->node_f[v];
    P->node_rec32[4 * v + 2] = (uint32_t)P->pred1[v];
    P->node_rec32[4 * v + 3] = (uint32_t)P->pred2[v];
    P->node_u2[2 * v] = P->pred1[v];
    P->node_u2[2 * v + 1] = P->pred2[v];
  }
}

}  // namespace mpb
