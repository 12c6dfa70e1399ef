// Host-side graph analysis behind mp_graph_upload: derives the tables the
// fused scorer needs so that, per candidate order, the device does the
// minimum number of random accesses. Every derivation is exact for VALID
// (topological) orders, which are the only ones whose scores are reported;
// validity itself is decided from an edge set with the same transitive
// closure as the reference's (graph.cpp:239-254 checks every (src, sink)
// pair; a pair implied by a path of other pairs cannot fail alone).
//
//   preds      per consumer node, its producer nodes minus redundant ones
//              (u -> w is dropped when another successor x of u reaches w;
//              exact bitsets up to kExactReachMaxNodes, a chain index above)
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
#include <climits>
#include <cstdlib>
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
  // MP_PREP_EXACT_MAX lowers the bitset limit (tests compare the chain index
  // against the exact closure on small graphs)
  int64_t exact_max = kExactReachMaxNodes;
  if (const char* e = std::getenv("MP_PREP_EXACT_MAX")) exact_max = std::atoll(e);
  const bool exact = acyclic && n <= exact_max;
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
  // Above the bitset limit: a chain index. Greedy chain cover along the Kahn
  // order (each node extends the longest chain ending at one of its producers),
  // then for the K longest chains c, minidx[v][c] = lowest chain index of a node of
  // c that v reaches (itself included). a reaches b on such a chain iff
  // minidx[a][c] <= idx(b): exact. Other targets are decided through their
  // producers (one level) and otherwise answered "no" - sound: a pair kept or a
  // sink kept as a candidate last consumer only costs a redundant check.
  std::vector<int32_t> chain_of, chain_idx, minidx;
  int32_t K = 0;
  if (acyclic && !exact && n > 0) {
    chain_of.assign(n, -1);
    chain_idx.assign(n, 0);
    std::vector<int32_t> tail, len;
    for (int32_t v : order) {
      int32_t best = -1;
      for (int32_t p : pred[v]) {
        const int32_t c = chain_of[p];
        if (tail[c] == p && (best < 0 || len[c] > len[best])) best = c;
      }
      if (best < 0) {
        best = (int32_t)tail.size();
        tail.push_back(v);
        len.push_back(0);
      }
      chain_of[v] = best;
      chain_idx[v] = len[best]++;
      tail[best] = v;
    }
    std::vector<int32_t> ids(len.size());
    std::iota(ids.begin(), ids.end(), 0);
    std::stable_sort(ids.begin(), ids.end(), [&](int32_t a, int32_t b) { return len[a] > len[b]; });
    const int32_t kmax = (int32_t)std::max<int64_t>(1, std::min<int64_t>(64, (int64_t{1} << 26) / n));
    std::vector<int32_t> slot(len.size(), -1);
    for (int32_t i = 0; i < (int32_t)ids.size() && K < kmax && len[ids[i]] >= 2; ++i) slot[ids[i]] = K++;
    for (int32_t v = 0; v < n; ++v) chain_of[v] = slot[chain_of[v]];  // -1: not indexed
    if (K > 0) {
      minidx.assign((size_t)n * K, INT32_MAX);
      for (int32_t i = n - 1; i >= 0; --i) {
        const int32_t v = order[i];
        int32_t* mv = &minidx[(size_t)v * K];
        for (int32_t x : succ[v]) {
          const int32_t* mx = &minidx[(size_t)x * K];
          for (int32_t c = 0; c < K; ++c) mv[c] = std::min(mv[c], mx[c]);
        }
        if (chain_of[v] >= 0) mv[chain_of[v]] = std::min(mv[chain_of[v]], chain_idx[v]);
      }
    }
  }
  auto reaches_idx = [&](int32_t a, int32_t b) -> int {  // 1 yes, 0 no, -1 unknown
    if (K == 0 || chain_of[b] < 0) return -1;
    return minidx[(size_t)a * K + chain_of[b]] <= chain_idx[b] && a != b ? 1 : 0;
  };
  auto reaches = [&](int32_t a, int32_t b) -> bool {
    if (exact) return (reach[(size_t)a * words + (b >> 6)] >> (b & 63)) & 1;
    if (a == b) return false;
    const int r = reaches_idx(a, b);
    if (r >= 0) return r == 1;
    if (std::binary_search(succ[a].begin(), succ[a].end(), b)) return true;
    for (int32_t p : pred[b]) {  // a reaches b iff a reaches (or is) one of b's producers
      if (p == a) return true;
      if (reaches_idx(a, p) == 1) return true;
    }
    for (int32_t x : succ[a])  // 2-hop
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
          if (reaches(x, w)) {
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
    bool m = !P->narrow;
    for (int32_t v = 0; v < n && m; ++v) {
      const int64_t xmax = (int64_t)alloc[v] - (int64_t)sfree[v];
      m = xmin[v] >= INT32_MIN && xmax <= INT32_MAX && fmax[v] <= (int64_t)UINT32_MAX &&
          alloc[v] <= (uint64_t)INT64_MAX / 2;
    }
    P->mid32 = m;
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
