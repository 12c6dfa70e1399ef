// Host planning of the node partition used by the large-graph scorer; see
// mp_parts.h for the idea and k_score_parts.cuh for the kernel.
#include "mp_parts.h"

#include <algorithm>
#include <utility>

namespace mpb {

namespace {

constexpr int32_t kChunk = 1 << kPartChunkBits;
constexpr size_t kPartsMiscSmem = 4096;  // static shared memory (~3.4 KB) + alignment (k_score_parts.cuh)
constexpr int32_t kMaxSlots = 32767;     // 15-bit slot field of xchk

// Weighted chunk graph: adjacency lists (neighbour, weight), merged duplicates.
std::vector<std::vector<std::pair<int32_t, int32_t>>> chunk_graph(const ScorePrep& S,
                                                                  int32_t nchunks) {
  std::vector<std::pair<int32_t, int32_t>> links;  // (a, b), a != b, both directions
  auto link = [&](int32_t u, int32_t w) {
    const int32_t a = u >> kPartChunkBits, b = w >> kPartChunkBits;
    if (a != b) {
      links.emplace_back(a, b);
      links.emplace_back(b, a);
    }
  };
  for (int32_t w = 0; w < S.n; ++w)
    if (S.pred1[w] >= 0) link(S.pred1[w], w);
  for (size_t i = 0; i < S.extra_u.size(); ++i) link(S.extra_u[i], S.extra_w[i]);
  for (size_t d = 0; d + 1 < S.dyn_off.size(); ++d)
    for (int32_t k = S.dyn_off[d] + 1; k < S.dyn_off[d + 1]; ++k)
      link(S.dyn_sinks[S.dyn_off[d]], S.dyn_sinks[k]);
  std::sort(links.begin(), links.end());
  std::vector<std::vector<std::pair<int32_t, int32_t>>> adj(nchunks);
  for (size_t i = 0; i < links.size();) {
    size_t j = i;
    while (j < links.size() && links[j] == links[i]) ++j;
    adj[links[i].first].emplace_back(links[i].second, (int32_t)(j - i));
    i = j;
  }
  for (auto& a : adj)  // heaviest neighbour first, then id (deterministic)
    std::sort(a.begin(), a.end(), [](const auto& x, const auto& y) {
      return x.second != y.second ? x.second > y.second : x.first < y.first;
    });
  return adj;
}

// BFS order of the whole chunk graph (every component), starting each component
// from a pseudo-peripheral chunk so the order sweeps along ladder-like graphs.
std::vector<int32_t> bfs_order(const std::vector<std::vector<std::pair<int32_t, int32_t>>>& adj) {
  const int32_t m = (int32_t)adj.size();
  std::vector<int32_t> order, mark(m, 0), queue;
  order.reserve(m);
  auto bfs = [&](int32_t s, int32_t stamp, std::vector<int32_t>* out) {
    queue.clear();
    queue.push_back(s);
    mark[s] = stamp;
    for (size_t h = 0; h < queue.size(); ++h)
      for (const auto& [v, w] : adj[queue[h]]) {
        (void)w;
        if (mark[v] != stamp && mark[v] >= 0) {
          mark[v] = stamp;
          queue.push_back(v);
        }
      }
    if (out) out->insert(out->end(), queue.begin(), queue.end());
    return queue.back();
  };
  int32_t stamp = 1;
  for (int32_t c = 0; c < m; ++c) {
    if (mark[c] < 0) continue;
    const int32_t far = bfs(c, ++stamp, nullptr);  // farthest chunk from c
    const size_t before = order.size();
    bfs(far, ++stamp, &order);
    for (size_t i = before; i < order.size(); ++i) mark[order[i]] = -1;  // placed
  }
  return order;
}

}  // namespace

size_t parts_smem_bytes(const PartPlan& p) {
  auto al = [](size_t b) { return (b + 15) & ~size_t(15); };
  return al((size_t)(p.nb_max + 2) * 4) + al((size_t)(p.nchunks + 1) * 4) + al((size_t)p.nslots * 4) +
         kPartsMiscSmem;
}

bool plan_parts(const ScorePrep& S, size_t smem_budget, int32_t max_chunks, PartPlan* out) {
  const int32_t n = S.n;
  if (n <= 0 || !S.tiny4 || n >= (1 << 24) - 1) return false;
  const int32_t nchunks = (n + kChunk - 1) / kChunk;
  const auto adj = chunk_graph(S, nchunks);
  const std::vector<int32_t> bfs = bfs_order(adj);

  // validity pairs (u before w) and multi-consumer tensors, as flat lists
  std::vector<std::pair<int32_t, int32_t>> pairs;
  pairs.reserve((size_t)n + S.extra_u.size());
  for (int32_t w = 0; w < n; ++w)
    if (S.pred1[w] >= 0) pairs.emplace_back(S.pred1[w], w);
  for (size_t i = 0; i < S.extra_u.size(); ++i) pairs.emplace_back(S.extra_u[i], S.extra_w[i]);
  const size_t ndyn = S.dyn_off.size() - 1;

  for (int32_t P = 1; P <= kPartMaxParts; ++P) {
    const int32_t per = (nchunks + P - 1) / P;  // chunks per part (the last may have fewer)
    // 16-bit local indices in the lists, two sentinel slots past the table
    if ((int64_t)per * kChunk > 65536 - kChunk) continue;
    if (per * kChunk % 16) continue;               // whole 16-byte groups of static bytes
    if (max_chunks > 0 && per > max_chunks) continue;
    PartPlan p;
    p.P = (nchunks + per - 1) / per;
    if (p.P > kPartMaxParts) continue;
    p.nchunks = nchunks;
    p.nb_max = per * kChunk;
    std::vector<int32_t> part(nchunks), base(nchunks);
    for (int32_t i = 0; i < nchunks; ++i) {
      part[bfs[i]] = i / per;
      base[bfs[i]] = (i % per) * kChunk;
    }
    auto pt = [&](int32_t v) { return part[v >> kPartChunkBits]; };
    auto loc = [&](int32_t v) { return (uint32_t)(base[v >> kPartChunkBits] + (v & (kChunk - 1))); };

    // count the stash slots first: they decide whether this P fits
    int32_t slots = 0, cross_pairs = 0, cross_dyn = 0;
    for (const auto& [u, w] : pairs)
      if (pt(u) != pt(w)) ++cross_pairs;
    for (size_t d = 0; d < ndyn; ++d) {
      const int32_t a = S.dyn_off[d], b = S.dyn_off[d + 1];
      bool same = b - a <= 4;
      for (int32_t k = a + 1; k < b && same; ++k) same = pt(S.dyn_sinks[k]) == pt(S.dyn_sinks[a]);
      if (!same) ++cross_dyn;
    }
    slots = cross_pairs + cross_dyn;
    if (slots > kMaxSlots) continue;
    p.nslots = slots;
    if (parts_smem_bytes(p) > smem_budget) continue;

    p.n_cross_pairs = cross_pairs;
    p.n_cross_dyn = cross_dyn;
    p.ctab.resize(nchunks + 1);
    for (int32_t c = 0; c < nchunks; ++c) p.ctab[c] = (uint32_t)part[c] << 24 | (uint32_t)base[c];
    p.ctab[nchunks] = 0xffu << 24;  // out-of-range ids: a part no pass owns
    // per-part lists, built in part order
    std::vector<std::vector<uint32_t>> intra(p.P), xput(p.P), xchk(p.P), xmax(p.P), dyn(p.P),
        dyn2(p.P);
    // one same-part producer per node is checked in node order beside the
    // permutation check (own slot read sequentially, one random read); the rest
    // go to the part's pair list, sorted by consumer so its reads run in order
    const uint32_t s0 = (uint32_t)p.nb_max, s1 = s0 + 1;  // sentinel slots: position 0 / kPos
    p.p1.assign((size_t)p.P * p.nb_max, (uint16_t)s0);
    int32_t slot = 0;
    for (const auto& [u, w] : pairs) {
      const int32_t a = pt(u), b = pt(w);
      if (a == b) {
        uint16_t& f = p.p1[(size_t)a * p.nb_max + loc(w)];
        if (f == (uint16_t)s0) f = (uint16_t)loc(u);
        else intra[a].push_back(loc(u) | loc(w) << 16);
        continue;
      }
      const uint32_t s = (uint32_t)slot++;
      if (a < b) {  // producer's part runs first: stash it, check when w's part runs
        xput[a].push_back(loc(u) | s << 16);
        xchk[b].push_back(loc(w) | s << 16);
      } else {      // consumer stashed first: require pos[u] < stash when u's part runs
        xput[b].push_back(loc(w) | s << 16);
        xchk[a].push_back(loc(u) | s << 16 | 1u << 31);
      }
    }
    for (size_t d = 0; d < ndyn; ++d) {
      const int32_t a = S.dyn_off[d], b = S.dyn_off[d + 1];
      bool same = b - a <= 4;
      for (int32_t k = a + 1; k < b && same; ++k) same = pt(S.dyn_sinks[k]) == pt(S.dyn_sinks[a]);
      const uint32_t sz = (uint32_t)S.dyn_size[d];
      if (same && b - a == 2) {  // the common case (a forward value read twice): 8 bytes
        auto& L = dyn2[pt(S.dyn_sinks[a])];
        L.push_back(loc(S.dyn_sinks[a]) | loc(S.dyn_sinks[a + 1]) << 16);
        L.push_back(sz);
        continue;
      }
      if (same) {
        uint32_t l[4] = {s0, s0, s0, s0};  // missing sinks read position 0
        for (int32_t k = a; k < b; ++k) l[k - a] = loc(S.dyn_sinks[k]);
        auto& L = dyn[pt(S.dyn_sinks[a])];
        L.push_back(l[0] | l[1] << 16);
        L.push_back(l[2] | l[3] << 16);
        L.push_back(sz);
        L.push_back(0);
        continue;
      }
      const uint32_t s = (uint32_t)slot++;
      p.slot_init_max.push_back((int32_t)s);
      for (int32_t k = a; k < b; ++k) xmax[pt(S.dyn_sinks[k])].push_back(loc(S.dyn_sinks[k]) | s << 16);
      p.xfree.push_back(s);
      p.xfree.push_back(sz);
    }
    for (auto& L : intra)
      std::sort(L.begin(), L.end(), [](uint32_t x, uint32_t y) {
        return (x >> 16) != (y >> 16) ? (x >> 16) < (y >> 16) : (x & 0xffffu) < (y & 0xffffu);
      });
    // static (x, f) bytes per local slot; padding slots stay inert (x = 0, f = 0)
    p.xtab.assign((size_t)p.P * p.nb_max, 8);
    for (int32_t v = 0; v < n; ++v) {
      const int64_t x = (int64_t)S.node_x[v];  // in [-8, 7] (tiny4), stored modular
      const uint32_t f = (uint32_t)S.node_f[v];
      p.xtab[(size_t)pt(v) * p.nb_max + loc(v)] = (uint8_t)(((uint32_t)(x + 8) & 0xfu) | f << 4);
    }
    p.desc.assign(p.P, PartDesc{});
    for (int32_t b = 0; b < p.P; ++b) {
      PartDesc& D = p.desc[b];
      D.nloc = std::min(per, nchunks - b * per) * kChunk;
      D.pad_lo = D.pad_hi = D.nloc;
      D.xtab_off = b * p.nb_max;
      // per-part lists start 16-byte aligned and are padded to whole uint4 groups
      // with 0xffffffff entries (skipped by the kernel); counts are in uint4 groups
      auto put = [](std::vector<uint32_t>& flat, const std::vector<uint32_t>& part_list,
                    int32_t* off, int32_t* cnt, int32_t unit) {
        *off = (int32_t)(flat.size() / 4);
        *cnt = (int32_t)((part_list.size() + 3) / 4);
        flat.insert(flat.end(), part_list.begin(), part_list.end());
        while (flat.size() % 4) flat.push_back(0xffffffffu);
        (void)unit;
      };
      put(p.intra, intra[b], &D.intra_off, &D.intra_n, 1);
      // intra pairs are checked without a padding test: pad with (s0, s1), never "later"
      for (size_t q = p.intra.size(); q > 0 && p.intra[q - 1] == 0xffffffffu; --q)
        p.intra[q - 1] = s0 | s1 << 16;
      put(p.xput, xput[b], &D.xput_off, &D.xput_n, 1);
      put(p.xchk, xchk[b], &D.xchk_off, &D.xchk_n, 1);
      put(p.xmax, xmax[b], &D.xmax_off, &D.xmax_n, 1);
      put(p.dyn4, dyn[b], &D.dyn_off, &D.dyn_n, 4);
      // two-sink records after the part's four-sink ones, padded with the sentinel pair
      // (position 0: no free) so the kernel tests nothing per record
      D.dyn2_off = (int32_t)(p.dyn4.size() / 4);
      D.dyn2_n = (int32_t)((dyn2[b].size() + 3) / 4);
      p.dyn4.insert(p.dyn4.end(), dyn2[b].begin(), dyn2[b].end());
      while (p.dyn4.size() % 4) {
        p.dyn4.push_back(s0 | s0 << 16);
        p.dyn4.push_back(0);
      }
    }
    if (n % kChunk) {  // the chunk holding the last node has unwritten tail slots
      const int32_t c = nchunks - 1;
      PartDesc& D = p.desc[part[c]];
      D.pad_lo = base[c] + (n % kChunk);
      D.pad_hi = base[c] + kChunk;
    }
    *out = std::move(p);
    return true;
  }
  return false;
}

}  // namespace mpb
