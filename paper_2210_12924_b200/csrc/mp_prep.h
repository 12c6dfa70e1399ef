// Host-side derivation of the fused scorer's tables (see mp_prep.cpp).
#pragma once

#include <cstdint>
#include <vector>

namespace mpb {

constexpr int32_t kExactReachMaxNodes = 32768;  // n^2/8 bytes of bitsets at most

struct ScorePrep {
  int32_t n = 0;
  bool exact_reach = false;
  bool narrow = true;           // total scaled bytes < 2^32: 32-bit arithmetic
  bool tiny8 = false;           // every node's x in [-128, 127] and f <= 255 for any order
  bool tiny4 = false;           // ... x in [-8, 7] and f <= 15
  uint64_t scale = 1;           // gcd of data sizes
  // node tables (scaled): x = alloc - static free, f = static free
  std::vector<uint64_t> node_x, node_f;
  std::vector<int32_t> pred1;   // first reduced producer of each node, -1 if none
  // remaining reduced validity pairs (u must run before w), flat
  std::vector<int32_t> extra_u, extra_w;
  // data edges whose last consumer depends on the order (>= 2 candidate sinks)
  std::vector<int32_t> dyn_off{0}, dyn_sinks;
  std::vector<uint64_t> dyn_size;   // scaled
  int64_t num_reduced_preds = 0;
  // packed forms read by the register-slot scorer:
  std::vector<int32_t> pred2;          // second reduced producer of each node, -1 if none
  std::vector<uint32_t> node_rec32;    // [4n] (x, f, pred1, pred2) for 32-bit graphs
  std::vector<int32_t> node_u2;        // [2n] (pred1, pred2) for 64-bit graphs
  std::vector<uint32_t> extra3_packed; // 3rd+ reduced producer pairs, u | w << 16 (n < 65536)
  // forms read by the tile scorer (any n):
  std::vector<int32_t> extra3_u, extra3_w;   // 3rd+ reduced producer pairs
  std::vector<int32_t> node_dyn_off{0};      // [n+1] per node: dynamic edges it may free last
  std::vector<int32_t> node_dyn;             // edge indexes into dyn_off / dyn_size
  // tile scorer node words (n < 2^24): z = pred1 (kNoNode if none) | min(#memberships,
  // 255) << 24, w = pred2 (kNoNode); memberships = (node v, dynamic edge d) pairs
  std::vector<uint32_t> tile_zw;             // [2n]
  std::vector<int32_t> out_off{0};           // [n+1] fanout(v) (graph.hpp:91), edge order
  std::vector<int32_t> out_edges;            // [E]
  std::vector<uint32_t> tile_rec32;          // [4n] (x, f, z, w) for 32-bit graphs
  std::vector<int32_t> tile_moff;            // [n] first membership of v
  std::vector<int32_t> tile_mother;          // [4 * m] other candidate sinks (kNoNode pad;
                                             //  kMoreSinks: > 4 others, use dyn_sinks)
  std::vector<int32_t> tile_medge;           // [m] the dynamic edge d
};

constexpr uint32_t kNoNode = 0xFFFFFFu;
constexpr int32_t kMoreSinks = -2;

void prepare_scoring(int32_t n, int32_t E, const int32_t* src, const int64_t* sink_off,
                     const int32_t* sinks, const uint64_t* size, ScorePrep* P);

}  // namespace mpb
