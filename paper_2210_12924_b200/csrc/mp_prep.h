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
  bool mid32 = false;           // not narrow, but every node's x fits int32 and f (with the
                                // order-dependent frees) uint32 for any order: 32-bit
                                // scan inputs, 64-bit sums
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
  std::vector<int32_t> extra3_u, extra3_w;   // the same pairs as int32 (any n)
  std::vector<int32_t> out_off{0};           // [n+1] fanout(v) (graph.hpp:91), edge order
  std::vector<int32_t> out_edges;            // [E]
};


void prepare_scoring(int32_t n, int32_t E, const int32_t* src, const int64_t* sink_off,
                     const int32_t* sinks, const uint64_t* size, ScorePrep* P);

}  // namespace mpb
