// Host-side derivation of the fused scorer's tables (see mp_prep.cpp).
#pragma once

#include <cstdint>
#include <vector>

namespace mpb {

constexpr int32_t kExactReachMaxNodes = 32768;  // n^2/8 bytes of bitsets at most
constexpr int kDynInline = 3;                   // other candidate-last sinks per record

// One "candidate last consumer" membership of a node in an order-dependent
// data edge: the node is the last consumer iff every other candidate sink
// runs before it.
struct DynMember {
  uint64_t size;                // scaled bytes
  int32_t cnt;                  // number of valid entries in others
  int32_t others[kDynInline];
};
static_assert(sizeof(DynMember) == 24, "DynMember layout");

struct ScorePrep {
  int32_t n = 0;
  bool exact_reach = false;
  bool narrow = true;           // total scaled bytes < 2^32: 32-bit arithmetic
  uint64_t scale = 1;           // gcd of data sizes
  std::vector<int32_t> pred_off, preds;
  std::vector<uint64_t> alloc, sfree;   // scaled
  std::vector<int32_t> dyn_off;
  std::vector<DynMember> dyn;
  std::vector<int32_t> big_off{0}, big_sinks;  // edges with > kDynInline+1 candidates
  std::vector<uint64_t> big_size;
  int32_t num_dyn_edges = 0;
};

void prepare_scoring(int32_t n, int32_t E, const int32_t* src, const int64_t* sink_off,
                     const int32_t* sinks, const uint64_t* size, ScorePrep* P);

}  // namespace mpb
