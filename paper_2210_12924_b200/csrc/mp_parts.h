// Node partition behind the large-graph scorer (k_score_parts.cuh).
//
// A candidate's positions (the inverse permutation of its order, 4 B per node:
// 533 KB at the 100k-tensor graph) do not fit one SM's shared memory, and
// scattering / gathering them through L2 costs a 32-byte sector per 4-byte
// access. Instead the nodes are split into P parts of at most ~45k nodes; the
// scorer streams the candidate's order P times (coalesced, L2-resident after the
// first pass) and in pass b keeps only part b's positions, in shared memory,
// where every producer check and last-consumer lookup of that part is a
// shared-memory access. Parts are unions of 64-node id chunks, so membership
// is one lookup in a small chunk table. The partition follows a BFS order of
// the chunk graph (edges = validity pairs and multi-consumer tensors), which
// for training graphs (forward/backward ladders) cuts only at layer
// boundaries; the few pairs that cross parts carry the earlier part's position
// in a shared-memory stash slot.
#pragma once

#include <cstdint>
#include <vector>

#include "mp_prep.h"

namespace mpb {

constexpr int kPartChunkBits = 6;  // 64-node id chunks
constexpr int kPartMaxParts = 16;
constexpr int32_t kPartsMinNodes = 16384;  // planned above this; used where smem variants do not fit

// Per-part descriptor read by the kernel. List offsets and counts are in uint4
// groups of four entries; padding entries are 0xffffffff (skipped), except in the
// intra list, padded with the sentinel pair (nb_max, nb_max + 1). Slots nb_max and
// nb_max + 1 are sentinels holding position 0 and "unwritten" (positions are 1-based).
struct PartDesc {
  int32_t nloc;       // local slots (64 per chunk)
  int32_t pad_lo;     // [pad_lo, pad_hi): local slots past the last node (never written)
  int32_t pad_hi;
  int32_t xtab_off;   // part-local static (x, f) bytes in the flat xtab; also the offset of
                      // the part's first-producer table p1 (uint16 local slot, nb_max none)
  int32_t intra_off, intra_n;  // u32 lu | lw << 16: pos[lu] < pos[lw] (beyond p1), by lw
  int32_t xput_off, xput_n;    // u32 l | slot << 16: stash[slot] = pos[l]
  int32_t xchk_off, xchk_n;    // u32 l | slot << 16 | dir << 31: compare with stash[slot]
  int32_t xmax_off, xmax_n;    // u32 l | slot << 16: stash[slot] = max(stash[slot], pos[l])
  int32_t dyn_off, dyn_n;      // uint4 {l1 | l2 << 16, l3 | l4 << 16, size, 0}, nb_max = none
  int32_t dyn2_off, dyn2_n;    // two-sink tensors, two per uint4 {l1 | l2 << 16, size}
                               // (in the dyn4 array; padded with the sentinel pair, size 0)
};

struct PartPlan {
  int32_t P = 0;
  int32_t nchunks = 0;
  int32_t nb_max = 0;          // max local slots over parts (smem array length)
  int32_t nslots = 0;          // stash slots
  int32_t n_cross_pairs = 0;   // validity pairs whose endpoints lie in different parts
  int32_t n_cross_dyn = 0;     // multi-consumer tensors whose candidates span parts
  std::vector<uint32_t> ctab;  // [nchunks + 1] part << 24 | local base; [nchunks]: no part
  std::vector<uint8_t> xtab;   // per part, per local slot: (x + 8) | f << 4
  std::vector<uint16_t> p1;    // per part, per local slot: one producer in the same part
  std::vector<PartDesc> desc;  // [P]
  std::vector<uint32_t> intra, xput, xchk, xmax;
  std::vector<uint32_t> dyn4;  // 4 words per record; the two-sink lists, 2 words per record
  std::vector<uint32_t> xfree; // 2 words per record: slot, size (after the last pass)
  std::vector<int32_t> slot_init_max;  // slots that accumulate a max (reset to 0 per candidate)
};

// Plans the partition for a tiny4 graph (every per-position (x, f) fits 4 bits);
// returns false when no P <= kPartMaxParts fits `smem_budget` bytes of shared
// memory (one 4-byte word per local slot, chunk table, stash).
// max_chunks > 0 caps the chunks per part (tests force several parts on small graphs).
bool plan_parts(const ScorePrep& S, size_t smem_budget, int32_t max_chunks, PartPlan* out);

// Shared-memory bytes the kernel needs for a plan (must match k_score_parts.cuh).
size_t parts_smem_bytes(const PartPlan& p);

}  // namespace mpb
