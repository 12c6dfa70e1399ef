// K8 - the joint-mode pair set: the pair loop of encode_joint (encode.cpp:401-408)
// over symbolic lifetimes, with its edge_precedes filter (analysis.cpp:94-113).
//
// edge_precedes(e1, e2) is true when the multiplicity windows mul[e1], mul[e2]
// (compute_bounds, analysis.cpp:33-62) are disjoint, or when e1 has sinks and
// every one of them is a proper ancestor of src(e2). (Its remaining checks -
// src(e2) or a sink of e2 among e1's endpoints - cannot fire once every sink
// of e1 reaches src(e2) in a DAG: each would close a cycle.) With
// AR(e) = the nodes every sink of e reaches (an intersection of descendant
// bitsets, built on the host per graph) a pair (i, j) of data edges is kept iff
//   mul[i] and mul[j] intersect  &&  src(j) not in AR(i)  &&  src(i) not in AR(j).
// One warp per row i: AR(i) is a short bit row read through L1, and
// "src(i) in AR(j)" for consecutive j is one word of the transposed matrix
// ARt[src(i)] shared by the 32 lanes. Count pass, exclusive scan, fill pass with
// ballot compaction - the lexicographic (i, j) order of the reference's loop.
#include <cuda_runtime.h>

#include <cstdint>

#include "mp_internal.h"

namespace mpb {
namespace {

__device__ __forceinline__ bool bit(const uint32_t* row, int k) {
  return (__ldg(row + (k >> 5)) >> (k & 31)) & 1u;
}

template <bool kFill>
__global__ void __launch_bounds__(256)
    joint_kernel(JointArgs a, int64_t* __restrict__ row_cnt, const int64_t* __restrict__ row_off,
                 int2* __restrict__ pairs) {
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  const unsigned lt_mask = (1u << lane) - 1u;
  for (int i = blockIdx.x * wpb + (threadIdx.x >> 5); i < a.E; i += gridDim.x * wpb) {
    int64_t cnt = 0;
    int64_t at = kFill ? row_off[i] : 0;
    if (a.size[i] > 0) {
      const int2 mi = a.mul[i];
      const int si = a.src[i];
      const uint32_t* ar_i = a.ar + (size_t)i * a.ar_words;
      const uint32_t* art_i = a.art + (size_t)si * a.art_words;
      for (int j0 = i + 1; j0 < a.E; j0 += 32) {
        const int j = j0 + lane;
        bool keep = false;
        if (j < a.E && a.size[j] > 0) {
          keep = true;
          if (a.filter) {
            const int2 mj = a.mul[j];
            const bool meet = mi.x <= mi.y && mj.x <= mj.y && mi.y >= mj.x && mj.y >= mi.x;
            keep = meet && !bit(ar_i, a.src[j]) && !bit(art_i, j);
          }
        }
        const unsigned m = __ballot_sync(0xffffffffu, keep);
        if (kFill) {
          if (keep) pairs[at + __popc(m & lt_mask)] = make_int2(i, j);
          at += __popc(m);
        } else {
          cnt += __popc(m);
        }
      }
    }
    if (!kFill && lane == 0) row_cnt[i] = cnt;
  }
}

// One warp per 32 x 32 bit block: lane r holds AR row (eb*32 + r), word vb; ballot
// of bit c across the lanes is ARt row (vb*32 + c), word eb.
__global__ void __launch_bounds__(256)
    joint_transpose_kernel(const uint32_t* __restrict__ ar, int32_t E, int32_t n, int ar_words,
                           int art_words, uint32_t* __restrict__ art) {
  const int lane = threadIdx.x & 31;
  const int64_t nblk_e = (E + 31) / 32;
  const int64_t nblocks = nblk_e * ar_words;
  for (int64_t blk = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); blk < nblocks;
       blk += (int64_t)gridDim.x * (blockDim.x >> 5)) {
    const int64_t eb = blk % nblk_e, vb = blk / nblk_e;
    const int64_t e = eb * 32 + lane;
    const uint32_t w = e < E ? __ldg(ar + (size_t)e * ar_words + vb) : 0u;
    uint32_t mine = 0;
#pragma unroll
    for (int c = 0; c < 32; ++c) {
      const uint32_t bal = __ballot_sync(0xffffffffu, (w >> c) & 1u);
      if (lane == c) mine = bal;
    }
    const int64_t v = vb * 32 + lane;
    if (v < n) art[(size_t)v * art_words + eb] = mine;
  }
}

}  // namespace

mp_status launch_joint_transpose(const uint32_t* d_ar, int32_t E, int32_t n, int ar_words,
                                 int art_words, uint32_t* d_art, cudaStream_t st) {
  if (E <= 0 || n <= 0) return MP_OK;
  joint_transpose_kernel<<<148 * 16, 256, 0, st>>>(d_ar, E, n, ar_words, art_words, d_art);
  MP_CUDA(cudaGetLastError());
  return MP_OK;
}

mp_status launch_joint(const JointArgs& a, int num_sms, int64_t* d_row_cnt,
                       const int64_t* d_row_off, int2* d_pairs, cudaStream_t st) {
  if (a.E <= 0) return MP_OK;
  int64_t grid = (a.E + 7) / 8;
  if (grid > (int64_t)num_sms * 8) grid = (int64_t)num_sms * 8;
  if (d_pairs)
    joint_kernel<true><<<(unsigned)grid, 256, 0, st>>>(a, nullptr, d_row_off, d_pairs);
  else
    joint_kernel<false><<<(unsigned)grid, 256, 0, st>>>(a, d_row_cnt, nullptr, nullptr);
  MP_CUDA(cudaGetLastError());
  return MP_OK;
}

}  // namespace mpb
