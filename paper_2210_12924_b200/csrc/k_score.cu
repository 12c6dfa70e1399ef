// K1+K3 fused: batched candidate-order scoring.
//
// For every candidate order (one row of int32[C][n]) one CTA computes, with
// no host round trip and no global intermediate when the graph is small
// enough for shared memory:
//   * the is_topological_order verdict          (graph.cpp:239-254)
//   * 1-based positions                         (schedule.cpp:23-31)
//   * lifetimes lo = pos[src], hi = last sink   (schedule.cpp:33-50)
//   * resident bytes per step and the peak      (schedule.cpp:69-88)
//   * the first step attaining the peak         (plan.cpp:135-141)
//
// Reformulation (exact): instead of the reference's
// O(sum of lifetime lengths) accumulation, each node's static allocation
// (sum of its data fanout) and the bytes freed after it by single-consumer
// edges are scattered to the node's position, multi-consumer edges add their
// size at the position of their last consumer, and RS(t) follows from one
// prefix sum:  RS(p) = sum_{q<=p} (alloc_q - free_q) + free_p.
// uint64 wrap-around arithmetic is exact because every RS(p) < 2^62
// (graph.cpp:122-128).
#include <cuda_runtime.h>

#include <climits>
#include <cstdint>

#include "mp_internal.h"

namespace mpb {
namespace {

struct ScoreGraph {
  int32_t n;
  int32_t M;
  const int32_t* __restrict__ pred_off;
  const int32_t* __restrict__ preds;
  const uint64_t* __restrict__ node_alloc;
  const uint64_t* __restrict__ node_sfree;
  const int32_t* __restrict__ multi_off;
  const int32_t* __restrict__ multi_sinks;
  const uint64_t* __restrict__ multi_size;
};

constexpr int kWarp = 32;

__device__ __forceinline__ uint64_t warp_incl_scan(uint64_t v, int lane) {
#pragma unroll
  for (int d = 1; d < kWarp; d <<= 1) {
    uint64_t o = __shfl_up_sync(0xffffffffu, v, d);
    if (lane >= d) v += o;
  }
  return v;
}

// (value, index) with "greater value, then smaller index" preference.
__device__ __forceinline__ void argmax_merge(uint64_t& v, int32_t& i, uint64_t v2, int32_t i2) {
  if (v2 > v || (v2 == v && i2 < i)) {
    v = v2;
    i = i2;
  }
}

template <int THREADS>
struct BlockShared {
  uint64_t warp_sum[THREADS / kWarp];
  uint64_t warp_max[THREADS / kWarp];
  int32_t warp_arg[THREADS / kWarp];
};

// Per-candidate state: X[n] (uint64), F[n] (uint64), pos[n] (int32), either
// in dynamic shared memory (kSmem) or in a per-CTA global scratch slice.
template <int THREADS, bool kSmem>
__global__ void __launch_bounds__(THREADS)
    score_kernel(ScoreGraph G, const int32_t* __restrict__ orders, int64_t C,
                 uint64_t* __restrict__ peak_out, int32_t* __restrict__ step_out,
                 uint8_t* __restrict__ valid_out, uint64_t* __restrict__ bytes_out,
                 unsigned long long* __restrict__ best_key, int64_t index_base,
                 char* __restrict__ gscratch, size_t gstride) {
  extern __shared__ __align__(16) char dyn_smem[];
  __shared__ BlockShared<THREADS> sh;

  const int n = G.n;
  const int tid = threadIdx.x;
  const int lane = tid & (kWarp - 1);
  const int warp = tid / kWarp;

  char* base = kSmem ? dyn_smem : gscratch + (size_t)blockIdx.x * gstride;
  uint64_t* X = reinterpret_cast<uint64_t*>(base);
  uint64_t* F = X + n;
  int32_t* pos = reinterpret_cast<int32_t*>(F + n);

  const int P = (n + THREADS - 1) / THREADS;  // blocked scan chunk
  const int my_begin = min(n, tid * P);
  const int my_end = min(n, my_begin + P);

  for (int64_t c = blockIdx.x; c < C; c += gridDim.x) {
    const int32_t* ord = orders + c * (int64_t)n;
    bool bad = false;

    // Phase 1 (order space): inverse permutation pos[order[k]] = k.
    for (int k = tid; k < n; k += THREADS) {
      int v = __ldg(ord + k);
      if ((unsigned)v >= (unsigned)n) bad = true;
      else pos[v] = k;
    }
    __syncthreads();

    // Phase 2a (order space): each node exactly once. With n slots and n
    // checks, pos[order[k]] == k for all k implies a permutation.
    for (int k = tid; k < n; k += THREADS) {
      int v = __ldg(ord + k);
      if ((unsigned)v < (unsigned)n && pos[v] != k) bad = true;
    }
    // Phase 2b (node space): every producer strictly before its consumer,
    // then the node's static bytes go to its position.
    for (int v = tid; v < n; v += THREADS) {
      int p = pos[v];
      if ((unsigned)p >= (unsigned)n) {
        bad = true;
        continue;
      }
      const int q0 = __ldg(G.pred_off + v), q1 = __ldg(G.pred_off + v + 1);
      for (int q = q0; q < q1; ++q)
        if (pos[__ldg(G.preds + q)] >= p) bad = true;
      const uint64_t sf = __ldg(G.node_sfree + v);
      X[p] = __ldg(G.node_alloc + v) - sf;
      F[p] = sf;
    }
    __syncthreads();

    // Phase 3: multi-consumer data edges free after their last consumer.
    for (int m = tid; m < G.M; m += THREADS) {
      int h = -1;
      const int s0 = __ldg(G.multi_off + m), s1 = __ldg(G.multi_off + m + 1);
      for (int s = s0; s < s1; ++s) h = max(h, pos[__ldg(G.multi_sinks + s)]);
      if ((unsigned)h < (unsigned)n) {
        const unsigned long long sz = __ldg(G.multi_size + m);
        atomicAdd(reinterpret_cast<unsigned long long*>(F + h), sz);
        atomicAdd(reinterpret_cast<unsigned long long*>(X + h), 0ull - sz);
      }
    }
    const bool any_bad = __syncthreads_or(bad);

    if (any_bad) {
      if (tid == 0) {
        peak_out[c] = 0;
        step_out[c] = 0;
        valid_out[c] = 0;
      }
      continue;  // the __syncthreads_or above already fenced this iteration
    }

    // Phase 4: blocked exclusive scan over positions, then RS and argmax.
    uint64_t local = 0;
    for (int p = my_begin; p < my_end; ++p) local += X[p];
    uint64_t incl = warp_incl_scan(local, lane);
    if (lane == kWarp - 1) sh.warp_sum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      uint64_t w = lane < THREADS / kWarp ? sh.warp_sum[lane] : 0;
      uint64_t wi = warp_incl_scan(w, lane);
      if (lane < THREADS / kWarp) sh.warp_sum[lane] = wi - w;  // exclusive
    }
    __syncthreads();
    uint64_t run = sh.warp_sum[warp] + incl - local;  // exclusive prefix of my chunk
    uint64_t best = 0;
    int32_t best_i = INT_MAX;
    for (int p = my_begin; p < my_end; ++p) {
      run += X[p];
      const uint64_t rs = run + F[p];
      if (bytes_out) bytes_out[c * (int64_t)n + p] = rs;
      if (best_i == INT_MAX || rs > best) {
        best = rs;
        best_i = p;
      }
    }
#pragma unroll
    for (int d = kWarp / 2; d > 0; d >>= 1) {
      uint64_t v2 = __shfl_xor_sync(0xffffffffu, best, d);
      int32_t i2 = __shfl_xor_sync(0xffffffffu, best_i, d);
      argmax_merge(best, best_i, v2, i2);
    }
    if (lane == 0) {
      sh.warp_max[warp] = best;
      sh.warp_arg[warp] = best_i;
    }
    __syncthreads();
    if (warp == 0) {
      best = lane < THREADS / kWarp ? sh.warp_max[lane] : 0;
      best_i = lane < THREADS / kWarp ? sh.warp_arg[lane] : INT_MAX;
#pragma unroll
      for (int d = kWarp / 2; d > 0; d >>= 1) {
        uint64_t v2 = __shfl_xor_sync(0xffffffffu, best, d);
        int32_t i2 = __shfl_xor_sync(0xffffffffu, best_i, d);
        argmax_merge(best, best_i, v2, i2);
      }
      if (lane == 0) {
        const bool empty = n == 0;
        const uint64_t pk = empty ? 0 : best;
        peak_out[c] = pk;
        step_out[c] = empty ? 0 : best_i + 1;  // first t with RS(t) == peak
        valid_out[c] = 1;
        // Fused first-minimum argmin: the packed key orders by (peak, index).
        if (best_key) {
          const uint64_t gi = (uint64_t)(c + index_base);
          const unsigned long long key =
              (pk < (1ull << 43) && gi < (1ull << 20)) ? ((pk << 20) | gi) : ~0ull - 1;
          atomicMin(best_key, key);
        }
      }
    }
    // sh.warp_* are rewritten only after two more barriers of the next
    // iteration; X/F/pos after at least one.
  }
}

template <int THREADS, bool kSmem>
mp_status run_score(const mp_graph* g, const int32_t* d_orders, int64_t C, uint64_t* d_peak,
                    int32_t* d_step, uint8_t* d_valid, uint64_t* d_bytes, uint64_t* d_key,
                    int64_t index_base, cudaStream_t st) {
  ScoreGraph G{g->n,           g->M,           g->d_pred_off,    g->d_preds,     g->d_node_alloc,
               g->d_node_sfree, g->d_multi_off, g->d_multi_sinks, g->d_multi_size};
  auto kern = score_kernel<THREADS, kSmem>;
  const size_t per = (size_t)g->n * 20 + 16;
  int blocks_per_sm = 0;
  const size_t smem = kSmem ? per : 0;
  if (kSmem) MP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)smem));
  MP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, kern, THREADS, smem));
  if (blocks_per_sm < 1) blocks_per_sm = 1;
  int64_t grid = (int64_t)g->ctx->num_sms * blocks_per_sm;
  char* gs = nullptr;
  size_t gstride = 0;
  if (!kSmem) {
    grid = (int64_t)g->ctx->num_sms * 2;
    gstride = (per + 255) & ~size_t(255);
    MP_TRY(g->ctx->scratch[3].reserve(gstride * grid));
    gs = static_cast<char*>(g->ctx->scratch[3].ptr);
  }
  if (grid > C) grid = C;
  if (grid < 1) return MP_OK;
  kern<<<(unsigned)grid, THREADS, smem, st>>>(G, d_orders, C, d_peak, d_step, d_valid, d_bytes,
                                              reinterpret_cast<unsigned long long*>(d_key),
                                              index_base, gs, gstride);
  MP_CUDA(cudaGetLastError());
  return MP_OK;
}

}  // namespace

mp_status score_configure(mp_graph* g) {
  const size_t per = (size_t)g->n * 20 + 16;
  g->smem_resident = per + 4096 <= g->ctx->max_smem_optin;
  g->score_smem_bytes = g->smem_resident ? per : 0;
  return MP_OK;
}

mp_status launch_score(const mp_graph* g, const int32_t* d_orders, int64_t C, uint64_t* d_peak,
                       int32_t* d_step, uint8_t* d_valid, uint64_t* d_bytes, uint64_t* d_key,
                       int64_t index_base, cudaStream_t st) {
  if (C <= 0) return MP_OK;
  if (g->smem_resident) {
    if (g->n <= 4096)
      return run_score<256, true>(g, d_orders, C, d_peak, d_step, d_valid, d_bytes, d_key,
                                  index_base, st);
    return run_score<1024, true>(g, d_orders, C, d_peak, d_step, d_valid, d_bytes, d_key,
                                 index_base, st);
  }
  return run_score<1024, false>(g, d_orders, C, d_peak, d_step, d_valid, d_bytes, d_key,
                                index_base, st);
}

// ---- argmin over candidates (single CTA; C is at most a few million) ------------
// Lexicographic (peak, index) minimum over valid candidates: the first
// minimum, as enumerate_min_peak keeps the first strictly smaller peak
// (oracle.cpp:78-81). out[0] = best index + base (or -1), out[1] = its
// peak, out[2] = packed key peak << 20 | index (UINT64_MAX when nothing is
// valid or the key would not fit) for a single allreduce(min) across GPUs.
namespace {
__device__ __forceinline__ void amin_merge(uint64_t& p, int64_t& i, uint64_t p2, int64_t i2) {
  if (i2 >= 0 && (i < 0 || p2 < p || (p2 == p && i2 < i))) {
    p = p2;
    i = i2;
  }
}

__global__ void __launch_bounds__(1024)
    argmin_kernel(const uint64_t* __restrict__ peak, const uint8_t* __restrict__ valid,
                  int64_t C, int64_t base, uint64_t* __restrict__ out) {
  uint64_t bp = 0;
  int64_t bi = -1;
  for (int64_t c = threadIdx.x; c < C; c += blockDim.x)
    if (valid[c]) amin_merge(bp, bi, peak[c], c);
  for (int d = 16; d > 0; d >>= 1) {
    uint64_t p2 = __shfl_xor_sync(0xffffffffu, bp, d);
    int64_t i2 = __shfl_xor_sync(0xffffffffu, bi, d);
    amin_merge(bp, bi, p2, i2);
  }
  __shared__ uint64_t wp[32];
  __shared__ int64_t wi[32];
  if ((threadIdx.x & 31) == 0) {
    wp[threadIdx.x >> 5] = bp;
    wi[threadIdx.x >> 5] = bi;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    const bool live = threadIdx.x < blockDim.x / 32;
    bp = live ? wp[threadIdx.x] : 0;
    bi = live ? wi[threadIdx.x] : -1;
    for (int d = 16; d > 0; d >>= 1) {
      uint64_t p2 = __shfl_xor_sync(0xffffffffu, bp, d);
      int64_t i2 = __shfl_xor_sync(0xffffffffu, bi, d);
      amin_merge(bp, bi, p2, i2);
    }
    if (threadIdx.x == 0) {
      const int64_t gi = bi < 0 ? -1 : bi + base;
      out[0] = (uint64_t)gi;
      out[1] = bp;
      const bool fits = gi >= 0 && gi < (1 << 20) && bp < (1ull << 43);
      out[2] = fits ? ((bp << 20) | (uint64_t)gi) : ~0ull;
    }
  }
}
}  // namespace

mp_status launch_argmin(const uint64_t* d_peak, const uint8_t* d_valid, int64_t C, int64_t base,
                        uint64_t* d_out3, cudaStream_t st) {
  argmin_kernel<<<1, 1024, 0, st>>>(d_peak, d_valid, C, base, d_out3);
  MP_CUDA(cudaGetLastError());
  return MP_OK;
}

}  // namespace mpb
