// K1 standalone (one order -> lifetimes), realized lifetimes, and the
// timeline over explicit lifetimes (K3 on intervals).
//
//   lifetimes_from_order     schedule.cpp:33-50 (+ is_topological_order graph.cpp:239-254)
//   realized_lifetimes       plan.cpp:101-120
//   timeline_from_lifetimes  plan.cpp:122-143 (bytes, peak_rs, peak_step)
#include <cuda_runtime.h>

#include <climits>
#include <cstdint>

#include "mp_internal.h"

namespace mpb {
namespace {

constexpr int kThreads = 256;

unsigned blocks_for(int64_t work, int64_t cap = 148 * 16) {
  int64_t b = (work + kThreads - 1) / kThreads;
  if (b < 1) b = 1;
  if (b > cap) b = cap;
  return (unsigned)b;
}

// pos[order[k]] = k + 1; out-of-range ids flag the order invalid.
__global__ void scatter_pos_kernel(const int32_t* __restrict__ order, int32_t n,
                                   int32_t* __restrict__ pos, int32_t* __restrict__ bad) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int v = order[k];
    if ((unsigned)v >= (unsigned)n) atomicOr(bad, 1);
    else pos[v] = (int32_t)k + 1;
  }
}

// Permutation check (order space) + per-edge lifetime and forward check.
__global__ void lifetimes_kernel(const int32_t* __restrict__ order, int32_t n, int32_t E,
                                 const int32_t* __restrict__ src,
                                 const int64_t* __restrict__ sink_off,
                                 const int32_t* __restrict__ sinks,
                                 const int32_t* __restrict__ pos, int32_t* __restrict__ lo,
                                 int32_t* __restrict__ hi, int32_t* __restrict__ bad) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  bool b = false;
  for (int64_t k = t0; k < n; k += stride) {
    const int v = order[k];
    if ((unsigned)v < (unsigned)n && pos[v] != (int32_t)k + 1) b = true;
  }
  for (int64_t e = t0; e < E; e += stride) {
    const int32_t l = pos[src[e]];
    int32_t h = l;
    const int64_t s0 = sink_off[e], s1 = sink_off[e + 1];
    if (s0 == s1) h = n;
    for (int64_t s = s0; s < s1; ++s) {
      const int32_t ps = pos[sinks[s]];
      if (ps <= l) b = true;
      h = max(h, ps);
    }
    lo[e] = l;
    hi[e] = h;
  }
  if (b) atomicOr(bad, 1);
}

__global__ void finalize_valid_kernel(const int32_t* __restrict__ bad, int32_t* __restrict__ valid) {
  valid[0] = bad[0] == 0 ? 1 : 0;
}

// realized_lifetimes: lo = t[src]; hi = horizon if no sinks else max(lo, t[sinks]).
// The smallest edge index touching a node without timestep is recorded; the
// host resolves which endpoint (source first, then sinks) in reference order.
__global__ void realized_kernel(int32_t E, const int32_t* __restrict__ src,
                                const int64_t* __restrict__ sink_off,
                                const int32_t* __restrict__ sinks,
                                const int32_t* __restrict__ ts, int32_t horizon,
                                int32_t* __restrict__ lo, int32_t* __restrict__ hi,
                                int32_t* __restrict__ first_bad_edge) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int32_t l = ts[src[e]];
    bool miss = l == 0;
    const int64_t s0 = sink_off[e], s1 = sink_off[e + 1];
    int32_t h = s0 == s1 ? horizon : l;
    for (int64_t s = s0; s < s1; ++s) {
      const int32_t t = ts[sinks[s]];
      miss |= t == 0;
      h = max(h, t);
    }
    lo[e] = l;
    hi[e] = h;
    if (miss) atomicMin(first_bad_edge, (int32_t)e);
  }
}

// Difference events of closed intervals clipped to [1, horizon]; control
// edges (size 0) and empty intervals contribute nothing (plan.cpp:128-133).
__global__ void timeline_events_kernel(int32_t E, const int32_t* __restrict__ lo,
                                       const int32_t* __restrict__ hi,
                                       const uint64_t* __restrict__ size, int32_t horizon,
                                       unsigned long long* __restrict__ diff) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E;
       e += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t sz = size[e];
    if (sz == 0) continue;
    const int32_t l = max(lo[e], 1), h = min(hi[e], horizon);
    if (l > h) continue;
    atomicAdd(diff + l, (unsigned long long)sz);
    atomicAdd(diff + h + 1, 0ull - (unsigned long long)sz);
  }
}

// One CTA: running prefix sum over t = 1..horizon, bytes out, first argmax.
__global__ void __launch_bounds__(1024)
    timeline_scan_kernel(const unsigned long long* __restrict__ diff, int32_t horizon,
                         uint64_t* __restrict__ bytes, uint64_t* __restrict__ peak_rs,
                         int32_t* __restrict__ peak_step) {
  __shared__ uint64_t wsum[32];
  __shared__ uint64_t wmax[32];
  __shared__ int32_t warg[32];
  __shared__ uint64_t carry_sh;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) carry_sh = 0;
  uint64_t best = 0;
  int32_t best_t = INT_MAX;
  for (int32_t base = 1; base <= horizon; base += 1024) {
    const int32_t t = base + tid;
    uint64_t v = t <= horizon ? (uint64_t)diff[t] : 0;
    uint64_t incl = v;
    for (int d = 1; d < 32; d <<= 1) {
      uint64_t o = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += o;
    }
    __syncthreads();  // carry_sh / wsum from the previous round are consumed
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      uint64_t w = wsum[lane];
      uint64_t wi = w;
      for (int d = 1; d < 32; d <<= 1) {
        uint64_t o = __shfl_up_sync(0xffffffffu, wi, d);
        if (lane >= d) wi += o;
      }
      wsum[lane] = wi - w;
    }
    __syncthreads();
    const uint64_t rs = carry_sh + wsum[warp] + incl;
    if (t <= horizon) {
      if (bytes) bytes[t - 1] = rs;
      if (best_t == INT_MAX || rs > best) {
        best = rs;
        best_t = t;
      }
    }
    __syncthreads();
    if (tid == 1023) carry_sh = rs;
  }
  for (int d = 16; d > 0; d >>= 1) {
    uint64_t v2 = __shfl_xor_sync(0xffffffffu, best, d);
    int32_t t2 = __shfl_xor_sync(0xffffffffu, best_t, d);
    if (v2 > best || (v2 == best && t2 < best_t)) {
      best = v2;
      best_t = t2;
    }
  }
  if (lane == 0) {
    wmax[warp] = best;
    warg[warp] = best_t;
  }
  __syncthreads();
  if (warp == 0) {
    best = wmax[lane];
    best_t = warg[lane];
    for (int d = 16; d > 0; d >>= 1) {
      uint64_t v2 = __shfl_xor_sync(0xffffffffu, best, d);
      int32_t t2 = __shfl_xor_sync(0xffffffffu, best_t, d);
      if (v2 > best || (v2 == best && t2 < best_t)) {
        best = v2;
        best_t = t2;
      }
    }
    if (lane == 0) {
      // plan.cpp:135-141: first strict increase over a running peak from 0,
      // i.e. the first argmax; all-zero gives step 1, an empty horizon 0.
      *peak_rs = horizon > 0 ? best : 0;
      *peak_step = horizon > 0 ? best_t : 0;
    }
  }
}

}  // namespace

mp_status launch_lifetimes(const mp_graph* g, const int32_t* d_order, int64_t order_len,
                           int32_t* d_lo, int32_t* d_hi, int32_t* d_valid, int32_t* d_pos,
                           cudaStream_t st) {
  int32_t* d_bad = reinterpret_cast<int32_t*>(g->ctx->d_small);
  MP_CUDA(cudaMemsetAsync(d_bad, 0, sizeof(int32_t), st));
  if (order_len != g->n) {
    MP_CUDA(cudaMemsetAsync(d_bad, 0xff, sizeof(int32_t), st));
  } else {
    if (g->n > 0) {
      scatter_pos_kernel<<<blocks_for(g->n), kThreads, 0, st>>>(d_order, g->n, d_pos, d_bad);
      MP_CUDA(cudaGetLastError());
    }
    const int64_t work = g->n > g->E ? g->n : g->E;
    if (work > 0) {
      lifetimes_kernel<<<blocks_for(work), kThreads, 0, st>>>(
          d_order, g->n, g->E, g->d_edge_src, g->d_sink_off, g->d_sinks, d_pos, d_lo, d_hi,
          d_bad);
      MP_CUDA(cudaGetLastError());
    }
  }
  finalize_valid_kernel<<<1, 1, 0, st>>>(d_bad, d_valid);
  MP_CUDA(cudaGetLastError());
  return MP_OK;
}

mp_status launch_realized(const mp_graph* g, const int32_t* d_ts, int32_t horizon, int32_t* d_lo,
                          int32_t* d_hi, int32_t* d_first_bad_edge, cudaStream_t st) {
  if (g->E == 0) return MP_OK;
  realized_kernel<<<blocks_for(g->E), kThreads, 0, st>>>(g->E, g->d_edge_src, g->d_sink_off,
                                                         g->d_sinks, d_ts, horizon, d_lo, d_hi,
                                                         d_first_bad_edge);
  MP_CUDA(cudaGetLastError());
  return MP_OK;
}

mp_status launch_timeline(int32_t E, const int32_t* d_lo, const int32_t* d_hi,
                          const uint64_t* d_size, int32_t horizon, uint64_t* d_bytes,
                          uint64_t* d_peak_rs, int32_t* d_peak_step, int64_t* d_diff,
                          cudaStream_t st) {
  const int32_t h = horizon > 0 ? horizon : 0;
  MP_CUDA(cudaMemsetAsync(d_diff, 0, sizeof(int64_t) * ((size_t)h + 2), st));
  if (E > 0 && h > 0) {
    timeline_events_kernel<<<blocks_for(E), kThreads, 0, st>>>(
        E, d_lo, d_hi, d_size, h, reinterpret_cast<unsigned long long*>(d_diff));
    MP_CUDA(cudaGetLastError());
  }
  timeline_scan_kernel<<<1, 1024, 0, st>>>(reinterpret_cast<const unsigned long long*>(d_diff), h,
                                           d_bytes, d_peak_rs, d_peak_step);
  MP_CUDA(cudaGetLastError());
  return MP_OK;
}

}  // namespace mpb
