// Batched candidate PLANS: the placement half of plan_once
// (proj/src/pipeline.cpp:236-285) composed per candidate order, so that a
// batch of schedules becomes a batch of checked address plans:
//
//   lifetimes_from_order        (schedule.cpp:33-50)      lifetimes_batch_kernel
//   preallocate_pyramid + greedy_pack (placement.cpp:25-62, 182-204)   K5 (k_place.cu)
//   peak_mem = max(addr + size) (pipeline.cpp:270-275)                  K5
//   addresses_feasible / validate_plan's below_above pairs
//                               (pipeline.cpp:146-160, plan.cpp:390-404) plan_check_kernel
//
// plus the scores of the schedules themselves (K3) and the first-minimum
// plan by peak_mem over the feasible ones (a fused atomicMin key).
#include <cuda_runtime.h>

#include <algorithm>

#include <climits>
#include <cstdint>

#include "mp_internal.h"

namespace mpb {
namespace {

constexpr int kLT = 512;  // threads per CTA, both kernels

// One CTA per candidate (persistent): positions in shared memory (1-based,
// 0 = never written), then per edge lo = pos[src], hi = n without sinks else
// max over sinks, and the reference's forward check on every (src, sink).
__global__ void __launch_bounds__(kLT)
    lifetimes_batch_kernel(const int32_t* __restrict__ orders, int64_t C, int32_t n, int32_t E,
                           const int32_t* __restrict__ src, const int64_t* __restrict__ sink_off,
                           const int32_t* __restrict__ sinks, int32_t* __restrict__ lo,
                           int32_t* __restrict__ hi, uint8_t* __restrict__ valid) {
  extern __shared__ __align__(16) int32_t pos[];
  for (int64_t c = blockIdx.x; c < C; c += gridDim.x) {
    const int32_t* ord = orders + c * (int64_t)n;
    for (int i = threadIdx.x; i < n; i += kLT) pos[i] = 0;
    __syncthreads();
    bool bad = false;
    for (int k = threadIdx.x; k < n; k += kLT) {
      const int v = __ldg(ord + k);
      if ((unsigned)v >= (unsigned)n) bad = true;
      else pos[v] = k + 1;
    }
    __syncthreads();
    for (int v = threadIdx.x; v < n; v += kLT) bad |= pos[v] == 0;  // n writes, n nodes
    int32_t* lo_c = lo + c * (int64_t)E;
    int32_t* hi_c = hi + c * (int64_t)E;
    for (int e = threadIdx.x; e < E; e += kLT) {
      const int32_t l = pos[__ldg(src + e)];
      const int64_t s0 = __ldg(sink_off + e), s1 = __ldg(sink_off + e + 1);
      int32_t h = s0 == s1 ? n : l;
      for (int64_t s = s0; s < s1; ++s) {
        const int32_t ps = pos[__ldg(sinks + s)];
        bad |= ps <= l;
        h = max(h, ps);
      }
      lo_c[e] = l;
      hi_c[e] = h;
    }
    const int any_bad = __syncthreads_or(bad);  // also: every read of pos is done
    if (threadIdx.x == 0) valid[c] = any_bad ? 0 : 1;
  }
}

// One CTA per plan: the candidate's (lifetime, address) records in shared
// memory, a warp per row i (round robin), lanes over j > i, counting the pairs
// that validate_plan reports as below_above: both data edges with an address,
// closed lifetimes intersecting, [addr, addr + size) ranges overlapping.
struct PlanRec {
  int32_t lo, hi;  // ineligible edges: lo = INT_MAX, hi = INT_MIN (never intersect)
  uint64_t a, s;
};

__global__ void __launch_bounds__(kLT)
    plan_check_kernel(int64_t C, int32_t E, const int32_t* __restrict__ lo,
                      const int32_t* __restrict__ hi, const uint64_t* __restrict__ size,
                      const uint8_t* __restrict__ has, const uint64_t* __restrict__ addr,
                      const uint8_t* __restrict__ valid, uint32_t* __restrict__ nviol,
                      uint64_t* __restrict__ peak_mem) {
  extern __shared__ __align__(16) PlanRec rec[];
  __shared__ uint32_t wcount[kLT / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t c = blockIdx.x; c < C; c += gridDim.x) {
    if (valid && !valid[c]) {  // an invalid order has no lifetimes, hence no plan
      if (threadIdx.x == 0) {
        nviol[c] = 0;
        if (peak_mem) peak_mem[c] = 0;
      }
      continue;
    }
    const int64_t base = c * (int64_t)E;
    for (int e = threadIdx.x; e < E; e += kLT) {
      const uint64_t s = __ldg(size + e);
      const bool ok = s > 0 && has[base + e];
      rec[e] = ok ? PlanRec{lo[base + e], hi[base + e], addr[base + e], s}
                  : PlanRec{INT_MAX, INT_MIN, 0, 0};
    }
    __syncthreads();
    uint32_t cnt = 0;
    for (int i = warp; i < E; i += kLT / 32) {
      const PlanRec r = rec[i];
      if (r.lo > r.hi) continue;  // warp-uniform: ineligible row
      for (int j = i + 1 + lane; j < E; j += 32) {
        const PlanRec q = rec[j];
        cnt += (r.lo <= q.hi && q.lo <= r.hi && r.a < q.a + q.s && q.a < r.a + r.s) ? 1u : 0u;
      }
    }
    for (int d = 16; d > 0; d >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, d);
    if (lane == 0) wcount[warp] = cnt;
    __syncthreads();
    if (warp == 0) {
      cnt = lane < kLT / 32 ? wcount[lane] : 0u;
      for (int d = 16; d > 0; d >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, d);
      if (lane == 0) nviol[c] = cnt;
    }
    __syncthreads();  // rec / wcount reused by the next plan
  }
}

// First minimum by peak_mem over the feasible plans (valid order, no conflicting
// pair): the same two-word key protocol as the fused scorer (k_score.cu).
__global__ void plan_key_kernel(int64_t C, const uint8_t* __restrict__ valid,
                                const uint32_t* __restrict__ nviol,
                                const uint64_t* __restrict__ peak_mem, int64_t index_base,
                                unsigned long long* __restrict__ key) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < C;
       c += (int64_t)gridDim.x * blockDim.x) {
    if (!valid[c] || nviol[c] != 0) continue;
    const uint64_t pk = peak_mem[c], gi = (uint64_t)(c + index_base);
    if (pk < (1ull << 42) && gi < (1ull << 20)) atomicMin(key, (unsigned long long)((pk << 20) | gi));
    else atomicMin(key + 1, 0ull);
  }
}

// Large graphs (launch_plans_large): one plan's conflict count, read from the K4 sweep's
// device total, clamped to 32 bits; an invalid order has no plan (count 0, peak_mem 0).
__global__ void plan_store_count_kernel(const int64_t* __restrict__ total,
                                        const uint8_t* __restrict__ valid, int64_t c,
                                        uint32_t* __restrict__ nviol, uint64_t* __restrict__ peak_mem) {
  if (threadIdx.x != 0) return;
  const bool ok = valid[c] != 0;
  const int64_t t = *total;
  nviol[c] = ok ? (uint32_t)(t < 0xffffffffll ? t : 0xffffffffll) : 0u;
  if (!ok && peak_mem) peak_mem[c] = 0;
}
__global__ void valid_narrow_kernel(const int32_t* __restrict__ v32, int64_t C,
                                    uint8_t* __restrict__ v8) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < C;
       c += (int64_t)gridDim.x * blockDim.x)
    v8[c] = v32[c] != 0 ? 1 : 0;
}

}  // namespace

size_t lifetimes_batch_smem(int32_t n) { return (size_t)n * 4; }
size_t plan_check_smem(int32_t E) { return (size_t)E * sizeof(PlanRec); }

mp_status launch_lifetimes_batch(const mp_graph* g, const int32_t* d_orders, int64_t C,
                                 int32_t* d_lo, int32_t* d_hi, uint8_t* d_valid, cudaStream_t st) {
  if (C <= 0) return MP_OK;
  const size_t smem = lifetimes_batch_smem(g->n);
  if (smem > g->ctx->max_smem_optin) return MP_E_CAPACITY;
  MP_CUDA(cudaFuncSetAttribute(lifetimes_batch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem));
  int per_sm = 0;
  MP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lifetimes_batch_kernel, kLT, smem));
  int64_t grid = (int64_t)g->ctx->num_sms * (per_sm > 0 ? per_sm : 1);
  if (grid > C) grid = C;
  lifetimes_batch_kernel<<<(unsigned)grid, kLT, smem, st>>>(
      d_orders, C, g->n, g->E, g->d_edge_src, g->d_sink_off, g->d_sinks, d_lo, d_hi, d_valid);
  MP_CUDA(cudaGetLastError());
  return MP_OK;
}

mp_status launch_plan_check(const mp_ctx* ctx, int64_t C, int32_t E, const int32_t* d_lo,
                            const int32_t* d_hi, const uint64_t* d_size, const uint8_t* d_has,
                            const uint64_t* d_addr, const uint8_t* d_valid, uint32_t* d_nviol,
                            uint64_t* d_peak_mem, cudaStream_t st) {
  if (C <= 0) return MP_OK;
  const size_t smem = plan_check_smem(E);
  if (smem > ctx->max_smem_optin) return MP_E_CAPACITY;
  MP_CUDA(cudaFuncSetAttribute(plan_check_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem));
  int per_sm = 0;
  MP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, plan_check_kernel, kLT, smem));
  int64_t grid = (int64_t)ctx->num_sms * (per_sm > 0 ? per_sm : 1);
  if (grid > C) grid = C;
  plan_check_kernel<<<(unsigned)grid, kLT, smem, st>>>(C, E, d_lo, d_hi, d_size, d_has, d_addr,
                                                       d_valid, d_nviol, d_peak_mem);
  MP_CUDA(cudaGetLastError());
  return MP_OK;
}

mp_status launch_plan_key(int64_t C, const uint8_t* d_valid, const uint32_t* d_nviol,
                          const uint64_t* d_peak_mem, int64_t index_base, uint64_t* d_key,
                          cudaStream_t st) {
  if (C <= 0 || !d_key) return MP_OK;
  const int64_t blocks = (C + 255) / 256;
  plan_key_kernel<<<(unsigned)(blocks < 1024 ? blocks : 1024), 256, 0, st>>>(
      C, d_valid, d_nviol, d_peak_mem, index_base, reinterpret_cast<unsigned long long*>(d_key));
  MP_CUDA(cudaGetLastError());
  return MP_OK;
}

// Candidate plans on graphs past the shared-memory kernels (the 100k-tensor graph):
// lifetimes per candidate with K1 (positions in global scratch), and each plan's address
// check with the K4 sweep over the whole GPU (validate_plan's below_above pairs),
// counted on the device. Placement (K5's global-memory variant) runs in between.
mp_status launch_lifetimes_large(const mp_graph* g, const int32_t* d_orders, int64_t C,
                                 int32_t* d_lo, int32_t* d_hi, int32_t* d_valid32,
                                 uint8_t* d_valid, int32_t* d_pos, cudaStream_t st) {
  const int64_t n = g->n, E = g->E;
  for (int64_t c = 0; c < C; ++c)
    MP_TRY(launch_lifetimes(g, d_orders + c * n, n, d_lo + c * E, d_hi + c * E, d_valid32 + c,
                            d_pos, st));
  valid_narrow_kernel<<<(unsigned)std::min<int64_t>((C + 255) / 256, 1024), 256, 0, st>>>(
      d_valid32, C, d_valid);
  MP_CUDA(cudaGetLastError());
  return MP_OK;
}

mp_status launch_plan_check_large(mp_ctx* ctx, int64_t C, int32_t E, const int32_t* d_lo,
                                  const int32_t* d_hi, const uint64_t* d_size,
                                  const uint8_t* d_has, const uint64_t* d_addr,
                                  const uint8_t* d_valid, uint32_t* d_nviol, uint64_t* d_peak_mem,
                                  int64_t* d_row_off, cudaStream_t st) {
  PairArgs a;
  a.num_edges = E;
  a.size = d_size;
  a.mode = 1;
  a.row_begin = 0;
  a.row_end = E;
  MP_TRY(ctx->scratch[2].reserve(pairs_scratch_bytes(a, ctx->num_sms)));
  for (int64_t c = 0; c < C; ++c) {
    a.lo = d_lo + c * E;
    a.hi = d_hi + c * E;
    a.mask = d_has + c * E;
    a.addr = d_addr + c * E;
    MP_TRY(pairs_count(a, ctx->num_sms, ctx->scratch[2].ptr, d_row_off, nullptr, st));
    plan_store_count_kernel<<<1, 32, 0, st>>>(pairs_device_total(a, ctx->num_sms, ctx->scratch[2].ptr),
                                              d_valid, c, d_nviol, d_peak_mem);
    MP_CUDA(cudaGetLastError());
  }
  return MP_OK;
}

}  // namespace mpb
