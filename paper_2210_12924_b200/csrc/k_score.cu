// K1+K3 fused: batched candidate-order scoring (one CTA per candidate in
// flight, persistent grid).
//
// For every candidate order (row of int32[C][n]) this computes
//   * the is_topological_order verdict          (graph.cpp:239-254)
//   * positions                                  (schedule.cpp:23-31)
//   * lifetimes lo = pos[src], hi = last sink    (schedule.cpp:33-50)
//   * resident bytes per step and the peak       (schedule.cpp:69-88)
//   * the first step attaining the peak          (plan.cpp:135-141)
//   * optionally the (peak, index) first-minimum over candidates (atomicMin)
//
// Reformulation (exact for valid orders). With node v at
// position p(v): RS(p) = sum_{q<=p} (alloc_q - free_q) + free_p, where
// alloc_q is the static fanout bytes of the node at q and free_q the bytes
// whose last consumer is that node. Host preprocessing (mp_prep.cpp) makes
// most frees static (single consumer, or every other consumer reaches this
// one) and drops redundant validity edges, so per candidate the device does:
//   phase 1 (order space)  pos[order[k]] = stamp|k                 n scatters
//   phase 2 (node space)   stamp check = permutation check,        n sequential reads
//                          producers-before-consumers,             |reduced preds| gathers
//                          order-dependent last consumers,         few gathers
//                          XF[p(v)] = (alloc - free, free)         n scatters
//   phase 3 (order space)  two-pass warp scan + first argmax       sequential
// Static per-node data lives in registers of the owning thread (node
// v = tid + j*T, j < J) for the whole persistent loop; the next candidate's
// order slice is prefetched into registers while the current one is scored.
// Values are in units of gcd(sizes); 32-bit when total/gcd < 2^32 (every
// RS then fits, and modular sums are exact).
#include <cuda_runtime.h>

#include <climits>
#include <cstdint>

#include "mp_internal.h"
#include "mp_prep.h"

namespace mpb {
namespace {

constexpr int kWarp = 32;

struct ScoreTables {
  int32_t n;
  int32_t npreds;
  int32_t ndyn;
  int32_t nbig;
  uint64_t scale;
  const int32_t* __restrict__ pred_off;
  const int32_t* __restrict__ preds;
  const uint64_t* __restrict__ alloc;
  const uint64_t* __restrict__ sfree;
  const int32_t* __restrict__ dyn_off;
  const DynMember* __restrict__ dyn;
  const int32_t* __restrict__ big_off;
  const int32_t* __restrict__ big_sinks;
  const uint64_t* __restrict__ big_size;
};

// Position word: stamp in the high half, position in the low half. Within one
// candidate all written words share the stamp, so comparing whole words
// compares positions; a stale stamp marks a node the order never wrote.
template <typename PW>
struct PosWord;
template <>
struct PosWord<uint32_t> {
  static constexpr uint32_t kMaxStamp = 0xffffu;
  __device__ static uint32_t make(uint32_t stamp, int k) { return (stamp << 16) | (uint32_t)k; }
  __device__ static uint32_t stamp(uint32_t w) { return w >> 16; }
  __device__ static int pos(uint32_t w) { return (int)(w & 0xffffu); }
};
template <>
struct PosWord<unsigned long long> {
  static constexpr uint32_t kMaxStamp = 0xffffffffu;
  __device__ static unsigned long long make(uint32_t stamp, int k) {
    return ((unsigned long long)stamp << 32) | (uint32_t)k;
  }
  __device__ static uint32_t stamp(unsigned long long w) { return (uint32_t)(w >> 32); }
  __device__ static int pos(unsigned long long w) { return (int)(uint32_t)w; }
};

template <typename VT>
struct XFPair {
  VT x, f;
};

template <typename VT>
__device__ __forceinline__ VT warp_sum(VT v) {
#pragma unroll
  for (int d = kWarp / 2; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
  return v;
}

template <typename VT>
__device__ __forceinline__ VT warp_incl_scan(VT v, int lane) {
#pragma unroll
  for (int d = 1; d < kWarp; d <<= 1) {
    VT o = __shfl_up_sync(0xffffffffu, v, d);
    if (lane >= d) v += o;
  }
  return v;
}

// max value, then smallest index
template <typename VT>
__device__ __forceinline__ void warp_argmax(VT& v, int& i) {
#pragma unroll
  for (int d = kWarp / 2; d > 0; d >>= 1) {
    VT v2 = __shfl_xor_sync(0xffffffffu, v, d);
    int i2 = __shfl_xor_sync(0xffffffffu, i, d);
    if (v2 > v || (v2 == v && i2 < i)) {
      v = v2;
      i = i2;
    }
  }
}

template <typename VT>
struct BlockScratch {
  VT wsum[32];
  VT wbest[32];
  int widx[32];
};

// J > 0: static node data in registers (node v = tid + j*T, T <= 512),
//        per-candidate buffers in shared memory.
// J == 0: node data read from global (coalesced, L1/L2-resident) per
//        candidate; buffers in shared memory (kSmem) or per-CTA global scratch.
// Node ranges are packed as offset << 12 | count (count < 4096, checked on
// the host; offsets < 2^20 in the shared-memory variants).
constexpr int kCntBits = 12;
constexpr int kCntMask = (1 << kCntBits) - 1;

template <typename VT, typename PW, int J, bool kSmem>
__global__ void __launch_bounds__(J > 0 ? 512 : 1024)
    score_kernel(ScoreTables G, const int32_t* __restrict__ orders, int64_t C,
                 uint64_t* __restrict__ peak_out, int32_t* __restrict__ step_out,
                 uint8_t* __restrict__ valid_out, uint64_t* __restrict__ bytes_out,
                 unsigned long long* __restrict__ best_key, int64_t index_base,
                 char* __restrict__ gscratch, size_t gstride) {
  using PWT = PosWord<PW>;
  extern __shared__ __align__(16) char smem[];
  __shared__ BlockScratch<VT> bs;

  const int n = G.n;
  const int T = blockDim.x;
  const int tid = threadIdx.x;
  const int lane = tid & (kWarp - 1);
  const int warp = tid >> 5;
  const int nwarps = T >> 5;

  // ---- buffers -------------------------------------------------------------
  const int32_t* preds;
  const DynMember* dyn;
  PW* pos;
  XFPair<VT>* XF;
  if (kSmem) {
    char* p = smem;
    int32_t* sp = reinterpret_cast<int32_t*>(p);
    p += ((size_t)G.npreds * 4 + 15) & ~size_t(15);
    DynMember* sd = reinterpret_cast<DynMember*>(p);
    p += ((size_t)G.ndyn * sizeof(DynMember) + 15) & ~size_t(15);
    pos = reinterpret_cast<PW*>(p);
    p += ((size_t)n * sizeof(PW) + 15) & ~size_t(15);
    XF = reinterpret_cast<XFPair<VT>*>(p);
    for (int i = tid; i < G.npreds; i += T) sp[i] = G.preds[i];
    const int32_t* gd = reinterpret_cast<const int32_t*>(G.dyn);
    int32_t* sdw = reinterpret_cast<int32_t*>(sd);
    for (int i = tid; i < G.ndyn * (int)(sizeof(DynMember) / 4); i += T) sdw[i] = gd[i];
    preds = sp;
    dyn = sd;
  } else {
    char* p = gscratch + (size_t)blockIdx.x * gstride;
    pos = reinterpret_cast<PW*>(p);
    p += ((size_t)n * sizeof(PW) + 255) & ~size_t(255);
    XF = reinterpret_cast<XFPair<VT>*>(p);
    preds = G.preds;
    dyn = G.dyn;
  }
  for (int i = tid; i < n; i += T) pos[i] = 0;  // stamp 0 is never used

  // ---- static per-node data in registers -------------------------------------
  constexpr int JR = J > 0 ? J : 1;
  VT ra[JR], rf[JR];
  uint32_t pr[JR], dr[JR];  // packed (offset << 12 | count)
  int ov[JR];
  if (J > 0) {
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const int v = tid + j * T;
      const bool in = v < n;
      ra[j] = in ? (VT)G.alloc[v] : (VT)0;
      rf[j] = in ? (VT)G.sfree[v] : (VT)0;
      pr[j] = in ? ((uint32_t)G.pred_off[v] << kCntBits) |
                       (uint32_t)(G.pred_off[v + 1] - G.pred_off[v])
                 : 0u;
      dr[j] = in ? ((uint32_t)G.dyn_off[v] << kCntBits) |
                       (uint32_t)(G.dyn_off[v + 1] - G.dyn_off[v])
                 : 0u;
      ov[j] = 0;
    }
    if ((int64_t)blockIdx.x < C) {
      const int32_t* ord = orders + (int64_t)blockIdx.x * n;
#pragma unroll
      for (int j = 0; j < J; ++j) {
        const int k = tid + j * T;
        ov[j] = k < n ? __ldg(ord + k) : 0;
      }
    }
  }
  __syncthreads();

  uint32_t stamp = 0;
  for (int64_t c = blockIdx.x; c < C; c += gridDim.x) {
    if (++stamp > PWT::kMaxStamp) {  // stamp wrap: forget every old position
      for (int i = tid; i < n; i += T) pos[i] = 0;
      stamp = 1;
      __syncthreads();
    }
    bool bad = false;

    // ---- phase 1: inverse permutation (order space) ----------------------------
    if (J > 0) {
#pragma unroll
      for (int j = 0; j < J; ++j) {
        const int k = tid + j * T;
        if (k < n) {
          const int v = ov[j];
          if ((unsigned)v >= (unsigned)n) bad = true;
          else pos[v] = PWT::make(stamp, k);
        }
      }
      // prefetch the next candidate's slice; it lands while this one is scored
      const int64_t cn = c + gridDim.x;
      if (cn < C) {
        const int32_t* ord = orders + cn * n;
#pragma unroll
        for (int j = 0; j < J; ++j) {
          const int k = tid + j * T;
          ov[j] = k < n ? __ldg(ord + k) : 0;
        }
      }
    } else {
      const int32_t* ord = orders + c * n;
      for (int k = tid; k < n; k += T) {
        const int v = __ldg(ord + k);
        if ((unsigned)v >= (unsigned)n) bad = true;
        else pos[v] = PWT::make(stamp, k);
      }
    }
    __syncthreads();

    // ---- phase 2: node space -----------------------------------------------------
    auto node = [&](int v, VT a, VT sf, int q0, int q1, int e0, int e1) {
      // q0..q1: reduced producers of v; e0..e1: v's order-dependent memberships
      const PW w = pos[v];
      if (PWT::stamp(w) != stamp) bad = true;  // never written: not a permutation
      for (int q = q0; q < q1; ++q)
        if (pos[preds[q]] >= w) bad = true;    // a producer does not run before v
      VT f = sf;
      for (int e = e0; e < e1; ++e) {
        const DynMember m = dyn[e];
        bool last = true;
        for (int i = 0; i < m.cnt; ++i) last &= pos[m.others[i]] < w;
        if (last) f += (VT)m.size;
      }
      const int p = PWT::pos(w);
      if (p < n) XF[p] = XFPair<VT>{(VT)(a - f), f};
    };
    if (J > 0) {
#pragma unroll
      for (int j = 0; j < J; ++j) {
        const int v = tid + j * T;
        if (v < n) {
          const int q0 = (int)(pr[j] >> kCntBits), e0 = (int)(dr[j] >> kCntBits);
          node(v, ra[j], rf[j], q0, q0 + (int)(pr[j] & kCntMask), e0,
               e0 + (int)(dr[j] & kCntMask));
        }
      }
    } else {
      for (int v = tid; v < n; v += T)
        node(v, (VT)G.alloc[v], (VT)G.sfree[v], G.pred_off[v], G.pred_off[v + 1], G.dyn_off[v],
             G.dyn_off[v + 1]);
    }
    if (G.nbig > 0) {  // order-dependent edges with many candidate consumers
      __syncthreads();
      for (int m = tid; m < G.nbig; m += T) {
        PW h = 0;
        for (int s = G.big_off[m]; s < G.big_off[m + 1]; ++s) h = max(h, pos[G.big_sinks[s]]);
        const int p = PWT::pos(h);
        if (p < n) {
          const VT sz = (VT)G.big_size[m];
          atomicAdd(&XF[p].f, sz);
          atomicAdd(&XF[p].x, (VT)0 - sz);
        }
      }
    }
    if (__syncthreads_or(bad)) {
      if (tid == 0) {
        peak_out[c] = 0;
        step_out[c] = 0;
        valid_out[c] = 0;
      }
      continue;
    }

    // ---- phase 3: order space, two-pass warp scan -------------------------------
    const int chunks = (n + kWarp - 1) / kWarp;
    const int per_warp = (chunks + nwarps - 1) / nwarps;
    const int w_begin = warp * per_warp * kWarp;
    const int w_end = min(n, w_begin + per_warp * kWarp);
    VT part = 0;
    for (int p = w_begin + lane; p < w_end; p += kWarp) part += XF[p].x;
    part = warp_sum(part);
    if (lane == 0) bs.wsum[warp] = part;
    __syncthreads();
    VT carry = lane < warp ? bs.wsum[lane] : (VT)0;
    carry = warp_sum(carry);
    VT best = 0;
    int best_i = INT_MAX;
    for (int base = w_begin; base < w_end; base += kWarp) {
      const int p = base + lane;
      const XFPair<VT> xf = p < w_end ? XF[p] : XFPair<VT>{0, 0};
      const VT incl = warp_incl_scan(xf.x, lane) + carry;
      const VT rs = incl + xf.f;
      if (p < w_end) {
        if (bytes_out) bytes_out[c * n + p] = (uint64_t)rs * G.scale;
        if (rs > best || best_i == INT_MAX) {
          best = rs;
          best_i = p;
        }
      }
      carry = __shfl_sync(0xffffffffu, incl, kWarp - 1);
    }
    warp_argmax(best, best_i);
    if (lane == 0) {
      bs.wbest[warp] = best;
      bs.widx[warp] = best_i;
    }
    __syncthreads();
    if (warp == 0) {
      best = lane < nwarps ? bs.wbest[lane] : (VT)0;
      best_i = lane < nwarps ? bs.widx[lane] : INT_MAX;
      warp_argmax(best, best_i);
      if (lane == 0) {
        const bool empty = n == 0;
        const uint64_t pk = empty ? 0 : (uint64_t)best * G.scale;
        peak_out[c] = pk;
        step_out[c] = empty ? 0 : best_i + 1;
        valid_out[c] = 1;
        if (best_key) {
          const uint64_t gi = (uint64_t)(c + index_base);
          const unsigned long long key =
              (pk < (1ull << 43) && gi < (1ull << 20)) ? ((pk << 20) | gi) : ~0ull - 1;
          atomicMin(best_key, key);
        }
      }
    }
    // bs.wsum/wbest are rewritten only after two more barriers of the next
    // candidate; XF after the next phase-1 barrier.
  }
}

template <typename VT>
size_t smem_bytes(const mp_graph* g) {
  return (((size_t)g->n_preds * 4 + 15) & ~size_t(15)) +
         (((size_t)g->n_dyn * sizeof(DynMember) + 15) & ~size_t(15)) +
         (((size_t)g->n * 4 + 15) & ~size_t(15)) + (size_t)g->n * 2 * sizeof(VT) + 64;
}

ScoreTables tables(const mp_graph* g) {
  ScoreTables G;
  G.n = g->n;
  G.npreds = (int32_t)g->n_preds;
  G.ndyn = g->n_dyn;
  G.nbig = g->n_big;
  G.scale = g->scale;
  G.pred_off = g->d_pred_off;
  G.preds = g->d_preds;
  G.alloc = g->d_node_alloc;
  G.sfree = g->d_node_sfree;
  G.dyn_off = g->d_dyn_off;
  G.dyn = reinterpret_cast<const DynMember*>(g->d_dyn);
  G.big_off = g->d_big_off;
  G.big_sinks = g->d_big_sinks;
  G.big_size = g->d_big_size;
  return G;
}

template <typename VT, typename PW, int J, bool kSmem>
mp_status run(const mp_graph* g, const int32_t* d_orders, int64_t C, uint64_t* d_peak,
              int32_t* d_step, uint8_t* d_valid, uint64_t* d_bytes, uint64_t* d_key,
              int64_t index_base, cudaStream_t st) {
  auto kern = score_kernel<VT, PW, J, kSmem>;
  const int T = g->score_threads;
  size_t smem = 0;
  char* gs = nullptr;
  size_t gstride = 0;
  int64_t grid;
  if (kSmem) {
    smem = smem_bytes<VT>(g);
    MP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    MP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, T, smem));
    grid = (int64_t)g->ctx->num_sms * (per_sm > 0 ? per_sm : 1);
  } else {
    grid = (int64_t)g->ctx->num_sms * 2;
    gstride = (((size_t)g->n * sizeof(PW) + 255) & ~size_t(255)) +
              (((size_t)g->n * 2 * sizeof(VT) + 255) & ~size_t(255));
    if (grid > C) grid = C;
    MP_TRY(g->ctx->scratch[3].reserve(gstride * (size_t)(grid > 0 ? grid : 1)));
    gs = static_cast<char*>(g->ctx->scratch[3].ptr);
  }
  if (grid > C) grid = C;
  if (grid < 1) return MP_OK;
  kern<<<(unsigned)grid, T, smem, st>>>(tables(g), d_orders, C, d_peak, d_step, d_valid, d_bytes,
                                        reinterpret_cast<unsigned long long*>(d_key), index_base,
                                        gs, gstride);
  MP_CUDA(cudaGetLastError());
  return MP_OK;
}

template <typename VT>
mp_status dispatch(const mp_graph* g, const int32_t* o, int64_t C, uint64_t* pk, int32_t* stp,
                   uint8_t* vl, uint64_t* by, uint64_t* key, int64_t base, cudaStream_t st) {
  switch (g->score_j) {
    case 4: return run<VT, uint32_t, 4, true>(g, o, C, pk, stp, vl, by, key, base, st);
    case 8: return run<VT, uint32_t, 8, true>(g, o, C, pk, stp, vl, by, key, base, st);
    default:
      if (g->smem_resident)
        return run<VT, uint32_t, 0, true>(g, o, C, pk, stp, vl, by, key, base, st);
      return run<VT, unsigned long long, 0, false>(g, o, C, pk, stp, vl, by, key, base, st);
  }
}

}  // namespace

mp_status score_configure(mp_graph* g, int max_pred_cnt, int max_dyn_cnt) {
  // Register slice J (nodes per thread) with T = ceil(n / J) <= 512 threads
  // when per-node counts fit the packed ranges; shared-memory buffers when
  // they fit; otherwise node tables from global and/or global scratch.
  const int n = g->n;
  const size_t need = g->narrow ? smem_bytes<uint32_t>(g) : smem_bytes<unsigned long long>(g);
  const bool smem = n < 65536 && need + 2048 <= g->ctx->max_smem_optin;
  const bool packable = max_pred_cnt <= kCntMask && max_dyn_cnt <= kCntMask &&
                        g->n_preds < (1 << 20) && g->n_dyn < (1 << 20);
  int J = 0, T = 1024;
  if (smem && packable) {
    for (int j : {4, 8}) {
      const int t = ((n + j - 1) / j + 31) / 32 * 32;
      if (t <= 512) {
        J = j;
        T = t < 32 ? 32 : t;
        break;
      }
    }
  }
  if (J == 0 && smem) T = n <= 8192 ? 512 : 1024;
  g->score_j = J;
  g->score_threads = T;
  g->smem_resident = smem;
  g->score_smem_bytes = smem ? need : 0;
  return MP_OK;
}

mp_status launch_score(const mp_graph* g, const int32_t* d_orders, int64_t C, uint64_t* d_peak,
                       int32_t* d_step, uint8_t* d_valid, uint64_t* d_bytes, uint64_t* d_key,
                       int64_t index_base, cudaStream_t st) {
  if (C <= 0) return MP_OK;
  if (g->narrow)
    return dispatch<uint32_t>(g, d_orders, C, d_peak, d_step, d_valid, d_bytes, d_key,
                              index_base, st);
  return dispatch<unsigned long long>(g, d_orders, C, d_peak, d_step, d_valid, d_bytes, d_key,
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
