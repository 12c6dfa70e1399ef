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
// most frees static (single consumer, or every other consumer reaches it) and
// drops redundant validity edges. Per candidate the device then does:
//   phase 1  (order space)  pos[order[k]] = stamp|k                      n scatters
//   phase 2a (node space)   stamp check (= permutation check),          n sequential reads
//                           first reduced producer before the node,     ~n gathers
//                           XF[p(v)] = (x_v, f_v)                        n scatters
//   phase 2b                remaining reduced producer pairs (flat)      few gathers
//   phase 2c                order-dependent last consumers: max pos over
//                           the candidate sinks, 2 smem atomics          few gathers
//   phase 3  (order space)  blocked two-pass scan + first argmax        sequential
// Static per-node data (x_v, f_v, first producer) lives in registers of the
// owning thread (node v = tid + j*T, j < J) for the whole persistent loop;
// the next candidate's order slice is prefetched into registers while the
// current one is scored. Values are in units of gcd(sizes); 32-bit when
// total/gcd < 2^32 (every RS then fits and modular sums are exact).
#include <cuda_runtime.h>

#include <climits>
#include <cstdlib>
#include <cstdint>
#include <string>

#include "mp_internal.h"
#include "mp_parts.h"
#include "mp_prep.h"

namespace mpb {
namespace {

constexpr int kWarp = 32;
// Packed argmin keys stay non-negative as int64 so an NCCL int64 MIN works.
// The fused key is two words {key, overflow}, both reset by one byte memset
// (0x7f): word 0 takes atomicMin(peak << 20 | index) for keys that fit (peak
// < 2^42, index < 2^20), word 1 drops to 0 when any candidate's key did not
// fit, so a MIN-reduction over shards can never hide an overflow.
constexpr unsigned long long kKeyNone = 0x7f7f7f7f7f7f7f7full;
constexpr unsigned long long kKeyOverflow = 0x7f7f7f7f7f7f7f7eull;  // mp_argmin_key_d out[2]
constexpr uint64_t kKeyMaxPeak = 1ull << 42;

__device__ __forceinline__ void record_key(unsigned long long* key, uint64_t pk, uint64_t gi) {
  if (pk < kKeyMaxPeak && gi < (1ull << 20)) atomicMin(key, (unsigned long long)((pk << 20) | gi));
  else atomicMin(key + 1, 0ull);
}

struct ScoreTables {
  int32_t n;
  int32_t nextra;
  int32_t ndyn;
  int32_t ndyn_sinks;
  int32_t P;  // scan chunk per thread (odd)
  uint64_t scale;
  const uint64_t* __restrict__ node_x;
  const uint64_t* __restrict__ node_f;
  const int32_t* __restrict__ pred1;
  const int32_t* __restrict__ extra_u;
  const int32_t* __restrict__ extra_w;
  const int32_t* __restrict__ dyn_off;
  const int32_t* __restrict__ dyn_sinks;
  const uint64_t* __restrict__ dyn_size;
  const uint4* __restrict__ node_rec32;      // (x, f, pred1, pred2), 32-bit graphs
  const int2* __restrict__ node_u2;          // (pred1, pred2)
  const uint32_t* __restrict__ extra3_packed;
  int32_t nextra3;
  const int4* __restrict__ dyn_sink4;        // [ndyn] candidate sinks, -1 padded (<= 4 each)
};

// Position word: stamp in the high half, position in the low half. Within one
// candidate all written words share the stamp, so comparing whole words
// compares positions; a stale stamp marks a node the order never wrote.
template <typename PW>
struct PosWord;
template <>
struct PosWord<uint32_t> {
  static constexpr uint32_t kMaxStamp = 0xffffu;
  __device__ static uint32_t tag(uint32_t stamp) { return stamp << 16; }
  __device__ static bool fresh(uint32_t w, uint32_t tag) { return (w & 0xffff0000u) == tag; }
  __device__ static int pos(uint32_t w) { return (int)(w & 0xffffu); }
};
// int32_t words: 24-bit position, 7-bit stamp (words stay non-negative, so
// signed compares order them like the unsigned variants). n < 2^24.
template <>
struct PosWord<int32_t> {
  static constexpr uint32_t kMaxStamp = 0x7fu;
  __device__ static int32_t tag(uint32_t stamp) { return (int32_t)(stamp << 24); }
  __device__ static bool fresh(int32_t w, int32_t tag) { return (w & 0x7f000000) == tag; }
  __device__ static int pos(int32_t w) { return w & 0xffffff; }
};
template <>
struct PosWord<unsigned long long> {
  static constexpr uint32_t kMaxStamp = 0xffffffffu;
  __device__ static unsigned long long tag(uint32_t stamp) {
    return (unsigned long long)stamp << 32;
  }
  __device__ static bool fresh(unsigned long long w, unsigned long long tag) {
    return (w & 0xffffffff00000000ull) == tag;
  }
  __device__ static int pos(unsigned long long w) { return (int)(uint32_t)w; }
};

template <typename VT>
struct XFPair {
  VT x, f;
};

// Storage of the per-position (x, f) scan inputs of the node-table scorer.
template <typename VT>
struct XFWide {  // one XFPair<VT> per position
  using E = XFPair<VT>;
  static constexpr bool kShared = false;
  __device__ static void store(E* a, int i, VT x, VT f) { a[i] = E{x, f}; }
  __device__ static void pad(E* a, int i) { a[i] = E{0, 0}; }
  __device__ static void free_at(E* a, int i, VT sz) {  // freed after position i
    atomicAdd(&a[i].f, sz);
    atomicAdd(&a[i].x, (VT)0 - sz);
  }
  __device__ static void load(const E* a, int i, VT& x, VT& f) {
    const E e = a[i];
    x = e.x;
    f = e.f;
  }
};
// Graphs whose per-node values fit a byte once every order-dependent free is
// counted (mp_prep.cpp `tiny8`, e.g. C5): 2 bytes per position, x + 128 in the
// low byte, f in the high byte - a quarter of the wide footprint, so the per-CTA
// scratch of the large-graph scorer stays L2-resident. A free adds 255*sz to
// the 16-bit entry (x -= sz, f += sz): no borrow or carry leaves the entry
// because the static bounds hold for every order.
struct XFTiny8 {
  using E = uint16_t;
  static constexpr bool kShared = false;
  __device__ static void store(E* a, int i, uint32_t x, uint32_t f) {
    a[i] = (E)(((x + 128u) & 0xffu) | (f << 8));
  }
  __device__ static void pad(E* a, int i) { a[i] = 128; }
  __device__ static void free_at(E* a, int i, uint32_t sz) {
    const uintptr_t at = reinterpret_cast<uintptr_t>(a + i);
    atomicAdd(reinterpret_cast<unsigned int*>(at & ~uintptr_t(3)), (sz * 255u) << ((at & 2) * 8));
  }
  __device__ static void load(const E* a, int i, uint32_t& x, uint32_t& f) {
    const uint32_t e = a[i];
    x = (e & 0xffu) - 128u;
    f = e >> 8;
  }
};

// Smaller still (`tiny4`: x in [-8, 7], f <= 15 for any order, e.g. C5): one byte
// per position, which fits the whole order-space array of the large-graph scorer
// in SHARED memory (133 KB at C5), leaving only the position words in global
// scratch. A free adds 15*sz to the byte through a 32-bit smem atomic.
struct XFTiny4 {
  using E = uint8_t;
  static constexpr bool kShared = true;
  __device__ static void store(E* a, int i, uint32_t x, uint32_t f) {
    a[i] = (E)(((x + 8u) & 0xfu) | (f << 4));
  }
  __device__ static void pad(E* a, int i) { a[i] = 8; }
  __device__ static void free_at(E* a, int i, uint32_t sz) {
    const uintptr_t at = reinterpret_cast<uintptr_t>(a + i);
    atomicAdd(reinterpret_cast<unsigned int*>(at & ~uintptr_t(3)), (sz * 15u) << ((at & 3) * 8));
  }
  __device__ static void load(const E* a, int i, uint32_t& x, uint32_t& f) {
    const uint32_t e = a[i];
    x = (e & 0xfu) - 8u;
    f = e >> 4;
  }
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

template <typename VT, typename PW, typename XS = XFWide<VT>>
struct Layout {
  // smem (or per-CTA global) layout: extra pairs, dyn tables, pos, XF
  static size_t bytes(int n, int T, int P, int nextra, int ndyn, int ndyn_sinks, bool tables) {
    size_t b = 0;
    if (tables) {
      b += ((size_t)nextra * 8 + 15) & ~size_t(15);
      b += ((size_t)(ndyn + 1) * 4 + 15) & ~size_t(15);
      b += ((size_t)ndyn_sinks * 4 + 15) & ~size_t(15);
      b += ((size_t)ndyn * sizeof(VT) + 15) & ~size_t(15);
    }
    b += ((size_t)n * sizeof(PW) + 15) & ~size_t(15);
    if (!XS::kShared) b += ((size_t)T * P * sizeof(typename XS::E) + 15) & ~size_t(15);
    return b + 16;
  }
};

// J > 0: node data in registers (node v = tid + j*T, T <= 512), buffers and
//        flat tables in shared memory.
// J == 0: node data read from global (coalesced) per candidate; buffers in
//        shared memory (kSmem) or in a per-CTA global scratch slice.
template <typename VT, typename PW, int J, bool kSmem, typename XS = XFWide<VT>>
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
  const int P = G.P;

  // ---- buffers -------------------------------------------------------------
  const int32_t* ex_u = G.extra_u;
  const int32_t* ex_w = G.extra_w;
  const int32_t* dy_off = G.dyn_off;
  const int32_t* dy_sinks = G.dyn_sinks;
  const uint64_t* dy_size64 = G.dyn_size;
  const VT* dy_size = nullptr;
  char* p = kSmem ? smem : gscratch + (size_t)blockIdx.x * gstride;
  if (kSmem) {
    int32_t* su = reinterpret_cast<int32_t*>(p);
    int32_t* sw = su + G.nextra;
    p += ((size_t)G.nextra * 8 + 15) & ~size_t(15);
    int32_t* so = reinterpret_cast<int32_t*>(p);
    p += ((size_t)(G.ndyn + 1) * 4 + 15) & ~size_t(15);
    int32_t* ss = reinterpret_cast<int32_t*>(p);
    p += ((size_t)G.ndyn_sinks * 4 + 15) & ~size_t(15);
    VT* sz = reinterpret_cast<VT*>(p);
    p += ((size_t)G.ndyn * sizeof(VT) + 15) & ~size_t(15);
    for (int i = tid; i < G.nextra; i += T) {
      su[i] = G.extra_u[i];
      sw[i] = G.extra_w[i];
    }
    for (int i = tid; i <= G.ndyn; i += T) so[i] = G.dyn_off[i];
    for (int i = tid; i < G.ndyn_sinks; i += T) ss[i] = G.dyn_sinks[i];
    for (int i = tid; i < G.ndyn; i += T) sz[i] = (VT)G.dyn_size[i];
    ex_u = su;
    ex_w = sw;
    dy_off = so;
    dy_sinks = ss;
    dy_size = sz;
  }
  PW* pos = reinterpret_cast<PW*>(p);
  p += ((size_t)n * sizeof(PW) + 15) & ~size_t(15);
  typename XS::E* XF = reinterpret_cast<typename XS::E*>(XS::kShared ? smem : p);
  for (int i = tid; i < n; i += T) pos[i] = 0;  // stamp 0 is never used
  for (int i = n + tid; i < T * P; i += T) XS::pad(XF, i);  // scan padding

  // ---- static per-node data in registers -------------------------------------
  constexpr int JR = J > 0 ? J : 1;
  VT rx[JR], rf[JR];
  int rp[JR];  // first reduced producer, -1 if none
  int ov[JR];  // next candidate's order slice
  if (J > 0) {
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const int v = tid + j * T;
      const bool in = v < n;
      rx[j] = in ? (VT)G.node_x[v] : (VT)0;
      rf[j] = in ? (VT)G.node_f[v] : (VT)0;
      rp[j] = in ? G.pred1[v] : -1;
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
    const PW tag = PWT::tag(stamp);
    bool bad = false;

    // ---- phase 1: inverse permutation (order space) ----------------------------
    if (J > 0) {
#pragma unroll
      for (int j = 0; j < J; ++j) {
        const int k = tid + j * T;
        if (k < n) {
          const int v = ov[j];
          if ((unsigned)v >= (unsigned)n) bad = true;
          else pos[v] = tag | (PW)k;
        }
      }
      const int64_t cn = c + gridDim.x;  // prefetch: lands while this one is scored
      if (cn < C) {
        const int32_t* ord = orders + cn * n;
#pragma unroll
        for (int j = 0; j < J; ++j) {
          const int k = tid + j * T;
          ov[j] = k < n ? __ldg(ord + k) : 0;
        }
      }
    } else {
      // batches of kB: all loads of a batch before its stores (the compiler cannot
      // reorder loads across stores to possibly aliasing buffers)
      constexpr int kB = kSmem ? 8 : 16;  // more loads in flight from HBM (scratch variant)
      const int32_t* ord = orders + c * n;
      for (int k0 = tid; k0 < n; k0 += T * kB) {
        int vv[kB];
#pragma unroll
        for (int u = 0; u < kB; ++u) {
          const int k = k0 + u * T;
          // global-scratch variant: orders are read once, evict-first (keep the scratch in L2)
          vv[u] = k < n ? (kSmem ? __ldg(ord + k) : __ldcs(ord + k)) : 0;
        }
#pragma unroll
        for (int u = 0; u < kB; ++u) {
          const int k = k0 + u * T;
          if (k < n) {
            if ((unsigned)vv[u] >= (unsigned)n) bad = true;
            else pos[vv[u]] = tag | (PW)k;
          }
        }
      }
    }
    __syncthreads();

    // ---- phase 2a: node space ------------------------------------------------------
    auto node = [&](int v, VT x, VT f, int u) {
      const PW w = pos[v];
      bad |= !PWT::fresh(w, tag);           // never written: not a permutation
      if (u >= 0) bad |= pos[u] >= w;       // producer not strictly before v
      const int u2 = __ldg(G.node_u2 + v).y;
      if (u2 >= 0) bad |= pos[u2] >= w;
      const int q = PWT::pos(w);
      if (q < n) XS::store(XF, q, x, f);
    };
    if (J > 0) {
#pragma unroll
      for (int j = 0; j < J; ++j) {
        const int v = tid + j * T;
        if (v < n) node(v, rx[j], rf[j], rp[j]);
      }
    } else {
      constexpr int kB = 8;
      for (int v0 = tid; v0 < n; v0 += T * kB) {
        // both first producers in node space: pos[v] is this node's own (coalesced)
        // word, so each needs one random gather (the flat list below needs two)
        PW w[kB], pu[kB], pu2[kB];
        VT xx[kB], ff[kB];
#pragma unroll
        for (int u = 0; u < kB; ++u) {
          const int v = v0 + u * T;
          const bool in = v < n;
          const int2 pr = in ? __ldg(G.node_u2 + v) : make_int2(-1, -1);
          w[u] = in ? pos[v] : tag;
          xx[u] = in ? (VT)__ldg(G.node_x + v) : (VT)0;
          ff[u] = in ? (VT)__ldg(G.node_f + v) : (VT)0;
          pu[u] = pr.x >= 0 ? pos[pr.x] : (PW)0;
          pu2[u] = pr.y >= 0 ? pos[pr.y] : (PW)0;
        }
#pragma unroll
        for (int u = 0; u < kB; ++u) {
          if (v0 + u * T < n) {
            bad |= !PWT::fresh(w[u], tag) || pu[u] >= w[u] || pu2[u] >= w[u];
            const int q = PWT::pos(w[u]);
            if (q < n) XS::store(XF, q, xx[u], ff[u]);
          }
        }
      }
    }
    // ---- phase 2b: 3rd+ reduced producer pairs (flat) --------------------------------
    {
      constexpr int kB = 8;
      for (int i0 = tid; i0 < G.nextra; i0 += T * kB) {
        PW a[kB], b[kB];
#pragma unroll
        for (int u = 0; u < kB; ++u) {
          const int i = i0 + u * T;
          const bool in = i < G.nextra;
          a[u] = in ? pos[ex_u[i]] : (PW)0;
          b[u] = in ? pos[ex_w[i]] : (PW)1;
        }
#pragma unroll
        for (int u = 0; u < kB; ++u) bad |= a[u] >= b[u];
      }
    }
    // ---- phase 2c: order-dependent last consumers --------------------------------------
    if (G.ndyn > 0) {
      __syncthreads();  // XF written by phase 2a
      constexpr int kB = 4;
      for (int d0 = tid; d0 < G.ndyn; d0 += T * kB) {
        PW h[kB];
        if (G.dyn_sink4 != nullptr) {  // <= 4 candidate sinks each: one 16-byte load per edge
          int4 sk[kB];
#pragma unroll
          for (int u = 0; u < kB; ++u) {
            const int d = d0 + u * T;
            sk[u] = d < G.ndyn ? __ldg(G.dyn_sink4 + d) : make_int4(-1, -1, -1, -1);
          }
#pragma unroll
          for (int u = 0; u < kB; ++u) {  // every gather of the batch before any atomic
            const PW a = sk[u].x >= 0 ? pos[sk[u].x] : (PW)0;
            const PW b = sk[u].y >= 0 ? pos[sk[u].y] : (PW)0;
            const PW c2 = sk[u].z >= 0 ? pos[sk[u].z] : (PW)0;
            const PW d2 = sk[u].w >= 0 ? pos[sk[u].w] : (PW)0;
            h[u] = max(max(a, b), max(c2, d2));
          }
        } else {
#pragma unroll
          for (int u = 0; u < kB; ++u) {  // gathers of kB edges before any atomic
            const int d = d0 + u * T;
            h[u] = 0;
            if (d < G.ndyn)
              for (int s = dy_off[d]; s < dy_off[d + 1]; ++s) h[u] = max(h[u], pos[dy_sinks[s]]);
          }
        }
#pragma unroll
        for (int u = 0; u < kB; ++u) {
          const int d = d0 + u * T;
          const int q = PWT::pos(h[u]);
          if (d < G.ndyn && q < n) {
            const VT sz = kSmem ? dy_size[d] : (VT)dy_size64[d];
            XS::free_at(XF, q, sz);
          }
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

    VT best = 0;
    int best_i = INT_MAX;
    if constexpr (kSmem) {
      // ---- phase 3: blocked two-pass scan (chunk [tid*P, tid*P+P), P odd) ----------
      const typename XS::E* mine = XF + tid * P;
      VT total = 0;
#pragma unroll 8
      for (int i = 0; i < P; ++i) {
        VT x, f;
        XS::load(mine, i, x, f);
        total += x;
      }
      const VT incl = warp_incl_scan(total, lane);
      if (lane == kWarp - 1) bs.wsum[warp] = incl;
      __syncthreads();
      VT run = warp_sum(lane < warp ? bs.wsum[lane] : (VT)0) + incl - total;
      const int p0 = tid * P;
      const int lim = min(P, n - p0);
      for (int i = 0; i < lim; ++i) {
        VT xx, ff;
        XS::load(mine, i, xx, ff);
        run += xx;
        const VT rs = run + ff;
        if (bytes_out) bytes_out[c * n + p0 + i] = (uint64_t)rs * G.scale;
        if (rs > best || best_i == INT_MAX) {
          best = rs;
          best_i = p0 + i;
        }
      }
    } else {
      // ---- phase 3, scan inputs in global scratch: warp rows -------------------------
      // Warp w owns positions [w*32P, (w+1)*32P) and reads them 128 at a time, four
      // consecutive per lane: each load instruction touches two lines instead of 32
      // (the blocked layout's per-thread chunks put every lane on its own line).
      const int wbeg = warp * kWarp * P, wend = wbeg + kWarp * P;
      VT tot = 0;
      for (int r = wbeg + 4 * lane; r < wend; r += 4 * kWarp)
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (r + q < wend) {
            VT xx, ff;
            XS::load(XF, r + q, xx, ff);
            tot += xx;
          }
      tot = warp_sum(tot);
      if (lane == 0) bs.wsum[warp] = tot;
      __syncthreads();
      VT carry = warp_sum(lane < warp ? bs.wsum[lane] : (VT)0);  // exclusive over warps
      for (int r0 = wbeg; r0 < wend; r0 += 4 * kWarp) {
        const int r = r0 + 4 * lane;
        VT xs[4], fs[4], t = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          xs[q] = 0;
          fs[q] = 0;
          if (r + q < wend) XS::load(XF, r + q, xs[q], fs[q]);
          t += xs[q];
        }
        const VT incl = warp_incl_scan(t, lane);
        VT run = carry + incl - t;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          run += xs[q];
          const VT rs = run + fs[q];
          const int k = r + q;
          if (k < n && k < wend) {
            if (bytes_out) bytes_out[c * n + k] = (uint64_t)rs * G.scale;
            if (best_i == INT_MAX || rs > best) {
              best = rs;
              best_i = k;
            }
          }
        }
        carry += __shfl_sync(0xffffffffu, incl, kWarp - 1);
      }
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
          record_key(best_key, pk, gi);
        }
      }
    }
    // bs.wsum is rewritten after >= 2 more barriers; XF after the next phase-1 barrier.
  }
}

#include "k_score_reg.cuh"
#include "k_score_warp.cuh"
#include "k_score_parts.cuh"

ScoreTables tables(const mp_graph* g) {
  ScoreTables G;
  G.n = g->n;
  G.nextra = g->n_extra;
  G.ndyn = g->n_dyn;
  G.ndyn_sinks = g->n_dyn_sinks;
  G.P = g->score_p;
  G.scale = g->scale;
  G.node_x = g->d_node_x;
  G.node_f = g->d_node_f;
  G.pred1 = g->d_pred1;
  G.extra_u = g->d_extra_u;
  G.extra_w = g->d_extra_w;
  G.dyn_off = g->d_dyn_off;
  G.dyn_sinks = g->d_dyn_sinks;
  G.dyn_size = g->d_dyn_size;
  G.node_rec32 = reinterpret_cast<const uint4*>(g->d_node_rec32);
  G.node_u2 = reinterpret_cast<const int2*>(g->d_node_u2);
  G.extra3_packed = g->d_extra3_packed;
  G.nextra3 = g->n_extra3;
  G.dyn_sink4 = reinterpret_cast<const int4*>(g->d_dyn_sink4);
  return G;
}

// An L2 persisting access-policy window over [base, base + bytes) for one launch
// (the per-CTA scratch of the large-graph scorers); false when unsupported.
bool l2_persist_window(const mp_ctx* ctx, void* base, size_t bytes, cudaLaunchAttribute* at) {
  int max_win = 0, persist_max = 0;
  cudaDeviceGetAttribute(&max_win, cudaDevAttrMaxAccessPolicyWindowSize, ctx->device);
  cudaDeviceGetAttribute(&persist_max, cudaDevAttrMaxPersistingL2CacheSize, ctx->device);
  if (max_win <= 0 || persist_max <= 0 || bytes == 0) return false;
  static bool limit_set = false;  // process-wide device limit, set once
  if (!limit_set) {
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)persist_max);
    limit_set = true;
  }
  const size_t win = bytes < (size_t)max_win ? bytes : (size_t)max_win;
  at->id = cudaLaunchAttributeAccessPolicyWindow;
  at->val.accessPolicyWindow.base_ptr = base;
  at->val.accessPolicyWindow.num_bytes = win;
  const double r = (double)persist_max / (double)win;
  at->val.accessPolicyWindow.hitRatio = (float)(r < 1.0 ? r : 1.0);
  at->val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
  at->val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  return true;
}

template <typename VT, typename PW, int J, bool kSmem, typename XS = XFWide<VT>>
mp_status run(const mp_graph* g, const int32_t* d_orders, int64_t C, uint64_t* d_peak,
              int32_t* d_step, uint8_t* d_valid, uint64_t* d_bytes, uint64_t* d_key,
              int64_t index_base, cudaStream_t st) {
  auto kern = score_kernel<VT, PW, J, kSmem, XS>;
  const int T = g->score_threads;
  const size_t per = Layout<VT, PW, XS>::bytes(g->n, T, g->score_p, g->n_extra, g->n_dyn,
                                           g->n_dyn_sinks, kSmem);
  size_t smem = 0;
  char* gs = nullptr;
  size_t gstride = 0;
  int64_t grid;
  if (kSmem) {
    smem = per;
    MP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    MP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, T, smem));
    grid = (int64_t)g->ctx->num_sms * (per_sm > 0 ? per_sm : 1);
  } else {
    // per-CTA scratch slices are the working set of the random scatters: a
    // grid of one CTA per SM keeps more of them L2-resident (MP_SCORE_GRID
    // overrides, for tuning)
    grid = (int64_t)g->ctx->num_sms;
    if (XS::kShared) {  // the order-space scan inputs live in shared memory
      smem = ((size_t)T * g->score_p * sizeof(typename XS::E) + 15) & ~size_t(15);
      MP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    }
    if (const char* e = std::getenv("MP_SCORE_GRID")) {
      const long v = std::atol(e);
      if (v > 0) grid = v;
    }
    if (grid > C) grid = C;
    gstride = (per + 255) & ~size_t(255);
    MP_TRY(g->ctx->scratch[3].reserve(gstride * (size_t)(grid > 0 ? grid : 1)));
    gs = static_cast<char*>(g->ctx->scratch[3].ptr);
  }
  if (grid > C) grid = C;
  if (grid < 1) return MP_OK;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(T);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  cfg.attrs = at;
  cfg.numAttrs = 0;
  // An L2 persisting window over this scratch measured 2.3x SLOWER at C5 (only 79 of its
  // 237 MB can persist; the rest turns evict-first): opt-in via MP_L2_WINDOW for tuning.
  if (!kSmem && std::getenv("MP_L2_WINDOW"))
    cfg.numAttrs = l2_persist_window(g->ctx, gs, gstride * (size_t)grid, &at[0]) ? 1 : 0;
  MP_CUDA(cudaLaunchKernelEx(&cfg, kern, tables(g), d_orders, C, d_peak, d_step, d_valid, d_bytes,
                             reinterpret_cast<unsigned long long*>(d_key), index_base, gs,
                             gstride));
  return MP_OK;
}

template <typename VT, int J, int KC, typename OT, typename AT = VT>
mp_status run_reg_t(const mp_graph* g, const OT* d_orders, int64_t C, uint64_t* d_peak,
                    int32_t* d_step, uint8_t* d_valid, uint64_t* d_bytes, uint64_t* d_key,
                    int64_t index_base, cudaStream_t st) {
  auto kern = score_reg_kernel<VT, J, KC, OT, AT>;
  const int T = g->score_threads;
  const size_t smem = reg_smem_bytes<VT>(g->n, T, g->score_p, J, KC);

  MP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  MP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, T, smem));
  int64_t grid = (int64_t)g->ctx->num_sms * (per_sm > 0 ? per_sm : 1);
  const int64_t groups = (C + KC - 1) / KC;
  if (grid > groups) grid = groups;
  kern<<<(unsigned)grid, T, smem, st>>>(tables(g), d_orders, C, d_peak, d_step, d_valid, d_bytes,
                                        reinterpret_cast<unsigned long long*>(d_key), index_base);
  MP_CUDA(cudaGetLastError());
  return MP_OK;
}

template <typename VT, int J, int KC, typename AT = VT>
mp_status run_reg(const mp_graph* g, const int32_t* d_orders, int64_t C, uint64_t* d_peak,
                  int32_t* d_step, uint8_t* d_valid, uint64_t* d_bytes, uint64_t* d_key,
                  int64_t index_base, cudaStream_t st, bool o16) {
  if (o16 && KC == 1)  // 16-bit orders (host-packed): same kernel, half the order bytes
    return run_reg_t<VT, J, KC, uint16_t, AT>(g, reinterpret_cast<const uint16_t*>(d_orders), C,
                                              d_peak, d_step, d_valid, d_bytes, d_key,
                                              index_base, st);
  if (o16) return MP_E_INVALID_ARG;
  return run_reg_t<VT, J, KC, int32_t, AT>(g, d_orders, C, d_peak, d_step, d_valid, d_bytes,
                                           d_key, index_base, st);
}

template <typename VT>
mp_status run_warp(const mp_graph* g, const int32_t* d_orders, int64_t C, uint64_t* d_peak,
                   int32_t* d_step, uint8_t* d_valid, uint64_t* d_bytes, uint64_t* d_key,
                   int64_t index_base, cudaStream_t st) {
  auto kern = score_warp_kernel<VT>;
  const int W = g->score_warps;
  const size_t smem = warp_smem_bytes<VT>(g->n, g->score_wp, W);
  MP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  MP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * W, smem));
  int64_t grid = (int64_t)g->ctx->num_sms * (per_sm > 0 ? per_sm : 1);
  const int64_t need = (C + W - 1) / W;
  if (grid > need) grid = need;
  ScoreTables G = tables(g);
  G.P = g->score_wp;
  kern<<<(unsigned)grid, 32 * W, smem, st>>>(G, d_orders, C, d_peak, d_step, d_valid, d_bytes,
                                             reinterpret_cast<unsigned long long*>(d_key),
                                             index_base);
  MP_CUDA(cudaGetLastError());
  return MP_OK;
}

mp_status run_parts(const mp_graph* g, const int32_t* d_orders, int64_t C, uint64_t* d_peak,
                    int32_t* d_step, uint8_t* d_valid, uint64_t* d_key, int64_t index_base,
                    cudaStream_t st, bool o24) {
  const auto& Q = g->parts;
  const bool vec = g->n % 4 == 0;
  if (o24 && !vec) return MP_E_INVALID_ARG;
  // deferred positions (one stream of the order) unless MP_PARTS_NO_DEFER
  const bool defer = vec && Q.P >= 2 && Q.P <= 7 && g->n <= 512 * kPartsMaxBlocks &&
                     !std::getenv("MP_PARTS_NO_DEFER");
  auto kern = o24 ? (defer ? score_parts_kernel<true, true, true> : score_parts_kernel<true, true>)
              : vec ? (defer ? score_parts_kernel<true, false, true> : score_parts_kernel<true>)
                    : score_parts_kernel<false>;
  MP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Q.smem));
  int64_t grid = g->ctx->num_sms;
  if (const char* e = std::getenv("MP_SCORE_GRID")) {
    const long v = std::atol(e);
    if (v > 0) grid = v;
  }
  if (grid > C) grid = C;
  if (grid < 1) return MP_OK;
  // per CTA: XF (1 byte per position) then, when deferring, 512 words per 512-position block
  const size_t xf_bytes = ((size_t)32 * Q.seg + 255) & ~size_t(255);
  const size_t gstride = xf_bytes + (defer ? (((size_t)g->n + 511) / 512) * 512 * 4 : 0);
  MP_TRY(g->ctx->scratch[3].reserve(gstride * (size_t)grid));
  PartArgs A;
  A.P = Q.P;
  A.nchunks = Q.nchunks;
  A.nb_max = Q.nb_max;
  A.nslots = Q.nslots;
  A.seg = Q.seg;
  A.n_slot_init = Q.n_slot_init;
  A.n_xfree = Q.n_xfree;
  A.desc = static_cast<const PartDesc*>(Q.d_desc);
  A.ctab = Q.d_ctab;
  A.xtab = Q.d_xtab;
  A.p1 = Q.d_p1;
  A.intra = Q.d_intra;
  A.xput = Q.d_xput;
  A.xchk = Q.d_xchk;
  A.xmax = Q.d_xmax;
  A.dyn4 = reinterpret_cast<const uint4*>(Q.d_dyn4);
  A.xfree = reinterpret_cast<const uint2*>(Q.d_xfree);
  A.slot_init = Q.d_slot_init;
  kern<<<(unsigned)grid, kPartsThreads, Q.smem, st>>>(
      A, g->n, d_orders, C, d_peak, d_step, d_valid,
      reinterpret_cast<unsigned long long*>(d_key), index_base, g->scale,
      static_cast<uint8_t*>(g->ctx->scratch[3].ptr), gstride, xf_bytes);
  MP_CUDA(cudaGetLastError());
  return MP_OK;
}

template <typename VT>
mp_status dispatch(const mp_graph* g, const int32_t* o, int64_t C, uint64_t* pk, int32_t* stp,
                   uint8_t* vl, uint64_t* by, uint64_t* key, int64_t base, cudaStream_t st,
                   int ofmt) {
  const bool o16 = ofmt == kOrdU16;
  if (o16 && !score_takes_u16(g)) return MP_E_INVALID_ARG;
  if (ofmt == kOrdU24 && !score_takes_u24(g)) return MP_E_INVALID_ARG;
  if (g->use_parts && by == nullptr)
    return run_parts(g, o, C, pk, stp, vl, key, base, st, ofmt == kOrdU24);
  if (g->score_warps > 0) return run_warp<VT>(g, o, C, pk, stp, vl, by, key, base, st);
  switch (g->score_j) {
    case 4:
      if (g->score_kc == 2) return run_reg<VT, 4, 2>(g, o, C, pk, stp, vl, by, key, base, st, o16);
      return run_reg<VT, 4, 1>(g, o, C, pk, stp, vl, by, key, base, st, o16);
    case 8:
      if (g->score_kc == 2) return run_reg<VT, 8, 2>(g, o, C, pk, stp, vl, by, key, base, st, o16);
      return run_reg<VT, 8, 1>(g, o, C, pk, stp, vl, by, key, base, st, o16);
    case 16:
      if (g->score_kc == 2) return run_reg<VT, 16, 2>(g, o, C, pk, stp, vl, by, key, base, st, o16);
      return run_reg<VT, 16, 1>(g, o, C, pk, stp, vl, by, key, base, st, o16);
    default:
      if (g->smem_resident)
        return run<VT, uint32_t, 0, true>(g, o, C, pk, stp, vl, by, key, base, st);
      if (g->n < (1 << 24) && !std::getenv("MP_SCORE_POS64")) {
        if constexpr (sizeof(VT) == 4) {
          const bool wide = std::getenv("MP_SCORE_WIDE_XF") != nullptr;
          const bool no4 = std::getenv("MP_SCORE_NO_TINY4") != nullptr;
          if (g->tiny4 && !wide && !no4 &&
              (size_t)g->score_threads * g->score_p + 64 <= g->ctx->max_smem_optin)
            return run<VT, int32_t, 0, false, XFTiny4>(g, o, C, pk, stp, vl, by, key, base, st);
          if (g->tiny8 && !wide)
            return run<VT, int32_t, 0, false, XFTiny8>(g, o, C, pk, stp, vl, by, key, base, st);
        }
        return run<VT, int32_t, 0, false>(g, o, C, pk, stp, vl, by, key, base, st);
      }
      return run<VT, unsigned long long, 0, false>(g, o, C, pk, stp, vl, by, key, base, st);
  }
}

}  // namespace

mp_status score_configure(mp_graph* g) {
  // Register slice J (nodes per thread): the smallest of {4, 8, 16} giving
  // T = ceil(n / J) <= 256 threads (512 for J = 16); shared-memory buffers
  // when they fit; otherwise node tables from global and/or global scratch.
  const int n = g->n;
  int J = 0, T = 1024;
  // MP_SCORE_J=4|8|16 forces the slot count (tuning experiments only).
  const char* force = std::getenv("MP_SCORE_J");
  const int fj = force ? std::atoi(force) : 0;
  for (int j : {4, 8, 16}) {
    if (fj && j != fj) continue;
    const int t = ((n + j - 1) / j + 31) / 32 * 32;
    if (t <= (j == 4 ? 256 : j == 8 ? MP_J8_MAXT : 512)) {  // RegBounds<J>::kMaxT
      J = j;
      T = t < 32 ? 32 : t;
      break;
    }
  }
  auto chunk = [&](int t) {
    int p = (n + t - 1) / t;
    if (p < 1) p = 1;
    return p | 1;  // odd stride: conflict-free blocked LDS
  };
  auto need = [&](int t) {
    return g->narrow ? Layout<uint32_t, uint32_t>::bytes(n, t, chunk(t), g->n_extra, g->n_dyn,
                                                          g->n_dyn_sinks, true)
                     : Layout<unsigned long long, uint32_t>::bytes(
                           n, t, chunk(t), g->n_extra, g->n_dyn, g->n_dyn_sinks, true);
  };
  // candidates scored together per CTA iteration (MP_SCORE_KC=1|2 forces it)
  const char* fkc = std::getenv("MP_SCORE_KC");
  int KC = fkc ? std::atoi(fkc) : 1;
  if (KC != 1 && KC != 2) KC = 1;
  auto reg_need = [&](int kc) {
    return g->narrow ? reg_smem_bytes<uint32_t>(n, T, chunk(T), J, kc)
                     : reg_smem_bytes<unsigned long long>(n, T, chunk(T), J, kc);
  };
  if (J > 0 && KC == 2 && reg_need(2) + 2048 > g->ctx->max_smem_optin) KC = 1;
  if (J == 8 && KC == 2 && T > 320) KC = 1;  // RegBounds<8, 2>::kMaxT
  const size_t need_reg = J == 0 ? 0 : reg_need(KC);


  if (J > 0 && need_reg + 2048 > g->ctx->max_smem_optin) J = 0;
  if (J > 0) T = ((n + J - 1) / J + 31) / 32 * 32, T = T < 32 ? 32 : T;
  bool smem = n < 65536 && need(J > 0 ? T : 1024) + 2048 <= g->ctx->max_smem_optin;
  if (J > 0) smem = true;
  if (J == 0) T = 1024;
  if (J == 0 && !smem) smem = false;
  // Warp-per-candidate variant for small graphs, opt-in (MP_SCORE_MODE=warp): on
  // the C2/C3 graphs it measured slower than the register-slot CTA variant.
  // as many warps per CTA as the per-warp buffers allow, up to 16.
  g->score_warps = 0;
  const char* mode = std::getenv("MP_SCORE_MODE");
  const bool want_warp = mode && std::string(mode) == "warp" && n <= kWarpMaxNodes;
  if (want_warp && n > 0 && n < 65535) {
    const int wp = ((n + 31) / 32) | 1;
    g->score_wp = wp;
    for (int w = 16; w >= 1; --w) {
      const size_t b = g->narrow ? warp_smem_bytes<uint32_t>(n, wp, w)
                                 : warp_smem_bytes<unsigned long long>(n, wp, w);
      if (b + 1024 <= g->ctx->max_smem_optin) {
        g->score_warps = w;
        break;
      }
    }
  }
  // the node-partitioned scorer wherever per-candidate state would otherwise go
  // through global scratch (MP_SCORE_PARTS: wherever a plan exists, for tests)
  g->use_parts = g->parts.P > 0 && ((J == 0 && !smem) || std::getenv("MP_SCORE_PARTS"));
  g->score_j = J;
  g->score_kc = KC;
  g->score_threads = T;
  g->score_p = chunk(T);
  g->smem_resident = smem;
  g->score_smem_bytes = smem ? need(T) : 0;
  return MP_OK;
}

bool score_takes_u24(const mp_graph* g) {
  return g->use_parts && g->n > 0 && g->n % 4 == 0 && g->n < 0xffffff;
}

bool score_takes_u16(const mp_graph* g) {
  return g->n > 0 && g->n < 65535 && g->score_j > 0 && g->score_warps == 0 && g->score_kc == 1 &&
         !g->use_parts;
}

mp_status launch_score(const mp_graph* g, const int32_t* d_orders, int64_t C, uint64_t* d_peak,
                       int32_t* d_step, uint8_t* d_valid, uint64_t* d_bytes, uint64_t* d_key,
                       int64_t index_base, cudaStream_t st, int ofmt) {
  if (C <= 0) return MP_OK;
  // mid32 graphs (64-bit totals, 32-bit per-node values): the register-slot kernel with
  // 32-bit scan inputs and 64-bit sums; per-step bytes and the other variants take the
  // 64-bit path
  if (g->mid32 && d_bytes == nullptr && g->score_warps == 0 && !g->use_parts &&
      ofmt != kOrdU24) {
    const bool o16 = ofmt == kOrdU16;
    if (o16 && !score_takes_u16(g)) return MP_E_INVALID_ARG;
    using U = unsigned long long;
    switch (g->score_j) {
      case 4:
        if (g->score_kc == 2) return run_reg<uint32_t, 4, 2, U>(g, d_orders, C, d_peak, d_step, d_valid, d_bytes, d_key, index_base, st, o16);
        return run_reg<uint32_t, 4, 1, U>(g, d_orders, C, d_peak, d_step, d_valid, d_bytes, d_key, index_base, st, o16);
      case 8:
        if (g->score_kc == 2) return run_reg<uint32_t, 8, 2, U>(g, d_orders, C, d_peak, d_step, d_valid, d_bytes, d_key, index_base, st, o16);
        return run_reg<uint32_t, 8, 1, U>(g, d_orders, C, d_peak, d_step, d_valid, d_bytes, d_key, index_base, st, o16);
      case 16:
        if (g->score_kc == 2) return run_reg<uint32_t, 16, 2, U>(g, d_orders, C, d_peak, d_step, d_valid, d_bytes, d_key, index_base, st, o16);
        return run_reg<uint32_t, 16, 1, U>(g, d_orders, C, d_peak, d_step, d_valid, d_bytes, d_key, index_base, st, o16);
      default:
        break;
    }
  }
  if (g->narrow)
    return dispatch<uint32_t>(g, d_orders, C, d_peak, d_step, d_valid, d_bytes, d_key,
                              index_base, st, ofmt);
  return dispatch<unsigned long long>(g, d_orders, C, d_peak, d_step, d_valid, d_bytes, d_key,
                                      index_base, st, ofmt);
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
      const bool fits = gi >= 0 && gi < (1 << 20) && bp < kKeyMaxPeak;
      out[2] = gi < 0 ? kKeyNone : fits ? ((bp << 20) | (uint64_t)gi) : kKeyOverflow;
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
