// K5 - placement heuristics over realized lifetimes, batched over problems:
//   preallocate_pyramid (placement.cpp:25-62) and greedy_pack
//   (placement.cpp:182-204), plus peak_mem = max(addr + size)
//   (pipeline.cpp:270-275) of the resulting address plan.
//
// One CTA per problem (a problem = one lifetime vector over the shared edge
// sizes, e.g. one candidate order). Both heuristics are sequential over edges,
// so the parallelism inside a CTA is over the already-placed tensors:
//
// greedy_pack places edge e at the lowest offset x >= 0 with no placed,
// lifetime-overlapping tensor w such that x < top_w && addr_w < x + size_e
// (the reference's bump loop reaches exactly that x: every offset it skips is
// covered by the tensor that made it jump, and it stops at a free one). In
// terms of L_w = addr_w - size_e and R_w = top_w the forbidden offsets are the
// open intervals (L_w, R_w); with the placed tensors kept sorted by address
// (hence by L), x is the first gap of their union: M = max(0, R over the
// prefix) up to the first conflicting w with L_w >= M. A CTA evaluates that
// with one block-wide exclusive prefix-max over per-thread chunks, a chunk
// sweep and a block min, then inserts e at its sorted position. Tensors stay
// in append-only slots; the address order is an index array `ord` that each
// thread shifts from its registers (4 bytes per entry). Per edge: O(placed/T)
// work and five barriers.
//
// preallocate_pyramid walks the problem's edges in preference order (duration, then
// size, then the edge id's rank in byte order; sorted by the launcher) with a cursor
// that only moves forward, since the window only narrows.
//
// Shared memory: the placed set, 28 bytes per tensor (address, top, lifetime,
// order index), so up to kPlaceMaxEntries tensors per problem.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cstdint>
#include <type_traits>

#include <cub/device/device_radix_sort.cuh>

#include "mp_internal.h"

namespace mpb {
namespace {

constexpr int kChMax = 16;    // entries per thread in registers
static_assert(512 * kChMax == kPlaceMaxEntries, "placed-set capacity");

// Threads per problem: the smallest of 128/256/512 whose chunks hold every
// tensor (16 per thread), so small graphs fit several problems per SM.
template <int kPT>
struct PlaceScratch {
  long long wmax[kPT / 32];
  int stop;
  int pos;
  long long x;
  long long allmax;
  int we[kPT / 32];  // pyramid: first qualifying index per warp
};

// `ord` is stored skewed (one pad word per 32 entries): thread t's chunk starts at
// t * ch, and with an even ch the unskewed words would sit in a few banks only.
__device__ __forceinline__ int sk(int i) { return i + (i >> 5); }

__device__ __forceinline__ bool disjoint(int alo, int ahi, int blo, int bhi) {
  return alo > ahi || blo > bhi || ahi < blo || bhi < alo;  // analysis.hpp:28-37
}

template <int kPT>
__global__ void __launch_bounds__(kPT, 512 / kPT)
    place_kernel(PlaceArgs a) {
  extern __shared__ __align__(16) char smem[];
  __shared__ PlaceScratch<kPT> ps;
  const int E = a.num_edges;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int kW = kPT / 32;
  const int cap = a.cap;
  // by slot: (address, top) together - the sweep reads both with one 16-byte load
  ulonglong2* e_at = reinterpret_cast<ulonglong2*>(smem);
  int2* e_life = reinterpret_cast<int2*>(e_at + cap);
  int* ord = reinterpret_cast<int*>(e_life + cap);          // slots in address order (skewed)
  uint8_t* flag = reinterpret_cast<uint8_t*>(ord + cap + (cap >> 5) + 1);  // [E] fixed / taken

  for (int64_t b = blockIdx.x; b < a.num_problems; b += gridDim.x) {
    const int32_t* lo = a.lo + b * (int64_t)E;
    const int32_t* hi = a.hi + b * (int64_t)E;
    uint64_t* out_addr = a.addr + b * (int64_t)E;
    uint8_t* out_has = a.has_addr + b * (int64_t)E;
    int k = 0;                // placed tensors
    unsigned long long peak = 0;
    for (int e = tid; e < E; e += kPT) {
      flag[e] = 0;
      out_has[e] = 0;
      out_addr[e] = 0;
    }
    __syncthreads();

    // Place one tensor (size s, lifetime [elo, ehi]) at x, or - when `search` -
    // at greedy_pack's lowest feasible offset; returns the offset.
    // CHT: compile-time bound on the per-thread chunk, chosen per step (2/4/8/16)
    // so early steps do not pay for 16 predicated-off register slots.
    auto place_ch = [&](auto cht, bool search, unsigned long long x, unsigned long long s,
                        int elo, int ehi) -> unsigned long long {
      constexpr int kCh = decltype(cht)::value;
      const int ch = (k + kPT - 1) / kPT;
      const int i0 = tid * ch;
      int o[kCh];
#pragma unroll
      for (int q = 0; q < kCh; ++q) o[q] = (q < ch && i0 + q < k) ? ord[sk(i0 + q)] : -1;
      if (search) {
        long long cm = LLONG_MIN;  // max top over this chunk's conflicting tensors
#pragma unroll
        for (int q = 0; q < kCh; ++q)
          if (o[q] >= 0) {
            const int2 l = e_life[o[q]];
            if (!disjoint(elo, ehi, l.x, l.y)) {
              const long long t = (long long)e_at[o[q]].y;
              cm = t > cm ? t : cm;
            }
          }
        // block exclusive prefix-max of cm (chunks are in address order)
        long long incl = cm;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const long long v = __shfl_up_sync(0xffffffffu, incl, d);
          if (lane >= d && v > incl) incl = v;
        }
        if (lane == 31) ps.wmax[warp] = incl;
        if (tid == 0) ps.stop = INT_MAX;
        __syncthreads();
        long long before = __shfl_up_sync(0xffffffffu, incl, 1);
        if (lane == 0) before = LLONG_MIN;
        for (int w = 0; w < warp; ++w) before = ps.wmax[w] > before ? ps.wmax[w] : before;
        // sweep the chunk: the first conflicting tensor with L >= M leaves a gap at M
        long long M = before > 0 ? before : 0;
        int stop = INT_MAX;
        long long xs = 0;
#pragma unroll
        for (int q = 0; q < kCh; ++q)
          if (stop == INT_MAX && o[q] >= 0) {
            const int2 l = e_life[o[q]];
            if (!disjoint(elo, ehi, l.x, l.y)) {
              const ulonglong2 at = e_at[o[q]];
              const long long L = (long long)at.x - (long long)s;
              const long long t = (long long)at.y;
              if (L >= M) {
                stop = i0 + q;
                xs = M;
              } else if (t > M) {
                M = t;
              }
            }
          }
        if (stop != INT_MAX) atomicMin(&ps.stop, stop);
        if (tid == kPT - 1) {
          long long all = incl;  // inclusive prefix at the last thread = max over all
          for (int w = 0; w < warp; ++w) all = ps.wmax[w] > all ? ps.wmax[w] : all;
          ps.allmax = all > 0 ? all : 0;
        }
        __syncthreads();
        if (stop != INT_MAX && stop == ps.stop) ps.x = xs;
        __syncthreads();
        x = ps.stop != INT_MAX ? (unsigned long long)ps.x : (unsigned long long)ps.allmax;
      }
      // insert at the first address-order index whose address is >= x
      int cnt = 0;
#pragma unroll
      for (int q = 0; q < kCh; ++q)
        if (o[q] >= 0) cnt += e_at[o[q]].x < x;
      if (tid == 0) ps.pos = 0;
      __syncthreads();
      cnt = __reduce_add_sync(0xffffffffu, cnt);
      if (lane == 0 && cnt) atomicAdd(&ps.pos, cnt);
      __syncthreads();
      const int p = ps.pos;
#pragma unroll
      for (int q = 0; q < kCh; ++q)
        if (o[q] >= 0 && i0 + q >= p) ord[sk(i0 + q + 1)] = o[q];
      if (tid == 0) {
        ord[sk(p)] = k;
        e_at[k] = make_ulonglong2(x, x + s);
        e_life[k] = make_int2(elo, ehi);
      }
      __syncthreads();
      ++k;
      return x;
    };
    auto place = [&](bool search, unsigned long long x, unsigned long long s, int elo,
                     int ehi) -> unsigned long long {
      const int ch = (k + kPT - 1) / kPT;
      if (ch <= 2) return place_ch(std::integral_constant<int, 2>{}, search, x, s, elo, ehi);
      if (ch <= 4) return place_ch(std::integral_constant<int, 4>{}, search, x, s, elo, ehi);
      if (ch <= 8) return place_ch(std::integral_constant<int, 8>{}, search, x, s, elo, ehi);
      return place_ch(std::integral_constant<int, kChMax>{}, search, x, s, elo, ehi);
    };

    // ---- fixed tensors: caller's preplaced map, or preallocate_pyramid ------------
    if (a.pyramid) {  // preference order with a forward-only cursor (see place_big_kernel)
      const int32_t* po = a.pyr_order + b * (int64_t)E;
      long long min_start = 0, max_end = LLONG_MAX;
      unsigned long long base = 0;
      for (int cur = 0; max_end > min_start && cur < E;) {
        const int i = cur + tid;
        bool ok = false;
        if (i < E) {
          const int e = po[i];
          ok = a.size[e] != 0 && lo[e] > min_start && hi[e] < max_end;
        }
        const int f = __reduce_min_sync(0xffffffffu, ok ? i : INT_MAX);
        if (lane == 0) ps.we[warp] = f;
        __syncthreads();
        int fm = INT_MAX;
        for (int w = 0; w < kW; ++w) fm = min(fm, ps.we[w]);
        __syncthreads();  // ps.we is rewritten by the next round
        if (fm == INT_MAX) {
          cur += kPT;
          continue;
        }
        cur = fm + 1;
        const int pick = po[fm];
        const unsigned long long s = a.size[pick];
        if (tid == 0) {
          flag[pick] = 1;
          out_addr[pick] = base;
          out_has[pick] = 1;
        }
        place(false, base, s, lo[pick], hi[pick]);
        base += s;
        peak = base > peak ? base : peak;
        min_start = lo[pick];
        max_end = hi[pick];
      }
      if (tid == 0 && a.pyramid_base) a.pyramid_base[b] = base;
    } else if (a.fixed) {
      for (int e = 0; e < E; ++e) {  // uniform loop: preplaced maps are small
        if (!a.fixed[e]) continue;
        const unsigned long long x = a.fixed_addr[e], s = a.size[e];
        if (tid == 0) {
          flag[e] = 1;
          out_addr[e] = x;
          out_has[e] = 1;
        }
        place(false, x, s, lo[e], hi[e]);
        peak = x + s > peak ? x + s : peak;
      }
    }
    __syncthreads();

    // ---- greedy_pack over the remaining data edges, in edge order -----------------
    if (!a.pyramid_only) {
      // the next edge's (size, lifetime) is loaded one step ahead (uniform loads)
      unsigned long long s_nx = E > 0 ? a.size[0] : 0;
      int lo_nx = E > 0 ? lo[0] : 0, hi_nx = E > 0 ? hi[0] : 0;
      for (int e = 0; e < E; ++e) {
        const unsigned long long s = s_nx;
        const int elo = lo_nx, ehi = hi_nx;
        if (e + 1 < E) {
          s_nx = a.size[e + 1];
          lo_nx = lo[e + 1];
          hi_nx = hi[e + 1];
        }
        if (s == 0 || flag[e]) continue;  // uniform: flags were fixed before this loop
        const unsigned long long x = place(true, 0, s, elo, ehi);
        if (tid == 0) {
          out_addr[e] = x;
          out_has[e] = 1;
        }
        peak = x + s > peak ? x + s : peak;
      }
    }
    if (tid == 0 && a.peak_mem) a.peak_mem[b] = peak;
    __syncthreads();
  }
}

// ---- warp per problem (many problems, E <= kPlaceWarpMaxEdges) -------------------
// The same heuristics with the placed set kept IN ADDRESS ORDER as three arrays in
// the warp's shared-memory slice (address, top, lifetime: 24 bytes per tensor), so
// the search reads 32 consecutive tensors per step with no index indirection and no
// bank conflicts, and no block barrier is ever needed:
//   search   rounds of 32 tensors in address order; pm = max(0, tops of the
//            lifetime-overlapping tensors before this one) is a carried value plus a
//            warp exclusive prefix-max; the first overlapping tensor with
//            addr - size >= pm leaves the gap at pm (ballot + ffs); if none, x = the
//            final pm. Rounds stop at the gap.
//   insert   the first index whose address is >= x (32-ary warp search), then the
//            tail shifts right by one, 32 tensors per step from the end.
// The CTA variant above keeps append-only slots and shifts a 4-byte index instead;
// its indirect random reads made half its shared-memory wavefronts bank conflicts.
// One warp per problem is latency-bound (a shuffle scan per 32 tensors): it wins
// only where many problems fit an SM (C2: 1.68e5 vs 1.51e5 placements/s).
constexpr int kPlaceWarpMaxEdges = 4096;

template <int W>
__global__ void __launch_bounds__(32 * W) place_warp_kernel(PlaceArgs a, size_t slice) {
  extern __shared__ __align__(16) char smem[];
  const int E = a.num_edges;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int cap = a.cap;
  char* base_p = smem + (size_t)warp * slice;
  unsigned long long* P_addr = reinterpret_cast<unsigned long long*>(base_p);
  unsigned long long* P_top = P_addr + cap;
  int2* P_life = reinterpret_cast<int2*>(P_top + cap);
  uint8_t* flag = reinterpret_cast<uint8_t*>(P_life + cap);

  for (int64_t b = (int64_t)blockIdx.x * W + warp; b < a.num_problems;
       b += (int64_t)gridDim.x * W) {
    const int32_t* lo = a.lo + b * (int64_t)E;
    const int32_t* hi = a.hi + b * (int64_t)E;
    uint64_t* out_addr = a.addr + b * (int64_t)E;
    uint8_t* out_has = a.has_addr + b * (int64_t)E;
    int k = 0;
    unsigned long long peak = 0;
    for (int e = lane; e < E; e += 32) {
      flag[e] = 0;
      out_has[e] = 0;
      out_addr[e] = 0;
    }
    __syncwarp();

    // insert (x, x + s, [elo, ehi]) at its address-order index
    auto insert = [&](unsigned long long x, unsigned long long s, int elo, int ehi) {
      // first index p with P_addr[p] >= x: 32-ary narrowing over [0, k)
      int lo_i = 0, n_i = k;
      while (n_i > 32) {
        const int step = (n_i + 31) / 32;
        const int probe = lo_i + lane * step;
        const bool below = probe < lo_i + n_i && P_addr[probe] < x;
        const int c = __popc(__ballot_sync(0xffffffffu, below));  // probes below x
        if (c == 0) {
          n_i = 0;
          break;
        }
        const int nlo = lo_i + (c - 1) * step;  // last probe below x: p is after it
        const int nhi = min(lo_i + c * step, lo_i + n_i);
        lo_i = nlo + 1;
        n_i = nhi - lo_i;
        if (n_i < 0) n_i = 0;
      }
      const bool below = lane < n_i && P_addr[lo_i + lane] < x;
      const int p = lo_i + __popc(__ballot_sync(0xffffffffu, below));
      // shift [p, k) right by one, 32 tensors per step from the end
      for (int r = k - 32; r > p - 32; r -= 32) {
        const int i = r + lane;
        const bool mv = i >= p && i >= 0 && i < k;
        unsigned long long ad = 0, tp = 0;
        int2 lf = make_int2(0, 0);
        if (mv) {
          ad = P_addr[i];
          tp = P_top[i];
          lf = P_life[i];
        }
        __syncwarp();
        if (mv) {
          P_addr[i + 1] = ad;
          P_top[i + 1] = tp;
          P_life[i + 1] = lf;
        }
        __syncwarp();
      }
      if (lane == 0) {
        P_addr[p] = x;
        P_top[p] = x + s;
        P_life[p] = make_int2(elo, ehi);
      }
      __syncwarp();
      ++k;
    };
    // greedy_pack's lowest feasible offset for (s, [elo, ehi]) (placement.cpp:187-200)
    auto search = [&](unsigned long long s, int elo, int ehi) -> unsigned long long {
      long long pm = 0;  // max(0, tops of the overlapping tensors before this round)
      for (int r = 0; r < k; r += 32) {
        const int i = r + lane;
        bool conf = false;
        long long t = LLONG_MIN, L = 0;
        if (i < k) {
          const int2 l = P_life[i];
          conf = !disjoint(elo, ehi, l.x, l.y);
          t = conf ? (long long)P_top[i] : LLONG_MIN;
          L = (long long)P_addr[i] - (long long)s;
        }
        long long incl = t;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const long long v = __shfl_up_sync(0xffffffffu, incl, d);
          if (lane >= d && v > incl) incl = v;
        }
        long long ex = __shfl_up_sync(0xffffffffu, incl, 1);
        if (lane == 0) ex = LLONG_MIN;
        const long long m = ex > pm ? ex : pm;
        const unsigned gap = __ballot_sync(0xffffffffu, conf && L >= m);
        if (gap) return (unsigned long long)__shfl_sync(0xffffffffu, m, __ffs(gap) - 1);
        const long long rm = __shfl_sync(0xffffffffu, incl, 31);
        pm = rm > pm ? rm : pm;
      }
      return (unsigned long long)pm;
    };

    // ---- fixed tensors: caller's preplaced map, or preallocate_pyramid ------------
    if (a.pyramid) {  // preference order with a forward-only cursor (see place_big_kernel)
      const int32_t* po = a.pyr_order + b * (int64_t)E;
      long long min_start = 0, max_end = LLONG_MAX;
      unsigned long long pbase = 0;
      for (int cur = 0; max_end > min_start && cur < E;) {
        const int i = cur + lane;
        bool ok = false;
        if (i < E) {
          const int e = po[i];
          ok = a.size[e] != 0 && lo[e] > min_start && hi[e] < max_end;
        }
        const unsigned m = __ballot_sync(0xffffffffu, ok);
        if (!m) {
          cur += 32;
          continue;
        }
        const int f = cur + __ffs(m) - 1;
        cur = f + 1;
        const int pick = po[f];
        const unsigned long long sz = a.size[pick];
        const int pl = lo[pick], ph = hi[pick];
        if (lane == 0) {
          flag[pick] = 1;
          out_addr[pick] = pbase;
          out_has[pick] = 1;
        }
        insert(pbase, sz, pl, ph);
        pbase += sz;
        peak = pbase > peak ? pbase : peak;
        min_start = pl;
        max_end = ph;
      }
      if (lane == 0 && a.pyramid_base) a.pyramid_base[b] = pbase;
    } else if (a.fixed) {
      for (int e = 0; e < E; ++e) {
        if (!a.fixed[e]) continue;
        const unsigned long long x = a.fixed_addr[e], sz = a.size[e];
        if (lane == 0) {
          flag[e] = 1;
          out_addr[e] = x;
          out_has[e] = 1;
        }
        insert(x, sz, lo[e], hi[e]);
        peak = x + sz > peak ? x + sz : peak;
      }
    }
    __syncwarp();

    // ---- greedy_pack over the remaining data edges, in edge order -----------------
    if (!a.pyramid_only) {
      // the next edge's (size, lifetime) is loaded one step ahead
      unsigned long long s_nx = a.size[0];
      int lo_nx = lo[0], hi_nx = hi[0];
      for (int e = 0; e < E; ++e) {
        const unsigned long long sz = s_nx;
        const int elo = lo_nx, ehi = hi_nx;
        if (e + 1 < E) {
          s_nx = a.size[e + 1];
          lo_nx = lo[e + 1];
          hi_nx = hi[e + 1];
        }
        if (sz == 0 || flag[e]) continue;
        const unsigned long long x = search(sz, elo, ehi);
        insert(x, sz, elo, ehi);
        if (lane == 0) {
          out_addr[e] = x;
          out_has[e] = 1;
        }
        peak = x + sz > peak ? x + sz : peak;
      }
    }
    if (lane == 0 && a.peak_mem) a.peak_mem[b] = peak;
    __syncwarp();
  }
}

// ---- one CTA per problem, placed set in global memory (E > kPlaceMaxEntries) -------
// The warp variant's address-ordered arrays (address, top, lifetime: 24 bytes per
// tensor) in a per-CTA global slice, L2-resident for one problem, scanned by 512
// threads in 4096-tensor tiles (8 consecutive tensors per thread, 16-byte loads):
//   search   per tile a block prefix-max of the overlapping tops (warp shuffles + one
//            word per warp), each thread's sweep of its 8 tensors from that prefix,
//            and a block min of the first gap; the scan stops at the tile holding it
//   insert   the first index whose address is >= x by a two-level 512-ary count
//            (__syncthreads_count), then the tail shifts right by one, 2048 tensors
//            per tile from the end
// Same results as the other variants (the placed set is the same set in the same
// order); for the 100k-tensor graph, whose placed sets do not fit shared memory.
constexpr int kBigT = 512, kBigR = 8, kBigTile = kBigT * kBigR;
constexpr int kBigW = kBigT / 32;

struct BigShared {
  long long wmax[32];
  int stop[2];
  long long x;
};
struct BigSet {  // the placed set in address order (a per-CTA global slice) and its size
  unsigned long long* addr;
  unsigned long long* top;
  int2* life;
  BigShared* s;
  int k;
  int gi;  // tiles scanned so far (selects the stop buffer)
};

// greedy_pack's lowest feasible offset for (s, [elo, ehi]) (placement.cpp:187-200)
__device__ __forceinline__ unsigned long long big_search(BigSet& P, unsigned long long s, int elo,
                                                         int ehi) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int k = P.k;
  long long carry = 0;  // max(0, overlapping tops of the earlier tiles)
  for (int b0 = 0; b0 < k; b0 += kBigTile, ++P.gi) {
    const int j0 = b0 + kBigR * tid;
    unsigned long long ad[kBigR], tp[kBigR];
    int2 lf[kBigR];
    if (j0 < k) {  // the slice is padded to whole tiles: no partial vectors
#pragma unroll
      for (int q = 0; q < kBigR; q += 2) {
        const ulonglong2 u = __ldcg(reinterpret_cast<const ulonglong2*>(P.addr + j0 + q));
        const ulonglong2 v = __ldcg(reinterpret_cast<const ulonglong2*>(P.top + j0 + q));
        const int4 l = __ldcg(reinterpret_cast<const int4*>(P.life + j0 + q));
        ad[q] = u.x, ad[q + 1] = u.y, tp[q] = v.x, tp[q + 1] = v.y;
        lf[q] = make_int2(l.x, l.y), lf[q + 1] = make_int2(l.z, l.w);
      }
    }
    bool cf[kBigR];
    long long cm = LLONG_MIN;  // max top over this thread's overlapping tensors
#pragma unroll
    for (int q = 0; q < kBigR; ++q) {
      cf[q] = j0 + q < k && !disjoint(elo, ehi, lf[q].x, lf[q].y);
      if (cf[q] && (long long)tp[q] > cm) cm = (long long)tp[q];
    }
    long long incl = cm;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const long long v = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d && v > incl) incl = v;
    }
    if (lane == 31) P.s->wmax[warp] = incl;
    __syncthreads();
    // the other buffer was last read before this barrier: reset it for the next tile
    if (tid == 0) P.s->stop[(P.gi + 1) & 1] = INT_MAX;
    long long before = __shfl_up_sync(0xffffffffu, incl, 1);
    if (lane == 0) before = LLONG_MIN;
    // the warps' totals: an inclusive max-scan over lanes 0 .. kBigW - 1
    long long wv = lane < kBigW ? P.s->wmax[lane] : LLONG_MIN;
#pragma unroll
    for (int d = 1; d < kBigW; d <<= 1) {
      const long long v = __shfl_up_sync(0xffffffffu, wv, d);
      if (lane >= d && v > wv) wv = v;
    }
    const long long wprev = __shfl_sync(0xffffffffu, wv, warp > 0 ? warp - 1 : 0);
    if (warp > 0 && wprev > before) before = wprev;
    const long long tmax = __shfl_sync(0xffffffffu, wv, kBigW - 1);
    long long M = before > carry ? before : carry;
    int stop = INT_MAX;
    long long xs = 0;
#pragma unroll
    for (int q = 0; q < kBigR; ++q)
      if (stop == INT_MAX && cf[q]) {
        const long long L = (long long)ad[q] - (long long)s;
        if (L >= M) {
          stop = j0 + q;
          xs = M;
        } else if ((long long)tp[q] > M) {
          M = (long long)tp[q];
        }
      }
    if (stop != INT_MAX) atomicMin(&P.s->stop[P.gi & 1], stop);
    __syncthreads();
    const int gs = P.s->stop[P.gi & 1];
    if (gs != INT_MAX) {
      if (stop == gs) P.s->x = xs;
      __syncthreads();
      ++P.gi;
      return (unsigned long long)P.s->x;  // rewritten only after two more barriers
    }
    if (tmax > carry) carry = tmax;
  }
  return (unsigned long long)carry;
}

// insert (x, x + s, [elo, ehi]) at the first index whose address is >= x
__device__ __forceinline__ void big_insert(BigSet& P, unsigned long long x, unsigned long long s,
                                           int elo, int ehi) {
  const int tid = threadIdx.x;
  const int k = P.k;
  int p = 0;
  if (k > 0) {
    const int step = (k + kBigT - 1) / kBigT;
    const int j = tid * step;
    const int c1 = __syncthreads_count(j < k && __ldcg(P.addr + j) < x);
    if (c1 > 0) {  // p in [(c1 - 1) * step + 1, min(c1 * step, k)]
      const int lo_i = (c1 - 1) * step + 1, hi_i = min(c1 * step, k);
      const int j2 = lo_i + tid;
      p = lo_i + __syncthreads_count(j2 < hi_i && __ldcg(P.addr + j2) < x);
    }
  }
  // [p, k) right by one, 2048 tensors per tile (4 per thread: the 8 of the search
  // would keep 48 addresses live across the barrier)
  constexpr int kShiftR = 4, kShiftTile = kBigT * kShiftR;
  for (int t_hi = k; t_hi > p; t_hi -= kShiftTile) {
    const int t_lo = max(p, t_hi - kShiftTile);
    unsigned long long ad[kShiftR], tp[kShiftR];
    int2 lf[kShiftR];
#pragma unroll
    for (int q = 0; q < kShiftR; ++q) {
      const int i = t_lo + tid + q * kBigT;
      if (i < t_hi) {
        ad[q] = __ldcg(P.addr + i);
        tp[q] = __ldcg(P.top + i);
        lf[q] = __ldcg(P.life + i);
      }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < kShiftR; ++q) {
      const int i = t_lo + tid + q * kBigT;
      if (i < t_hi) {
        __stcg(P.addr + i + 1, ad[q]);
        __stcg(P.top + i + 1, tp[q]);
        __stcg(P.life + i + 1, lf[q]);
      }
    }
    __syncthreads();
  }
  if (tid == 0) {
    __stcg(P.addr + p, x);
    __stcg(P.top + p, x + s);
    __stcg(P.life + p, make_int2(elo, ehi));
  }
  __syncthreads();
  ++P.k;
}

__global__ void __launch_bounds__(kBigT, 1)
    place_big_kernel(PlaceArgs a, char* __restrict__ scratch, size_t stride, int cap) {
  __shared__ BigShared sh;
  __shared__ int s_wd[32];
  const int E = a.num_edges;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  char* base_p = scratch + (size_t)blockIdx.x * stride;
  BigSet P;
  P.addr = reinterpret_cast<unsigned long long*>(base_p);
  P.top = P.addr + cap;
  P.life = reinterpret_cast<int2*>(P.top + cap);
  P.s = &sh;
  P.gi = 0;
  uint8_t* flag = reinterpret_cast<uint8_t*>(P.life + cap);
  if (tid < 2) sh.stop[tid] = INT_MAX;

  for (int64_t b = blockIdx.x; b < a.num_problems; b += gridDim.x) {
    const int32_t* lo = a.lo + b * (int64_t)E;
    const int32_t* hi = a.hi + b * (int64_t)E;
    uint64_t* out_addr = a.addr + b * (int64_t)E;
    uint8_t* out_has = a.has_addr + b * (int64_t)E;
    P.k = 0;
    unsigned long long peak = 0;
    for (int e = tid; e < E; e += kBigT) {
      flag[e] = 0;
      out_has[e] = 0;
      out_addr[e] = 0;
    }
    __syncthreads();

    // ---- fixed tensors: caller's preplaced map, or preallocate_pyramid ------------
    // The pyramid walks this problem's edges in preference order (duration desc, size
    // desc, id rank asc: pyr_order, sorted by the launcher): the pick is the first edge
    // from the cursor inside the window. The window only shrinks (min_start rises to the
    // pick's lo, max_end falls to its hi), so the edges skipped on the way never qualify
    // again and the cursor only moves forward: O(E) checks for all picks together.
    if (a.pyramid) {
      const int32_t* po = a.pyr_order + b * (int64_t)E;
      long long min_start = 0, max_end = LLONG_MAX;
      unsigned long long pbase = 0;
      int cur = 0;
      while (max_end > min_start && cur < E) {
        const int i = cur + tid;
        bool ok = false;
        if (i < E) {
          const int e = po[i];
          ok = a.size[e] != 0 && lo[e] > min_start && hi[e] < max_end;
        }
        const int f = __reduce_min_sync(0xffffffffu, ok ? i : INT_MAX);
        if (lane == 0) s_wd[warp] = f;
        __syncthreads();
        int fm = INT_MAX;
        for (int w = 0; w < kBigW; ++w) fm = min(fm, s_wd[w]);
        __syncthreads();  // s_wd is rewritten by the next round
        if (fm == INT_MAX) {
          cur += kBigT;
          continue;
        }
        const int pick = po[fm];
        cur = fm + 1;
        const unsigned long long sz = a.size[pick];
        if (tid == 0) {
          flag[pick] = 1;
          out_addr[pick] = pbase;
          out_has[pick] = 1;
        }
        big_insert(P, pbase, sz, lo[pick], hi[pick]);  // its barriers also publish flag[pick]
        pbase += sz;
        peak = pbase > peak ? pbase : peak;
        min_start = lo[pick];
        max_end = hi[pick];
      }
      if (tid == 0 && a.pyramid_base) a.pyramid_base[b] = pbase;
    } else if (a.fixed) {
      for (int e = 0; e < E; ++e) {  // uniform loop: preplaced maps are small
        if (!a.fixed[e]) continue;
        const unsigned long long x = a.fixed_addr[e], sz = a.size[e];
        if (tid == 0) {
          flag[e] = 1;
          out_addr[e] = x;
          out_has[e] = 1;
        }
        big_insert(P, x, sz, lo[e], hi[e]);
        peak = x + sz > peak ? x + sz : peak;
      }
    }
    __syncthreads();

    // ---- greedy_pack over the remaining data edges, in edge order -----------------
    if (!a.pyramid_only) {
      for (int e = 0; e < E; ++e) {
        const unsigned long long sz = a.size[e];
        if (sz == 0 || flag[e]) continue;  // uniform: flags were fixed before this loop
        const int elo = lo[e], ehi = hi[e];
        const unsigned long long x = big_search(P, sz, elo, ehi);
        big_insert(P, x, sz, elo, ehi);
        if (tid == 0) {
          out_addr[e] = x;
          out_has[e] = 1;
        }
        peak = x + sz > peak ? x + sz : peak;
      }
    }
    if (tid == 0 && a.peak_mem) a.peak_mem[b] = peak;
    __syncthreads();
  }
}

// pyramid preference order for the global-memory variant (sorted by the launcher with
// stable radix sorts): edges by id rank, then by size descending (static), then per
// problem by duration descending
__global__ void pyr_key_rank(int E, const int32_t* __restrict__ id_rank, uint32_t* key,
                             int32_t* val) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < E; i += gridDim.x * blockDim.x) {
    key[i] = id_rank ? (uint32_t)id_rank[i] : (uint32_t)i;
    val[i] = i;
  }
}
__global__ void pyr_key_size(int E, const uint64_t* __restrict__ size,
                             const int32_t* __restrict__ by_rank, uint64_t* key, int32_t* val) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < E; i += gridDim.x * blockDim.x) {
    const int e = by_rank[i];
    key[i] = ~size[e];  // ascending sort = size descending
    val[i] = e;
  }
}
__global__ void pyr_key_dur(int E, int64_t nb, const int32_t* __restrict__ lo,
                            const int32_t* __restrict__ hi, const int32_t* __restrict__ order0,
                            uint64_t* key, int32_t* val) {
  const int64_t N = nb * (int64_t)E;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < N;
       x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = x / E;
    const int e = order0[x - b * E];
    const uint32_t d = (uint32_t)(hi[b * E + e] - lo[b * E + e]) ^ 0x80000000u;  // signed order
    key[x] = (uint64_t)b << 32 | (0xffffffffu - d);  // by problem, then duration descending
    val[x] = e;
  }
}

size_t place_big_stride(int num_edges, int* cap) {
  // whole tiles (search loads 8 tensors per thread unguarded) plus the one-past shift
  *cap = ((num_edges + 1 + kBigTile - 1) / kBigTile) * kBigTile;
  return ((size_t)*cap * (8 + 8 + 8) + (size_t)num_edges + 255) & ~size_t(255);
}

size_t place_warp_slice(int num_edges) {
  const size_t cap = (size_t)num_edges + 1;
  return ((cap * (8 + 8 + 8) + (size_t)num_edges) + 15) & ~size_t(15);
}

}  // namespace

size_t place_smem_bytes(int num_edges) {
  const int cap = num_edges < kPlaceMaxEntries ? num_edges + 1 : kPlaceMaxEntries;
  return (size_t)cap * (8 + 8 + 8 + 4) + 4 * ((size_t)(cap >> 5) + 1) + (size_t)num_edges + 16;
}

template <int kPT>
mp_status launch_place_t(const PlaceArgs& in, mp_ctx* ctx, cudaStream_t st) {
  PlaceArgs a = in;
  a.cap = in.num_edges < kPlaceMaxEntries ? in.num_edges + 1 : kPlaceMaxEntries;
  const size_t smem = place_smem_bytes(in.num_edges);
  auto kern = place_kernel<kPT>;
  MP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  MP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kPT, smem));
  int64_t grid = (int64_t)ctx->num_sms * (per_sm > 0 ? per_sm : 1);
  if (grid > in.num_problems) grid = in.num_problems;
  kern<<<(unsigned)grid, kPT, smem, st>>>(a);
  MP_CUDA(cudaGetLastError());
  return MP_OK;
}

// The pyramid's preference order per problem (every K5 variant walks it with a cursor):
// stable radix sorts by id rank and by size descending once per call, then per group of
// problems by (problem, duration descending). Buffers are carved from one scratch slot.
struct PyrSort {
  int E = 0;
  int64_t group = 0;
  size_t temp = 0;
  int32_t* order0 = nullptr;
  uint32_t *k32 = nullptr, *k32o = nullptr;
  int32_t* v32 = nullptr;
  uint64_t *k64 = nullptr, *keys = nullptr, *keys_o = nullptr;
  int32_t *vals = nullptr, *porder = nullptr;
  void* tmp = nullptr;
  static size_t al(size_t b) { return (b + 255) & ~size_t(255); }
  mp_status size(int e, int64_t g, size_t* bytes, cudaStream_t st) {
    E = e;
    group = g;
    const size_t ng = (size_t)g * e;
    size_t t1 = 0, t2 = 0;
    MP_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, t1, (const uint64_t*)nullptr,
                                            (uint64_t*)nullptr, (const int32_t*)nullptr,
                                            (int32_t*)nullptr, (int64_t)std::max<size_t>(ng, e),
                                            0, 64, st));
    MP_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, t2, (const uint32_t*)nullptr,
                                            (uint32_t*)nullptr, (const int32_t*)nullptr,
                                            (int32_t*)nullptr, e, 0, 32, st));
    temp = al(std::max(t1, t2));
    *bytes = 4 * al(4 * (size_t)e) + al(8 * (size_t)e) + 2 * al(8 * ng) + 2 * al(4 * ng) + temp;
    return MP_OK;
  }
  void carve(char* p) {
    auto take = [&](size_t b) {
      char* r = p;
      p += al(b);
      return r;
    };
    const size_t ng = (size_t)group * E;
    order0 = reinterpret_cast<int32_t*>(take(4 * (size_t)E));
    k32 = reinterpret_cast<uint32_t*>(take(4 * (size_t)E));
    k32o = reinterpret_cast<uint32_t*>(take(4 * (size_t)E));
    v32 = reinterpret_cast<int32_t*>(take(4 * (size_t)E));
    k64 = reinterpret_cast<uint64_t*>(take(8 * (size_t)E));
    keys = reinterpret_cast<uint64_t*>(take(8 * ng));
    keys_o = reinterpret_cast<uint64_t*>(take(8 * ng));
    vals = reinterpret_cast<int32_t*>(take(4 * ng));
    porder = reinterpret_cast<int32_t*>(take(4 * ng));
    tmp = take(temp);
  }
  mp_status statics(const int32_t* id_rank, const uint64_t* size, cudaStream_t st) {
    const int eb = (int)std::min<int64_t>((E + 255) / 256, 4096);
    pyr_key_rank<<<eb, 256, 0, st>>>(E, id_rank, k32, v32);
    size_t tb = temp;
    MP_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, k32, k32o, v32, vals, E, 0, 32, st));
    pyr_key_size<<<eb, 256, 0, st>>>(E, size, vals, k64, v32);
    tb = temp;
    MP_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, k64, keys_o, v32, order0, E, 0, 64, st));
    return MP_OK;
  }
  mp_status problems(const int32_t* lo, const int32_t* hi, int64_t nb, cudaStream_t st) {
    const int64_t n_items = nb * (int64_t)E;
    int bits = 1;
    while ((int64_t(1) << bits) < nb) ++bits;
    const int kb = (int)std::min<int64_t>((n_items + 255) / 256, 8192);
    pyr_key_dur<<<kb, 256, 0, st>>>(E, nb, lo, hi, order0, keys, vals);
    size_t tb = temp;
    MP_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, keys, keys_o, vals, porder, n_items, 0,
                                            32 + bits, st));
    return MP_OK;
  }
};

static mp_status launch_group(const PlaceArgs& a, mp_ctx* ctx, cudaStream_t st, char* slices,
                              size_t stride, int cap) {
  if (slices) {  // placed sets past shared memory: one 512-thread CTA per problem
    place_big_kernel<<<(unsigned)a.num_problems, kBigT, 0, st>>>(a, slices, stride, cap);
    MP_CUDA(cudaGetLastError());
    return MP_OK;
  }
  // many problems of a modest graph: one warp per problem, placed set in address order
  // (MP_PLACE_CTA forces the CTA variant, MP_PLACE_WARP the warp variant)
  const bool force_cta = std::getenv("MP_PLACE_CTA") != nullptr;
  const bool force_warp = std::getenv("MP_PLACE_WARP") != nullptr;
  const size_t slice = place_warp_slice(a.num_edges);
  // measured: +11% at C2 (7 warps per SM), 2x slower at C3 (3 warps per SM): only where
  // at least six problems' placed sets fit one SM
  const bool warp_ok = force_warp || (a.num_problems > ctx->num_sms && slice * 6 <= 228 * 1024);
  if (!force_cta && a.num_edges <= kPlaceWarpMaxEdges && warp_ok &&
      slice <= (size_t)ctx->max_smem_optin) {
    PlaceArgs w = a;
    w.cap = a.num_edges + 1;
    // one-warp CTAs: as many per SM as their placed sets fit (up to 32)
    auto kern = place_warp_kernel<1>;
    MP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)slice));
    int per_sm = 0;
    MP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32, slice));
    int64_t grid = (int64_t)ctx->num_sms * (per_sm > 0 ? per_sm : 1);
    if (grid > a.num_problems) grid = a.num_problems;
    kern<<<(unsigned)grid, 32, slice, st>>>(w, slice);
    MP_CUDA(cudaGetLastError());
    return MP_OK;
  }
  // + preplaced entries never exceed num_edges: the placed set holds <= E tensors
  // few problems (latency): the widest CTA, short chunks; many (throughput): the
  // narrowest CTA that holds the placed set, several problems per SM
  if (a.num_problems <= ctx->num_sms) return launch_place_t<512>(a, ctx, st);
  if (a.num_edges <= 128 * kChMax) return launch_place_t<128>(a, ctx, st);
  if (a.num_edges <= 256 * kChMax) return launch_place_t<256>(a, ctx, st);
  return launch_place_t<512>(a, ctx, st);
}

mp_status launch_place(const PlaceArgs& in, mp_ctx* ctx, cudaStream_t st) {
  if (in.num_problems <= 0 || in.num_edges == 0) return MP_OK;
  const int E = in.num_edges;
  // placed sets past shared memory (MP_PLACE_BIG forces it: tests)
  const bool big = E > kPlaceMaxEntries || std::getenv("MP_PLACE_BIG");
  int cap = 0;
  const size_t stride = big ? place_big_stride(E, &cap) : 0;
  // problems per launch: one per SM for the global-memory variant; otherwise as many as
  // keep the pyramid's sort buffers (24 bytes per edge and problem) under ~1.5 GB
  const int64_t group =
      big ? std::min<int64_t>(in.num_problems, ctx->num_sms)
          : std::min<int64_t>(in.num_problems, std::max<int64_t>(1, (int64_t(1) << 26) / E));
  const size_t slices = PyrSort::al(stride * (size_t)group);
  PyrSort ps;
  size_t sort_bytes = 0;
  if (in.pyramid) MP_TRY(ps.size(E, group, &sort_bytes, st));
  if (slices + sort_bytes > 0) MP_TRY(ctx->scratch[7].reserve(slices + sort_bytes));
  char* base = static_cast<char*>(ctx->scratch[7].ptr);
  if (in.pyramid) {
    ps.carve(base + slices);
    MP_TRY(ps.statics(in.id_rank, in.size, st));
  }
  for (int64_t g0 = 0; g0 < in.num_problems; g0 += group) {
    const int64_t nb = std::min<int64_t>(group, in.num_problems - g0);
    PlaceArgs a = in;
    a.num_problems = nb;
    a.lo = in.lo + g0 * E;
    a.hi = in.hi + g0 * E;
    a.addr = in.addr + g0 * E;
    a.has_addr = in.has_addr + g0 * E;
    if (in.peak_mem) a.peak_mem = in.peak_mem + g0;
    if (in.pyramid_base) a.pyramid_base = in.pyramid_base + g0;
    if (in.pyramid) {
      MP_TRY(ps.problems(a.lo, a.hi, nb, st));
      a.pyr_order = ps.porder;
    }
    MP_TRY(launch_group(a, ctx, st, big ? base : nullptr, stride, cap));
  }
  return MP_OK;
}

}  // namespace mpb
