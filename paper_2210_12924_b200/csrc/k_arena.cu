// K6 - the arena baseline run_baseline (placement.cpp:150-180), batched over
// candidate orders: the free-list allocator (placement.cpp:69-148) replayed
// over each order, reporting the allocator high-water mark (mr_peak), the live
// bytes when it was set (rs_at_peak) and their fragmentation (placement.cpp:64-67).
//
// One warp per candidate, its state in shared memory:
//   pos[n]            1-based position of each node (order validity, lifetimes)
//   fstart[n+3]       frees bucketed by timestep (hi + 1), stable in edge order,
//   flist[E]          as placement.cpp:155-158 builds them
//   blk[E]            (kBlk) the block index of each allocated edge, kept current
//                     through every shift, so Arena::release finds its block in O(1)
//                     instead of a ballot search; used when its 2E bytes do not cost
//                     a round of resident candidates (launch_arena_t)
//   blocks[cap]       the arena: (size, edge or -1 when free), address-sorted and
//                     contiguous, so addresses are implicit and top() is a sum
// The block list gets kArenaCap entries first (the live-block count is far
// below its 2E + 2 bound on real graphs); a candidate that would overflow it is
// marked and replayed again by a second launch with the full bound. pos and
// the block list share storage (pos is dead once the frees are bucketed).
// Each allocate / release is warp-cooperative over the block list: a ballot
// finds the first fit (or an arg-min the best fit) or the released edge, and
// splits / coalescing shift the list 32 entries per step. The replay itself is
// sequential in time, as the reference's is; the GPU's parallelism is the
// candidates (thousands of orders at once) and the 32 lanes per operation.
#include <cuda_runtime.h>

#include <climits>
#include <cstdint>
#include <cstdlib>

#include "mp_internal.h"

namespace mpb {
namespace {

constexpr int kArenaWarps = 1;  // candidates per CTA (shared memory bound)
constexpr uint8_t kOverflow = 2;  // valid[] marker: replay again with the full block list

// IT: the index type of pos / fstart / flist / block edges - 16-bit when n and E
// are below 65535 (half the state, twice the candidates per SM), else 32-bit.
struct ArenaLayout {
  int n, E, cap, ib, sb, bk;  // ib = sizeof(IT), sb = sizeof(ST) (block sizes), bk = kBlk
  __host__ __device__ size_t fstart_off() const { return 0; }
  __host__ __device__ size_t flist_off() const {
    return align(fstart_off() + ib * ((size_t)n + 3));
  }
  __host__ __device__ size_t blk_off() const { return align(flist_off() + ib * (size_t)E); }
  // pos [n] and the block list (size [cap], edge [cap]) share this region
  __host__ __device__ size_t pos_off() const { return align(blk_off() + bk * ib * (size_t)E); }
  __host__ __device__ size_t bsize_off() const { return pos_off(); }
  __host__ __device__ size_t bedge_off() const {
    return align(bsize_off() + sb * (size_t)cap4());
  }
  __host__ __device__ size_t cap4() const { return ((size_t)cap + 3) & ~size_t(3); }
  __host__ __device__ size_t bytes() const {
    const size_t blocks = align(bedge_off() + ib * cap4());
    const size_t p = align(pos_off() + ib * (size_t)n);
    return blocks > p ? blocks : p;
  }
  __host__ __device__ static size_t align(size_t x) { return (x + 15) & ~size_t(15); }
};

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// pos[v] = k + 1 unless already set (returns the previous value: nonzero = a repeat)
__device__ __forceinline__ int set_pos(int* p, int v, int val) { return atomicExch(p + v, val); }
__device__ __forceinline__ int set_pos(uint16_t* p, int v, int val) {
  const uintptr_t at = reinterpret_cast<uintptr_t>(p + v);
  const int sh = (int)(at & 2) * 8;
  const unsigned old =
      atomicOr(reinterpret_cast<unsigned*>(at & ~uintptr_t(3)), (unsigned)val << sh);
  return (int)((old >> sh) & 0xffffu);
}
__device__ __forceinline__ void count1(int* p, int t) { atomicAdd(p + t, 1); }
__device__ __forceinline__ void count1(uint16_t* p, int t) {
  const uintptr_t at = reinterpret_cast<uintptr_t>(p + t);
  atomicAdd(reinterpret_cast<unsigned*>(at & ~uintptr_t(3)), 1u << ((at & 2) * 8));
}

// ST: the block-size type - 32-bit sizes in units of the graph's gcd when the
// scaled total fits (mp_graph::narrow), which shrinks the block list by a third
// and raises the resident warps per SM; 64-bit byte sizes otherwise.
template <typename ST>
__device__ __forceinline__ ST size_of(const ArenaArgs& a, int e) {
  if constexpr (sizeof(ST) == 4) return __ldg(a.edge_size32 + e);
  else return __ldg(a.edge_size + e);
}

// Fit mask of blocks [i, i + 4) (bit k: block i + k is free, below nb, and holds
// s), for 16-bit edges: i is a multiple of 4, so the loads are aligned (16-byte
// size loads, one 8-byte edge load); entries at or past nb are masked (the list
// storage is padded to 4).
__device__ __forceinline__ unsigned fit4(const uint32_t* bsz, const uint16_t* bed, int i, int nb,
                                         uint32_t s) {
  const uint4 z = *reinterpret_cast<const uint4*>(bsz + i);
  const uint2 e = *reinterpret_cast<const uint2*>(bed + i);
  unsigned f = 0;
  f |= ((e.x & 0xffffu) == 0xffffu && z.x >= s) ? 1u : 0u;
  f |= ((e.x >> 16) == 0xffffu && z.y >= s) ? 2u : 0u;
  f |= ((e.y & 0xffffu) == 0xffffu && z.z >= s) ? 4u : 0u;
  f |= ((e.y >> 16) == 0xffffu && z.w >= s) ? 8u : 0u;
  const int left = nb - i;
  return left >= 4 ? f : f & ((1u << left) - 1u);
}
__device__ __forceinline__ unsigned fit4(const unsigned long long*, const int*, int, int,
                                         unsigned long long) {
  return 0;  // 64-bit sizes / 32-bit edges use the scalar scan
}
__device__ __forceinline__ unsigned fit4(const unsigned long long* bsz, const uint16_t* bed,
                                         int i, int nb, unsigned long long s) {
  const ulonglong2 z0 = *reinterpret_cast<const ulonglong2*>(bsz + i);
  const ulonglong2 z1 = *reinterpret_cast<const ulonglong2*>(bsz + i + 2);
  const uint2 e = *reinterpret_cast<const uint2*>(bed + i);
  unsigned f = 0;
  f |= ((e.x & 0xffffu) == 0xffffu && z0.x >= s) ? 1u : 0u;
  f |= ((e.x >> 16) == 0xffffu && z0.y >= s) ? 2u : 0u;
  f |= ((e.y & 0xffffu) == 0xffffu && z1.x >= s) ? 4u : 0u;
  f |= ((e.y >> 16) == 0xffffu && z1.y >= s) ? 8u : 0u;
  const int left = nb - i;
  return left >= 4 ? f : f & ((1u << left) - 1u);
}
__device__ __forceinline__ unsigned fit4(const uint32_t*, const int*, int, int, uint32_t) {
  return 0;
}

template <typename IT, typename ST, bool kBlk>
__global__ void __launch_bounds__(32 * kArenaWarps)
    arena_kernel(ArenaArgs a) {
  constexpr bool kVec4 = sizeof(IT) == 2;  // 16-bit edges; 32- or 64-bit sizes
  extern __shared__ __align__(16) char smem[];
  const int n = a.n, E = a.E;
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  const ArenaLayout Lo{n, E, a.cap, (int)sizeof(IT), (int)sizeof(ST), kBlk ? 1 : 0};
  constexpr IT kFree = (IT)-1;  // block edge of a free block
  constexpr IT kTomb = (IT)-2;  // an erased entry (edge ids are < E < kTomb)
#ifndef MP_TOMB_MAX
#define MP_TOMB_MAX 96
#endif
  constexpr int kTombMax = MP_TOMB_MAX;  // tombstones tolerated before a compaction
  char* base = smem + (size_t)wid * Lo.bytes();
  IT* pos = reinterpret_cast<IT*>(base + Lo.pos_off());
  IT* fstart = reinterpret_cast<IT*>(base + Lo.fstart_off());
  IT* flist = reinterpret_cast<IT*>(base + Lo.flist_off());
  IT* blk = reinterpret_cast<IT*>(base + Lo.blk_off());
  ST* bsz = reinterpret_cast<ST*>(base + Lo.bsize_off());
  IT* bed = reinterpret_cast<IT*>(base + Lo.bedge_off());

  for (int64_t c = (int64_t)blockIdx.x * kArenaWarps + wid; c < a.num_orders;
       c += (int64_t)gridDim.x * kArenaWarps) {
    if (a.retry && a.valid[c] != kOverflow) continue;  // uniform per warp
    const int32_t* order = a.orders + c * n;
    // ---- positions: a permutation of [0, n) (duplicates via the returned word)
    for (int v = lane; v < n; v += 32) pos[v] = 0;
    __syncwarp();
    bool bad = false;
    for (int k = lane; k < n; k += 32) {
      const int v = order[k];
      if ((unsigned)v >= (unsigned)n) bad = true;
      else bad |= set_pos(pos, v, k + 1) != 0;
    }
    __syncwarp();
    // ---- lifetimes hi[e] (schedule.cpp:33-50) and validity (graph.cpp:239-254);
    //      count the frees per timestep hi + 1 (placement.cpp:155-158)
    for (int t = lane; t < n + 3; t += 32) fstart[t] = 0;
    __syncwarp();
    for (int e = lane; e < E; e += 32) {
      const int lo = bad ? 0 : pos[a.edge_src[e]];
      int hi = lo;
      const int64_t s0 = a.sink_off[e], s1 = a.sink_off[e + 1];
      for (int64_t q = s0; q < s1; ++q) {
        const int ps = bad ? 0 : pos[a.sinks[q]];
        bad |= ps <= lo;
        hi = ps > hi ? ps : hi;
      }
      if (s1 == s0) hi = n;
      if (!bad && a.edge_size[e] > 0) count1(fstart, hi + 2);
    }
    bad = __any_sync(0xffffffffu, bad);
    if (bad) {
      if (lane == 0) {
        a.mr_peak[c] = 0;
        a.rs_at_peak[c] = 0;
        a.frag[c] = 0.0;
        a.valid[c] = 0;
      }
      __syncwarp();
      continue;
    }
    __syncwarp();
    // exclusive scan: fstart[t + 1] = first free at timestep t (t = 0 .. n + 1)
    {
      int carry = 0;
      for (int t0 = 0; t0 < n + 3; t0 += 32) {
        const int t = t0 + lane;
        int v = t < n + 3 ? fstart[t] : 0;
        int incl = v;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const int o = __shfl_up_sync(0xffffffffu, incl, d);
          if (lane >= d) incl += o;
        }
        __syncwarp();
        if (t < n + 3) fstart[t] = carry + incl - v;
        carry += __shfl_sync(0xffffffffu, incl, 31);
      }
    }
    __syncwarp();
    // stable fill in edge order: within a 32-edge chunk, rank lanes with the same t
    for (int e0 = 0; e0 < E; e0 += 32) {
      const int e = e0 + lane;
      int t = -1;
      if (e < E && a.edge_size[e] > 0) {
        const int32_t* sk = a.sinks + a.sink_off[e];
        const int64_t ns = a.sink_off[e + 1] - a.sink_off[e];
        int hi = ns == 0 ? n : pos[a.edge_src[e]];
        for (int64_t q = 0; q < ns; ++q) hi = pos[sk[q]] > hi ? pos[sk[q]] : hi;
        t = hi + 1;
      }
      const unsigned peers = __match_any_sync(0xffffffffu, t);
      const int rank = __popc(peers & lanemask_lt());
      int at = 0;
      if (t >= 0) at = fstart[t + 1] + rank;
      __syncwarp();
      if (t >= 0) {
        flist[at] = e;
        if (rank == 0) fstart[t + 1] += __popc(peers);
      }
      __syncwarp();
    }
    // fstart[t + 1] now points past bucket t; bucket t = [fstart[t], fstart[t + 1])
    // ---- replay (placement.cpp:160-177) ------------------------------------------
    // Erased entries become tombstones (edge kTomb, size 0) instead of shifting the
    // list: they never fit, never match an edge, and are skipped when looking for a
    // block's neighbours, so the live entries are always the reference's list in
    // order. A split reuses the nearest tombstone after it (shifting only up to
    // there); a compaction past kTombMax (96) tombstones (or at the capacity) removes
    // them, and trailing ones are trimmed at once (bed[nb - 1] is always live).
    int nb = 0, ntomb = 0;
    bool overflow = false;  // warp-uniform
    unsigned long long top = 0, live = 0, mr = 0, rs = 0;
    auto next_live = [&](int b) -> int {
      for (int i0 = b + 1; i0 < nb; i0 += 32) {
        const int i = i0 + lane;
        const unsigned m = __ballot_sync(0xffffffffu, i < nb && bed[i] != kTomb);
        if (m) return i0 + __ffs(m) - 1;
      }
      return -1;
    };
    auto prev_live = [&](int b) -> int {
      for (int i1 = b - 1; i1 >= 0; i1 -= 32) {
        const int i = i1 - lane;
        const unsigned m = __ballot_sync(0xffffffffu, i >= 0 && bed[i] != kTomb);
        if (m) return i1 - (__ffs(m) - 1);
      }
      return -1;
    };
    auto compact = [&]() {  // stable, in place: writes never pass the reads
      int w = 0;
      for (int i0 = 0; i0 < nb; i0 += 32) {
        const int i = i0 + lane;
        ST sz = 0;
        IT ed = kTomb;
        if (i < nb) {
          sz = bsz[i];
          ed = bed[i];
        }
        const bool keep = ed != kTomb;
        const unsigned m = __ballot_sync(0xffffffffu, keep);
        const int to = w + __popc(m & lanemask_lt());
        __syncwarp();
        if (keep) {
          bsz[to] = sz;
          bed[to] = ed;
          if (kBlk && ed != kFree) blk[ed] = (IT)to;
        }
        __syncwarp();
        w += __popc(m);
      }
      nb = w;
      ntomb = 0;
    };
    for (int t = 1; t <= n && !overflow; ++t) {
      const int f0 = fstart[t], f1 = fstart[t + 1];
      for (int q = f0; q < f1; ++q) {  // Arena::release (placement.cpp:103-111)
        const int e = flist[q];
        int b = -1;
        if constexpr (kBlk) {
          b = (int)blk[e];
          if (b < 0 || b >= nb || (int)bed[b] != e) b = -1;  // stale: never allocated
        } else if constexpr (kVec4) {  // 4 edges per lane, 128 blocks per ballot
          for (int i0 = 0; i0 < nb && b < 0; i0 += 128) {
            const int i = i0 + 4 * lane;
            unsigned f = 0;
            if (i < nb) {
              const uint2 w = *reinterpret_cast<const uint2*>(bed + i);
              f = ((int)(w.x & 0xffffu) == e ? 1u : 0u) | ((int)(w.x >> 16) == e ? 2u : 0u) |
                  ((int)(w.y & 0xffffu) == e ? 4u : 0u) | ((int)(w.y >> 16) == e ? 8u : 0u);
              if (nb - i < 4) f &= (1u << (nb - i)) - 1u;
            }
            const unsigned m = __ballot_sync(0xffffffffu, f != 0);
            if (m) {
              const int src = __ffs(m) - 1;
              b = i0 + 4 * src + __ffs(__shfl_sync(0xffffffffu, f, src)) - 1;
            }
          }
        } else {
          for (int i0 = 0; i0 < nb && b < 0; i0 += 32) {
            const unsigned m =
                __ballot_sync(0xffffffffu, i0 + lane < nb && (int)bed[i0 + lane] == e);
            if (m) b = i0 + __ffs(m) - 1;
          }
        }
        live -= size_of<ST>(a, e);
        if (b < 0) continue;
        __syncwarp();
        if (lane == 0) bed[b] = kFree;
        __syncwarp();
        // coalesce (placement.cpp:130-139): the next live block, then the previous
        // one; a merged-away entry becomes a tombstone
        const int nx = next_live(b);
        if (nx >= 0 && bed[nx] == kFree) {
          if (lane == 0) {
            bsz[b] += bsz[nx];
            bed[nx] = kTomb;
            bsz[nx] = 0;
          }
          ++ntomb;
        }
        __syncwarp();
        const int pv = prev_live(b);
        if (pv >= 0 && bed[pv] == kFree) {
          if (lane == 0) {
            bsz[pv] += bsz[b];
            bed[b] = kTomb;
            bsz[b] = 0;
          }
          ++ntomb;
        }
        __syncwarp();
        while (nb > 0 && bed[nb - 1] == kTomb) {  // keep bed[nb - 1] live
          --nb;
          --ntomb;
        }
      }
      const int v = order[t - 1];
      const int o0 = a.out_off[v], o1 = a.out_off[v + 1];
      for (int q = o0; q < o1; ++q) {  // fanout(v) in edge order
        const int e = a.out_edges[q];
        const unsigned long long s = size_of<ST>(a, e);
        if (s == 0) continue;
        if (ntomb > kTombMax || (ntomb > 0 && nb >= a.cap - 1)) compact();
        // Arena::allocate (placement.cpp:80-101): first fit, or the smallest fit
        int pick = -1;
        if (!a.best_fit && kVec4) {
          // 4 blocks per lane (one 16-byte size load + one 8-byte edge load): a
          // 128-block window per ballot; the first lane with a fit, then its first
          for (int i0 = 0; i0 < nb && pick < 0; i0 += 128) {
            const int i = i0 + 4 * lane;
            const unsigned f = i < nb ? fit4(bsz, bed, i, nb, (ST)s) : 0u;
            const unsigned m = __ballot_sync(0xffffffffu, f != 0);
            if (m) {
              const int src = __ffs(m) - 1;
              const unsigned fs = __shfl_sync(0xffffffffu, f, src);
              pick = i0 + 4 * src + __ffs(fs) - 1;
            }
          }
        } else if (!a.best_fit) {
          for (int i0 = 0; i0 < nb && pick < 0; i0 += 32) {
            const int i = i0 + lane;
            const unsigned m =
                __ballot_sync(0xffffffffu, i < nb && bed[i] == kFree && bsz[i] >= s);
            if (m) pick = i0 + __ffs(m) - 1;
          }
        } else {
          unsigned long long best = ULLONG_MAX;
          int bi = INT_MAX;
          for (int i0 = 0; i0 < nb; i0 += 32) {
            const int i = i0 + lane;
            if (i < nb && bed[i] == kFree && bsz[i] >= s && bsz[i] < best) {
              best = bsz[i];
              bi = i;
            }
          }
#pragma unroll
          for (int d = 16; d > 0; d >>= 1) {
            const unsigned long long b2 = __shfl_xor_sync(0xffffffffu, best, d);
            const int i2 = __shfl_xor_sync(0xffffffffu, bi, d);
            if (b2 < best || (b2 == best && i2 < bi)) {
              best = b2;
              bi = i2;
            }
          }
          pick = bi == INT_MAX ? -1 : bi;
        }
        __syncwarp();
        if (pick < 0) {  // grow (placement.cpp:117-128)
          if (nb > 0 && bed[nb - 1] == kFree) {
            const unsigned long long old = bsz[nb - 1];
            __syncwarp();
            if (lane == 0) {
              bsz[nb - 1] = (ST)s;
              bed[nb - 1] = e;
              if (kBlk) blk[e] = (IT)(nb - 1);
            }
            top = top - old + s;
          } else {
            if (nb == a.cap) {
              overflow = true;
              break;
            }
            if (lane == 0) {
              bsz[nb] = (ST)s;
              bed[nb] = e;
              if (kBlk) blk[e] = (IT)nb;
            }
            ++nb;
            top += s;
          }
        } else {
          const unsigned long long bsize = bsz[pick];
          __syncwarp();
          if (bsize > s) {  // split: the rest stays free right after pick
            int tpos = -1;  // the first tombstone after pick: the shift stops there
            for (int i0 = pick + 1; ntomb > 0 && i0 < nb && tpos < 0; i0 += 32) {
              const unsigned m =
                  __ballot_sync(0xffffffffu, i0 + lane < nb && bed[i0 + lane] == kTomb);
              if (m) tpos = i0 + __ffs(m) - 1;
            }
            if (tpos < 0 && nb == a.cap) {  // (compacted above: no tombstone to reuse)
              overflow = true;
              break;
            }
            const int end = tpos >= 0 ? tpos : nb;  // shift [pick + 1, end) right by one
            for (int i0 = ((end - 1 - (pick + 1)) / 32) * 32 + pick + 1;
                 end > pick + 1 && i0 >= pick + 1; i0 -= 32) {
              const int i = i0 + lane;
              ST sz = 0;
              IT ed = 0;
              if (i < end) {
                sz = bsz[i];
                ed = bed[i];
              }
              __syncwarp();
              if (i < end) {
                bsz[i + 1] = sz;
                bed[i + 1] = ed;
                if (kBlk && ed != kFree) blk[ed] = (IT)(i + 1);
              }
              __syncwarp();
            }
            if (lane == 0) {
              bsz[pick + 1] = (ST)(bsize - s);
              bed[pick + 1] = kFree;
            }
            if (tpos >= 0) --ntomb;
            else ++nb;
          }
          if (lane == 0) {
            bsz[pick] = (ST)s;
            bed[pick] = e;
            if (kBlk) blk[e] = (IT)pick;
          }
        }
        __syncwarp();
        live += s;
        if (top > mr) {
          mr = top;
          rs = live;
        }
      }
    }
    mr *= a.scale;  // back to bytes (scale = 1 for 64-bit sizes)
    rs *= a.scale;
    if (lane == 0) {
      a.mr_peak[c] = overflow ? 0 : mr;
      a.rs_at_peak[c] = overflow ? 0 : rs;
      a.frag[c] = (overflow || mr == 0) ? 0.0 : (double)(mr - rs) / (double)mr;  // :64-67
      a.valid[c] = overflow ? kOverflow : 1;
    }
    __syncwarp();
  }
}

}  // namespace

static bool arena_narrow(int n, int E) { return n < 65535 && 2 * E + 2 < 65535; }

size_t arena_smem_bytes(int n, int E, int cap, int sb, int bk) {
  const bool narrow = arena_narrow(n, E) && !std::getenv("MP_ARENA_WIDE");
  return ArenaLayout{n, E, cap, narrow ? 2 : 4, sb, bk}.bytes() * kArenaWarps;
}

template <typename IT, typename ST, bool kBlk>
int arena_per_sm(const ArenaArgs& in, size_t* smem) {
  *smem = arena_smem_bytes(in.n, in.E, in.cap, (int)sizeof(ST), kBlk ? 1 : 0);
  auto kern = arena_kernel<IT, ST, kBlk>;
  int per_sm = 0;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)*smem) !=
          cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * kArenaWarps, *smem) !=
          cudaSuccess) {
    (void)cudaGetLastError();  // too big for shared memory: not an error, just not usable
    return 0;
  }
  return per_sm;
}

template <typename IT, typename ST>
mp_status launch_arena_t(const ArenaArgs& in, const mp_ctx* ctx, cudaStream_t st) {
  // The edge -> block index (kBlk) removes the release search (~20% of the scalar
  // replay's instructions) but adds 2E bytes per candidate: use it unless the lost
  // resident candidates cost more than that, i.e. it adds more than ~20% rounds.
  size_t smem0 = 0, smem1 = 0;
  const int occ0 = arena_per_sm<IT, ST, false>(in, &smem0);
  const int occ1 = arena_per_sm<IT, ST, true>(in, &smem1);
  const int64_t per_sm_work =
      (in.num_orders + (int64_t)ctx->num_sms * kArenaWarps - 1) / ((int64_t)ctx->num_sms * kArenaWarps);
  auto rounds = [&](int occ) { return occ > 0 ? (per_sm_work + occ - 1) / occ : INT64_MAX; };
  // with 16-bit edges the search itself is 4 blocks per lane, so the index only
  // pays when it costs no round (measured with tombstones: C2 +13%, C3 +12% with
  // it; C4, one round more, 15% slower)
  bool blk = occ1 > 0 && (sizeof(IT) == 2 ? rounds(occ1) <= rounds(occ0)
                                          : 5 * rounds(occ1) <= 6 * rounds(occ0));
  if (const char* e = std::getenv("MP_ARENA_BLK")) blk = std::atoi(e) != 0 && occ1 > 0;
  const int per_sm = blk ? occ1 : occ0;
  if (per_sm <= 0) {
    set_error("Capacity: run_baseline state exceeds shared memory");
    return MP_E_CAPACITY;
  }
  int64_t grid = (int64_t)ctx->num_sms * (per_sm > 0 ? per_sm : 1);
  const int64_t need = (in.num_orders + kArenaWarps - 1) / kArenaWarps;
  if (grid > need) grid = need;
  if (blk)
    arena_kernel<IT, ST, true><<<(unsigned)grid, 32 * kArenaWarps, smem1, st>>>(in);
  else
    arena_kernel<IT, ST, false><<<(unsigned)grid, 32 * kArenaWarps, smem0, st>>>(in);
  MP_CUDA(cudaGetLastError());
  return MP_OK;
}

mp_status launch_arena_pass(const ArenaArgs& in, const mp_ctx* ctx, cudaStream_t st) {
  const bool s32 = in.edge_size32 != nullptr;
  if (arena_narrow(in.n, in.E) && !std::getenv("MP_ARENA_WIDE"))
    return s32 ? launch_arena_t<uint16_t, uint32_t>(in, ctx, st)
               : launch_arena_t<uint16_t, unsigned long long>(in, ctx, st);
  return s32 ? launch_arena_t<int, uint32_t>(in, ctx, st)
             : launch_arena_t<int, unsigned long long>(in, ctx, st);
}

mp_status launch_arena(const ArenaArgs& in, const mp_ctx* ctx, cudaStream_t st) {
  if (in.num_orders <= 0) return MP_OK;
  const int full = 2 * in.E + 2;  // used + free blocks never exceed this
  ArenaArgs a = in;
  int first = kArenaCap;
  if (const char* e = std::getenv("MP_ARENA_CAP")) first = std::atoi(e) > 0 ? std::atoi(e) : first;
  a.cap = full < first ? full : first;  // MP_ARENA_CAP: tests of the overflow path
  a.retry = 0;
  MP_TRY(launch_arena_pass(a, ctx, st));
  if (a.cap < full) {  // candidates whose block list overflowed, with the full bound
    a.cap = full;
    a.retry = 1;
    MP_TRY(launch_arena_pass(a, ctx, st));
  }
  return MP_OK;
}

}  // namespace mpb
