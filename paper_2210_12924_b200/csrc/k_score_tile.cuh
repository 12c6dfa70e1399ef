// Tile scorer for graphs whose per-candidate state does not fit on chip
// (the 100k-tensor C5 graph: n = 133,336), included by k_score.cu inside
// namespace mpb::{anon}.
//
// One CTA scores one candidate at a time (persistent grid, one CTA per SM),
// walking the order in position tiles of T*PT; thread t owns the PT
// consecutive positions [tile + t*PT, tile + t*PT + PT) in registers:
//   (a) pos[v] = stamp|k for its positions by atomicExch on a per-CTA word
//       array in global memory (L2-resident: one n-word slice per SM). The
//       old word must be stale: a fresh one means v occurred earlier in this
//       order. n in-range ids without a repeat are a permutation.
//   (b) barrier (the tile's words are visible to the whole CTA), then per
//       position the node record (alloc - static free, static free, first two
//       reduced producers) from the shared read-only table, and the producers'
//       words: a producer is "strictly earlier" iff its word is fresh AND its
//       position < k. Words of later tiles are still stale, so checking while
//       walking the order is exact. The same fact decides order-dependent
//       frees: node v at k frees dynamic edge d iff every other candidate
//       last consumer of d already has a fresh word with position < k.
//   (c) block scan of the x's with the carry of earlier tiles: RS(k) = S(k-1)
//       + x_k + f_k exactly in VT (modular sums of a value < 2^32 / 2^62), and
//       the first maximum, kept across tiles (strict >).
// Afterwards the 3rd+ reduced producer pairs are checked from the finished words.
// Random traffic per candidate: n atomics + n record reads + ~1 word read per
// reduced producer, all in L2 (the word slices total grid*n*4 bytes, e.g. 79 MB
// at C5); only the order row comes from HBM. Compare the node-space kernel
// (score_kernel, kSmem = false) whose XF scatter doubled the working set.
// Measured at C5 (1,024 candidates, one B200): 2.77 ms vs 2.62 ms for the
// node-space kernel, with 1.7 GB instead of 12.3 GB of DRAM traffic. Both are
// bound by the L1TEX pipe's rate for warp-wide random accesses (~32 wavefronts
// per instruction); this kernel makes ~5.5 random accesses per position (the
// atomic, the record, producer words, and C5's 33k order-dependent frees)
// against ~3 there, so it is opt-in (MP_SCORE_MODE=tile). DESIGN.md §3.
// The order row is read with an evict-first hint and the word slices are
// launched under an L2 persisting access-policy window, so the streamed
// orders do not push the words out of L2 between candidates.

constexpr int kTileT = 512;

template <typename VT>
struct TileScratch {
  VT wsum[32];
  VT wbest[32];
  int widx[32];
  VT carry;      // S(tile start - 1)
  VT best;       // running first maximum over earlier tiles
  int best_i;
};

template <typename VT>
__device__ __forceinline__ void tile_rec(const ScoreTables& G, int v, VT& x, VT& f, uint32_t& z,
                                         uint32_t& w) {
  if constexpr (sizeof(VT) == 4) {
    const uint4 r = __ldg(G.tile_rec32 + v);
    x = r.x;
    f = r.y;
    z = r.z;
    w = r.w;
  } else {
    x = (VT)__ldg(G.node_x + v);
    f = (VT)__ldg(G.node_f + v);
    const uint2 zw = __ldg(G.tile_zw + v);
    z = zw.x;
    w = zw.y;
  }
}

// fresh word with a position < k  <=>  (word - tagw) < k as unsigned (stale words wrap high)
__device__ __forceinline__ bool earlier(const uint32_t* words, uint32_t node, uint32_t tagw,
                                        uint32_t k) {
  return node == kNoNode || (__ldcg(words + node) - tagw) < k;
}

template <typename VT, int PT>
__global__ void __launch_bounds__(kTileT, 1)
    score_tile_kernel(ScoreTables G, const int32_t* __restrict__ orders, int64_t C,
                      uint64_t* __restrict__ peak_out, int32_t* __restrict__ step_out,
                      uint8_t* __restrict__ valid_out, uint64_t* __restrict__ bytes_out,
                      unsigned long long* __restrict__ best_key, int64_t index_base,
                      uint32_t* __restrict__ words_all, int slices) {
  __shared__ TileScratch<VT> bs;
  const int n = G.n;
  const int tid = threadIdx.x;
  const int lane = tid & (kWarp - 1);
  const int warp = tid >> 5;
  constexpr int kWarps = kTileT / kWarp;
  constexpr int TS = kTileT * PT;
  uint32_t* words = words_all + (size_t)blockIdx.x * n;
  uint32_t* stamp_slot = words_all + (size_t)slices * n + blockIdx.x;
  uint32_t stamp = *stamp_slot;  // persists across launches (0 = freshly zeroed)

  for (int64_t c = blockIdx.x; c < C; c += gridDim.x) {
    if (++stamp > 0xffu) {  // 8-bit stamps: clear the slice every 255 candidates
      for (int i = tid; i < n; i += kTileT) words[i] = 0;
      stamp = 1;
      __syncthreads();
    }
    const uint32_t tagw = stamp << 24;
    bool bad = false;
    if (tid == 0) {
      bs.carry = 0;
      bs.best = 0;
      bs.best_i = INT_MAX;
    }
    const int32_t* row = orders + c * n;
    // (a) for one tile: ids (evict-first loads) and their words by atomicExch.
    // Tile t+1 is issued before tile t is checked, so its atomics overlap the
    // checks; a check only needs every EARLIER position written, and a later
    // one reads either stale or fresh-with-a-larger-position: both "not earlier".
    int ov[PT];
    uint32_t old[PT];
    auto place = [&](int t0, int* o, uint32_t* od) {
      const int k0 = t0 + tid * PT;
#pragma unroll
      for (int j = 0; j < PT; ++j) o[j] = k0 + j < n ? __ldcs(row + k0 + j) : 0;
#pragma unroll
      for (int j = 0; j < PT; ++j) {
        od[j] = 0;
        if (k0 + j < n) {
          if ((unsigned)o[j] >= (unsigned)n) {
            bad = true;
            o[j] = 0;
          } else {
            od[j] = atomicExch(words + o[j], tagw | (uint32_t)(k0 + j));
          }
        }
      }
    };
    place(0, ov, old);
    for (int t0 = 0; t0 < n; t0 += TS) {
      int ovn[PT] = {};
      uint32_t oldn[PT] = {};
      if (t0 + TS < n) place(t0 + TS, ovn, oldn);
#pragma unroll
      for (int j = 0; j < PT; ++j) bad |= (old[j] >> 24) == stamp;  // v placed twice
      __syncthreads();  // every word of tiles <= t0 is written and visible
      const int k0 = t0 + tid * PT;
      // (b) node records, producers' words, order-dependent frees
      VT x[PT], f[PT];
      uint32_t z[PT], w[PT];
#pragma unroll
      for (int j = 0; j < PT; ++j) {
        x[j] = 0;
        f[j] = 0;
        z[j] = kNoNode;
        w[j] = kNoNode;
        if (k0 + j < n) tile_rec<VT>(G, ov[j], x[j], f[j], z[j], w[j]);
      }
#pragma unroll
      for (int j = 0; j < PT; ++j) {
        const uint32_t k = (uint32_t)(k0 + j);
        bad |= !earlier(words, z[j] & kNoNode, tagw, k) || !earlier(words, w[j], tagw, k);
      }
      if (G.ndyn > 0) {
        // node v at k frees dynamic edge d iff every other candidate last
        // consumer of d is already placed earlier (exactly one does, if valid)
        int m0[PT];
#pragma unroll
        for (int j = 0; j < PT; ++j) m0[j] = (z[j] >> 24) ? __ldg(G.tile_moff + ov[j]) : -1;
#pragma unroll
        for (int j = 0; j < PT; ++j) {
          const uint32_t cnt = z[j] >> 24;
          if (cnt == 0) continue;
          const uint32_t k = (uint32_t)(k0 + j);
          const int m1 = cnt < 255 ? m0[j] + (int)cnt : __ldg(G.node_dyn_off + ov[j] + 1);
          for (int m = m0[j]; m < m1; ++m) {
            const int4 o = __ldg(G.tile_mother + m);
            const int d = __ldg(G.tile_medge + m);
            bool last = earlier(words, (uint32_t)o.x, tagw, k) &&
                        earlier(words, (uint32_t)o.y, tagw, k) &&
                        earlier(words, (uint32_t)o.z, tagw, k);
            if (o.w == kMoreSinks) {  // > 4 other candidates: walk the edge's sink list
              const int s1 = __ldg(G.dyn_off + d + 1);
              for (int s = __ldg(G.dyn_off + d); s < s1; ++s) {
                const int x2 = __ldg(G.dyn_sinks + s);
                if (x2 != ov[j]) last &= earlier(words, (uint32_t)x2, tagw, k);
              }
            } else {
              last &= earlier(words, (uint32_t)o.w, tagw, k);
            }
            if (last) {  // RS(k) still holds the edge; it is gone from k + 1 on
              const VT sz = (VT)__ldg(G.dyn_size + d);
              x[j] -= sz;
              f[j] += sz;
            }
          }
        }
      }
      // (c) block scan with the carry of earlier tiles
      VT tot = 0;
#pragma unroll
      for (int j = 0; j < PT; ++j) tot += x[j];
      const VT incl = warp_incl_scan(tot, lane);
      if (lane == kWarp - 1) bs.wsum[warp] = incl;
      __syncthreads();
      VT run = bs.carry + warp_sum(lane < warp ? bs.wsum[lane] : (VT)0) + incl - tot;
      VT best = 0;
      int best_i = INT_MAX;
#pragma unroll
      for (int j = 0; j < PT; ++j) {
        const int k = k0 + j;
        run += x[j];
        const VT rs = run + f[j];
        if (k < n) {
          if (bytes_out) bytes_out[c * n + k] = (uint64_t)rs * G.scale;
          if (best_i == INT_MAX || rs > best) {
            best = rs;
            best_i = k;
          }
        }
      }
      warp_argmax(best, best_i);
      if (lane == 0) {
        bs.wbest[warp] = best;
        bs.widx[warp] = best_i;
      }
      __syncthreads();
      if (warp == 0) {
        VT b = lane < kWarps ? bs.wbest[lane] : (VT)0;
        int bi = lane < kWarps ? bs.widx[lane] : INT_MAX;
        VT tsum = lane < kWarps ? bs.wsum[lane] : (VT)0;
        warp_argmax(b, bi);
        tsum = warp_sum(tsum);
        if (lane == 0) {
          if (bi != INT_MAX && (bs.best_i == INT_MAX || b > bs.best)) {
            bs.best = b;
            bs.best_i = bi;
          }
          bs.carry += tsum;
        }
      }
      // bs.wsum / wbest are rewritten after the next tile's first barrier, which
      // warp 0 reaches only after this update.
#pragma unroll
      for (int j = 0; j < PT; ++j) {
        ov[j] = ovn[j];
        old[j] = oldn[j];
      }
    }
    // remaining reduced producer pairs, from the finished words
    for (int i = tid; i < G.nextra3w; i += kTileT) {
      const uint32_t a = __ldcg(words + __ldg(G.extra3_u + i));
      const uint32_t b = __ldcg(words + __ldg(G.extra3_w + i));
      bad |= a >= b;
    }
    bad = __syncthreads_or(bad);
    if (tid == 0) {
      const bool empty = n == 0;
      const uint64_t pk = (bad || empty) ? 0 : (uint64_t)bs.best * G.scale;
      peak_out[c] = pk;
      step_out[c] = (bad || empty) ? 0 : bs.best_i + 1;
      valid_out[c] = bad ? 0 : 1;
      if (best_key && !bad) {
        const uint64_t gi = (uint64_t)(c + index_base);
        const unsigned long long key =
            (pk < (1ull << 43) && gi < (1ull << 20)) ? ((pk << 20) | gi) : kKeyOverflow;
        atomicMin(best_key, key);
      }
    }
    __syncthreads();  // bs.carry/best reset by the next candidate
  }
  if (tid == 0) *stamp_slot = stamp;
}
