// Register-slot variant of the fused scorer (n up to ~8k nodes), included by
// k_score.cu inside namespace mpb::{anon}. See k_score.cu for the math.
//
// Slot j of a thread covers order position AND node k = (warp*J + j)*32 + lane,
// k < TJ = T*J: warp-contiguous, so global loads coalesce and every per-slot
// shared-memory address is the thread's base plus an immediate. Per slot the
// thread keeps in registers the node's static bytes (x, f) and the pos
// indexes of its first two reduced producers - shared by KC candidates that
// the CTA scores together (KC independent chains per barrier and per
// instruction stream), each with its own order registers and smem buffers.
//
// Padding slots (k >= n) behave as inert nodes instead of branching: they
// write pos[k] = tag|k in phase 1 (so they read back fresh), carry x = f = 0
// (so their scatter leaves the scan padding at zero) and have "no producer"
// (pos[TJ+1], never written, always 0). pos[TJ] absorbs out-of-range ids of
// invalid orders. XF[n .. T*P) is scan padding (0, 0) and XF[T*P] absorbs
// scatters of stale positions (invalid orders only).
// Permutation check: stamps only grow (until a wrap clears pos), so a word is
// fresh iff w >= tag; n writes reaching all n nodes = a permutation.

template <typename VT>
struct RegLayout {
  int n, T, P, J;
  __host__ __device__ int TJ() const { return T * J; }
  __host__ __device__ size_t pos_words() const { return ((size_t)T * J + 2 + 3) & ~size_t(3); }
  __host__ __device__ size_t pos_bytes() const { return pos_words() * 4; }
  __host__ __device__ size_t xf_bytes() const {
    return ((size_t)(T * P + 1) * sizeof(XFPair<VT>) + 15) & ~size_t(15);
  }
  __host__ __device__ size_t per_candidate() const { return pos_bytes() + xf_bytes(); }
};

// Register budgets (65536 / (kMaxT * kMinBlocks) per thread):
//   J=4: T <= 256, 64 regs (KC=1) / 85 (KC=2);  J=8: T <= 384, 85 (KC=1) / 102 (KC=2, T <= 320)
//   J=16: T <= 512, 128.  score_configure picks T within kMaxT.
template <int J, int KC>
struct RegBounds {
#ifndef MP_J8_MAXT
#define MP_J8_MAXT 384
#endif
#ifndef MP_J8_MINB
#define MP_J8_MINB 2
#endif
  static constexpr int kMaxT = J == 4 ? 256 : J == 8 ? (KC == 1 ? MP_J8_MAXT : 320) : 512;
  static constexpr int kMinBlocks = J == 4 ? (KC == 1 ? 4 : 3) : J == 8 ? (KC == 1 ? MP_J8_MINB : 2) : 1;
};

template <typename VT, int KC>
struct RegScratch {
  VT wsum[KC][32];
  VT wbest[KC][32];
  int widx[KC][32];
  uint32_t bad[2];  // per-iteration-parity bitmask of invalid candidates
};

// x as a signed 64-bit value: 32-bit scan inputs are int32 bit patterns
__device__ __forceinline__ long long sx64(uint32_t v) { return (long long)(int32_t)v; }
__device__ __forceinline__ long long sx64(unsigned long long v) { return (long long)v; }

// OT: the order element type - int32 (the reference's layout) or uint16 (the host
// call packs orders of graphs with n < 65535 to halve the PCIe bytes; values
// outside [0, n) arrive as 0xffff, still out of range).
// AT: the sum type. AT = VT, or VT = uint32 with AT = uint64 ("mid32" graphs:
// total bytes past 2^32 in gcd units, but every node's x fits int32 and f uint32
// for any order) - half the registers and shared bytes of the 64-bit variant,
// exact 64-bit sums in the one-pass scan (peak/step only; no per-step bytes).
template <typename VT, int J, int KC, typename OT = int32_t, typename AT = VT>
__global__ void __launch_bounds__(RegBounds<J, KC>::kMaxT, RegBounds<J, KC>::kMinBlocks)
    score_reg_kernel(ScoreTables G, const OT* __restrict__ orders, int64_t C,
                     uint64_t* __restrict__ peak_out, int32_t* __restrict__ step_out,
                     uint8_t* __restrict__ valid_out, uint64_t* __restrict__ bytes_out,
                     unsigned long long* __restrict__ best_key, int64_t index_base) {
  extern __shared__ __align__(16) char smem[];
  __shared__ RegScratch<AT, KC> bs;

  const int n = G.n;
  const int T = blockDim.x;
  const int tid = threadIdx.x;
  const int lane = tid & (kWarp - 1);
  const int warp = tid >> 5;
  const int nwarps = T >> 5;
  const int P = G.P;
  const int TP = T * P;
  const RegLayout<VT> L{n, T, P, J};
  const int TJ = L.TJ();

  uint32_t* pos[KC];
  XFPair<VT>* XF[KC];
#pragma unroll
  for (int k = 0; k < KC; ++k) {
    char* b = smem + k * L.per_candidate();
    pos[k] = reinterpret_cast<uint32_t*>(b);
    XF[k] = reinterpret_cast<XFPair<VT>*>(b + L.pos_bytes());
    uint4* z = reinterpret_cast<uint4*>(pos[k]);  // pos = 0: stamp 0 is never used
    for (int i = tid; i < (int)(L.pos_words() / 4); i += T) z[i] = make_uint4(0, 0, 0, 0);
    for (int i = n + tid; i <= TP; i += T) XF[k][i] = XFPair<VT>{0, 0};  // scan padding
  }
  if (tid < 2) bs.bad[tid] = 0;

  const int base = warp * J * kWarp + lane;  // slot j: k = base + 32*j
  uint32_t real = 0;                          // bit j: slot j is a real node / position
  VT rx[J], rf[J];
  int ru[J], ru2[J];  // pos indexes of the first two reduced producers (TJ+1: none)
#pragma unroll
  for (int j = 0; j < J; ++j) {
    const int v = base + kWarp * j;
    const bool in = v < n;
    real |= (in ? 1u : 0u) << j;
    int u1 = -1, u2 = -1;
    rx[j] = 0;
    rf[j] = 0;
    if (in) {
      if constexpr (sizeof(VT) == 4) {
        const uint4 rec = __ldg(G.node_rec32 + v);  // (x, f, pred1, pred2): one load
        rx[j] = rec.x;
        rf[j] = rec.y;
        u1 = (int)rec.z;
        u2 = (int)rec.w;
      } else {
        rx[j] = (VT)__ldg(G.node_x + v);
        rf[j] = (VT)__ldg(G.node_f + v);
        const int2 uu = __ldg(G.node_u2 + v);
        u1 = uu.x;
        u2 = uu.y;
      }
    }
    ru[j] = u1 >= 0 ? u1 : TJ + 1;
    ru2[j] = u2 >= 0 ? u2 : TJ + 1;
  }
  // bit j: some lane of this warp has a second producer in slot j (warp-uniform),
  // so slots without any skip the gather (most nodes have at most one)
  uint32_t has2 = 0;
#pragma unroll
  for (int j = 0; j < J; ++j) has2 |= (__any_sync(0xffffffffu, ru2[j] != TJ + 1) ? 1u : 0u) << j;

  // Candidate groups: group g covers candidates [g*KC, g*KC + KC).
  const int64_t ngroups = (C + KC - 1) / KC;
  int ov[KC][J];
  auto load_group = [&](int64_t g) {
#pragma unroll
    for (int k = 0; k < KC; ++k) {
      const int64_t c = g * KC + k;
      const OT* row = orders + c * n + base;
#pragma unroll
      for (int j = 0; j < J; ++j)
        ov[k][j] = ((real >> j & 1) && c < C) ? (int)__ldg(row + kWarp * j) : base + kWarp * j;
    }
  };
  if ((int64_t)blockIdx.x < ngroups) load_group(blockIdx.x);
  __syncthreads();

  uint32_t stamp = 0;
  int parity = 0;
  for (int64_t g = blockIdx.x; g < ngroups; g += gridDim.x, parity ^= 1) {
    if (++stamp > 0xffffu) {
      for (int k = 0; k < KC; ++k)
        for (int i = tid; i < (int)L.pos_words(); i += T) pos[k][i] = 0;
      stamp = 1;
      __syncthreads();
    }
    const uint32_t tag = stamp << 16;
    const uint32_t tagbase = tag + (uint32_t)base;
    uint32_t bad = 0;  // bit k: candidate k of the group is invalid

    // ---- phase 1: pos[order[k]] = tag | k --------------------------------------------
#pragma unroll
    for (int k = 0; k < KC; ++k)
#pragma unroll
      for (int j = 0; j < J; ++j) {
        const uint32_t v = (uint32_t)ov[k][j];
        bad |= (((real >> j) & 1u) & (v >= (uint32_t)n ? 1u : 0u)) << k;
        pos[k][min(v, (uint32_t)TJ)] = tagbase + kWarp * j;
      }
    if (g + gridDim.x < ngroups) load_group(g + gridDim.x);  // lands while this group is scored
    __syncthreads();

    // ---- phase 2a: node slots -----------------------------------------------------------
    // all loads of the slots first, then the scatters (pos and XF alias as far
    // as the compiler knows, so it would not hoist a load above a store)
#pragma unroll
    for (int k = 0; k < KC; ++k) {
      uint32_t w[J], pu[J], pu2[J];
#pragma unroll
      for (int j = 0; j < J; ++j) {
        w[j] = pos[k][base + kWarp * j];
        pu[j] = pos[k][ru[j]];
        pu2[j] = (has2 >> j & 1u) ? pos[k][ru2[j]] : 0u;
      }
#pragma unroll
      for (int j = 0; j < J; ++j) {
        // stale word (not a permutation) / a producer not strictly earlier
        bad |= ((w[j] < tag || pu[j] >= w[j] || pu2[j] >= w[j]) ? 1u : 0u) << k;
        XF[k][min((int)(w[j] & 0xffffu), TP)] = XFPair<VT>{rx[j], rf[j]};
      }
    }
    // ---- phase 2b: 3rd+ reduced producer pairs (flat) ----------------------------------
    for (int i = tid; i < G.nextra3; i += T) {
      const uint32_t e = __ldg(G.extra3_packed + i);
#pragma unroll
      for (int k = 0; k < KC; ++k)
        bad |= ((pos[k][e & 0xffffu] >= pos[k][e >> 16]) ? 1u : 0u) << k;
    }
    // ---- phase 2c: order-dependent last consumers -----------------------------------
    if (G.ndyn > 0) {
      __syncthreads();
      // edges spread over the warps (d = i*T + lane*nwarps + warp) so no warp
      // reaches the barrier late; <= 4 candidate sinks come as one 16-byte record
      for (int d = lane * nwarps + warp; d < G.ndyn; d += T) {
        uint32_t h[KC];
#pragma unroll
        for (int k = 0; k < KC; ++k) h[k] = 0;
        if (G.dyn_sink4 != nullptr) {
          const int4 sk = __ldg(G.dyn_sink4 + d);
#pragma unroll
          for (int k = 0; k < KC; ++k) {
            const uint32_t a = sk.x >= 0 ? pos[k][sk.x] : 0u, b = sk.y >= 0 ? pos[k][sk.y] : 0u;
            const uint32_t c2 = sk.z >= 0 ? pos[k][sk.z] : 0u, d2 = sk.w >= 0 ? pos[k][sk.w] : 0u;
            h[k] = max(max(a, b), max(c2, d2));
          }
        } else {
          const int s1 = __ldg(G.dyn_off + d + 1);
          for (int s = __ldg(G.dyn_off + d); s < s1; ++s) {
            const int x = __ldg(G.dyn_sinks + s);
#pragma unroll
            for (int k = 0; k < KC; ++k) h[k] = max(h[k], pos[k][x]);
          }
        }
        const VT sz = (VT)__ldg(G.dyn_size + d);
#pragma unroll
        for (int k = 0; k < KC; ++k) {
          const int q = (int)(h[k] & 0xffffu);
          if (q < n) {
            atomicAdd(&XF[k][q].f, sz);
            atomicAdd(&XF[k][q].x, (VT)0 - sz);
          }
        }
      }
    }
    // per-candidate verdicts: warp ballots, one atomicOr per warp that saw any
    {
      uint32_t wb = 0;
#pragma unroll
      for (int k = 0; k < KC; ++k) wb |= (__ballot_sync(0xffffffffu, (bad >> k) & 1u) ? 1u : 0u) << k;
      if (lane == 0 && wb) atomicOr(&bs.bad[parity], wb);
    }
    __syncthreads();
    const uint32_t badmask = bs.bad[parity];
    const int64_t c0 = g * KC;

    if constexpr (sizeof(AT) == 8) {
      if (bytes_out == nullptr || sizeof(VT) != sizeof(AT)) {  // the mid variant: never bytes
        // ---- phase 3, 64-bit values: ONE pass over the chunk [p0, p0 + P) -----------
        // x = alloc - free is exact as int64 (|x| <= total < 2^62), so chunk-relative
        // RS values are exact: each thread finds its chunk's first maximum relative to
        // the chunk start, a warp scan of the chunk sums makes it warp-relative, and
        // warp 0 combines the per-warp (sum, best, index) triples after one barrier.
        const int p0 = tid * P;
#pragma unroll
        for (int k = 0; k < KC; ++k) {
          const XFPair<VT>* mine = XF[k] + p0;
          XFPair<VT> xf = mine[0];
          long long l = sx64(xf.x);
          long long lb = l + (long long)(AT)xf.f;
          int li = 0;
          for (int i = 1; i < P; ++i) {
            xf = mine[i];
            l += sx64(xf.x);
            const long long rs = l + (long long)(AT)xf.f;
            const bool better = rs > lb;
            lb = better ? rs : lb;
            li = better ? i : li;
          }
          const long long incl = warp_incl_scan(l, lane);
          long long cand = incl - l + lb;
          int ci = p0 < n ? p0 + li : INT_MAX;  // a chunk made only of padding
          warp_argmax(cand, ci);
          if (lane == 0) {
            bs.wbest[k][warp] = (AT)cand;
            bs.widx[k][warp] = ci;
          }
          if (lane == kWarp - 1) bs.wsum[k][warp] = (AT)incl;
        }
        __syncthreads();
        if (tid == 0) bs.bad[parity ^ 1] = 0;  // next iteration's flags
        if (warp == 0) {
#pragma unroll
          for (int k = 0; k < KC; ++k) {
            const bool live = lane < nwarps;
            const long long wt = live ? (long long)bs.wsum[k][lane] : 0;
            const long long incl = warp_incl_scan(wt, lane);
            long long b = live ? incl - wt + (long long)bs.wbest[k][lane] : LLONG_MIN;
            int bi = live ? bs.widx[k][lane] : INT_MAX;
            warp_argmax(b, bi);
            const int64_t c = c0 + k;
            if (lane == 0 && c < C) {
              const bool ok = !((badmask >> k) & 1u);
              const bool empty = n == 0;
              const uint64_t pk = (!ok || empty) ? 0 : (uint64_t)b * G.scale;
              peak_out[c] = pk;
              step_out[c] = (!ok || empty) ? 0 : bi + 1;
              valid_out[c] = ok ? 1 : 0;
              if (best_key && ok) {
                const uint64_t gi = (uint64_t)(c + index_base);
                record_key(best_key, pk, gi);
              }
            }
          }
        }
        continue;
      }
    }
    // ---- phase 3: blocked two-pass scan over [tid*P, tid*P + P), P odd -------------
    VT run[KC], best[KC];
    int best_i[KC];
    const int p0 = tid * P;
    // KC == 1, J <= 8: pass 1 keeps the chunk (P <= J + 1 entries) in registers for
    // pass 2 (J = 16 would spill)
    constexpr bool kRegChunk = KC == 1 && J <= 8;
    constexpr int PM = kRegChunk ? J + 1 : 1;
    VT xr[PM], fr[PM];
#pragma unroll
    for (int k = 0; k < KC; ++k) {
      const XFPair<VT>* mine = XF[k] + p0;
      VT total = 0;
      if constexpr (kRegChunk) {
#pragma unroll
        for (int i = 0; i < PM; ++i) {
          xr[i] = 0;
          fr[i] = 0;
          if (i < P) {
            const XFPair<VT> e = mine[i];
            xr[i] = e.x;
            fr[i] = e.f;
          }
          total += xr[i];
        }
      } else {
        for (int i = 0; i < P; ++i) total += mine[i].x;
      }
      const VT incl = warp_incl_scan(total, lane);
      if (lane == kWarp - 1) bs.wsum[k][warp] = incl;
      run[k] = incl - total;
    }
    __syncthreads();
    if (tid == 0) bs.bad[parity ^ 1] = 0;  // next iteration's flags (last read a barrier ago)
#pragma unroll
    for (int k = 0; k < KC; ++k) {
      run[k] += warp_sum(lane < warp ? bs.wsum[k][lane] : (VT)0);
      const XFPair<VT>* mine = XF[k] + p0;
      if (kRegChunk && bytes_out == nullptr) {
        // from the registers of pass 1 (entries past P are (0, 0) and never win:
        // strict > keeps the first maximum)
        VT r = run[k] + xr[0];
        VT b = r + fr[0];
        int bi = 0;
#pragma unroll
        for (int i = 1; i < PM; ++i) {
          r += xr[i];
          const VT rs = r + fr[i];
          const bool better = rs > b;
          b = better ? rs : b;
          bi = better ? i : bi;
        }
        best[k] = b;
        best_i[k] = p0 < n ? p0 + bi : INT_MAX;  // a chunk made only of padding
      } else if (bytes_out == nullptr) {
        // First element initialises (best, index); strict > keeps the first
        // maximum. Padding entries are (0, 0): their RS equals S(n-1) <= RS(n-1),
        // so they never replace a real position.
        XFPair<VT> xf = mine[0];
        VT r = run[k] + xf.x;
        VT b = r + xf.f;
        int bi = 0;
        for (int i = 1; i < P; ++i) {
          xf = mine[i];
          r += xf.x;
          const VT rs = r + xf.f;
          const bool better = rs > b;
          b = better ? rs : b;
          bi = better ? i : bi;
        }
        best[k] = b;
        best_i[k] = p0 < n ? p0 + bi : INT_MAX;  // a chunk made only of padding
      } else {
        VT r = run[k], b = 0;
        int bi = INT_MAX;
        const int64_t c = c0 + k;
        const int lim = min(P, n - p0);
        for (int i = 0; i < lim; ++i) {
          const XFPair<VT> xf = mine[i];
          r += xf.x;
          const VT rs = r + xf.f;
          if (c < C) bytes_out[c * n + p0 + i] = (uint64_t)rs * G.scale;
          if (rs > b || bi == INT_MAX) {
            b = rs;
            bi = p0 + i;
          }
        }
        best[k] = b;
        best_i[k] = bi;
      }
      warp_argmax(best[k], best_i[k]);
      if (lane == 0) {
        bs.wbest[k][warp] = best[k];
        bs.widx[k][warp] = best_i[k];
      }
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
      for (int k = 0; k < KC; ++k) {
        VT b = lane < nwarps ? bs.wbest[k][lane] : (VT)0;
        int bi = lane < nwarps ? bs.widx[k][lane] : INT_MAX;
        warp_argmax(b, bi);
        const int64_t c = c0 + k;
        if (lane == 0 && c < C) {
          const bool ok = !((badmask >> k) & 1u);
          const bool empty = n == 0;
          const uint64_t pk = (!ok || empty) ? 0 : (uint64_t)b * G.scale;
          peak_out[c] = pk;
          step_out[c] = (!ok || empty) ? 0 : bi + 1;
          valid_out[c] = ok ? 1 : 0;
          if (best_key && ok) {
            const uint64_t gi = (uint64_t)(c + index_base);
            record_key(best_key, pk, gi);
          }
        }
      }
    }
  }
}

template <typename VT>
size_t reg_smem_bytes(int n, int T, int P, int J, int KC) {
  return RegLayout<VT>{n, T, P, J}.per_candidate() * KC + 16;
}
