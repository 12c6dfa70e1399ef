// Register-slot variant of the fused scorer (n up to ~8k nodes), included by
// k_score.cu inside namespace mpb::{anon}. See k_score.cu for the math.
//
// Slot j of a thread covers order position AND node k = (warp*J + j)*32 + lane:
// warp-contiguous, so global loads coalesce, node-table reads are
// conflict-free, and per-slot offsets are immediates. Only the next
// candidate's order values live in registers (ov[J]); the static node tables
// (x, f, first producer) sit in shared memory once per CTA.
//
// Absorbing slots instead of branches:
//   pos[n]    written by padding slots (k >= n) and by out-of-range ids
//             (which already flag the order); padding node slots read it
//   pos[n+1]  never written, stays 0: "no producer", always earlier
//   XF[T*P]   garbage entry for scatters of stale (invalid-order) positions;
//             XF[n .. T*P) is scan padding and stays (0, 0)
// Permutation check: stamps only grow (until a wrap clears pos), so a word
// is fresh iff w >= tag; n writes reaching all n nodes = a permutation.

template <typename VT>
struct RegLayout {
  int n, T, P, nextra, ndyn, ndyn_sinks;
  __host__ __device__ size_t pos_bytes() const { return ((size_t)(n + 2) * 4 + 15) & ~size_t(15); }
  __host__ __device__ size_t xf_bytes() const {
    return ((size_t)(T * P + 1) * sizeof(XFPair<VT>) + 15) & ~size_t(15);
  }
  __host__ __device__ size_t node_bytes() const {  // NXF[n+1] pairs + NU[n+1]
    return (((size_t)(n + 1) * sizeof(XFPair<VT>) + 15) & ~size_t(15)) +
           (((size_t)(n + 1) * 4 + 15) & ~size_t(15));
  }
  __host__ __device__ size_t table_bytes() const {
    return (((size_t)nextra * 4 + 15) & ~size_t(15)) + (((size_t)(ndyn + 1) * 4 + 15) & ~size_t(15)) +
           (((size_t)ndyn_sinks * 4 + 15) & ~size_t(15)) +
           (((size_t)ndyn * sizeof(VT) + 15) & ~size_t(15));
  }
  __host__ __device__ size_t total() const { return pos_bytes() + xf_bytes() + 16; }
};

// Register caps: J=4/8 run with T <= 256 and >= 4 CTAs per SM (<= 64 regs),
// J=16 with T <= 512 and >= 2 CTAs per SM.
template <int J>
struct RegBounds {
  static constexpr int kMaxT = J <= 8 ? 256 : 512;
  static constexpr int kMinBlocks = J <= 8 ? 4 : 2;
};

template <typename VT, int J>
__global__ void __launch_bounds__(RegBounds<J>::kMaxT, RegBounds<J>::kMinBlocks)
    score_reg_kernel(ScoreTables G, const int32_t* __restrict__ orders, int64_t C,
                     uint64_t* __restrict__ peak_out, int32_t* __restrict__ step_out,
                     uint8_t* __restrict__ valid_out, uint64_t* __restrict__ bytes_out,
                     unsigned long long* __restrict__ best_key, int64_t index_base) {
  extern __shared__ __align__(16) char smem[];
  __shared__ BlockScratch<VT> bs;

  const int n = G.n;
  const int T = blockDim.x;
  const int tid = threadIdx.x;
  const int lane = tid & (kWarp - 1);
  const int warp = tid >> 5;
  const int nwarps = T >> 5;
  const int P = G.P;
  const int TP = T * P;
  const RegLayout<VT> L{n, T, P, G.nextra, G.ndyn, G.ndyn_sinks};

  // ---- shared memory: only the per-candidate buffers; the static tables are
  // read through L1 (prepared on the host in their final packed form, so a
  // CTA that scores only a few candidates pays no copy-in).
  char* p = smem;
  uint32_t* pos = reinterpret_cast<uint32_t*>(p);
  p += L.pos_bytes();
  XFPair<VT>* XF = reinterpret_cast<XFPair<VT>*>(p);
  const XFPair<VT>* __restrict__ NXF = reinterpret_cast<const XFPair<VT>*>(
      sizeof(VT) == 4 ? (const void*)G.node_xf32 : (const void*)G.node_xf64);  // [n+1]
  const int32_t* __restrict__ NU = G.node_u;        // [n+1], n+1 = no producer
  const uint32_t* __restrict__ ex = G.extra_packed;  // u | w << 16
  const int32_t* __restrict__ dyo = G.dyn_off;
  const int32_t* __restrict__ dys = G.dyn_sinks;
  const uint64_t* __restrict__ dyz = G.dyn_size;
  for (int i = tid; i < n + 2; i += T) pos[i] = 0;
  for (int i = tid; i <= TP; i += T) XF[i] = XFPair<VT>{0, 0};

  const int base = warp * J * kWarp + lane;  // slot j: k = base + 32*j
  uint32_t inmask = 0;
#pragma unroll
  for (int j = 0; j < J; ++j) inmask |= (base + kWarp * j < n ? 1u : 0u) << j;
  int ov[J];
#pragma unroll
  for (int j = 0; j < J; ++j) ov[j] = -1;
  if ((int64_t)blockIdx.x < C) {
    const int32_t* row = orders + (int64_t)blockIdx.x * n + base;
#pragma unroll
    for (int j = 0; j < J; ++j)
      if (inmask >> j & 1) ov[j] = __ldg(row + kWarp * j);
  }
  __syncthreads();

  uint32_t stamp = 0;
  for (int64_t c = blockIdx.x; c < C; c += gridDim.x) {
    if (++stamp > 0xffffu) {
      for (int i = tid; i < n + 2; i += T) pos[i] = 0;
      stamp = 1;
      __syncthreads();
    }
    const uint32_t tag = stamp << 16;
    const uint32_t tagbase = tag + (uint32_t)base;
    uint32_t bad = 0;

    // ---- phase 1: pos[order[k]] = tag | k --------------------------------------------
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const uint32_t v = (uint32_t)ov[j];
      const bool ok = v < (uint32_t)n;                 // padding slots carry -1
      bad |= (ok || !((inmask >> j) & 1u)) ? 0u : 1u;
      pos[ok ? v : (uint32_t)n] = tagbase + kWarp * j;
    }
    {
      const int64_t cn = c + gridDim.x;  // prefetch the next candidate's slice
      if (cn < C) {
        const int32_t* row = orders + cn * n + base;
#pragma unroll
        for (int j = 0; j < J; ++j)
          if (inmask >> j & 1) ov[j] = __ldg(row + kWarp * j);
      }
    }
    __syncthreads();

    // ---- phase 2a: node slots -----------------------------------------------------------
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const int v = min(base + kWarp * j, n);        // padding slots -> node n
      const uint32_t w = pos[v];
      const XFPair<VT> nxf = NXF[v];
      const uint32_t pu = pos[__ldg(NU + v)];
      bad |= (w < tag || pu >= w) ? 1u : 0u;         // stale (not a permutation) / producer late
      XF[min((int)(w & 0xffffu), TP)] = nxf;
    }
    // ---- phase 2b: remaining reduced producer pairs -----------------------------------
    for (int i = tid; i < G.nextra; i += T) {
      const uint32_t e = __ldg(ex + i);
      bad |= (pos[e & 0xffffu] >= pos[e >> 16]) ? 1u : 0u;
    }
    // ---- phase 2c: order-dependent last consumers -----------------------------------
    if (G.ndyn > 0) {
      __syncthreads();
      for (int d = tid; d < G.ndyn; d += T) {
        uint32_t h = 0;
        for (int s = __ldg(dyo + d); s < __ldg(dyo + d + 1); ++s) h = max(h, pos[__ldg(dys + s)]);
        const int q = (int)(h & 0xffffu);
        if (q < n) {
          const VT sz = (VT)__ldg(dyz + d);
          atomicAdd(&XF[q].f, sz);
          atomicAdd(&XF[q].x, (VT)0 - sz);
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

    // ---- phase 3: blocked two-pass scan over [tid*P, tid*P + P), P odd -------------
    const XFPair<VT>* mine = XF + tid * P;
    VT total = 0;
    for (int i = 0; i < P; ++i) total += mine[i].x;
    const VT incl = warp_incl_scan(total, lane);
    if (lane == kWarp - 1) bs.wsum[warp] = incl;
    __syncthreads();
    VT run = warp_sum(lane < warp ? bs.wsum[lane] : (VT)0) + incl - total;
    VT best = 0;
    int best_i = INT_MAX;
    const int p0 = tid * P;
    if (bytes_out == nullptr) {
      // padding entries are (0, 0): their RS never exceeds RS(n-1), so a strict
      // comparison never lets them replace a real position.
      for (int i = 0; i < P; ++i) {
        const XFPair<VT> xf = mine[i];
        run += xf.x;
        const VT rs = run + xf.f;
        const bool better = rs > best || best_i == INT_MAX;
        best = better ? rs : best;
        best_i = better ? p0 + i : best_i;
      }
      if (best_i >= n) best_i = INT_MAX;  // a chunk made only of padding
    } else {
      const int lim = min(P, n - p0);
      for (int i = 0; i < lim; ++i) {
        const XFPair<VT> xf = mine[i];
        run += xf.x;
        const VT rs = run + xf.f;
        bytes_out[c * n + p0 + i] = (uint64_t)rs * G.scale;
        if (rs > best || best_i == INT_MAX) {
          best = rs;
          best_i = p0 + i;
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
              (pk < (1ull << 43) && gi < (1ull << 20)) ? ((pk << 20) | gi) : kKeyOverflow;
          atomicMin(best_key, key);
        }
      }
    }
  }
}

template <typename VT>
size_t reg_smem_bytes(int n, int T, int P, int nextra, int ndyn, int ndyn_sinks) {
  return RegLayout<VT>{n, T, P, nextra, ndyn, ndyn_sinks}.total();
}
