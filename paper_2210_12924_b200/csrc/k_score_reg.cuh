// Register-slot variant of the fused scorer (n up to ~8k nodes), included by
// k_score.cu inside namespace mpb::{anon}. See k_score.cu for the math.
//
// Slot j of a thread covers order position AND node k = (warp*J + j)*32 + lane,
// k < TJ = T*J: warp-contiguous, so global loads coalesce and every per-slot
// shared-memory address is the thread's base plus an immediate. Per slot the
// thread keeps in registers: the next candidate's order value ov, the node's
// static bytes (x, f) and the pos index of its first reduced producer.
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
  __host__ __device__ size_t total() const { return pos_bytes() + xf_bytes() + 16; }
};

// Register budgets per slot count: J=4 -> T <= 256, 64 regs; J=8 -> T <= 384,
// 85 regs; J=16 -> T <= 512, 128 regs (score_configure picks the smallest J).
template <int J>
struct RegBounds {
  static constexpr int kMaxT = J == 4 ? 256 : J == 8 ? 384 : 512;
  static constexpr int kMinBlocks = J == 4 ? 4 : J == 8 ? 2 : 1;
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
  const RegLayout<VT> L{n, T, P, J};
  const int TJ = L.TJ();

  uint32_t* pos = reinterpret_cast<uint32_t*>(smem);
  XFPair<VT>* XF = reinterpret_cast<XFPair<VT>*>(smem + L.pos_bytes());
  {
    uint4* z = reinterpret_cast<uint4*>(pos);  // pos = 0: stamp 0 is never used
    for (int i = tid; i < (int)(L.pos_words() / 4); i += T) z[i] = make_uint4(0, 0, 0, 0);
    for (int i = n + tid; i <= TP; i += T) XF[i] = XFPair<VT>{0, 0};  // scan padding
  }

  const int base = warp * J * kWarp + lane;  // slot j: k = base + 32*j
  uint32_t real = 0;                          // bit j: slot j is a real node / position
  int ov[J];
  VT rx[J], rf[J];
  int ru[J], ru2[J];  // pos indexes of the first two reduced producers (TJ+1: none)
#pragma unroll
  for (int j = 0; j < J; ++j) {
    const int k = base + kWarp * j;
    const bool in = k < n;
    real |= (in ? 1u : 0u) << j;
    int u1 = -1, u2 = -1;
    rx[j] = 0;
    rf[j] = 0;
    if (in) {
      if constexpr (sizeof(VT) == 4) {
        const uint4 rec = __ldg(G.node_rec32 + k);  // (x, f, pred1, pred2): one load
        rx[j] = rec.x;
        rf[j] = rec.y;
        u1 = (int)rec.z;
        u2 = (int)rec.w;
      } else {
        rx[j] = (VT)__ldg(G.node_x + k);
        rf[j] = (VT)__ldg(G.node_f + k);
        const int2 uu = __ldg(G.node_u2 + k);
        u1 = uu.x;
        u2 = uu.y;
      }
    }
    ru[j] = u1 >= 0 ? u1 : TJ + 1;
    ru2[j] = u2 >= 0 ? u2 : TJ + 1;
    ov[j] = k;  // padding slots keep their own index forever
  }
  const int32_t* nrow = orders + (int64_t)blockIdx.x * n + base;  // row of the next candidate
  const int64_t rowstep = (int64_t)gridDim.x * n;
  if ((int64_t)blockIdx.x < C) {
#pragma unroll
    for (int j = 0; j < J; ++j)
      if (real >> j & 1) ov[j] = __ldg(nrow + kWarp * j);
  }
  nrow += rowstep;
  __syncthreads();

  uint32_t stamp = 0;
  for (int64_t c = blockIdx.x; c < C; c += gridDim.x, nrow += rowstep) {
    if (++stamp > 0xffffu) {
      for (int i = tid; i < (int)L.pos_words(); i += T) pos[i] = 0;
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
      bad |= ((real >> j) & 1u) & (v >= (uint32_t)n ? 1u : 0u);
      pos[min(v, (uint32_t)TJ)] = tagbase + kWarp * j;
    }
    if (c + gridDim.x < C) {  // prefetch the next candidate's slice
#pragma unroll
      for (int j = 0; j < J; ++j)
        if (real >> j & 1) ov[j] = __ldg(nrow + kWarp * j);
    }
    __syncthreads();

    // ---- phase 2a: node slots -----------------------------------------------------------
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const uint32_t w = pos[base + kWarp * j];
      const uint32_t pu = pos[ru[j]];
      const uint32_t pu2 = pos[ru2[j]];
      // stale word (not a permutation) / a producer not strictly earlier
      bad |= (w < tag || pu >= w || pu2 >= w) ? 1u : 0u;
      XF[min((int)(w & 0xffffu), TP)] = XFPair<VT>{rx[j], rf[j]};
    }
    // ---- phase 2b: 3rd+ reduced producer pairs (flat) ----------------------------------
    for (int i = tid; i < G.nextra3; i += T) {
      const uint32_t e = __ldg(G.extra3_packed + i);
      bad |= (pos[e & 0xffffu] >= pos[e >> 16]) ? 1u : 0u;
    }
    // ---- phase 2c: order-dependent last consumers -----------------------------------
    if (G.ndyn > 0) {
      __syncthreads();
      for (int d = tid; d < G.ndyn; d += T) {
        uint32_t h = 0;
        const int s1 = __ldg(G.dyn_off + d + 1);
        for (int s = __ldg(G.dyn_off + d); s < s1; ++s) h = max(h, pos[__ldg(G.dyn_sinks + s)]);
        const int q = (int)(h & 0xffffu);
        if (q < n) {
          const VT sz = (VT)__ldg(G.dyn_size + d);
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
    const int p0 = tid * P;
    VT best;
    int best_i;
    if (bytes_out == nullptr) {
      // First element initialises (best, index); strict > keeps the first
      // maximum. Padding entries are (0, 0): their RS equals S(n-1) <= RS(n-1),
      // so they never replace a real position.
      XFPair<VT> xf = mine[0];
      run += xf.x;
      best = run + xf.f;
      best_i = 0;
      for (int i = 1; i < P; ++i) {
        xf = mine[i];
        run += xf.x;
        const VT rs = run + xf.f;
        const bool better = rs > best;
        best = better ? rs : best;
        best_i = better ? i : best_i;
      }
      best_i = p0 < n ? p0 + best_i : INT_MAX;  // a chunk made only of padding
    } else {
      best = 0;
      best_i = INT_MAX;
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
size_t reg_smem_bytes(int n, int T, int P, int J) {
  return RegLayout<VT>{n, T, P, J}.total();
}
