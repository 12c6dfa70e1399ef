// Warp-per-candidate variant of the fused scorer (n up to kWarpMaxNodes),
// included by k_score.cu inside namespace mpb::{anon}. Same math and the
// same absorbing-slot conventions as the register variant (k_score_reg.cuh),
// but each WARP scores its own candidates end to end: no block barriers, one
// warp scan and one warp argmax per candidate, and ~n/32 independent slots per
// lane in every phase (ILP instead of barrier-separated CTA phases).
//
// Shared memory per CTA:
//   node table (shared by the CTA's warps, filled once):
//     NX[n+1]  (x, f) pairs   NP[n+1]  (pred1 | pred2 << 16), 0xffff = none
//   per warp:
//     pos[n+2]   stamped positions; pos[n] absorbs bad ids, pos[n+1] == 0
//     XF[32P+1]  scattered (x, f); [n, 32P) scan padding, [32P] garbage slot
//     buf[n]     the next candidate's order row (cp.async prefetch)
// Requires n < 65535 (16-bit producer ids and positions).

constexpr int kWarpMaxNodes = 2048;

__device__ __forceinline__ void cp_async4(void* smem_dst, const void* gmem_src) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(d), "l"(gmem_src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n"); }

template <typename VT>
struct WarpLayout {
  int n, P, W;  // P = per-lane scan chunk (odd), W = warps per CTA
  __host__ __device__ size_t nx_bytes() const {
    return ((size_t)(n + 1) * sizeof(XFPair<VT>) + 15) & ~size_t(15);
  }
  __host__ __device__ size_t np_bytes() const { return ((size_t)(n + 1) * 4 + 15) & ~size_t(15); }
  __host__ __device__ size_t pos_bytes() const { return ((size_t)(n + 2) * 4 + 15) & ~size_t(15); }
  __host__ __device__ size_t xf_bytes() const {
    return ((size_t)(32 * P + 1) * sizeof(XFPair<VT>) + 15) & ~size_t(15);
  }
  __host__ __device__ size_t buf_bytes() const { return ((size_t)n * 4 + 15) & ~size_t(15); }
  __host__ __device__ size_t per_warp() const { return pos_bytes() + xf_bytes() + buf_bytes(); }
  __host__ __device__ size_t total() const { return nx_bytes() + np_bytes() + W * per_warp() + 16; }
};

template <typename VT>
__global__ void __launch_bounds__(512)
    score_warp_kernel(ScoreTables G, const int32_t* __restrict__ orders, int64_t C,
                      uint64_t* __restrict__ peak_out, int32_t* __restrict__ step_out,
                      uint8_t* __restrict__ valid_out, uint64_t* __restrict__ bytes_out,
                      unsigned long long* __restrict__ best_key, int64_t index_base) {
  extern __shared__ __align__(16) char smem[];
  const int n = G.n;
  const int W = blockDim.x >> 5;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int P = G.P;
  const int TP = 32 * P;
  const WarpLayout<VT> L{n, P, W};

  XFPair<VT>* NX = reinterpret_cast<XFPair<VT>*>(smem);
  uint32_t* NP = reinterpret_cast<uint32_t*>(smem + L.nx_bytes());
  char* mine = smem + L.nx_bytes() + L.np_bytes() + (size_t)warp * L.per_warp();
  uint32_t* pos = reinterpret_cast<uint32_t*>(mine);
  XFPair<VT>* XF = reinterpret_cast<XFPair<VT>*>(mine + L.pos_bytes());
  int32_t* buf = reinterpret_cast<int32_t*>(mine + L.pos_bytes() + L.xf_bytes());

  // ---- CTA setup: node table, per-warp buffers --------------------------------------
  for (int v = threadIdx.x; v <= n; v += blockDim.x) {
    const bool in = v < n;
    NX[v] = XFPair<VT>{in ? (VT)G.node_x[v] : (VT)0, in ? (VT)G.node_f[v] : (VT)0};
    uint32_t u1 = 0xffffu, u2 = 0xffffu;
    if (in) {
      const int2 uu = __ldg(G.node_u2 + v);
      if (uu.x >= 0) u1 = (uint32_t)uu.x;
      if (uu.y >= 0) u2 = (uint32_t)uu.y;
    }
    NP[v] = u1 | (u2 << 16);
  }
  for (int i = lane; i < n + 2; i += 32) pos[i] = 0;
  for (int i = n + lane; i <= TP; i += 32) XF[i] = XFPair<VT>{0, 0};
  // "no producer" (0xffff) must read as pos 0: pos[n+1] is 0, so map 0xffff -> n+1
  const uint32_t none = (uint32_t)(n + 1);

  const int64_t wstride = (int64_t)gridDim.x * W;
  int64_t c = (int64_t)blockIdx.x * W + warp;
  if (c < C) {
    const int32_t* row = orders + c * n;
    for (int k = lane; k < n; k += 32) cp_async4(buf + k, row + k);
  }
  cp_async_commit();
  __syncthreads();  // node table visible to every warp

  uint32_t stamp = 0;
  for (; c < C; c += wstride) {
    if (++stamp > 0xffffu) {
      for (int i = lane; i < n + 2; i += 32) pos[i] = 0;
      stamp = 1;
    }
    const uint32_t tag = stamp << 16;
    uint32_t bad = 0;
    cp_async_wait_all();
    __syncwarp();

    // ---- phase 1: pos[order[k]] = tag | k ------------------------------------------
    // Batches of kB: every load of a batch is issued before any store (the
    // buffers alias as far as the compiler knows, so it would not reorder).
    constexpr int kB = 8;
    for (int k0 = lane; k0 < n; k0 += 32 * kB) {
      uint32_t v[kB];
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        const int k = k0 + 32 * u;
        v[u] = k < n ? (uint32_t)buf[k] : (uint32_t)n;  // past the end: absorb slot
      }
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        const int k = k0 + 32 * u;
        bad |= (k < n && v[u] >= (uint32_t)n) ? 1u : 0u;
        pos[min(v[u], (uint32_t)n)] = tag | (uint32_t)k;
      }
    }
    __syncwarp();  // buf consumed, pos written
    {
      const int64_t cn = c + wstride;  // prefetch the next candidate's row
      if (cn < C) {
        const int32_t* row = orders + cn * n;
#pragma unroll 8
        for (int k = lane; k < n; k += 32) cp_async4(buf + k, row + k);
      }
      cp_async_commit();
    }

    // ---- phase 2a: node space ---------------------------------------------------------
    for (int v0 = lane; v0 < n; v0 += 32 * kB) {
      uint32_t w[kB], pu[kB], pu2[kB];
      XFPair<VT> nx[kB];
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        const int v = min(v0 + 32 * u, n);  // past the end: node n (pos[n] absorbs)
        w[u] = pos[v];
        const uint32_t pp = NP[v];
        nx[u] = NX[v];
        const uint32_t a = pp & 0xffffu, b = pp >> 16;
        pu[u] = pos[a == 0xffffu ? none : a];
        pu2[u] = pos[b == 0xffffu ? none : b];
      }
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        if (v0 + 32 * u < n) {
          bad |= (w[u] < tag || pu[u] >= w[u] || pu2[u] >= w[u]) ? 1u : 0u;
          XF[min((int)(w[u] & 0xffffu), TP)] = nx[u];
        }
      }
    }
    // ---- phase 2b: 3rd+ reduced producer pairs ------------------------------------------
    for (int i = lane; i < G.nextra3; i += 32) {
      const uint32_t e = __ldg(G.extra3_packed + i);
      bad |= (pos[e & 0xffffu] >= pos[e >> 16]) ? 1u : 0u;
    }
    // ---- phase 2c: order-dependent last consumers ------------------------------------
    if (G.ndyn > 0) {
      __syncwarp();
      for (int d = lane; d < G.ndyn; d += 32) {
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
    __syncwarp();
    const bool invalid = __any_sync(0xffffffffu, bad != 0);

    // ---- phase 3: lane-blocked two-pass scan over [lane*P, lane*P + P), P odd -------
    const XFPair<VT>* ch = XF + lane * P;
    VT total = 0;
#pragma unroll 8
    for (int i = 0; i < P; ++i) total += ch[i].x;
    const VT incl = warp_incl_scan(total, lane);
    VT r = incl - total;
    const int p0 = lane * P;
    VT best;
    int best_i;
    if (bytes_out == nullptr) {
      XFPair<VT> xf = ch[0];
      r += xf.x;
      best = r + xf.f;
      int bi = 0;
#pragma unroll 8
      for (int i = 1; i < P; ++i) {
        xf = ch[i];
        r += xf.x;
        const VT rs = r + xf.f;
        const bool better = rs > best;
        best = better ? rs : best;
        bi = better ? i : bi;
      }
      best_i = p0 < n ? p0 + bi : INT_MAX;
    } else {
      best = 0;
      best_i = INT_MAX;
      const int lim = min(P, n - p0);
      for (int i = 0; i < lim; ++i) {
        const XFPair<VT> xf = ch[i];
        r += xf.x;
        const VT rs = r + xf.f;
        bytes_out[c * n + p0 + i] = (uint64_t)rs * G.scale;
        if (rs > best || best_i == INT_MAX) {
          best = rs;
          best_i = p0 + i;
        }
      }
    }
    warp_argmax(best, best_i);
    if (lane == 0) {
      const bool empty = n == 0;
      const uint64_t pk = (invalid || empty) ? 0 : (uint64_t)best * G.scale;
      peak_out[c] = pk;
      step_out[c] = (invalid || empty) ? 0 : best_i + 1;
      valid_out[c] = invalid ? 0 : 1;
      if (best_key && !invalid) {
        const uint64_t gi = (uint64_t)(c + index_base);
        record_key(best_key, pk, gi);
      }
    }
    __syncwarp();  // XF reads done before the next candidate scatters
  }
  cp_async_wait_all();
}

template <typename VT>
size_t warp_smem_bytes(int n, int P, int W) {
  return WarpLayout<VT>{n, P, W}.total();
}
