// K2 (liveness-overlap pairs) and K4 (address-plan validation) as one
// row-parallel pairwise sweep with warp-ballot compaction.
//
//   mode 0  encode_addresses pair loop   encode.cpp:347-367
//           (size>0 both, not both pinned, closed intervals intersect)
//   mode 1  validate_plan pairwise part  plan.cpp:390-404 / addresses_feasible
//           pipeline.cpp:146-160 (has address, size>0, lifetimes intersect,
//           [addr, addr+size) ranges overlap)
//
// Output order is the reference's lexicographic (i, j): a count pass writes
// per-row totals, an exclusive scan turns them into row offsets, and the
// fill pass writes each row's j's in increasing order at its offset (no
// sort, deterministic for any grid size).
#include <cuda_runtime.h>

#include <climits>
#include <cstdint>

#include "mp_internal.h"

namespace mpb {
namespace {

constexpr int kThreads = 256;
constexpr int kWarpsPerBlock = kThreads / 32;

struct PairRec {
  int2* lh;           // {lo, hi}; ineligible or empty -> {INT_MAX, INT_MIN}
  ulonglong2* as;     // mode 1: {addr, size}
  uint8_t* pin;       // mode 0: pinned (may be null)
};

// Ineligible or empty intervals get a sentinel that fails both comparisons
// of the intersection test (analysis.hpp:35-37).
__global__ void pack_kernel(int32_t E, const int32_t* __restrict__ lo,
                            const int32_t* __restrict__ hi, const uint64_t* __restrict__ size,
                            const uint8_t* __restrict__ mask, const uint64_t* __restrict__ addr,
                            int mode, int2* __restrict__ lh, ulonglong2* __restrict__ as) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int32_t l = lo[e], h = hi[e];
    bool ok = size[e] > 0 && l <= h;
    if (mode == 1) ok = ok && mask[e] != 0;
    lh[e] = ok ? make_int2(l, h) : make_int2(INT_MAX, INT_MIN);
    if (mode == 1) as[e] = make_ulonglong2(addr[e], size[e]);
  }
}

template <int MODE, bool PINNED>
__device__ __forceinline__ bool pair_pred(const int2 a, const int2 b, const ulonglong2 aa,
                                          const PairRec& R, int32_t j, bool pin_i) {
  bool ok = b.x <= a.y && a.x <= b.y;
  if (MODE == 0) {
    if (PINNED) ok = ok && !(pin_i && R.pin[j]);
  } else {
    if (ok) {
      const ulonglong2 bb = R.as[j];
      ok = aa.x < bb.x + bb.y && bb.x < aa.x + aa.y;
    }
  }
  return ok;
}

// One warp per row i (rows interleaved over all warps of the grid so the
// triangular work balances), 32 consecutive j per step.
template <int MODE, bool PINNED, bool FILL>
__global__ void __launch_bounds__(kThreads)
    pair_sweep_kernel(int32_t E, PairRec R, int64_t row_begin, int64_t row_end,
                      int64_t* __restrict__ row_off, int2* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t warp_global = (int64_t)blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  const int64_t num_warps = (int64_t)gridDim.x * kWarpsPerBlock;
  const unsigned lt_mask = (1u << lane) - 1u;
  for (int64_t r = row_begin + warp_global; r < row_end; r += num_warps) {
    const int32_t i = (int32_t)r;
    const int2 a = R.lh[i];
    int64_t cnt = 0;
    int64_t off = FILL ? row_off[r - row_begin] : 0;
    if (a.x <= a.y) {
      const ulonglong2 aa = MODE == 1 ? R.as[i] : make_ulonglong2(0, 0);
      const bool pin_i = PINNED ? R.pin[i] != 0 : false;
      for (int32_t j0 = i + 1; j0 < E; j0 += 32) {
        const int32_t j = j0 + lane;
        bool p = false;
        if (j < E) p = pair_pred<MODE, PINNED>(a, R.lh[j], aa, R, j, pin_i);
        const unsigned m = __ballot_sync(0xffffffffu, p);
        if (FILL) {
          if (p) out[off + __popc(m & lt_mask)] = make_int2(i, j);
          off += __popc(m);
        } else {
          cnt += __popc(m);
        }
      }
    }
    if (!FILL && lane == 0) row_off[r - row_begin + 1] = cnt;
  }
}

// In-place inclusive scan of row_off[1..rows] with row_off[0] = 0 (one CTA).
__global__ void __launch_bounds__(1024)
    offsets_scan_kernel(int64_t* __restrict__ row_off, int64_t rows,
                        int64_t* __restrict__ total) {
  __shared__ int64_t wsum[32];
  __shared__ int64_t carry_sh;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    carry_sh = 0;
    row_off[0] = 0;
  }
  for (int64_t base = 1; base <= rows; base += 1024) {
    const int64_t t = base + tid;
    int64_t v = t <= rows ? row_off[t] : 0;
    int64_t incl = v;
    for (int d = 1; d < 32; d <<= 1) {
      int64_t o = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += o;
    }
    __syncthreads();
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      int64_t w = wsum[lane], wi = w;
      for (int d = 1; d < 32; d <<= 1) {
        int64_t o = __shfl_up_sync(0xffffffffu, wi, d);
        if (lane >= d) wi += o;
      }
      wsum[lane] = wi - w;
    }
    __syncthreads();
    const int64_t s = carry_sh + wsum[warp] + incl;
    if (t <= rows) row_off[t] = s;
    __syncthreads();
    if (tid == 1023) carry_sh = s;
  }
  __syncthreads();
  if (tid == 0) *total = carry_sh;
}

__global__ void peak_mem_kernel(int32_t E, const uint64_t* __restrict__ size,
                                const uint8_t* __restrict__ has,
                                const uint64_t* __restrict__ addr,
                                unsigned long long* __restrict__ out) {
  unsigned long long best = 0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E;
       e += (int64_t)gridDim.x * blockDim.x)
    if (has[e]) best = max(best, (unsigned long long)(addr[e] + size[e]));
  for (int d = 16; d > 0; d >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, d));
  if ((threadIdx.x & 31) == 0 && best) atomicMax(out, best);
}

PairRec carve(const PairArgs& a, void* scratch) {
  char* p = static_cast<char*>(scratch);
  PairRec R;
  R.lh = reinterpret_cast<int2*>(p);
  p += ((size_t)a.num_edges * sizeof(int2) + 255) & ~size_t(255);
  R.as = reinterpret_cast<ulonglong2*>(p);
  R.pin = const_cast<uint8_t*>(a.mask);
  return R;
}

unsigned sweep_grid(int64_t rows, int num_sms) {
  int64_t want = (rows + kWarpsPerBlock - 1) / kWarpsPerBlock;
  int64_t cap = (int64_t)num_sms * 16;
  if (want > cap) want = cap;
  if (want < 1) want = 1;
  return (unsigned)want;
}

mp_status pack(const PairArgs& a, const PairRec& R, cudaStream_t st) {
  if (a.num_edges == 0) return MP_OK;
  int64_t b = (a.num_edges + kThreads - 1) / kThreads;
  if (b > 148 * 16) b = 148 * 16;
  pack_kernel<<<(unsigned)b, kThreads, 0, st>>>(a.num_edges, a.lo, a.hi, a.size, a.mask, a.addr,
                                                a.mode, R.lh, R.as);
  MP_CUDA(cudaGetLastError());
  return MP_OK;
}

template <bool FILL>
mp_status sweep(const PairArgs& a, int num_sms, const PairRec& R, int64_t* row_off, int2* out,
                cudaStream_t st) {
  const int64_t rows = a.row_end - a.row_begin;
  if (rows <= 0) return MP_OK;
  const unsigned grid = sweep_grid(rows, num_sms);
  if (a.mode == 0) {
    if (a.mask)
      pair_sweep_kernel<0, true, FILL><<<grid, kThreads, 0, st>>>(a.num_edges, R, a.row_begin,
                                                                  a.row_end, row_off, out);
    else
      pair_sweep_kernel<0, false, FILL><<<grid, kThreads, 0, st>>>(a.num_edges, R, a.row_begin,
                                                                   a.row_end, row_off, out);
  } else {
    pair_sweep_kernel<1, false, FILL><<<grid, kThreads, 0, st>>>(a.num_edges, R, a.row_begin,
                                                                 a.row_end, row_off, out);
  }
  MP_CUDA(cudaGetLastError());
  return MP_OK;
}

}  // namespace

size_t pairs_scratch_bytes(const PairArgs& a, int) {
  return (((size_t)a.num_edges * sizeof(int2) + 255) & ~size_t(255)) +
         (size_t)a.num_edges * sizeof(ulonglong2) + 512;
}

mp_status pairs_count(const PairArgs& a, int num_sms, void* scratch, int64_t* d_row_off,
                      int64_t* h_total, cudaStream_t st) {
  PairRec R = carve(a, scratch);
  MP_TRY(pack(a, R, st));
  const int64_t rows = a.row_end - a.row_begin;
  MP_TRY(sweep<false>(a, num_sms, R, d_row_off, nullptr, st));
  int64_t* d_total = reinterpret_cast<int64_t*>(reinterpret_cast<char*>(scratch) +
                                                pairs_scratch_bytes(a, num_sms) - 256);
  offsets_scan_kernel<<<1, 1024, 0, st>>>(d_row_off, rows > 0 ? rows : 0, d_total);
  MP_CUDA(cudaGetLastError());
  MP_CUDA(cudaMemcpyAsync(h_total, d_total, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  MP_CUDA(cudaStreamSynchronize(st));
  return MP_OK;
}

mp_status pairs_fill(const PairArgs& a, int num_sms, void* scratch, const int64_t* d_row_off,
                     int32_t* d_pairs, cudaStream_t st) {
  PairRec R = carve(a, scratch);  // packed by pairs_count
  return sweep<true>(a, num_sms, R, const_cast<int64_t*>(d_row_off),
                     reinterpret_cast<int2*>(d_pairs), st);
}

mp_status launch_peak_mem(int32_t E, const uint64_t* d_size, const uint8_t* d_has,
                          const uint64_t* d_addr, uint64_t* d_out, cudaStream_t st) {
  MP_CUDA(cudaMemsetAsync(d_out, 0, sizeof(uint64_t), st));
  if (E == 0) return MP_OK;
  int64_t b = (E + kThreads - 1) / kThreads;
  if (b > 148 * 8) b = 148 * 8;
  peak_mem_kernel<<<(unsigned)b, kThreads, 0, st>>>(E, d_size, d_has, d_addr,
                                                    reinterpret_cast<unsigned long long*>(d_out));
  MP_CUDA(cudaGetLastError());
  return MP_OK;
}

}  // namespace mpb
