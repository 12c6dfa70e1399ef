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
#include <cstdlib>

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

// Tiled sweep: a CTA owns RPW rows per warp (kept in registers) and streams
// the columns j > first row through shared memory in tiles of kTileCols, so
// every column record is read from L2 once per CTA instead of once per row.
// Each lane evaluates its column of a 32-wide chunk against all of its warp's
// rows (RPW ballots per loaded column); the count pass accumulates popc per
// row, the fill pass writes each row's matches at off + popc(ballot & lt) in
// increasing j (the reference's lexicographic order). Ineligible rows are
// sentinels that match nothing.
constexpr int kTileCols = 1024;

template <int MODE, bool PINNED, bool FILL, int RPW>
__global__ void __launch_bounds__(kThreads)
    pair_tile_kernel(int32_t E, PairRec R, int64_t row_begin, int64_t row_end,
                     int64_t* __restrict__ row_off, int2* __restrict__ out, int64_t cap) {
  __shared__ int2 slh[kTileCols];
  __shared__ ulonglong2 sas[MODE == 1 ? kTileCols : 1];
  __shared__ uint8_t spin[PINNED ? kTileCols : 1];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const unsigned lt_mask = (1u << lane) - 1u;
  const int64_t r0 = row_begin + (int64_t)blockIdx.x * kWarpsPerBlock * RPW;

  int2 a[RPW];
  ulonglong2 aa[RPW];
  bool pin_i[RPW];
  int64_t acc[RPW];  // FILL: running output offset; count: matches
  int32_t ri[RPW];
  bool any = false;
#pragma unroll
  for (int t = 0; t < RPW; ++t) {
    const int64_t i = r0 + warp * RPW + t;
    const bool in = i < row_end;
    ri[t] = (int32_t)i;
    a[t] = in ? R.lh[i] : make_int2(INT_MAX, INT_MIN);
    any |= a[t].x <= a[t].y;
    if (MODE == 1) aa[t] = in ? R.as[i] : make_ulonglong2(0, 0);
    if (PINNED) pin_i[t] = in ? R.pin[i] != 0 : false;
    acc[t] = (FILL && in) ? row_off[i - row_begin] : 0;
  }
  const bool warp_any = __any_sync(0xffffffffu, any);

  for (int64_t j0 = r0 + 1; j0 < E; j0 += kTileCols) {
    for (int q = threadIdx.x; q < kTileCols; q += kThreads) {
      const int64_t j = j0 + q;
      const bool in = j < E;
      slh[q] = in ? R.lh[j] : make_int2(INT_MAX, INT_MIN);
      if (MODE == 1) sas[q] = in ? R.as[j] : make_ulonglong2(0, 0);
      if (PINNED) spin[q] = in ? R.pin[j] : 0;
    }
    __syncthreads();
    if (warp_any) {
      const int cols = (int)min((int64_t)kTileCols, E - j0);
      for (int c = 0; c < cols; c += 32) {
        const int q = c + lane;
        const int32_t j = (int32_t)(j0 + q);
        const int2 b = slh[q];
        ulonglong2 bb;
        if (MODE == 1) bb = sas[q];
        const bool pj = PINNED ? spin[q] != 0 : false;
#pragma unroll
        for (int t = 0; t < RPW; ++t) {
          bool p = b.x <= a[t].y && a[t].x <= b.y && j > ri[t];
          if (MODE == 0 && PINNED) p = p && !(pin_i[t] && pj);
          if (MODE == 1) p = p && aa[t].x < bb.x + bb.y && bb.x < aa[t].x + aa[t].y;
          const unsigned m = __ballot_sync(0xffffffffu, p);
          if (FILL) {
            if (p) {
              const int64_t o = acc[t] + __popc(m & lt_mask);
              if (o < cap) out[o] = make_int2(ri[t], j);  // capacity: the first cap pairs
            }
          }
          acc[t] += __popc(m);
        }
      }
    }
    __syncthreads();
  }
  if (!FILL && lane == 0) {
#pragma unroll
    for (int t = 0; t < RPW; ++t) {
      const int64_t i = r0 + warp * RPW + t;
      if (i < row_end) row_off[i - row_begin + 1] = acc[t];
    }
  }
}

// ---- mode 0 count without the O(E^2) sweep ------------------------------------
// For row i and a column tile lying entirely after i, the overlapping eligible j are
//   #{lo_j <= hi_i} - #{hi_j < lo_i}
// (hi_j < lo_i <= hi_i implies lo_j <= hi_i, so the second set is inside the first):
// two binary searches in the tile's sorted lo and hi arrays (ineligible columns sort
// to the end as INT_MAX and are never counted). Only the tile holding row i itself
// is swept column by column (j > i). The per-row totals are identical to the
// sweep's; the fill pass still walks every tile to emit the pairs in (i, j) order.
constexpr int kSortT = 512;
constexpr int32_t kSortedCountMinEdges = 8 * kTileCols;  // C2-C4 (<= 4,180 edges) sweep

// One CTA per column tile: sorted lo / hi of the eligible columns (and, for pinned
// mode, of the eligible UNPINNED columns), bitonic in shared memory.
template <bool PINNED>
__global__ void __launch_bounds__(kSortT)
    tile_sort_kernel(int32_t E, PairRec R, int32_t* __restrict__ sorted) {
  constexpr int NA = PINNED ? 4 : 2;
  __shared__ int32_t s[NA][kTileCols];
  const int t = blockIdx.x;
  for (int q = threadIdx.x; q < kTileCols; q += kSortT) {
    const int64_t j = (int64_t)t * kTileCols + q;
    const int2 b = j < E ? R.lh[j] : make_int2(INT_MAX, INT_MIN);
    const bool el = b.x <= b.y;
    s[0][q] = el ? b.x : INT_MAX;
    s[1][q] = el ? b.y : INT_MAX;
    if (PINNED) {
      const bool up = el && !(j < E && R.pin[j] != 0);
      s[2][q] = up ? b.x : INT_MAX;
      s[3][q] = up ? b.y : INT_MAX;
    }
  }
  __syncthreads();
  for (int k = 2; k <= kTileCols; k <<= 1)
    for (int jj = k >> 1; jj > 0; jj >>= 1) {
      for (int i = threadIdx.x; i < kTileCols; i += kSortT) {
        const int ixj = i ^ jj;
        if (ixj > i) {
          const bool asc = (i & k) == 0;
#pragma unroll
          for (int a = 0; a < NA; ++a) {
            const int x = s[a][i], y = s[a][ixj];
            if ((x > y) == asc) {
              s[a][i] = y;
              s[a][ixj] = x;
            }
          }
        }
      }
      __syncthreads();
    }
  int32_t* out = sorted + (size_t)t * NA * kTileCols;
  for (int a = 0; a < NA; ++a)
    for (int q = threadIdx.x; q < kTileCols; q += kSortT) out[a * kTileCols + q] = s[a][q];
}

// entries <= x (LE) or < x (!LE) in a sorted 1024-entry shared array
template <bool LE>
__device__ __forceinline__ int rank_in(const int32_t* S, int x) {
  int pos = 0;
#pragma unroll
  for (int step = kTileCols / 2; step > 0; step >>= 1)
    if (LE ? S[pos + step - 1] <= x : S[pos + step - 1] < x) pos += step;
  // the steps sum to 1023: a tile whose every entry qualifies ends at 1023
  if (LE ? S[pos] <= x : S[pos] < x) ++pos;
  return pos;
}

constexpr int kCountT = 256;

template <bool PINNED>
__global__ void __launch_bounds__(kCountT)
    pair_count_sorted_kernel(int32_t E, PairRec R, const int32_t* __restrict__ sorted,
                             int64_t row_begin, int64_t row_end, int64_t* __restrict__ row_off) {
  constexpr int NA = PINNED ? 4 : 2;
  __shared__ int32_t ss[NA][kTileCols];
  __shared__ int2 slh[kTileCols];
  __shared__ uint8_t spin[PINNED ? kTileCols : 1];
  const int64_t b0 = row_begin + (int64_t)blockIdx.x * kCountT;
  const int64_t r = b0 + threadIdx.x;
  const bool in = r < row_end;
  const int2 a = in ? R.lh[r] : make_int2(INT_MAX, INT_MIN);
  const bool pin = PINNED && in && R.pin[r] != 0;
  const bool el = a.x <= a.y;
  const int tr = (int)(r / kTileCols);
  const int64_t blast = min(row_end, b0 + kCountT) - 1;
  const int ntiles = (E + kTileCols - 1) / kTileCols;
  int64_t cnt = 0;
  for (int t = (int)(b0 / kTileCols); t < ntiles; ++t) {
    const bool diag = t <= (int)(blast / kTileCols);  // some row of this CTA lies in tile t
    __syncthreads();
    const int32_t* src = sorted + (size_t)t * NA * kTileCols;
    for (int q = threadIdx.x; q < NA * kTileCols; q += kCountT) (&ss[0][0])[q] = __ldg(src + q);
    if (diag)
      for (int q = threadIdx.x; q < kTileCols; q += kCountT) {
        const int64_t j = (int64_t)t * kTileCols + q;
        slh[q] = j < E ? R.lh[j] : make_int2(INT_MAX, INT_MIN);
        if (PINNED) spin[q] = j < E ? R.pin[j] : 0;
      }
    __syncthreads();
    if (!el || !in) continue;
    if (t > tr) {
      const int32_t* SL = ss[pin ? 2 : 0];
      const int32_t* SH = ss[pin ? 3 : 1];
      cnt += rank_in<true>(SL, a.y) - rank_in<false>(SH, a.x);
    } else if (t == tr) {
      const int cols = (int)min((int64_t)kTileCols, (int64_t)E - (int64_t)t * kTileCols);
      for (int q = (int)(r - (int64_t)t * kTileCols) + 1; q < cols; ++q) {
        const int2 b = slh[q];
        bool p = b.x <= a.y && a.x <= b.y;
        if (PINNED) p = p && !(pin && spin[q] != 0);
        cnt += p ? 1 : 0;
      }
    }
  }
  if (in) row_off[r - row_begin + 1] = cnt;
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
  R.as = reinterpret_cast<ulonglong2*>(p);  // mode 1; the sorted tiles follow it
  R.pin = const_cast<uint8_t*>(a.mask);
  return R;
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

template <int MODE, bool PINNED, bool FILL, int RPW>
void launch_tile(const PairArgs& a, const PairRec& R, int64_t* row_off, int2* out,
                 int64_t cap, cudaStream_t st) {
  const int64_t rows = a.row_end - a.row_begin;
  const int64_t per_block = (int64_t)kWarpsPerBlock * RPW;
  const unsigned grid = (unsigned)((rows + per_block - 1) / per_block);
  pair_tile_kernel<MODE, PINNED, FILL, RPW>
      <<<grid, kThreads, 0, st>>>(a.num_edges, R, a.row_begin, a.row_end, row_off, out, cap);
}

template <bool FILL>
mp_status sweep(const PairArgs& a, int num_sms, const PairRec& R, int64_t* row_off, int2* out,
                int64_t cap, cudaStream_t st) {
  const int64_t rows = a.row_end - a.row_begin;
  if (rows <= 0) return MP_OK;
  // 8 rows per warp once there are enough rows to fill the GPU twice over
  const bool big = rows >= (int64_t)num_sms * kWarpsPerBlock * 8 * 2;
  if (a.mode == 0) {
    if (a.mask) {
      big ? launch_tile<0, true, FILL, 8>(a, R, row_off, out, cap, st)
          : launch_tile<0, true, FILL, 1>(a, R, row_off, out, cap, st);
    } else {
      big ? launch_tile<0, false, FILL, 8>(a, R, row_off, out, cap, st)
          : launch_tile<0, false, FILL, 1>(a, R, row_off, out, cap, st);
    }
  } else {
    big ? launch_tile<1, false, FILL, 8>(a, R, row_off, out, cap, st)
        : launch_tile<1, false, FILL, 1>(a, R, row_off, out, cap, st);
  }
  MP_CUDA(cudaGetLastError());
  return MP_OK;
}

}  // namespace

// scratch: packed {lo,hi} | {addr,size} | mode-0 sorted tiles | 256 B (device total)
size_t sorted_bytes(const PairArgs& a) {
  if (a.mode != 0) return 0;
  const size_t tiles = ((size_t)a.num_edges + kTileCols - 1) / kTileCols;
  return tiles * (a.mask ? 4 : 2) * kTileCols * sizeof(int32_t);
}
size_t pairs_scratch_bytes(const PairArgs& a, int) {
  return (((size_t)a.num_edges * sizeof(int2) + 255) & ~size_t(255)) +
         (((size_t)a.num_edges * sizeof(ulonglong2) + 255) & ~size_t(255)) + sorted_bytes(a) +
         512;
}

mp_status pairs_count(const PairArgs& a, int num_sms, void* scratch, int64_t* d_row_off,
                      int64_t* h_total, cudaStream_t st) {
  PairRec R = carve(a, scratch);
  MP_TRY(pack(a, R, st));
  const int64_t rows = a.row_end - a.row_begin;
  // per-row totals from sorted column tiles (no O(E^2) sweep) once there are enough
  // tiles to amortise the sort and the serial in-tile count; small graphs sweep
  const bool force_sorted = std::getenv("MP_PAIRS_SORTED") != nullptr;  // tests
  if (a.mode == 0 && rows > 0 && (a.num_edges >= kSortedCountMinEdges || force_sorted)) {
    int32_t* sorted = reinterpret_cast<int32_t*>(
        reinterpret_cast<char*>(scratch) +
        (((size_t)a.num_edges * sizeof(int2) + 255) & ~size_t(255)) +
        (((size_t)a.num_edges * sizeof(ulonglong2) + 255) & ~size_t(255)));
    const unsigned tiles = (unsigned)((a.num_edges + kTileCols - 1) / kTileCols);
    const unsigned grid = (unsigned)((rows + kCountT - 1) / kCountT);
    if (a.mask) {
      tile_sort_kernel<true><<<tiles, kSortT, 0, st>>>(a.num_edges, R, sorted);
      pair_count_sorted_kernel<true>
          <<<grid, kCountT, 0, st>>>(a.num_edges, R, sorted, a.row_begin, a.row_end, d_row_off);
    } else {
      tile_sort_kernel<false><<<tiles, kSortT, 0, st>>>(a.num_edges, R, sorted);
      pair_count_sorted_kernel<false>
          <<<grid, kCountT, 0, st>>>(a.num_edges, R, sorted, a.row_begin, a.row_end, d_row_off);
    }
    MP_CUDA(cudaGetLastError());
  } else {
    MP_TRY(sweep<false>(a, num_sms, R, d_row_off, nullptr, 0, st));
  }
  int64_t* d_total = pairs_device_total(a, num_sms, scratch);
  offsets_scan_kernel<<<1, 1024, 0, st>>>(d_row_off, rows > 0 ? rows : 0, d_total);
  MP_CUDA(cudaGetLastError());
  if (h_total) {
    MP_CUDA(cudaMemcpyAsync(h_total, d_total, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    MP_CUDA(cudaStreamSynchronize(st));
  }
  return MP_OK;
}

int64_t* pairs_device_total(const PairArgs& a, int num_sms, void* scratch) {
  return reinterpret_cast<int64_t*>(reinterpret_cast<char*>(scratch) +
                                    pairs_scratch_bytes(a, num_sms) - 256);
}

mp_status pairs_fill(const PairArgs& a, int num_sms, void* scratch, const int64_t* d_row_off,
                     int32_t* d_pairs, cudaStream_t st, int64_t cap) {
  PairRec R = carve(a, scratch);  // packed by pairs_count
  return sweep<true>(a, num_sms, R, const_cast<int64_t*>(d_row_off),
                     reinterpret_cast<int2*>(d_pairs), cap, st);
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
