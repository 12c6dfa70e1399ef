// K7 - non-overlap row emission straight from the GPU pair list: the text of
// write_lp (lp_format.cpp:88-121) for the rows encode_addresses emits per
// overlapping pair (encode.cpp:358-365 and 277-291):
//   c<3p>_live_pair:  +1 below +1 above = 1
//   c<3p+1>_below:    [+1 addr_i] [-1 addr_j] +M below <= M - size_i - v_i + v_j
//   c<3p+2>_above:    [+1 addr_i] [-1 addr_j] -M above >= size_j - M - v_i + v_j
// (a pinned address contributes its value v to the constant instead of a
// term, encode.cpp:46-50), and the two binaries of each pair for the
// "Binaries" section. One thread per pair: a length pass, an exclusive scan
// of the lengths, and a write pass that formats the integers itself into a
// per-warp shared stage stored out with 16-byte writes. The output is byte
// text, so the roofline is HBM writes of the text.
#include <cuda_runtime.h>

#include <cstdint>

#include "mp_internal.h"

namespace mpb {
namespace {

__device__ __forceinline__ int digits_u64(unsigned long long v) {
  int d = 1;
  while (v >= 10) {
    v /= 10;
    ++d;
  }
  return d;
}

__device__ __forceinline__ int digits_i64(long long v) {
  return v < 0 ? 1 + digits_u64((unsigned long long)(-v)) : digits_u64((unsigned long long)v);
}

__device__ __forceinline__ char* put_u64(char* p, unsigned long long v) {
  const int d = digits_u64(v);
  for (int k = d - 1; k >= 0; --k) {
    p[k] = (char)('0' + v % 10);
    v /= 10;
  }
  return p + d;
}

__device__ __forceinline__ char* put_i64(char* p, long long v) {
  if (v < 0) {
    *p++ = '-';
    return put_u64(p, (unsigned long long)(-v));
  }
  return put_u64(p, (unsigned long long)v);
}

__device__ __forceinline__ char* put_str(char* p, const char* s, int n) {
  for (int k = 0; k < n; ++k) p[k] = s[k];
  return p + n;
}

template <int N>
__device__ __forceinline__ char* put_lit(char* p, const char (&s)[N]) {
  return put_str(p, s, N - 1);
}

struct PairText {
  int li, lj;                 // sanitized id lengths
  const char* si;
  const char* sj;
  bool pi, pj;                // pinned
  long long rhs_below, rhs_above;
};

__device__ __forceinline__ PairText pair_text(const LpArgs& a, int i, int j) {
  PairText t;
  t.si = a.names + a.name_off[i];
  t.sj = a.names + a.name_off[j];
  t.li = (int)(a.name_off[i + 1] - a.name_off[i]);
  t.lj = (int)(a.name_off[j + 1] - a.name_off[j]);
  t.pi = a.pinned && a.pinned[i];
  t.pj = a.pinned && a.pinned[j];
  const long long vi = t.pi ? (long long)a.pinned_addr[i] : 0;
  const long long vj = t.pj ? (long long)a.pinned_addr[j] : 0;
  // Row::emit: rhs - constant, constant = +1*v_i - 1*v_j (encode.cpp:277-291)
  t.rhs_below = a.M - (long long)a.size[i] - vi + vj;
  t.rhs_above = (long long)a.size[j] - a.M - vi + vj;
  return t;
}

// below_<si>_<sj>_ / above_<si>_<sj>_ : 6 + li + 1 + lj + 1
__device__ __forceinline__ int pair_name_len(const PairText& t) { return t.li + t.lj + 8; }

__device__ __forceinline__ char* put_pair_name(char* p, bool below, const PairText& t) {
  p = below ? put_lit(p, "below_") : put_lit(p, "above_");
  p = put_str(p, t.si, t.li);
  *p++ = '_';
  p = put_str(p, t.sj, t.lj);
  *p++ = '_';
  return p;
}

__device__ __forceinline__ long long rows_len(const LpArgs& a, const PairText& t, long long p) {
  const int nl = pair_name_len(t);
  const int dm = digits_u64((unsigned long long)a.M);
  const int terms = (t.pi ? 0 : 4 + t.li + 6) + (t.pj ? 0 : 4 + t.lj + 6);
  long long n = 0;
  n += 2 + digits_u64(3 * p) + 11 + 4 + nl + 4 + nl + 5;                               // live_pair
  n += 2 + digits_u64(3 * p + 1) + 7 + terms + 3 + dm + nl + 4 + digits_i64(t.rhs_below) + 1;
  n += 2 + digits_u64(3 * p + 2) + 7 + terms + 3 + dm + nl + 4 + digits_i64(t.rhs_above) + 1;
  return n;
}

__device__ __forceinline__ char* put_terms(char* q, const PairText& t) {
  if (!t.pi) {
    q = put_lit(q, " +1 addr_");
    q = put_str(q, t.si, t.li);
    *q++ = '_';
  }
  if (!t.pj) {
    q = put_lit(q, " -1 addr_");
    q = put_str(q, t.sj, t.lj);
    *q++ = '_';
  }
  return q;
}

__global__ void lp_len_kernel(LpArgs a) {
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < a.P;
       p += (long long)gridDim.x * blockDim.x) {
    const int2 ij = a.pairs[p];
    const PairText t = pair_text(a, ij.x, ij.y);
    a.row_len[p] = rows_len(a, t, p);
    a.bin_len[p] = 2 * (1 + pair_name_len(t) + 1);
  }
}

__device__ __forceinline__ char* put_rows(char* q, const LpArgs& a, const PairText& t,
                                          long long p) {
  // c<3p>_live_pair: +1 below +1 above = 1
  q = put_lit(q, " c");
  q = put_u64(q, 3 * p);
  q = put_lit(q, "_live_pair: +1 ");
  q = put_pair_name(q, true, t);
  q = put_lit(q, " +1 ");
  q = put_pair_name(q, false, t);
  q = put_lit(q, " = 1\n");
  // c<3p+1>_below: ... +M below <= rhs
  q = put_lit(q, " c");
  q = put_u64(q, 3 * p + 1);
  q = put_lit(q, "_below:");
  q = put_terms(q, t);
  q = put_lit(q, " +");
  q = put_u64(q, (unsigned long long)a.M);
  *q++ = ' ';
  q = put_pair_name(q, true, t);
  q = put_lit(q, " <= ");
  q = put_i64(q, t.rhs_below);
  *q++ = '\n';
  // c<3p+2>_above: ... -M above >= rhs
  q = put_lit(q, " c");
  q = put_u64(q, 3 * p + 2);
  q = put_lit(q, "_above:");
  q = put_terms(q, t);
  q = put_lit(q, " -");
  q = put_u64(q, (unsigned long long)a.M);
  *q++ = ' ';
  q = put_pair_name(q, false, t);
  q = put_lit(q, " >= ");
  q = put_i64(q, t.rhs_above);
  *q++ = '\n';
  return q;
}

// Binaries section: below, then above (variable creation order, encode.cpp:263-272)
__device__ __forceinline__ char* put_bins(char* q, const PairText& t) {
  *q++ = ' ';
  q = put_pair_name(q, true, t);
  *q++ = '\n';
  *q++ = ' ';
  q = put_pair_name(q, false, t);
  *q++ = '\n';
  return q;
}

constexpr int kLpWarps = 4;
constexpr int kLpStage = 16384;  // bytes of staged text per warp

// Copy len bytes from shared src to global dst with the warp: byte head up to a
// 16-byte boundary of dst, then 16-byte stores whose words are funnel-shifted out
// of aligned shared words, then a byte tail.
__device__ __forceinline__ void warp_copy(char* __restrict__ dst, const char* src, int len,
                                          int lane) {
  const int head = min(len, (int)((16 - (reinterpret_cast<uintptr_t>(dst) & 15)) & 15));
  if (lane < head) dst[lane] = src[lane];
  const int body = (len - head) & ~15;
  const char* s0 = src + head;
  const uint32_t* sw = reinterpret_cast<const uint32_t*>(reinterpret_cast<uintptr_t>(s0) & ~uintptr_t(3));
  const int sh = (int)(reinterpret_cast<uintptr_t>(s0) & 3) * 8;
  uint4* d4 = reinterpret_cast<uint4*>(dst + head);
  for (int j = lane; j < body / 16; j += 32) {
    const uint32_t* w = sw + 4 * j;
    uint32_t x[5];
#pragma unroll
    for (int k = 0; k < 5; ++k) x[k] = (k < 4 || sh) ? w[k] : 0u;
    uint4 o;
    o.x = __funnelshift_r(x[0], x[1], sh);
    o.y = __funnelshift_r(x[1], x[2], sh);
    o.z = __funnelshift_r(x[2], x[3], sh);
    o.w = __funnelshift_r(x[3], x[4], sh);
    d4[j] = o;
  }
  for (int k = head + body + lane; k < len; k += 32) dst[k] = src[k];
}

// One warp per 32 consecutive pairs: each lane formats its pair into a
// contiguous shared staging area (the pairs' texts are contiguous in the
// output), then the warp stores it with 16-byte writes - the byte-at-a-time
// global stores of a per-thread formatter made this kernel L1-bound. Pairs
// whose 32 texts exceed the stage are formatted straight to global memory.
__global__ void __launch_bounds__(32 * kLpWarps)
    lp_write_kernel(LpArgs a, char* __restrict__ rows, char* __restrict__ bins) {
  extern __shared__ __align__(16) char stage[];  // [kLpWarps][kLpStage + 16]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  char* st = stage + (size_t)w * (kLpStage + 16);
  const long long nwarps = (long long)gridDim.x * kLpWarps;
  for (long long p0 = ((long long)blockIdx.x * kLpWarps + w) * 32; p0 < a.P; p0 += nwarps * 32) {
    const long long p = p0 + lane;
    const bool live = p < a.P;
    const long long last = (p0 + 32 < a.P ? p0 + 32 : a.P) - 1;
    PairText t;
    if (live) t = pair_text(a, a.pairs[p].x, a.pairs[p].y);
    // rows
    {
      const long long base = a.row_off[p0];
      const long long span = a.row_off[last] + a.row_len[last] - base;
      if (span <= kLpStage) {
        if (live) put_rows(st + (a.row_off[p] - base), a, t, p);
        __syncwarp();
        warp_copy(rows + base, st, (int)span, lane);
        __syncwarp();
      } else if (live) {
        put_rows(rows + a.row_off[p], a, t, p);
      }
    }
    // binaries
    {
      const long long base = a.bin_off[p0];
      const long long span = a.bin_off[last] + a.bin_len[last] - base;
      if (span <= kLpStage) {
        if (live) put_bins(st + (a.bin_off[p] - base), t);
        __syncwarp();
        warp_copy(bins + base, st, (int)span, lane);
        __syncwarp();
      } else if (live) {
        put_bins(bins + a.bin_off[p], t);
      }
    }
  }
}

// ---- exclusive scan of int64 lengths (reduce -> one-CTA scan of block sums -> down) -
constexpr int kScanT = 512;
constexpr int kScanPer = 8;  // elements per thread per block

__global__ void scan_reduce_kernel(const int64_t* __restrict__ in, int64_t n,
                                   int64_t* __restrict__ sums) {
  __shared__ long long ws[kScanT / 32];
  const int64_t b0 = (int64_t)blockIdx.x * kScanT * kScanPer;
  long long s = 0;
  for (int k = 0; k < kScanPer; ++k) {
    const int64_t i = b0 + (int64_t)k * kScanT + threadIdx.x;
    if (i < n) s += in[i];
  }
  for (int d = 16; d > 0; d >>= 1) s += __shfl_xor_sync(0xffffffffu, s, d);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    s = threadIdx.x < kScanT / 32 ? ws[threadIdx.x] : 0;
    for (int d = 16; d > 0; d >>= 1) s += __shfl_xor_sync(0xffffffffu, s, d);
    if (threadIdx.x == 0) sums[blockIdx.x] = s;
  }
}

__global__ void scan_sums_kernel(int64_t* __restrict__ sums, int64_t nb, int64_t* total) {
  __shared__ long long carry;
  __shared__ long long ws[32];
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t i0 = 0; i0 < nb; i0 += blockDim.x) {
    const int64_t i = i0 + threadIdx.x;
    const long long v = i < nb ? sums[i] : 0;
    long long x = v;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int d = 1; d < 32; d <<= 1) {
      const long long o = __shfl_up_sync(0xffffffffu, x, d);
      if (lane >= d) x += o;
    }
    if (lane == 31) ws[w] = x;
    __syncthreads();
    long long before = 0;
    for (int k = 0; k < w; ++k) before += ws[k];
    const long long c = carry;
    if (i < nb) sums[i] = c + before + x - v;  // exclusive
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = c + before + x;
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = carry;
}

__global__ void scan_down_kernel(const int64_t* __restrict__ in, int64_t n,
                                 const int64_t* __restrict__ sums, int64_t* __restrict__ out) {
  __shared__ long long ws[kScanT / 32];
  __shared__ long long carry;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t b0 = (int64_t)blockIdx.x * kScanT * kScanPer;
  if (threadIdx.x == 0) carry = sums[blockIdx.x];
  __syncthreads();
  for (int k = 0; k < kScanPer; ++k) {
    const int64_t i = b0 + (int64_t)k * kScanT + threadIdx.x;
    const long long v = i < n ? in[i] : 0;
    long long x = v;
    for (int d = 1; d < 32; d <<= 1) {
      const long long o = __shfl_up_sync(0xffffffffu, x, d);
      if (lane >= d) x += o;
    }
    if (lane == 31) ws[w] = x;
    __syncthreads();
    long long before = 0;
    for (int q = 0; q < w; ++q) before += ws[q];
    const long long c = carry;
    if (i < n) out[i] = c + before + x - v;
    __syncthreads();
    if (threadIdx.x == kScanT - 1) carry = c + before + x;
    __syncthreads();
  }
}

}  // namespace

size_t lp_scan_scratch(int64_t n) {
  return (size_t)((n + kScanT * kScanPer - 1) / (kScanT * kScanPer) + 1) * 8;
}

mp_status scan_exclusive_i64(const int64_t* d_in, int64_t n, int64_t* d_out, int64_t* d_sums,
                             int64_t* d_total, cudaStream_t st) {
  const int64_t nb = (n + kScanT * kScanPer - 1) / (kScanT * kScanPer);
  if (nb > 0) scan_reduce_kernel<<<(unsigned)nb, kScanT, 0, st>>>(d_in, n, d_sums);
  scan_sums_kernel<<<1, 1024, 0, st>>>(d_sums, nb, d_total);
  if (nb > 0) scan_down_kernel<<<(unsigned)nb, kScanT, 0, st>>>(d_in, n, d_sums, d_out);
  MP_CUDA(cudaGetLastError());
  return MP_OK;
}

mp_status launch_lp_len(const LpArgs& a, int num_sms, cudaStream_t st) {
  if (a.P <= 0) return MP_OK;
  int64_t grid = (a.P + 255) / 256;
  if (grid > (int64_t)num_sms * 16) grid = (int64_t)num_sms * 16;
  lp_len_kernel<<<(unsigned)grid, 256, 0, st>>>(a);
  MP_CUDA(cudaGetLastError());
  return MP_OK;
}

mp_status launch_lp_write(const LpArgs& a, char* d_rows, char* d_bins, int num_sms,
                          cudaStream_t st) {
  if (a.P <= 0) return MP_OK;
  int64_t grid = (a.P + 32 * kLpWarps - 1) / (32 * kLpWarps);
  if (grid > (int64_t)num_sms * 3) grid = (int64_t)num_sms * 3;
  const int smem = kLpWarps * (kLpStage + 16);
  MP_CUDA(cudaFuncSetAttribute(lp_write_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  lp_write_kernel<<<(unsigned)grid, 32 * kLpWarps, smem, st>>>(a, d_rows, d_bins);
  MP_CUDA(cudaGetLastError());
  return MP_OK;
}

}  // namespace mpb
