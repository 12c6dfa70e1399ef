// Microbenchmark: random 4-byte shared-memory traffic, local vs distributed
// shared memory (cluster of CS CTAs), to size the C5 scorer design.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dsmem_rand dsmem_rand.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t mix(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16; return x;
}

// mode 0: stores, mode 1: loads (8 independent per batch)
template <int CS, int MODE>
__global__ void k_rand(int words, int iters, uint32_t* out) {
  extern __shared__ uint32_t s[];
  for (int i = threadIdx.x; i < words; i += blockDim.x) s[i] = i;
  cg::cluster_group cl = cg::this_cluster();
  if (CS > 1) cl.sync(); else __syncthreads();
  uint32_t h = mix(blockIdx.x * 1024 + threadIdx.x + 1);
  uint32_t acc = 0;
  const uint32_t mask = words - 1;
  for (int it = 0; it < iters; ++it) {
    uint32_t* p[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      h = h * 1664525u + 1013904223u;
      uint32_t* base = s;
      if (CS > 1) base = cl.map_shared_rank(s, (h >> 28) % CS);
      p[u] = base + ((h >> 8) & mask);
    }
    if (MODE == 0) {
#pragma unroll
      for (int u = 0; u < 8; ++u) *p[u] = h + u;
    } else {
      uint32_t v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = *(volatile uint32_t*)p[u];
#pragma unroll
      for (int u = 0; u < 8; ++u) acc += v[u];
    }
  }
  if (CS > 1) cl.sync(); else __syncthreads();
  if (acc == 0x12345678) out[0] = acc;
}

template <int CS, int MODE>
void run(int T, int words, const char* name) {
  auto kern = k_rand<CS, MODE>;
  size_t smem = words * 4;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (CS > 1) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int grid = (sms / CS) * CS;
  uint32_t* out; cudaMalloc(&out, 4);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid); cfg.blockDim = dim3(T); cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CS; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  int iters = 256;
  cudaLaunchKernelEx(&cfg, kern, words, iters, out);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) cudaLaunchKernelEx(&cfg, kern, words, iters, out);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  cudaError_t e = cudaGetLastError();
  double reqs = 5.0 * grid * T * iters * 8;
  double per_sm_per_ns = reqs / (ms * 1e6) / grid;
  printf("%-28s CS=%d T=%4d words=%6d : %.3f ms  %.2f req/ns/SM (%.2f req/clk/SM @1.965GHz) %s\n",
         name, CS, T, words, ms / 5, per_sm_per_ns, per_sm_per_ns / 1.965, e ? cudaGetErrorString(e) : "");
}

int main() {
  run<1, 0>(1024, 32768, "local store");
  run<1, 1>(1024, 32768, "local load");
  run<2, 0>(1024, 32768, "dsmem store");
  run<2, 1>(1024, 32768, "dsmem load");
  run<4, 0>(1024, 32768, "dsmem store");
  run<4, 1>(1024, 32768, "dsmem load");
  run<8, 0>(1024, 32768, "dsmem store");
  run<8, 1>(1024, 32768, "dsmem load");
  run<16, 0>(1024, 32768, "dsmem store");
  run<16, 1>(1024, 32768, "dsmem load");
  return 0;
}
