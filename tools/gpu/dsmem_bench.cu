// Microbenchmark: scattered 4-byte stores into the shared memory of the CTAs of a
// cluster (st.shared::cluster) vs local scattered stores, at the node-partitioned
// scorer's shape (1024 threads, ~180 KB of slots per CTA, one CTA per SM).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dsmem_bench tools/gpu/dsmem_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kNW = 44000;

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
  return x;
}

template <int kMode>
__global__ void __launch_bounds__(1024, 1) k(int iters, int cs, uint32_t* out) {
  extern __shared__ uint32_t s[];
  for (int i = threadIdx.x; i < kNW; i += 1024) s[i] = 0;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(s);
  uint32_t seed = (blockIdx.x * 1024 + threadIdx.x) * 0x9e3779b9u;
  uint32_t acc = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll 8
    for (int j = 0; j < 16; ++j) {
      const uint32_t x = hash32(seed + it * 16 + j);
      const uint32_t loc = (x >> 8) % kNW;
      const uint32_t a = base + 4u * loc;
      if (kMode == 0) {  // local scattered store
        asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(x) : "memory");
      } else if (kMode == 1) {  // local read-modify-write
        uint32_t w;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(w) : "r"(a) : "memory");
        asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"((w & 0xff000000u) | x) : "memory");
      } else {
        const uint32_t r = kMode == 2 ? (x & 0xffu) % cs : kMode == 3 ? rank : ((threadIdx.x >> 5) + it) % cs;
        uint32_t ra;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(r));
        asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(ra), "r"(x) : "memory");
      }
    }
  }
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  for (int i = threadIdx.x; i < kNW; i += 1024) acc += s[i];
  if (acc == 0x12345678u) out[0] = acc;
}

template <int kMode>
float run(int cs, int iters) {
  auto f = k<kMode>;
  const size_t smem = kNW * 4;
  cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(1024);
  cfg.dynamicSmemBytes = smem;
  cfg.attrs = at; cfg.numAttrs = 1;
  int ncl = 0;
  cfg.gridDim = dim3(cs * 64);
  cudaOccupancyMaxActiveClusters(&ncl, f, &cfg);
  cfg.gridDim = dim3(cs * ncl);
  uint32_t* out; cudaMalloc(&out, 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaLaunchKernelEx(&cfg, f, iters, cs, out);
  cudaEventRecord(e0);
  cudaLaunchKernelEx(&cfg, f, iters, cs, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double stores_per_sm = (double)iters * 16 * 1024;
  const cudaError_t err = cudaGetLastError();
  printf("mode %d cs %d clusters %d (%d SMs): %.3f ms, %.2f stores/cycle/SM at 1.9 GHz %s\n", kMode, cs,
         ncl, ncl * cs, ms, stores_per_sm / (ms * 1e-3 * 1.9e9), err ? cudaGetErrorString(err) : "");
  cudaFree(out);
  return ms;
}

int main() {
  const int iters = 2000;
  for (int cs : {1, 2, 3, 4}) {
    run<0>(cs, iters);
    run<1>(cs, iters);
    run<2>(cs, iters);
    run<3>(cs, iters);
    run<4>(cs, iters);
  }
  return 0;
}
