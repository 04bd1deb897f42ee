// Microbenchmark: cycles per tcgen05.mma.cta_group::2.kind::i8 (M = 256 over a
// CTA pair, K = 32 bytes, both operands in shared memory, SW32 K-major): each
// CTA holds its 128 rows of A and N/2 rows of B.  Compare with mma_rate.cu
// (cta_group::1, M = 128): the pair form reads (4 KB + N/2 * 32 B) of shared
// memory per SM per MMA instead of (4 KB + N * 32 B).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2603_17230_b200/csrc \
//        scripts/mma_rate2.cu -o /tmp/mma_rate2 && /tmp/mma_rate2
#include <cstdio>
#include <cuda_runtime.h>

#include "kan_ptx.cuh"

using namespace kan;

__device__ __forceinline__ uint32_t crank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void csync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__global__ void __cluster_dims__(2, 1, 1) mma_rate2(int n_mma, int N, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint32_t s_tmem;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = i * 2654435761u;
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar), 1);
    mbar_fence_init();
  }
  if (warp == 0) tmem_alloc2(smem_u32(&s_tmem), 512);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  csync();
  tc_fence_after();
  const uint32_t tmem = s_tmem;
  if (threadIdx.x == 0) {
    unsigned long long t0 = clock64();
    if (crank() == 0) {
      const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
      const uint64_t ad = umma_desc_sw32(a), bd = umma_desc_sw32(b);
      const uint32_t idesc = idesc_i8_m(N, true, 256);
      for (int i = 0; i < n_mma; ++i) mma_i8_2cta(tmem, ad + 2 * (i & 7), bd + 2 * (i & 3), idesc, i > 0 ? 1u : 0u);
      tc_commit2_mc(smem_u32(&bar), 3);
    }
    mbar_wait(smem_u32(&bar), 0);
    unsigned long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  csync();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc2(tmem, 512);
  }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * sizeof(unsigned long long));
  cudaFuncSetAttribute(mma_rate2, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
  for (int grid : {2, 148})
    for (int N : {64, 128, 256}) {
      const int n = 4096;
      mma_rate2<<<grid, 128, 80 * 1024>>>(n, N, d);
      mma_rate2<<<grid, 128, 80 * 1024>>>(n, N, d);
      cudaError_t e = cudaDeviceSynchronize();
      unsigned long long c[148];
      cudaMemcpy(c, d, grid * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
      unsigned long long mx = 0;
      for (int i = 0; i < grid; ++i) mx = c[i] > mx ? c[i] : mx;
      const double cyc = static_cast<double>(mx) / n;
      const double macs = 128.0 * N * 32;  // per SM
      printf("pair grid %3d SW32 N=%3d: %6.1f cycles/MMA (M=256), %7.0f MAC/clk/SM (%s)\n", grid, N, cyc, macs / cyc,
             e == cudaSuccess ? "ok" : cudaGetErrorString(e));
    }
  return 0;
}
