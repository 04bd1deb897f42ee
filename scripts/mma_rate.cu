// Microbenchmark: cycles per tcgen05.mma.cta_group::1.kind::i8 (M = 128,
// K = 32 bytes) with both operands in shared memory, for N = 64 / 128 / 256,
// SW32 vs SW128 K-major layouts, and with A from TMEM (TS mode), issued
// back-to-back by one thread into one accumulator.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2603_17230_b200/csrc \
//        scripts/mma_rate.cu -o /tmp/mma_rate && /tmp/mma_rate
#include <cstdio>
#include <cuda_runtime.h>

#include "kan_ptx.cuh"

using namespace kan;

__global__ void mma_rate(int n_mma, int N, int sw, unsigned long long* out) {
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
  if (warp == 0) tmem_alloc(smem_u32(&s_tmem), 512);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;
  if (threadIdx.x == 0) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
    const uint64_t ad = sw == 32 ? umma_desc_sw32(a) : umma_desc_sw128(a);
    const uint64_t bd = sw == 32 ? umma_desc_sw32(b) : umma_desc_sw128(b);
    const uint32_t idesc = idesc_i8(N, true);
    unsigned long long t0 = clock64();
    for (int i = 0; i < n_mma; ++i) mma_i8(tmem, ad + 2 * (i & 7), bd + 2 * (i & 3), idesc, i > 0 ? 1u : 0u);
    tc_commit(smem_u32(&bar));
    mbar_wait(smem_u32(&bar), 0);
    unsigned long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * sizeof(unsigned long long));
  cudaFuncSetAttribute(mma_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
  for (int grid : {1, 148})
    for (int sw : {32, 128})
      for (int N : {64, 128, 256}) {
        const int n = 4096;
        mma_rate<<<grid, 128, 80 * 1024>>>(n, N, sw, d);
        mma_rate<<<grid, 128, 80 * 1024>>>(n, N, sw, d);
        cudaError_t e = cudaDeviceSynchronize();
        unsigned long long c[148];
        cudaMemcpy(c, d, grid * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
        unsigned long long mx = 0;
        for (int i = 0; i < grid; ++i) mx = c[i] > mx ? c[i] : mx;
        const double cyc = static_cast<double>(mx) / n;
        const double macs = 128.0 * N * 32;
        printf("grid %3d SW%-3d N=%3d: %6.1f cycles/MMA, %7.0f MAC/clk/SM (%s)\n", grid, sw, N, cyc, macs / cyc,
               e == cudaSuccess ? "ok" : cudaGetErrorString(e));
      }
  return 0;
}
