// Microbenchmark: what a tcgen05.commit per group of MMAs costs the issue
// stream.  One thread issues groups of `g` SS-mode kind::i8 MMAs (M = 128,
// K = 32 B, SW32) followed by `c` commits onto rotating mbarriers (never
// waited on, except the final one); prints cycles per MMA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2603_17230_b200/csrc \
//        scripts/mma_commit.cu -o scripts/mma_commit.bin && scripts/mma_commit.bin
#include <cstdio>
#include <cuda_runtime.h>

#include "kan_ptx.cuh"

using namespace kan;

__global__ void mma_commit(int n_groups, int g, int c, int N, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint32_t s_tmem;
  __shared__ __align__(8) uint64_t bars[9];
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = i * 2654435761u;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 9; ++i) mbar_init(smem_u32(&bars[i]), 1);
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
    const uint64_t ad = umma_desc_sw32(a), bd = umma_desc_sw32(b);
    const uint32_t idesc = idesc_i8(N, true);
    unsigned long long t0 = clock64();
    int k = 0;
    for (int gi = 0; gi < n_groups; ++gi) {
      for (int i = 0; i < g; ++i, ++k) mma_i8(tmem, ad + 16 * (k & 15), bd + 2 * (k & 3), idesc, k > 0 ? 1u : 0u);
      for (int j = 0; j < c; ++j) tc_commit(smem_u32(&bars[(2 * gi + j) & 7]));
    }
    tc_commit(smem_u32(&bars[8]));
    mbar_wait(smem_u32(&bars[8]), 0);
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
  cudaFuncSetAttribute(mma_commit, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
  for (int N : {64, 128, 192})
    for (int g : {9, 18, 36})
      for (int c : {0, 1, 2}) {
        const int groups = 4096 / g;
        mma_commit<<<148, 128, 80 * 1024>>>(groups, g, c, N, d);
        mma_commit<<<148, 128, 80 * 1024>>>(groups, g, c, N, d);
        cudaError_t e = cudaDeviceSynchronize();
        unsigned long long cc[148];
        cudaMemcpy(cc, d, 148 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
        unsigned long long mx = 0;
        for (int i = 0; i < 148; ++i) mx = cc[i] > mx ? cc[i] : mx;
        printf("N=%3d group %2d commits %d: %6.1f cycles/MMA (%s)\n", N, g, c, static_cast<double>(mx) / (groups * g),
               e == cudaSuccess ? "ok" : cudaGetErrorString(e));
      }
  return 0;
}
