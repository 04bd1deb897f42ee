// Microbenchmark: what tcgen05.commit and the single issuing thread cost the
// MMA stream.  `nt` threads (one per warp) each issue groups of `g` SS-mode
// kind::i8 MMAs (M = 128, K = 32 B, SW32) into their OWN accumulator, followed
// by `c` commits onto rotating mbarriers (never waited on, except the final
// ones); prints cycles per MMA over all threads.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2603_17230_b200/csrc \
//        scripts/mma_commit.cu -o scripts/mma_commit.bin && scripts/mma_commit.bin
#include <cstdio>
#include <cuda_runtime.h>

#include "kan_ptx.cuh"

using namespace kan;

template <int G>
__global__ void mma_commit(int n_groups, int c, int N, int nt, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint32_t s_tmem;
  __shared__ __align__(8) uint64_t bars[20];
  __shared__ unsigned long long t_end[2];
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = i * 2654435761u;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 20; ++i) mbar_init(smem_u32(&bars[i]), 1);
    mbar_fence_init();
  }
  if (warp == 0) tmem_alloc(smem_u32(&s_tmem), 512);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;
  unsigned long long t0 = clock64();
  if ((threadIdx.x & 31) == 0 && warp < nt) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
    const uint64_t ad = umma_desc_sw32(a), bd = umma_desc_sw32(b);
    const uint32_t idesc = idesc_i8(N, true);
    const uint32_t d = tmem + static_cast<uint32_t>(warp) * 256u;
    for (int gi = 0; gi < n_groups; ++gi) {
#pragma unroll
      for (int i = 0; i < G; ++i)
        mma_i8(d, ad + 16 * ((i + warp) & 15), bd + 2 * (i & 3), idesc, (gi | i) != 0 ? 1u : 0u);
      for (int j = 0; j < c; ++j) tc_commit(smem_u32(&bars[8 * warp + ((2 * gi + j) & 7)]));
    }
    tc_commit(smem_u32(&bars[16 + warp]));
    mbar_wait(smem_u32(&bars[16 + warp]), 0);
    t_end[warp] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = nt == 2 && t_end[1] > t_end[0] ? t_end[1] : t_end[0];
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * sizeof(unsigned long long));
  cudaFuncSetAttribute(mma_commit<9>, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
  cudaFuncSetAttribute(mma_commit<18>, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
  for (int N : {64, 128, 192})
    for (int nt : {1, 2})
      for (int c : {0, 1, 2}) {
        // the same 18 MMAs per group in all: one thread x 18, or two threads x 9
        const int groups = 256;
        for (int rep = 0; rep < 2; ++rep) {
          if (nt == 1)
            mma_commit<18><<<148, 128, 80 * 1024>>>(groups, c, N, nt, d);
          else
            mma_commit<9><<<148, 128, 80 * 1024>>>(groups, c, N, nt, d);
        }
        cudaError_t e = cudaDeviceSynchronize();
        unsigned long long cc[148];
        cudaMemcpy(cc, d, 148 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
        unsigned long long mx = 0;
        for (int i = 0; i < 148; ++i) mx = cc[i] > mx ? cc[i] : mx;
        printf("N=%3d issuing threads %d (18 MMAs per group in all) commits per thread per group %d: %6.1f cycles/MMA (%s)\n", N,
               nt, c, static_cast<double>(mx) / (groups * 18), e == cudaSuccess ? "ok" : cudaGetErrorString(e));
      }
  return 0;
}
