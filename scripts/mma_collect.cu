// Microbenchmark: does the A-operand collector hint (collector::a::fill/use/lastuse)
// or the weight-stationary form (tcgen05.mma.ws, B collector) lower the cycles per
// SS-mode kind::i8 MMA (M = 128, K = 32 bytes) when consecutive MMAs share an operand?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2603_17230_b200/csrc \
//        scripts/mma_collect.cu -o /tmp/mma_collect && /tmp/mma_collect
#include <cstdio>
#include <cuda_runtime.h>

#include "kan_ptx.cuh"

using namespace kan;

#define MMA_VARIANT(name, suffix)                                                                  \
  __device__ __forceinline__ void name(uint32_t d, uint64_t ad, uint64_t bd, uint32_t idesc,      \
                                       uint32_t acc) {                                             \
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"                                 \
                 "tcgen05.mma.cta_group::1.kind::i8" suffix " [%0], %1, %2, %3, p;\n\t}" ::"r"(d), \
                 "l"(ad), "l"(bd), "r"(idesc), "r"(acc)                                            \
                 : "memory");                                                                      \
  }
MMA_VARIANT(mma_fill, ".collector::a::fill")
MMA_VARIANT(mma_use, ".collector::a::use")
MMA_VARIANT(mma_last, ".collector::a::lastuse")
MMA_VARIANT(mma_disc, ".collector::a::discard")

// mode 0: plain, distinct A each MMA.  mode 1: plain, groups of `grp` MMAs share A (no hint).
// mode 2: groups share A with fill/use/lastuse hints.  Each MMA of a group has its own B and
// its own accumulator (as the window-shared conv issues them).
__global__ void mma_rate(int n_mma, int N, int mode, int grp, unsigned long long* out) {
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
    const uint64_t ad = umma_desc_sw32(a);
    const uint64_t bd = umma_desc_sw32(b);
    const uint32_t idesc = idesc_i8(N, true);
    unsigned long long t0 = clock64();
    for (int i = 0; i < n_mma; i += grp) {
      const uint64_t ag = ad + 2 * ((mode == 0 ? i : i / grp) & 7) * (mode == 0 ? 1 : 16);
      for (int g = 0; g < grp; ++g) {
        const uint64_t aa = mode == 0 ? ad + 2 * ((i + g) & 7) * 16 : ag;
        const uint64_t bb = bd + 2 * ((i + g) & 3) * 16;
        const uint32_t dd = tmem + (g & 3) * N;
        const uint32_t acc = i > 0 ? 1u : 0u;
        if (mode != 2) mma_i8(dd, aa, bb, idesc, acc);
        else if (g == 0) mma_fill(dd, aa, bb, idesc, acc);
        else if (g == grp - 1) mma_last(dd, aa, bb, idesc, acc);
        else mma_use(dd, aa, bb, idesc, acc);
      }
    }
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
  for (int N : {64, 128})
    for (int mode : {0, 1, 2})
      for (int grp : {2, 3, 4}) {
        if (mode == 0 && grp != 2) continue;
        const int n = 4096 / grp * grp;
        mma_rate<<<148, 128, 80 * 1024>>>(n, N, mode, grp, d);
        mma_rate<<<148, 128, 80 * 1024>>>(n, N, mode, grp, d);
        cudaError_t e = cudaDeviceSynchronize();
        unsigned long long c[148];
        cudaMemcpy(c, d, 148 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
        unsigned long long mx = 0;
        for (int i = 0; i < 148; ++i) mx = c[i] > mx ? c[i] : mx;
        const double cyc = static_cast<double>(mx) / n;
        printf("N=%3d mode %d (%s) grp %d: %6.1f cycles/MMA (%s)\n", N, mode,
               mode == 0 ? "distinct A" : mode == 1 ? "shared A, no hint" : "shared A, collector hints", grp, cyc,
               e == cudaSuccess ? "ok" : cudaGetErrorString(e));
      }
  return 0;
}
