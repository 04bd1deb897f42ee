// Tuning microbenchmark (not product code): per-SM issue cost of the fp64 ops
// the epilogue uses, and of try_wait polling.  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dfma(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0000001, c = 1e-9;
  double x0 = a, x1 = a + 1, x2 = a + 2, x3 = a + 3;
  for (int i = 0; i < iters; ++i) {
    x0 = fma(x0, b, c); x1 = fma(x1, b, c); x2 = fma(x2, b, c); x3 = fma(x3, b, c);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3;
}
__global__ void k_ffma(float* out, int iters) {
  float a = threadIdx.x * 1e-3f, b = 1.0000001f, c = 1e-9f;
  float x0 = a, x1 = a + 1, x2 = a + 2, x3 = a + 3;
  for (int i = 0; i < iters; ++i) {
    x0 = fmaf(x0, b, c); x1 = fmaf(x1, b, c); x2 = fmaf(x2, b, c); x3 = fmaf(x3, b, c);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3;
}
__global__ void k_ddiv(double* out, int iters) {
  double x = threadIdx.x + 1.5, s = 0.0015625;
  double acc = 0;
  for (int i = 0; i < iters; ++i) { acc += __ddiv_rn(x + i, s); }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void k_d2ll(long long* out, int iters) {
  double x = threadIdx.x + 0.25;
  long long acc = 0;
  for (int i = 0; i < iters; ++i) { acc += __double2ll_rz(x + i); }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <class F>
float timeit(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  f();
  cudaEventRecord(a); f(); cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms;
}

int main() {
  const int blocks = 148 * 4, threads = 256, iters = 4096;
  double* d; float* f; long long* l;
  cudaMalloc(&d, blocks * threads * 8); cudaMalloc(&f, blocks * threads * 4); cudaMalloc(&l, blocks * threads * 8);
  const double n = double(blocks) * threads * iters;
  float ms = timeit([&] { k_dfma<<<blocks, threads>>>(d, iters); });
  printf("DFMA: %.1f Gop/s (%.2f TFLOP/s)\n", 4 * n / ms / 1e6, 8 * n / ms / 1e9);
  ms = timeit([&] { k_ffma<<<blocks, threads>>>(f, iters); });
  printf("FFMA: %.1f Gop/s (%.2f TFLOP/s)\n", 4 * n / ms / 1e6, 8 * n / ms / 1e9);
  ms = timeit([&] { k_ddiv<<<blocks, threads>>>(d, iters); });
  printf("DDIV: %.2f Gop/s\n", n / ms / 1e6);
  ms = timeit([&] { k_d2ll<<<blocks, threads>>>(l, iters); });
  printf("D2LL: %.2f Gop/s\n", n / ms / 1e6);
  return 0;
}
