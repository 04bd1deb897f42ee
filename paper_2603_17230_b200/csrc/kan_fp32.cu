// kan_fp32.cu -- fp32 Cox-de Boor KAN layer on CUDA cores (accuracy baseline).
//
// Replaces kan_linear_forward<RecursiveBasis> (proj/include/kantize/layers.hpp:
// 99-121): the basis triangle (grid.hpp:124-140) is evaluated in fp32 for the
// P+1 supported functions, scattered into a dense smem tile, and contracted
// with the coefficients in fp32 FFMA (no TF32: its 1e-3 error would break the
// 1e-4 tolerance this path is held to).  A 64x64 output tile per CTA,
// 4x4 outputs per thread, K chunks of 8 inputs x NBP basis columns.
#include <cuda_runtime.h>

#include "kan_internal.h"

namespace kan {

template <int PMAX>
__device__ __forceinline__ int basis_f32_local(float x, float lo, float hi_open, float inv_delta,
                                               int G, int P, float (&N)[PMAX + 1]) {
  x = fminf(fmaxf(x, lo), hi_open);
  const float xi = (x - lo) * inv_delta + static_cast<float>(P);
  int j = static_cast<int>(floorf(xi));
  j = min(max(j, P), G + P - 1);
#pragma unroll
  for (int r = 0; r <= PMAX; ++r) N[r] = 0.f;
  N[PMAX] = 1.f;
#pragma unroll
  for (int d = 1; d <= PMAX; ++d) {
    if (d > P) break;
    const float rd = 1.0f / static_cast<float>(d);
#pragma unroll
    for (int r = 0; r <= d; ++r) {
      const int i = j - d + r;
      const float left = (r == 0) ? 0.f : N[PMAX - d + r];
      const float right = (r == d) ? 0.f : N[PMAX - d + r + 1];
      N[PMAX - d + r] = ((xi - static_cast<float>(i)) * rd) * left +
                        ((static_cast<float>(i + d + 1) - xi) * rd) * right;
    }
  }
  if (P < PMAX) {
#pragma unroll
    for (int r = 0; r <= PMAX; ++r) N[r] = (r + PMAX - P <= PMAX) ? N[r + PMAX - P] : 0.f;
  }
  return j - P;
}

template <int NBP>
__global__ void __launch_bounds__(256) kan_fp32_kernel(const Fp32Params p) {
  constexpr int TM = 64, TN = 64, CI = 64 / NBP, KC = CI * NBP;
  __shared__ float Bs[TM][KC + 1];
  __shared__ __align__(16) float Ws[KC][TN];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int m0 = blockIdx.y * TM, n0 = blockIdx.x * TN;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;

  auto mma_chunk = [&](int kc) {
#pragma unroll 4
    for (int kk = 0; kk < kc; ++kk) {
      const float4 b = *reinterpret_cast<const float4*>(&Ws[kk][tx * 4]);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float a = Bs[ty * 4 + i][kk];
        acc[i][0] += a * b.x;
        acc[i][1] += a * b.y;
        acc[i][2] += a * b.z;
        acc[i][3] += a * b.w;
      }
    }
  };

  // spline segment
  for (int i0 = 0; i0 < p.n_in; i0 += CI) {
    for (int q = tid; q < TM * CI; q += 256) {
      const int r = q / CI, ii = q % CI;
      const int row = m0 + r, in = i0 + ii;
      float vals[NBP];
#pragma unroll
      for (int b = 0; b < NBP; ++b) vals[b] = 0.f;
      if (row < p.M && in < p.n_in) {
        float N[4];
        const int jj = basis_f32_local<3>(p.x[static_cast<size_t>(row) * p.ld_x + in], p.lo,
                                          p.hi_open, p.inv_delta, p.G, p.P, N);
#pragma unroll
        for (int b = 0; b < NBP; ++b) {
          const int rr = b - jj;
          float v = 0.f;
#pragma unroll
          for (int t = 0; t < 4; ++t) v = (rr == t) ? N[t] : v;
          vals[b] = v;
        }
      }
#pragma unroll
      for (int b = 0; b < NBP; ++b) Bs[r][ii * NBP + b] = vals[b];
    }
    for (int q = tid; q < KC * TN / 4; q += 256) {
      const int kr = q / (TN / 4), c4 = q % (TN / 4);
      const int krow = i0 * NBP + kr;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (krow < p.n_in * NBP)
        v = *reinterpret_cast<const float4*>(p.w + static_cast<size_t>(krow) * p.Npad + n0 + c4 * 4);
      *reinterpret_cast<float4*>(&Ws[kr][c4 * 4]) = v;
    }
    __syncthreads();
    mma_chunk(KC);
    __syncthreads();
  }
  // SiLU base segment: silu(clamp(x)) . w_base
  if (p.wb) {
    for (int i0 = 0; i0 < p.n_in; i0 += KC) {
      for (int q = tid; q < TM * KC; q += 256) {
        const int r = q / KC, ii = q % KC;
        const int row = m0 + r, in = i0 + ii;
        float v = 0.f;
        if (row < p.M && in < p.n_in) {
          const float xc =
              fminf(fmaxf(p.x[static_cast<size_t>(row) * p.ld_x + in], p.lo), p.hi_open);
          v = xc / (1.0f + expf(-xc));
        }
        Bs[r][ii] = v;
      }
      for (int q = tid; q < KC * TN / 4; q += 256) {
        const int kr = q / (TN / 4), c4 = q % (TN / 4);
        const int krow = i0 + kr;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (krow < p.n_in)
          v = *reinterpret_cast<const float4*>(p.wb + static_cast<size_t>(krow) * p.Npad + n0 +
                                               c4 * 4);
        *reinterpret_cast<float4*>(&Ws[kr][c4 * 4]) = v;
      }
      __syncthreads();
      mma_chunk(KC);
      __syncthreads();
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int row = m0 + ty * 4 + i;
    if (row >= p.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int col = n0 + tx * 4 + j;
      if (col < p.N) p.out[static_cast<size_t>(row) * p.ld_out + col] = acc[i][j];
    }
  }
}

cudaError_t launch_fp32_layer(const Fp32Params& p, cudaStream_t st) {
  if (p.M == 0) return cudaSuccess;
  dim3 grid(p.Npad / 64, (p.M + 63) / 64);
  if (p.NBP == 8)
    kan_fp32_kernel<8><<<grid, 256, 0, st>>>(p);
  else
    kan_fp32_kernel<16><<<grid, 256, 0, st>>>(p);
  return cudaGetLastError();
}

}  // namespace kan

// ---------------------------------------------------------------------------
// fp32 conv models (EvalMode::kFp32 on conv / maxpool / flatten stacks): the
// reference's convkan_forward = im2col (layers.hpp:126-154) + the dense layer
// on the patch rows, NCHW activations throughout (flatten is a view).
namespace kan {

// rows [n_img*Ho*Wo][C*K*K], column c*K*K + ky*K + kx; out-of-image taps 0.0
__global__ void __launch_bounds__(256) kan_im2col_f32_kernel(const float* __restrict__ in, int64_t n_img, int C,
                                                             int H, int W, int K, int stride, int pad, int Ho,
                                                             int Wo, float* __restrict__ out) {
  const int ncol = C * K * K;
  const int64_t total = n_img * Ho * Wo * static_cast<int64_t>(ncol);
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int col = static_cast<int>(t % ncol);
    const int64_t rowi = t / ncol;
    const int ox = static_cast<int>(rowi % Wo);
    const int oy = static_cast<int>((rowi / Wo) % Ho);
    const int64_t img = rowi / (static_cast<int64_t>(Wo) * Ho);
    const int c = col / (K * K), kk = col % (K * K), ky = kk / K, kx = kk % K;
    const int iy = oy * stride + ky - pad, ix = ox * stride + kx - pad;
    out[t] = (iy >= 0 && iy < H && ix >= 0 && ix < W) ? in[((img * C + c) * H + iy) * W + ix] : 0.f;
  }
}

// rows [n_img*HW][N] -> NCHW [n_img][N][HW] (convkan_forward's reshape, layers.hpp:179-184)
__global__ void __launch_bounds__(256) kan_rows_to_nchw_kernel(const float* __restrict__ rows, int64_t n_img,
                                                               int HW, int N, float* __restrict__ out) {
  const int64_t total = n_img * HW * static_cast<int64_t>(N);
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int p = static_cast<int>(t % HW);
    const int64_t q = t / HW;
    const int j = static_cast<int>(q % N);
    const int64_t img = q / N;
    out[t] = rows[(img * HW + p) * N + j];
  }
}

// maxpool2 (layers.hpp:193-205) on NCHW fp32 planes
__global__ void __launch_bounds__(256) kan_maxpool_f32_kernel(const float* __restrict__ in, int64_t planes, int H,
                                                              int W, int win, float* __restrict__ out) {
  const int Ho = H / win, Wo = W / win;
  const int64_t total = planes * Ho * Wo;
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t pl = t / (Ho * Wo);
    const int q = static_cast<int>(t % (Ho * Wo));
    const int oy = q / Wo, ox = q % Wo;
    const float* src = in + pl * H * W + static_cast<int64_t>(oy * win) * W + ox * win;
    float m = src[0];
    for (int dy = 0; dy < win; ++dy)
      for (int dx = 0; dx < win; ++dx) m = fmaxf(m, src[dy * W + dx]);
    out[t] = m;
  }
}

static unsigned fp_blocks(int64_t n) {
  const int64_t b = (n + 255) / 256;
  return static_cast<unsigned>(b < 148 * 32 ? b : 148 * 32);
}

cudaError_t launch_im2col_f32(const float* in, int64_t n_img, int C, int H, int W, int K, int stride, int pad, int Ho,
                              int Wo, float* out, cudaStream_t st) {
  const int64_t n = n_img * Ho * Wo * static_cast<int64_t>(C) * K * K;
  if (n == 0) return cudaSuccess;
  kan_im2col_f32_kernel<<<fp_blocks(n), 256, 0, st>>>(in, n_img, C, H, W, K, stride, pad, Ho, Wo, out);
  return cudaGetLastError();
}

cudaError_t launch_rows_to_nchw(const float* rows, int64_t n_img, int HW, int N, float* out, cudaStream_t st) {
  const int64_t n = n_img * HW * static_cast<int64_t>(N);
  if (n == 0) return cudaSuccess;
  kan_rows_to_nchw_kernel<<<fp_blocks(n), 256, 0, st>>>(rows, n_img, HW, N, out);
  return cudaGetLastError();
}

cudaError_t launch_maxpool_f32(const float* in, int64_t planes, int H, int W, int win, float* out, cudaStream_t st) {
  const int64_t n = planes * (H / win) * (W / win);
  if (n == 0) return cudaSuccess;
  kan_maxpool_f32_kernel<<<fp_blocks(n), 256, 0, st>>>(in, planes, H, W, win, out);
  return cudaGetLastError();
}

}  // namespace kan
