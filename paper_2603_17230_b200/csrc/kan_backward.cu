// kan_backward.cu -- training backward of a linear KAN layer, fp32.
//
// Replaces the reference's training math (proj/include/kantize/train.hpp):
//   kan_linear_backward_with (:84-129)  -> kan_bw_dcoeffs_kernel, kan_bw_dinputs_kernel
//   basis_derivative_at_coord (:24-51)  -> bw_basis (degree P-1 triangle, differenced)
//   softmax_cross_entropy (:139-160)    -> kan_softmax_ce_kernel
// d_coeffs = B^T dY over the clamped activations' basis rows; d_inputs[m,i] =
// sum_k b'_k(x) (dY[m] . W[i*nb+k]), zero where clamp_to_domain moved x.  The
// basis is local (P+1 non-zeros), so both are scatter/gather loops over the
// support instead of dense GEMMs; fp32 throughout (held to 1e-4 of the fp64
// reference).
#include <cuda_runtime.h>

#include <cstdint>

namespace kan {

struct BwParams {
  int64_t M;
  int n_in, n_out, G, P;
  const float* x;  // [M][ld_x]
  int64_t ld_x;
  const float* dy;  // [M][n_out]
  const float* w;   // [n_in*nb][n_out] (reference layout)
  float* dcoeffs;   // [n_in*nb][n_out]
  float* dinputs;   // [M][n_in] or null
  float lo, hi_open, inv_delta;
};

// Local basis of degree P at x (already clamped): N[r] = B_{j-P+r}, returns
// jj = j - P (first supported basis); with deriv, D[r] = B'_{j-P+r} in x units
// (degree P-1 triangle, (B_{i,P-1} - B_{i+1,P-1}) / delta, train.hpp:46-50).
__device__ __forceinline__ int bw_basis(float x, const BwParams& p, float (&N)[4], float (&D)[4], bool deriv) {
  const float xi = (x - p.lo) * p.inv_delta + static_cast<float>(p.P);
  int j = static_cast<int>(floorf(xi));
  j = min(max(j, p.P), p.G + p.P - 1);
  // triangle: T[q] at degree d holds B_{j-d+q}, q = 0..d
  float T[4] = {1.f, 0.f, 0.f, 0.f};
  float M[4] = {0.f, 0.f, 0.f, 0.f};  // degree P-1 values B_{j-P+1+q}
  for (int d = 1; d <= p.P; ++d) {
    if (d == p.P) {
#pragma unroll
      for (int q = 0; q < 4; ++q) M[q] = T[q];
    }
    const float rd = 1.0f / static_cast<float>(d);
    float U[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (q > d) break;
      const int i = j - d + q;
      const float left = q == 0 ? 0.f : T[q - 1];
      const float right = q == d ? 0.f : T[q];
      U[q] = ((xi - static_cast<float>(i)) * rd) * left + ((static_cast<float>(i + d + 1) - xi) * rd) * right;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) T[q] = U[q];
  }
  if (p.P == 0) M[0] = 0.f;
#pragma unroll
  for (int r = 0; r < 4; ++r) N[r] = r <= p.P ? T[r] : 0.f;
  if (deriv) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      // B'_{j-P+r} = (B_{j-P+r,P-1} - B_{j-P+r+1,P-1}) / delta, with M[q] = B_{j-P+1+q,P-1}
      const float a = (r >= 1 && r - 1 < p.P) ? M[r - 1] : 0.f;
      const float b = (r < p.P) ? M[r] : 0.f;
      D[r] = r <= p.P ? (a - b) * p.inv_delta : 0.f;
    }
  }
  return j - p.P;
}

// d_coeffs: CTA (input i, 128 outputs), thread j sums over the batch rows
__global__ void __launch_bounds__(128) kan_bw_dcoeffs_kernel(const BwParams p) {
  const int i = blockIdx.x;
  const int j = blockIdx.y * 128 + threadIdx.x;
  const int nb = p.G + p.P;
  float acc[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) acc[k] = 0.f;
  for (int64_t m = 0; m < p.M; ++m) {
    const float x = fminf(fmaxf(__ldg(p.x + m * p.ld_x + i), p.lo), p.hi_open);
    float N[4], D[4];
    const int jj = bw_basis(x, p, N, D, false);
    const float g = j < p.n_out ? __ldg(p.dy + m * p.n_out + j) : 0.f;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const int r = k - jj;
      const float b = r == 0 ? N[0] : (r == 1 ? N[1] : (r == 2 ? N[2] : (r == 3 ? N[3] : 0.f)));
      acc[k] = fmaf(b, g, acc[k]);
    }
  }
  if (j < p.n_out)
#pragma unroll
    for (int k = 0; k < 16; ++k)
      if (k < nb) p.dcoeffs[(static_cast<int64_t>(i) * nb + k) * p.n_out + j] = acc[k];
}

// d_inputs: thread per (m, i)
__global__ void __launch_bounds__(256) kan_bw_dinputs_kernel(const BwParams p) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= p.M * p.n_in) return;
  const int64_t m = t / p.n_in;
  const int i = static_cast<int>(t % p.n_in);
  const int nb = p.G + p.P;
  const float x = __ldg(p.x + m * p.ld_x + i);
  const float cx = fminf(fmaxf(x, p.lo), p.hi_open);
  if (cx != x) {  // the clamp blocks the gradient (train.hpp:113)
    p.dinputs[m * p.n_in + i] = 0.f;
    return;
  }
  float N[4], D[4];
  const int jj = bw_basis(cx, p, N, D, true);
  const float* g = p.dy + m * p.n_out;
  float acc = 0.f;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    if (r > p.P || jj + r >= nb || D[r] == 0.f) continue;
    const float* wr = p.w + (static_cast<int64_t>(i) * nb + jj + r) * p.n_out;
    float dot = 0.f;
    for (int j = 0; j < p.n_out; ++j) dot = fmaf(__ldg(wr + j), __ldg(g + j), dot);
    acc = fmaf(D[r], dot, acc);
  }
  p.dinputs[m * p.n_in + i] = acc;
}

// softmax_cross_entropy: per row loss (log-sum-exp) and dL/dlogits = (p - y) / M
__global__ void __launch_bounds__(256) kan_softmax_ce_kernel(const float* __restrict__ logits,
                                                             const int32_t* __restrict__ labels, int64_t M,
                                                             int n, float* __restrict__ loss_rows,
                                                             float* __restrict__ dlogits) {
  const int64_t m = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (m >= M) return;
  const float* row = logits + m * n;
  float mx = row[0];
  for (int j = 1; j < n; ++j) mx = fmaxf(mx, row[j]);
  float den = 0.f;
  for (int j = 0; j < n; ++j) den += expf(row[j] - mx);
  const int y = labels[m];
  loss_rows[m] = logf(den) - (row[y] - mx);
  const float inv_m = 1.0f / static_cast<float>(M);
  for (int j = 0; j < n; ++j) dlogits[m * n + j] = (expf(row[j] - mx) / den - (j == y ? 1.f : 0.f)) * inv_m;
}

// SGD with momentum on a layer's coefficients (train.hpp:361-366, 401-404):
// v = momentum * v - lr * g; w += v, in fp64 on the device-resident master
// copy (nothing fused, the reference's operation order), then the two fp32
// working copies: the reference layout [n_in * nb][N] the backward reads and
// the padded layout [(i * nbp + b) * Npad + j] the fp32 forward reads.
__global__ void kan_sgd_step_kernel(double* __restrict__ w, double* __restrict__ v, const float* __restrict__ g,
                                    float* __restrict__ w_bw, float* __restrict__ w32, long long n, int nb, int nbp,
                                    int N, int Npad, double lr, double momentum) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const double vn = __dsub_rn(__dmul_rn(momentum, v[i]), __dmul_rn(lr, static_cast<double>(g[i])));
    const double wn = __dadd_rn(w[i], vn);
    v[i] = vn;
    w[i] = wn;
    const float wf = static_cast<float>(wn);
    if (w_bw) w_bw[i] = wf;
    if (w32) {
      const long long r = i / N;  // = input * nb + basis
      const int j = static_cast<int>(i - r * N);
      const long long in = r / nb;
      const int b = static_cast<int>(r - in * nb);
      w32[(in * nbp + b) * Npad + j] = wf;
    }
  }
}

cudaError_t launch_sgd_step(double* w, double* v, const float* g, float* w_bw, float* w32, long long n, int nb,
                            int nbp, int N, int Npad, double lr, double momentum, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const unsigned blocks = static_cast<unsigned>(std::min<long long>((n + 255) / 256, 148 * 8));
  kan_sgd_step_kernel<<<blocks, 256, 0, st>>>(w, v, g, w_bw, w32, n, nb, nbp, N, Npad, lr, momentum);
  return cudaGetLastError();
}

cudaError_t launch_linear_backward(const BwParams& p, cudaStream_t st) {
  if (p.M == 0) return cudaSuccess;
  kan_bw_dcoeffs_kernel<<<dim3(static_cast<unsigned>(p.n_in), static_cast<unsigned>((p.n_out + 127) / 128)), 128, 0,
                          st>>>(p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || !p.dinputs) return e;
  const int64_t n = p.M * p.n_in;
  kan_bw_dinputs_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_softmax_ce(const float* logits, const int32_t* labels, int64_t M, int n, float* loss_rows,
                              float* dlogits, cudaStream_t st) {
  if (M == 0) return cudaSuccess;
  kan_softmax_ce_kernel<<<static_cast<unsigned>((M + 255) / 256), 256, 0, st>>>(logits, labels, M, n, loss_rows,
                                                                                  dlogits);
  return cudaGetLastError();
}

}  // namespace kan

// ---------------------------------------------------------------------------
// conv / pooling backward (train.hpp:367-431)
namespace kan {

// NCHW [n_img][N][HW] -> rows [n_img*HW][N]
__global__ void __launch_bounds__(256) kan_nchw_to_rows_kernel(const float* __restrict__ in, int64_t n_img, int HW,
                                                               int N, float* __restrict__ rows) {
  const int64_t total = n_img * HW * static_cast<int64_t>(N);
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int j = static_cast<int>(t % N);
    const int64_t r = t / N;
    const int p = static_cast<int>(r % HW);
    const int64_t img = r / HW;
    rows[t] = in[(img * N + j) * HW + p];
  }
}

// col2im_add (train.hpp:221-243) as a gather: every input pixel sums the
// patch-gradient entries that read it (deterministic, no atomics)
__global__ void __launch_bounds__(256) kan_col2im_kernel(const float* __restrict__ dpatch, int64_t n_img, int C,
                                                         int H, int W, int K, int stride, int pad, int Ho, int Wo,
                                                         float* __restrict__ din) {
  const int64_t total = n_img * C * static_cast<int64_t>(H) * W;
  const int ncol = C * K * K;
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int ix = static_cast<int>(t % W);
    const int iy = static_cast<int>((t / W) % H);
    const int c = static_cast<int>((t / (static_cast<int64_t>(W) * H)) % C);
    const int64_t img = t / (static_cast<int64_t>(W) * H * C);
    float acc = 0.f;
    for (int ky = 0; ky < K; ++ky) {
      const int ny = iy + pad - ky;
      if (ny < 0 || ny % stride) continue;
      const int oy = ny / stride;
      if (oy >= Ho) continue;
      for (int kx = 0; kx < K; ++kx) {
        const int nx = ix + pad - kx;
        if (nx < 0 || nx % stride) continue;
        const int ox = nx / stride;
        if (ox >= Wo) continue;
        acc += dpatch[((img * Ho + oy) * Wo + ox) * ncol + (c * K + ky) * K + kx];
      }
    }
    din[t] = acc;
  }
}

// maxpool2 backward (train.hpp:407-431): each output's gradient goes to the
// first strict maximum of its window (row-major scan); windows do not overlap
__global__ void __launch_bounds__(256) kan_maxpool_bw_kernel(const float* __restrict__ in, int64_t planes, int H,
                                                             int W, int win, const float* __restrict__ dout,
                                                             float* __restrict__ din) {
  const int Ho = H / win, Wo = W / win;
  const int64_t total = planes * Ho * Wo;
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t pl = t / (Ho * Wo);
    const int q = static_cast<int>(t % (Ho * Wo));
    const int y = q / Wo, x = q % Wo;
    const float* src = in + pl * H * W;
    int by = y * win, bx = x * win;
    float best = src[by * W + bx];
    for (int dy = 0; dy < win; ++dy)
      for (int dx = 0; dx < win; ++dx) {
        const float v = src[(y * win + dy) * W + x * win + dx];
        if (v > best) {
          best = v;
          by = y * win + dy;
          bx = x * win + dx;
        }
      }
    din[pl * H * W + by * W + bx] = dout[t];  // din zeroed by the launcher
  }
}

static unsigned bw_blocks(int64_t n) {
  const int64_t b = (n + 255) / 256;
  return static_cast<unsigned>(b < 148 * 32 ? b : 148 * 32);
}

cudaError_t launch_nchw_to_rows(const float* in, int64_t n_img, int HW, int N, float* rows, cudaStream_t st) {
  const int64_t n = n_img * HW * static_cast<int64_t>(N);
  if (n == 0) return cudaSuccess;
  kan_nchw_to_rows_kernel<<<bw_blocks(n), 256, 0, st>>>(in, n_img, HW, N, rows);
  return cudaGetLastError();
}

cudaError_t launch_col2im(const float* dpatch, int64_t n_img, int C, int H, int W, int K, int stride, int pad, int Ho,
                          int Wo, float* din, cudaStream_t st) {
  const int64_t n = n_img * C * static_cast<int64_t>(H) * W;
  if (n == 0) return cudaSuccess;
  kan_col2im_kernel<<<bw_blocks(n), 256, 0, st>>>(dpatch, n_img, C, H, W, K, stride, pad, Ho, Wo, din);
  return cudaGetLastError();
}

cudaError_t launch_maxpool_bw(const float* in, int64_t planes, int H, int W, int win, const float* dout, float* din,
                              cudaStream_t st) {
  const int64_t n_in = planes * H * static_cast<int64_t>(W);
  cudaError_t e = cudaMemsetAsync(din, 0, static_cast<size_t>(n_in) * sizeof(float), st);
  const int64_t n = planes * (H / win) * (W / win);
  if (e != cudaSuccess || n == 0) return e;
  kan_maxpool_bw_kernel<<<bw_blocks(n), 256, 0, st>>>(in, planes, H, W, win, dout, din);
  return cudaGetLastError();
}

}  // namespace kan
