// kan_spline_table.cu -- spline-table mode: per-connection table gather + integer add.
//
// Replaces the reference's EvalMode::kSplineTable path (proj/include/kantize/
// spline_table.hpp):
//   build_spline_tables  (:38-95)   -> st_sample_kernel (two passes, fp64)
//   spline_table_forward (:90-107)  -> kan_st_layer_kernel (linear rows)
//   spline_table_forward (:110-123) -> kan_st_layer_kernel (conv, implicit im2col)
//
// Table build.  Every spline phi_{i,j} is sampled at the 2^bits_a dequantized
// input levels in fp64 with the reference's operation order (basis from the
// host, acc += basis[k] * coeff[i*nb+k][j] in k order with explicit
// __dmul_rn/__dadd_rn, so nothing is contracted into an FMA).  Pass 0 folds the
// layer's min/max (ordered-integer atomics; the fold is order-free), the host
// derives the zero-spanning h-bit quantizer exactly as RangeCalibrator +
// zero_spanning + compute_quant_params do, and pass 1 re-evaluates the same
// samples and writes llround(v / s + z) (correctly rounded __ddiv_rn) clamped
// to [0, 2^h - 1].  The device layout is [i][level][Np] (Np = n_out padded to
// 16): the row one activation selects is Np contiguous bytes.
//
// Forward.  out[m, j] = s_out * sum_i (T[i][level(m,i)][j] - z_out): a lane
// owns 16 output columns (one 16-byte row slice per input), adds the bytes as
// packed 16-bit pairs (byte_perm + IADD, flushed to int32 every <= 256 inputs,
// so no lane can overflow: 256 * 255 < 65536), and the integer sum is exact in
// any order.  Hidden outputs leave as the next layer's u8 input levels
// (quantize_value of the fp64 output, correctly rounded), the model output as
// fp32.  The hot loop is one 16-byte L1/L2 gather plus 16 integer ops per
// (row, input, 16 columns): gather-bound, no tensor cores.
#include <cuda_runtime.h>

#include <cstdint>

#include "kan_internal.h"
#include "kan_ptx.cuh"

namespace kan {

// ordered-integer encoding of doubles: key order == value order (NaN excluded)
__device__ __forceinline__ unsigned long long dkey(double v) {
  const unsigned long long u = static_cast<unsigned long long>(__double_as_longlong(v));
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

// Samples of phi_{i,j} at every input level, thread per (i, j).
//   pass 0: min/max fold into mm[0] (min key) / mm[1] (max key)
//   pass 1: T[(i*Lv + m)*Np + j] = clamp(llround(v / s + z), 0, qhi)
template <int NBMAX>
__global__ void __launch_bounds__(256) st_sample_kernel(const double* __restrict__ basis,
                                                        const double* __restrict__ coeffs, int n_in,
                                                        int n_out, int nb, int Lv, int pass,
                                                        unsigned long long* mm, uint8_t* __restrict__ T,
                                                        int Np, double s, double zd, long long qhi) {
  extern __shared__ double sb[];  // basis [Lv][nb]
  for (int t = threadIdx.x; t < Lv * nb; t += blockDim.x) sb[t] = basis[t];
  __syncthreads();
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const bool ok = idx < static_cast<int64_t>(n_in) * n_out;
  unsigned long long kmin = ~0ull, kmax = 0ull;
  if (ok) {
    const int i = static_cast<int>(idx / n_out), j = static_cast<int>(idx % n_out);
    double w[NBMAX];
#pragma unroll
    for (int k = 0; k < NBMAX; ++k)
      w[k] = k < nb ? coeffs[(static_cast<int64_t>(i) * nb + k) * n_out + j] : 0.0;
    for (int m = 0; m < Lv; ++m) {
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < NBMAX; ++k)
        if (k < nb) acc = __dadd_rn(acc, __dmul_rn(sb[m * nb + k], w[k]));
      if (pass == 0) {
        if (acc == acc) {  // NaN never wins std::min / std::max against a number
          const unsigned long long key = dkey(acc);
          kmin = key < kmin ? key : kmin;
          kmax = key > kmax ? key : kmax;
        }
      } else {
        long long q = llround(__dadd_rn(__ddiv_rn(acc, s), zd));
        q = q < 0 ? 0 : (q > qhi ? qhi : q);
        T[(static_cast<int64_t>(i) * Lv + m) * Np + j] = static_cast<uint8_t>(q);
      }
    }
  }
  if (pass == 0) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long a = __shfl_xor_sync(0xffffffffu, kmin, o);
      const unsigned long long b = __shfl_xor_sync(0xffffffffu, kmax, o);
      kmin = a < kmin ? a : kmin;
      kmax = b > kmax ? b : kmax;
    }
    if ((threadIdx.x & 31) == 0 && kmin != ~0ull) {
      atomicMin(&mm[0], kmin);
      atomicMax(&mm[1], kmax);
    }
  }
}

// quantize_value(x, in_qp) of an fp32 activation through exact thresholds:
// thr[n] = smallest fp32 x with level >= n (n = 1..Lv-1).  The fp32 estimate
// is within one level of the exact fp64 rounding, the thresholds settle it.
// x >= ovf (thr[qhi+1]) overflows llround on the reference's x86-64 build,
// whose out-of-range result (LLONG_MIN) clamps to level 0, as NaN does.
__device__ __forceinline__ int st_level_f32(float x, const float* thr, float inv_s, float zf, int qhi) {
  if (!(x < thr[qhi + 1])) return 0;
  int n = __float2int_rn(fmaf(x, inv_s, zf));
  n = n < 0 ? 0 : (n > qhi ? qhi : n);
  if (n > 0 && x < thr[n])
    --n;
  else if (n < qhi && x >= thr[n + 1])
    ++n;
  return n;
}

// level of the fp64 layer output y under the consumer's quantizer
__device__ __forceinline__ uint8_t st_level_f64(double y, double in_s, double in_zd, long long qhi) {
  const double v = __dadd_rn(__ddiv_rn(y, in_s), in_zd);
  if (!(v < 9223372036854775808.0)) return 0;  // NaN / llround overflow -> LLONG_MIN -> q_lo
  long long q = llround(v);
  return static_cast<uint8_t>(q < 0 ? 0 : (q > qhi ? qhi : q));
}

struct Acc16 {
  uint32_t pk[8];  // packed 16-bit pairs: pk[2t] = (b0, b1), pk[2t+1] = (b2, b3) of word t
  int a[16];
  __device__ __forceinline__ void clear_pk() {
#pragma unroll
    for (int t = 0; t < 8; ++t) pk[t] = 0u;
  }
  __device__ __forceinline__ void add(const uint4 w) {
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      pk[2 * t] += __byte_perm(ws[t], 0u, 0x4140);
      pk[2 * t + 1] += __byte_perm(ws[t], 0u, 0x4342);
    }
  }
  __device__ __forceinline__ void flush() {
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      a[4 * t + 0] += static_cast<int>(pk[2 * t] & 0xffffu);
      a[4 * t + 1] += static_cast<int>(pk[2 * t] >> 16);
      a[4 * t + 2] += static_cast<int>(pk[2 * t + 1] & 0xffffu);
      a[4 * t + 3] += static_cast<int>(pk[2 * t + 1] >> 16);
    }
    clear_pk();
  }
};

__device__ __forceinline__ uint4 ldg_row(const uint8_t* p) {
  return __ldg(reinterpret_cast<const uint4*>(p));
}

// Epilogue of one row's 16 columns.
__device__ __forceinline__ void st_epilogue(const StParams& p, int64_t r, int c0, const int (&a)[16]) {
  if (p.conv) {
    const int64_t hw = static_cast<int64_t>(p.Ho) * p.Wo;
    const int64_t img = r / hw, pp = r % hw;
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      const int j = c0 + t;
      if (j >= p.n_out) break;
      const long long v = static_cast<long long>(a[t]) - p.corr;
      const int64_t o = (img * p.n_out + j) * hw + pp;
      if (p.epi == EPI_RAW) {
        static_cast<int*>(p.out)[o] = static_cast<int>(v);
      } else {
        const double y = __dmul_rn(p.out_s, static_cast<double>(v));
        if (p.epi == EPI_LEVEL)
          static_cast<uint8_t*>(p.out)[o] = st_level_f64(y, p.in_s, p.in_zd, p.in_qhi);
        else
          static_cast<float*>(p.out)[o] = static_cast<float>(y);
      }
    }
    return;
  }
  const int64_t o = r * p.ld_out + c0;
  if (p.epi == EPI_LEVEL) {
    uint8_t q[16];
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      const long long v = static_cast<long long>(a[t]) - p.corr;
      q[t] = st_level_f64(__dmul_rn(p.out_s, static_cast<double>(v)), p.in_s, p.in_zd, p.in_qhi);
    }
    uint8_t* dst = static_cast<uint8_t*>(p.out) + o;
    if (c0 + 16 <= p.n_out && (p.ld_out & 15) == 0) {
      uint4 w;
      w.x = q[0] | (q[1] << 8) | (q[2] << 16) | (static_cast<uint32_t>(q[3]) << 24);
      w.y = q[4] | (q[5] << 8) | (q[6] << 16) | (static_cast<uint32_t>(q[7]) << 24);
      w.z = q[8] | (q[9] << 8) | (q[10] << 16) | (static_cast<uint32_t>(q[11]) << 24);
      w.w = q[12] | (q[13] << 8) | (q[14] << 16) | (static_cast<uint32_t>(q[15]) << 24);
      *reinterpret_cast<uint4*>(dst) = w;
    } else {
#pragma unroll
      for (int t = 0; t < 16; ++t)
        if (c0 + t < p.n_out) dst[t] = q[t];
    }
  } else if (p.epi == EPI_RAW) {
    int* dst = static_cast<int*>(p.out) + o;
#pragma unroll
    for (int t = 0; t < 16; ++t)
      if (c0 + t < p.n_out) dst[t] = static_cast<int>(static_cast<long long>(a[t]) - p.corr);
  } else {
    float y[16];
#pragma unroll
    for (int t = 0; t < 16; ++t)
      y[t] = static_cast<float>(__dmul_rn(p.out_s, static_cast<double>(static_cast<long long>(a[t]) - p.corr)));
    float* dst = static_cast<float*>(p.out) + o;
    if (c0 + 16 <= p.n_out && (p.ld_out & 3) == 0) {
#pragma unroll
      for (int t = 0; t < 4; ++t)
        reinterpret_cast<float4*>(dst)[t] = make_float4(y[4 * t], y[4 * t + 1], y[4 * t + 2], y[4 * t + 3]);
    } else {
#pragma unroll
      for (int t = 0; t < 16; ++t)
        if (c0 + t < p.n_out) dst[t] = y[t];
    }
  }
}

// One spline-table layer.  A CTA of 256 threads runs RP = 256 / lpr rows at a
// time, lpr lanes per row, each lane 16 columns of column tile blockIdx.y.
// Dense rows stage their input levels (u8 rows, or fp32 rows quantized on the
// way in) in shared memory, IC inputs at a time; conv rows read the u8 NCHW
// input levels directly (implicit im2col, padded taps = level of 0.0).
__global__ void __launch_bounds__(256) kan_st_layer_kernel(const StParams p) {
  extern __shared__ __align__(16) uint8_t st_smem[];
  pdl_trigger();
  const int lpr = p.lpr;
  const int RP = 256 / lpr;
  const int g = threadIdx.x / lpr, l = threadIdx.x % lpr;
  const int c0 = (static_cast<int>(blockIdx.y) * lpr + l) * 16;
  const bool col_ok = c0 < p.Np;
  const int IC = p.ic;
  const int lds = IC + 4;  // staged row pitch (odd word count: conflict-free)
  float* thr = reinterpret_cast<float*>(st_smem + RP * lds);
  if (p.in_kind == ST_IN_F32)
    for (int t = threadIdx.x; t <= p.in_qhi + 1; t += blockDim.x) thr[t] = p.thr[t];
  const uint8_t* T = p.T + (col_ok ? c0 : 0);
  const int64_t row_stride = static_cast<int64_t>(p.Lv) * p.Np;  // bytes per input
  pdl_wait();
  for (int64_t rb = blockIdx.x; rb * RP < p.rows; rb += gridDim.x) {
    const int64_t r = rb * RP + g;
    const bool row_ok = r < p.rows;
    Acc16 acc;
    acc.clear_pk();
#pragma unroll
    for (int t = 0; t < 16; ++t) acc.a[t] = 0;
    if (!p.conv) {
      for (int i0 = 0; i0 < p.n_in; i0 += IC) {
        const int cnt = min(IC, p.n_in - i0);
        __syncthreads();  // the previous chunk's levels are consumed
        if (p.in_kind == ST_IN_F32) {
          const float* x = static_cast<const float*>(p.x);
          for (int t = threadIdx.x; t < RP * IC; t += blockDim.x) {
            const int rr = t / IC, ii = t % IC;
            const int64_t row = rb * RP + rr;
            int lv = 0;
            if (ii < cnt && row < p.rows)
              lv = st_level_f32(x[row * p.ld_x + i0 + ii], thr, p.inv_s, p.zf, p.in_qhi);
            st_smem[rr * lds + ii] = static_cast<uint8_t>(lv);
          }
        } else {
          const uint8_t* x = static_cast<const uint8_t*>(p.x);
          for (int t = threadIdx.x; t < RP * IC; t += blockDim.x) {
            const int rr = t / IC, ii = t % IC;
            const int64_t row = rb * RP + rr;
            st_smem[rr * lds + ii] = (ii < cnt && row < p.rows) ? x[row * p.ld_x + i0 + ii] : 0;
          }
        }
        __syncthreads();
        if (row_ok && col_ok) {
          const uint8_t* lv = st_smem + g * lds;
          const uint8_t* Ti = T + static_cast<int64_t>(i0) * row_stride;
          int ii = 0;
          for (; ii + 4 <= cnt; ii += 4) {
            const uint32_t l4 = *reinterpret_cast<const uint32_t*>(lv + ii);
            const uint4 w0 = ldg_row(Ti + (l4 & 0xffu) * p.Np);
            const uint4 w1 = ldg_row(Ti + row_stride + ((l4 >> 8) & 0xffu) * p.Np);
            const uint4 w2 = ldg_row(Ti + 2 * row_stride + ((l4 >> 16) & 0xffu) * p.Np);
            const uint4 w3 = ldg_row(Ti + 3 * row_stride + (l4 >> 24) * p.Np);
            acc.add(w0);
            acc.add(w1);
            acc.add(w2);
            acc.add(w3);
            Ti += 4 * row_stride;
          }
          for (; ii < cnt; ++ii) {
            acc.add(ldg_row(Ti + lv[ii] * p.Np));
            Ti += row_stride;
          }
          acc.flush();  // IC <= 256 inputs per chunk
        }
      }
    } else if (row_ok && col_ok) {
      const int64_t hw = static_cast<int64_t>(p.Ho) * p.Wo;
      const int64_t img = r / hw, pp = r % hw;
      const int oy = static_cast<int>(pp / p.Wo), ox = static_cast<int>(pp % p.Wo);
      const int iy0 = oy * p.cstride - p.pad, ix0 = ox * p.cstride - p.pad;
      const uint8_t* xin = static_cast<const uint8_t*>(p.x) + img * p.C * static_cast<int64_t>(p.H) * p.W;
      const uint8_t* Ti = T;
      const int kk = p.K * p.K;
      const int cpf = max(1, 256 / kk);  // channels between flushes (<= 256 inputs)
      for (int c = 0; c < p.C; ++c) {
        const uint8_t* xc = xin + static_cast<int64_t>(c) * p.H * p.W;
        for (int ky = 0; ky < p.K; ++ky) {
          const int iy = iy0 + ky;
          const bool yok = iy >= 0 && iy < p.H;
          for (int kx = 0; kx < p.K; ++kx) {
            const int ix = ix0 + kx;
            const int lv = (yok && ix >= 0 && ix < p.W) ? __ldg(xc + iy * p.W + ix) : p.lvl0;
            acc.add(ldg_row(Ti + lv * p.Np));
            Ti += row_stride;
          }
          if (kk > 256) acc.flush();  // very large kernels: one flush per kernel row
        }
        if ((c + 1) % cpf == 0) acc.flush();
      }
      acc.flush();
    }
    if (row_ok && col_ok) st_epilogue(p, r, c0, acc.a);
  }
}

// fp32 -> u8 input levels (the NCHW model input of a conv model; parity probes)
__global__ void __launch_bounds__(256) kan_st_levels_kernel(const float* __restrict__ x, int64_t n,
                                                            const float* __restrict__ thr_g, float inv_s,
                                                            float zf, int qhi, void* __restrict__ out,
                                                            int out_u16) {
  __shared__ float thr[258];
  pdl_trigger();
  for (int t = threadIdx.x; t <= qhi + 1; t += blockDim.x) thr[t] = thr_g[t];
  __syncthreads();
  pdl_wait();
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int lv = st_level_f32(x[i], thr, inv_s, zf, qhi);
    if (out_u16)
      static_cast<uint16_t*>(out)[i] = static_cast<uint16_t>(lv);
    else
      static_cast<uint8_t*>(out)[i] = static_cast<uint8_t>(lv);
  }
}

// u16 -> u8 levels (parity probe input)
__global__ void kan_u16_to_u8_kernel(const uint16_t* __restrict__ in, int64_t n, uint8_t* __restrict__ out) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = static_cast<uint8_t>(in[i]);
}

// maxpool2 (layers.hpp:193-205) over u8 NCHW levels: the level is monotone in
// the value, so the max of levels is the level of the max
__global__ void __launch_bounds__(256) kan_st_maxpool_kernel(const uint8_t* __restrict__ in, int64_t planes,
                                                             int H, int W, int win, uint8_t* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  const int Ho = H / win, Wo = W / win;
  const int64_t n = planes * Ho * Wo;
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < n;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t pl = t / (Ho * Wo);
    const int q = static_cast<int>(t % (Ho * Wo));
    const int oy = q / Wo, ox = q % Wo;
    const uint8_t* src = in + pl * H * W + static_cast<int64_t>(oy * win) * W + ox * win;
    uint8_t m = 0;
    for (int dy = 0; dy < win; ++dy)
      for (int dx = 0; dx < win; ++dx) {
        const uint8_t v = src[dy * W + dx];
        m = v > m ? v : m;
      }
    out[t] = m;
  }
}

// ---------------------------------------------------------------------------
// host-side launchers (called from kan_engine.cpp)

template <class... KArgs, class... Args>
static cudaError_t st_launch(void (*kfn)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                             Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kfn, std::forward<Args>(args)...);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

static int st_sm_count() {
  static int n_sm = 0;
  if (n_sm == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    if (n_sm <= 0) n_sm = 148;
  }
  return n_sm;
}

cudaError_t launch_st_sample(const double* basis, const double* coeffs, int n_in, int n_out, int nb, int Lv,
                             int pass, unsigned long long* mm, uint8_t* T, int Np, double s, double zd,
                             long long qhi, cudaStream_t st) {
  const int64_t n = static_cast<int64_t>(n_in) * n_out;
  if (n == 0) return cudaSuccess;
  const size_t smem = static_cast<size_t>(Lv) * nb * sizeof(double);
  const dim3 grid(static_cast<unsigned>((n + 255) / 256));
  cudaError_t e;
  if (nb <= 16) {
    e = cudaFuncSetAttribute(st_sample_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    st_sample_kernel<16><<<grid, 256, smem, st>>>(basis, coeffs, n_in, n_out, nb, Lv, pass, mm, T, Np, s, zd, qhi);
  } else if (nb <= 32) {
    e = cudaFuncSetAttribute(st_sample_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    st_sample_kernel<32><<<grid, 256, smem, st>>>(basis, coeffs, n_in, n_out, nb, Lv, pass, mm, T, Np, s, zd, qhi);
  } else {
    return cudaErrorInvalidValue;  // the engine rejects G+P > 32 in spline-table mode
  }
  return cudaGetLastError();
}

size_t st_layer_smem(const StParams& p) {
  const int RP = 256 / p.lpr;
  return static_cast<size_t>(RP) * (p.ic + 4) + 258 * sizeof(float);
}

cudaError_t launch_st_layer(const StParams& p, cudaStream_t st) {
  if (p.rows == 0) return cudaSuccess;
  const size_t smem = st_layer_smem(p);
  static size_t configured = 0;
  if (smem > configured) {
    cudaError_t e = cudaFuncSetAttribute(kan_st_layer_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  const int RP = 256 / p.lpr;
  const int64_t blocks = (p.rows + RP - 1) / RP;
  const int64_t cap = static_cast<int64_t>(st_sm_count()) * 8;
  const dim3 grid(static_cast<unsigned>(blocks < cap ? blocks : cap), static_cast<unsigned>(p.col_tiles));
  return st_launch(kan_st_layer_kernel, grid, dim3(256), smem, st, p);
}

cudaError_t launch_st_levels(const float* x, int64_t n, const float* thr, float inv_s, float zf, int qhi,
                             void* out, int out_u16, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  const int64_t blocks = (n + 255) / 256;
  const int64_t cap = static_cast<int64_t>(st_sm_count()) * 16;
  return st_launch(kan_st_levels_kernel, dim3(static_cast<unsigned>(blocks < cap ? blocks : cap)), dim3(256), 0,
                   st, x, n, thr, inv_s, zf, qhi, out, out_u16);
}

cudaError_t launch_u16_to_u8(const uint16_t* in, int64_t n, uint8_t* out, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  const int64_t blocks = (n + 255) / 256;
  kan_u16_to_u8_kernel<<<static_cast<unsigned>(blocks < 4096 ? blocks : 4096), 256, 0, st>>>(in, n, out);
  return cudaGetLastError();
}

cudaError_t launch_st_maxpool(const uint8_t* in, int64_t planes, int H, int W, int win, uint8_t* out,
                              cudaStream_t st) {
  const int64_t n = planes * (H / win) * (W / win);
  if (n == 0) return cudaSuccess;
  const int64_t blocks = (n + 255) / 256;
  const int64_t cap = static_cast<int64_t>(st_sm_count()) * 16;
  return st_launch(kan_st_maxpool_kernel, dim3(static_cast<unsigned>(blocks < cap ? blocks : cap)), dim3(256), 0,
                   st, in, planes, H, W, win, out);
}

}  // namespace kan
