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
#include <type_traits>

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
//   pass 2: fp32 T[(i*Lv + m)*(Np/4) + j] = v (fake-quant float tables; Np in bytes)
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
      } else if (pass == 2) {  // fake-quant float tables: the fp64 sample rounded once
        reinterpret_cast<float*>(T)[(static_cast<int64_t>(i) * Lv + m) * (Np / 4) + j] = __double2float_rn(acc);
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

// fake-quant float tables: a lane's 16-byte row slice is 4 fp32 columns
struct AccF {
  float a[4];
  __device__ __forceinline__ void clear_pk() {}
  __device__ __forceinline__ void add(const uint4 w) {
    a[0] += __uint_as_float(w.x);
    a[1] += __uint_as_float(w.y);
    a[2] += __uint_as_float(w.z);
    a[3] += __uint_as_float(w.w);
  }
  __device__ __forceinline__ void flush() {}
};

// L2 eviction-priority policies: the tables are re-read by every row and
// should stay L2-resident while the activation stream passes through
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// one 16-byte table row slice; L1 is bypassed (rows are rarely re-hit there)
__device__ __forceinline__ uint4 ldg_row(const uint8_t* p, uint64_t pol) {
  uint4 v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
      : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
      : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ float4 ldg_stream_f4(const float4* p, uint64_t pol) {
  float4 v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
      : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
      : "l"(p), "l"(pol));
  return v;
}

// Next-layer level of an integer sum v (v = sum - corr): quantize_value of
// s_out * v is monotone in v, so the host's exact integer thresholds
// vthr[n] = smallest v with level >= n settle an fp32 estimate (no fp64 divide).
__device__ __forceinline__ uint8_t st_level_of_sum(const StParams& p, int v) {
  int n = __float2int_rn(fmaf(static_cast<float>(v), p.ratio_f, p.zf));
  n = n < 0 ? 0 : (n > p.in_qhi ? static_cast<int>(p.in_qhi) : n);
  if (n > 0 && v < __ldg(p.vthr + n))
    --n;
  else if (n < p.in_qhi && v >= __ldg(p.vthr + n + 1))
    ++n;
  return static_cast<uint8_t>(n);
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
        if (p.epi == EPI_LEVEL)
          static_cast<uint8_t*>(p.out)[o] = st_level_of_sum(p, static_cast<int>(v));
        else
          static_cast<float*>(p.out)[o] = static_cast<float>(__dmul_rn(p.out_s, static_cast<double>(v)));
      }
    }
    return;
  }
  const int64_t o = r * p.ld_out + c0;
  if (p.epi == EPI_LEVEL) {
    uint8_t q[16];
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      q[t] = st_level_of_sum(p, static_cast<int>(static_cast<long long>(a[t]) - p.corr));
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

// Epilogue of one row's 4 fp32 columns (fake-quant float tables): fp32 values,
// or the next layer's input level of the value (exact fp32 thresholds)
__device__ __forceinline__ void st_epilogue_f(const StParams& p, int64_t r, int col0, const float (&a)[4]) {
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const int j = col0 + t;
    if (j >= p.n_out) break;
    int64_t o;
    if (p.conv) {
      const int64_t hw = static_cast<int64_t>(p.Ho) * p.Wo;
      o = ((r / hw) * p.n_out + j) * hw + r % hw;
    } else {
      o = r * p.ld_out + j;
    }
    if (p.epi == EPI_LEVEL)
      static_cast<uint8_t*>(p.out)[o] = static_cast<uint8_t>(st_level_f32(a[t], p.o_thr, p.o_inv_s, p.o_zf, p.o_qhi));
    else
      static_cast<float*>(p.out)[o] = a[t];
  }
}

// One spline-table layer.  A CTA of 256 threads runs RP rows at a time; each
// row is split over S input slices x lpr lanes (16 columns each, column tile
// blockIdx.y), so even a few thousand rows fill the GPU with independent
// gathers.  Dense rows: slice s owns the 4-input quads q = s mod S; its lanes
// read the quad's levels straight from the input row (one u32 of u8 levels, or
// one float4 of fp32 values whose levels the group's lanes split and exchange
// by shuffles) and issue eight 16-byte gathers per step (two quads).  Conv
// rows read the u8 NCHW input levels directly (implicit im2col, padded taps =
// level of 0.0); slice s owns channels c = s mod S.  The S partial sums of a
// row meet by warp shuffles when the row's lpr*S threads share a warp, else in
// shared memory.
// Raw input of one 4-input quad: fp32 values, or u8 levels in .x
template <bool F32>
__device__ __forceinline__ float4 st_quad_raw(const StParams& p, const void* xrow, int q) {
  if (!F32) {
    const uint8_t* xr = static_cast<const uint8_t*>(xrow);
    uint32_t w = 0;
    if (4 * q + 3 < p.n_in && (p.ld_x & 3) == 0) {
      w = __ldg(reinterpret_cast<const uint32_t*>(xr) + q);
    } else {
#pragma unroll
      for (int t = 0; t < 4; ++t)
        if (4 * q + t < p.n_in) w |= static_cast<uint32_t>(__ldg(xr + 4 * q + t)) << (8 * t);
    }
    return make_float4(__uint_as_float(w), 0.f, 0.f, 0.f);
  }
  const float* xr = static_cast<const float*>(xrow);
  if (4 * q + 3 < p.n_in && (p.ld_x & 3) == 0)
    return ldg_stream_f4(reinterpret_cast<const float4*>(xr) + q, l2_policy_evict_first());
  float v[4];
#pragma unroll
  for (int t = 0; t < 4; ++t) v[t] = 4 * q + t < p.n_in ? __ldg(xr + 4 * q + t) : 0.f;
  return make_float4(v[0], v[1], v[2], v[3]);
}

// The quad's four levels packed in a u32.  fp32 inputs: element t is
// quantized by lane t % lpr of the group (slot t / lpr) and exchanged by
// shuffles among the group's lanes (which share row, slice and trip count).
template <int LPR, bool F32>
__device__ __forceinline__ uint32_t st_quad_levels(const StParams& p, float4 f, int q, int lane,
                                                   const float* thr) {
  if (!F32) return __float_as_uint(f.x);
  constexpr int lpr = LPR;
  const float v[4] = {f.x, f.y, f.z, f.w};
  const int l = lane % lpr;
  int mine[4] = {0, 0, 0, 0};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int t = l + k * lpr;
    const float vt = t == 0 ? v[0] : (t == 1 ? v[1] : (t == 2 ? v[2] : v[3]));
    mine[k] = (t < 4 && 4 * q + t < p.n_in) ? st_level_f32(vt, thr, p.inv_s, p.zf, p.in_qhi) : 0;
    if (k * lpr + lpr >= 4) break;
  }
  if constexpr (lpr == 1) return mine[0] | (mine[1] << 8) | (mine[2] << 16) | (static_cast<uint32_t>(mine[3]) << 24);
  const int base = lane - l;
  const unsigned mask = (lpr == 32) ? 0xffffffffu : (((1u << lpr) - 1u) << base);
  uint32_t w = 0;
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const int src = base + (t % lpr);
    const int mv = lpr >= 4 ? mine[0] : (t / lpr == 0 ? mine[0] : mine[1]);  // lpr == 2: slots 0, 1
    const int lv = __shfl_sync(mask, mv, src);
    w |= static_cast<uint32_t>(lv) << (8 * t);
  }
  return w;
}

// KIND: 0 dense u8 levels, 1 dense fp32 values, 2 conv u8 NCHW.  FT: fp32
// tables (fake-quant mode): a lane's 16-byte slice is 4 fp32 columns summed in
// fp32, no output quantizer.
template <int LPR, int KIND, bool FT>
__global__ void __launch_bounds__(256, 3) kan_st_layer_kernel(const StParams p) {
  extern __shared__ __align__(16) uint8_t st_smem[];
  pdl_trigger();
  constexpr int lpr = LPR;
  constexpr bool F32 = KIND == 1;
  const int S = p.slices;
  const int RP = 256 / (lpr * S);
  const int lane = threadIdx.x & 31;
  const int l = threadIdx.x % lpr, s = (threadIdx.x / lpr) % S, g = threadIdx.x / (lpr * S);
  const int c0 = (static_cast<int>(blockIdx.y) * lpr + l) * 16;
  const bool col_ok = c0 < p.Np;
  int* red = reinterpret_cast<int*>(st_smem);                    // [8 warps][32][16] partial sums (S*lpr > 32)
  float* thr = reinterpret_cast<float*>(st_smem + 256 * 16 * 4);  // [qhi + 2]
  if (F32)
    for (int t = threadIdx.x; t <= p.in_qhi + 1; t += blockDim.x) thr[t] = p.thr[t];
  __syncthreads();
  const uint8_t* T = p.T + (col_ok ? c0 : 0);
  const int64_t row_stride = static_cast<int64_t>(p.Lv) * p.Np;  // bytes per input
  const uint64_t pol_t = l2_policy_evict_last();
  pdl_wait();
  for (int64_t rb = blockIdx.x; rb * RP < p.rows; rb += gridDim.x) {
    const int64_t r = rb * RP + g;
    const bool row_ok = r < p.rows;
    constexpr int NC = FT ? 4 : 16;  // columns per lane
    std::conditional_t<FT, AccF, Acc16> acc;
    acc.clear_pk();
#pragma unroll
    for (int t = 0; t < NC; ++t) acc.a[t] = 0;
    if constexpr (KIND != 2) {
      if (row_ok) {  // group-uniform: the lpr lanes of a (row, slice) share the trip count
        constexpr int esz = F32 ? 4 : 1;
        const uint8_t* xrow = static_cast<const uint8_t*>(p.x) + r * p.ld_x * esz;
        const int nq = (p.n_in + 3) >> 2;
        int q = s, since = 0;
        // the next step's inputs are loaded while this step's gathers are in flight
        float4 ra = q < nq ? st_quad_raw<F32>(p, xrow, q) : make_float4(0.f, 0.f, 0.f, 0.f);
        float4 rb2 = q + S < nq ? st_quad_raw<F32>(p, xrow, q + S) : make_float4(0.f, 0.f, 0.f, 0.f);
        for (; q + S < nq; q += 2 * S) {  // two quads in flight: eight 16-byte gathers
          const uint32_t la = st_quad_levels<LPR, F32>(p, ra, q, lane, thr);
          const uint32_t lb = st_quad_levels<LPR, F32>(p, rb2, q + S, lane, thr);
          if (q + 2 * S < nq) ra = st_quad_raw<F32>(p, xrow, q + 2 * S);
          if (q + 3 * S < nq) rb2 = st_quad_raw<F32>(p, xrow, q + 3 * S);
          const uint8_t* Ta = T + static_cast<int64_t>(4 * q) * row_stride;
          const uint8_t* Tb = T + static_cast<int64_t>(4 * (q + S)) * row_stride;
          uint4 w[8];
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            w[t] = ldg_row(Ta + t * row_stride + ((la >> (8 * t)) & 0xffu) * p.Np, pol_t);
            w[4 + t] = ldg_row(Tb + t * row_stride + ((lb >> (8 * t)) & 0xffu) * p.Np, pol_t);
          }
#pragma unroll
          for (int t = 0; t < 8; ++t) acc.add(w[t]);
          since += 2;
          if (since >= 62) {  // <= 256 inputs per flush: the 16-bit pairs cannot overflow
            acc.flush();
            since = 0;
          }
        }
        if (q < nq) {
          const uint32_t la = st_quad_levels<LPR, F32>(p, ra, q, lane, thr);
          const uint8_t* Ta = T + static_cast<int64_t>(4 * q) * row_stride;
          uint4 w[4];
#pragma unroll
          for (int t = 0; t < 4; ++t) w[t] = ldg_row(Ta + t * row_stride + ((la >> (8 * t)) & 0xffu) * p.Np, pol_t);
#pragma unroll
          for (int t = 0; t < 4; ++t) acc.add(w[t]);
        }
        acc.flush();
      }
    } else if (row_ok) {
      const int64_t hw = static_cast<int64_t>(p.Ho) * p.Wo;
      const int64_t img = r / hw, pp = r % hw;
      const int oy = static_cast<int>(pp / p.Wo), ox = static_cast<int>(pp % p.Wo);
      const int iy0 = oy * p.cstride - p.pad, ix0 = ox * p.cstride - p.pad;
      const uint8_t* xin = static_cast<const uint8_t*>(p.x) + img * p.C * static_cast<int64_t>(p.H) * p.W;
      const int kk = p.K * p.K;
      const int cpf = max(1, 256 / kk);  // own channels between flushes (<= 256 inputs)
      int since = 0;
      if (p.K == 3) {  // 3x3: tap offsets / padding masks hoisted, nine gathers in flight
        int off[9];
        bool ok[9];
#pragma unroll
        for (int t = 0; t < 9; ++t) {
          const int iy = iy0 + t / 3, ix = ix0 + t % 3;
          ok[t] = iy >= 0 && iy < p.H && ix >= 0 && ix < p.W;
          off[t] = ok[t] ? iy * p.W + ix : 0;
        }
        const int64_t plane = static_cast<int64_t>(p.H) * p.W;
        for (int c = s; c < p.C; c += S) {
          const uint8_t* xc = xin + c * plane;
          const uint8_t* Ti = T + static_cast<int64_t>(c) * 9 * row_stride;
          int lv[9];
#pragma unroll
          for (int t = 0; t < 9; ++t) lv[t] = ok[t] ? __ldg(xc + off[t]) : p.lvl0;
          uint4 w[9];
#pragma unroll
          for (int t = 0; t < 9; ++t) w[t] = ldg_row(Ti + t * row_stride + lv[t] * p.Np, pol_t);
#pragma unroll
          for (int t = 0; t < 9; ++t) acc.add(w[t]);
          if (++since == 28) {  // 252 inputs per flush
            acc.flush();
            since = 0;
          }
        }
      } else {
        for (int c = s; c < p.C; c += S) {
          const uint8_t* xc = xin + static_cast<int64_t>(c) * p.H * p.W;
          const uint8_t* Ti = T + static_cast<int64_t>(c) * kk * row_stride;
          for (int ky = 0; ky < p.K; ++ky) {
            const int iy = iy0 + ky;
            const bool yok = iy >= 0 && iy < p.H;
            for (int kx = 0; kx < p.K; ++kx) {
              const int ix = ix0 + kx;
              const int lv = (yok && ix >= 0 && ix < p.W) ? __ldg(xc + iy * p.W + ix) : p.lvl0;
              acc.add(ldg_row(Ti + lv * p.Np, pol_t));
              Ti += row_stride;
            }
            if (kk > 256) acc.flush();  // very large kernels: one flush per kernel row
          }
          if (++since == cpf) {
            acc.flush();
            since = 0;
          }
        }
      }
      acc.flush();
    }
    // the S slices of a row meet: warp shuffles over the slices inside a warp,
    // then (rows wider than a warp) shared memory across the row's warps
    if (S > 1) {
      const int span = lpr * S < 32 ? lpr * S : 32;
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1)
        if (o >= lpr && o < span)
#pragma unroll
          for (int t = 0; t < NC; ++t) acc.a[t] += __shfl_xor_sync(0xffffffffu, acc.a[t], o);
      if (lpr * S > 32) {
        const int wpr = lpr * S / 32;  // warps per row
        __syncthreads();
        if (lane < lpr) {
#pragma unroll
          for (int t = 0; t < NC; ++t)
            red[((threadIdx.x >> 5) * 32 + lane) * 16 + ((t + lane) & 15)] =
                (FT ? __float_as_int(static_cast<float>(acc.a[t])) : static_cast<int>(acc.a[t]));
        }
        __syncthreads();
        if (s == 0) {
          for (int o = 1; o < wpr; ++o) {
            const int src = ((threadIdx.x >> 5) + o) * 32 + lane;
#pragma unroll
            for (int t = 0; t < NC; ++t) {
              const int bits = red[src * 16 + ((t + lane) & 15)];
              if constexpr (FT)
                acc.a[t] += __int_as_float(bits);
              else
                acc.a[t] += bits;
            }
          }
        }
      }
    }
    if constexpr (KIND != 2 && !FT) {
      if (p.f_on) {  // fused output layer: the row's first warp (lpr * S >= 32) runs it
        if ((threadIdx.x % (lpr * S)) >= 32) continue;  // warp-uniform
        uint8_t* hid = st_smem + 256 * 16 * 4 + 258 * 4 + g * 512;
        if (s == 0 && col_ok) {
#pragma unroll
          for (int t = 0; t < 16; ++t)
            if (c0 + t < p.n_out) hid[c0 + t] = st_level_of_sum(p, static_cast<int>(acc.a[t] - p.corr));
        }
        __syncwarp();
        Acc16 acc2;
        acc2.clear_pk();
#pragma unroll
        for (int t = 0; t < 16; ++t) acc2.a[t] = 0;
        if (row_ok)
          for (int j = lane; j < p.f_n_in; j += 32)
            acc2.add(ldg_row(p.f_T + (static_cast<int64_t>(j) * p.f_Lv + hid[j]) * 16, pol_t));
        acc2.flush();  // <= 16 inputs per lane for n_in <= 512
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1)
#pragma unroll
          for (int t = 0; t < 16; ++t) acc2.a[t] += __shfl_xor_sync(0xffffffffu, acc2.a[t], o);
        if (lane < p.f_n_out && row_ok) {
          int v = acc2.a[0];
#pragma unroll
          for (int t = 1; t < 16; ++t) v = lane == t ? acc2.a[t] : v;
          p.f_out[r * p.f_ld_out + lane] =
              static_cast<float>(__dmul_rn(p.f_out_s, static_cast<double>(static_cast<long long>(v) - p.f_corr)));
        }
        __syncwarp();
        continue;
      }
    }
    if (s == 0 && row_ok && col_ok) {
      if constexpr (FT)
        st_epilogue_f(p, r, c0 / 4, acc.a);
      else
        st_epilogue(p, r, c0, acc.a);
    }
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

// evaluate_accuracy (eval.hpp:279-287): number of rows whose prediction equals the label
__global__ void __launch_bounds__(256) kan_count_equal_kernel(const int32_t* __restrict__ a,
                                                              const int32_t* __restrict__ b, int64_t n,
                                                              unsigned long long* count) {
  unsigned long long c = 0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    c += a[i] == b[i] ? 1ull : 0ull;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, c);
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

static int st_sm_count() { return device_sm_count(); }

cudaError_t launch_st_sample(const double* basis, const double* coeffs, int n_in, int n_out, int nb, int Lv,
                             int pass, unsigned long long* mm, uint8_t* T, int Np, double s, double zd,
                             long long qhi, cudaStream_t st) {
  const int64_t n = static_cast<int64_t>(n_in) * n_out;
  if (n == 0) return cudaSuccess;
  const size_t smem = static_cast<size_t>(Lv) * nb * sizeof(double);
  const dim3 grid(static_cast<unsigned>((n + 255) / 256));
  cudaError_t e;
  if (nb <= 16) {
    static std::atomic<unsigned long long> optin{0};
    if ((e = smem_optin(st_sample_kernel<16>, optin)) != cudaSuccess) return e;
    st_sample_kernel<16><<<grid, 256, smem, st>>>(basis, coeffs, n_in, n_out, nb, Lv, pass, mm, T, Np, s, zd, qhi);
  } else if (nb <= 32) {
    static std::atomic<unsigned long long> optin{0};
    if ((e = smem_optin(st_sample_kernel<32>, optin)) != cudaSuccess) return e;
    st_sample_kernel<32><<<grid, 256, smem, st>>>(basis, coeffs, n_in, n_out, nb, Lv, pass, mm, T, Np, s, zd, qhi);
  } else {
    return cudaErrorInvalidValue;  // the engine rejects G+P > 32 in spline-table mode
  }
  return cudaGetLastError();
}

size_t st_layer_smem(const StParams& p) {
  return 256 * 16 * sizeof(int) + 258 * sizeof(float) + (p.f_on ? 8 * 512 : 0);
}

template <int LPR, int KIND, bool FT>
static cudaError_t launch_st_layer_t(const StParams& p, dim3 grid, size_t smem, cudaStream_t st) {
  auto kfn = kan_st_layer_kernel<LPR, KIND, FT>;
  static std::atomic<unsigned long long> optin{0};  // per instantiation, per device
  if (cudaError_t e = smem_optin(kfn, optin); e != cudaSuccess) return e;
  return st_launch(kfn, grid, dim3(256), smem, st, p);
}

template <int KIND, bool FT>
static cudaError_t launch_st_kind(const StParams& p, dim3 grid, size_t smem, cudaStream_t st) {
  switch (p.lpr) {
    case 1: return launch_st_layer_t<1, KIND, FT>(p, grid, smem, st);
    case 2: return launch_st_layer_t<2, KIND, FT>(p, grid, smem, st);
    case 4: return launch_st_layer_t<4, KIND, FT>(p, grid, smem, st);
    case 8: return launch_st_layer_t<8, KIND, FT>(p, grid, smem, st);
    case 16: return launch_st_layer_t<16, KIND, FT>(p, grid, smem, st);
    case 32: return launch_st_layer_t<32, KIND, FT>(p, grid, smem, st);
    default: return cudaErrorInvalidValue;
  }
}

template <bool FT>
static cudaError_t launch_st_ft(const StParams& p, dim3 grid, size_t smem, cudaStream_t st) {
  if (p.conv) return launch_st_kind<2, FT>(p, grid, smem, st);
  return p.in_kind == ST_IN_F32 ? launch_st_kind<1, FT>(p, grid, smem, st) : launch_st_kind<0, FT>(p, grid, smem, st);
}

cudaError_t launch_st_layer(const StParams& p, cudaStream_t st) {
  if (p.rows == 0) return cudaSuccess;
  const size_t smem = st_layer_smem(p);
  const int RP = 256 / (p.lpr * p.slices);
  const int64_t blocks = (p.rows + RP - 1) / RP;
  const int64_t cap = static_cast<int64_t>(st_sm_count()) * 8;
  const dim3 grid(static_cast<unsigned>(blocks < cap ? blocks : cap), static_cast<unsigned>(p.col_tiles));
  return p.ft ? launch_st_ft<true>(p, grid, smem, st) : launch_st_ft<false>(p, grid, smem, st);
}

cudaError_t launch_st_levels(const float* x, int64_t n, const float* thr, float inv_s, float zf, int qhi,
                             void* out, int out_u16, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  const int64_t blocks = (n + 255) / 256;
  const int64_t cap = static_cast<int64_t>(st_sm_count()) * 16;
  return st_launch(kan_st_levels_kernel, dim3(static_cast<unsigned>(blocks < cap ? blocks : cap)), dim3(256), 0,
                   st, x, n, thr, inv_s, zf, qhi, out, out_u16);
}

cudaError_t launch_count_equal(const int32_t* a, const int32_t* b, int64_t n, unsigned long long* count,
                               cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(count, 0, sizeof(unsigned long long), st);
  if (e != cudaSuccess || n == 0) return e;
  const int64_t blocks = (n + 255) / 256;
  kan_count_equal_kernel<<<static_cast<unsigned>(blocks < 1184 ? blocks : 1184), 256, 0, st>>>(a, b, n, count);
  return cudaGetLastError();
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
