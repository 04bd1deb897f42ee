/*
 * kan_oracle.c -- CPU restatement of the reference KAN-layer hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see kan_oracle.h).  Compiled with
 * -O2 -ffp-contract=off and no -march flags so every double operation is a
 * single IEEE-754 round-to-nearest step in the reference's order.
 *
 * Parity status: PINNED.  tests/test_oracle_pins.py checks this file
 * bit-for-bit against the reference compiled from /root/reference
 * (oracle/_ref/libkantize_ref.so, built by oracle/Makefile) and against the
 * committed golden vectors in tests/golden/ generated from that build.
 */
#include "kan_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* grid.hpp                                                                  */
/* ------------------------------------------------------------------------ */

/* build_grid, proj/include/kantize/grid.hpp:72-96 (delta = (hi-lo)/G, :82) */
int kor_grid_build(int G, int P, double lo, double hi, kor_grid* g) {
  if (G < 1 || P < 0 || !(hi > lo)) return -1;
  g->intervals = G;
  g->degree = P;
  g->lo = lo;
  g->hi = hi;
  g->delta = (hi - lo) / G;
  return 0;
}

/* GridSpec::knot_coord, grid.hpp:44 */
double kor_knot_coord(const kor_grid* g, double x) { return (x - g->lo) / g->delta + g->degree; }

/* GridSpec::clamp_to_domain, grid.hpp:49-56.  std::max(x, lo) is
 * (x < lo ? lo : x) and std::min(a, b) is (b < a ? b : a): NaN passes
 * through both, exactly as in libstdc++. */
double kor_clamp(const kor_grid* g, double x) {
  const double hi_open = nextafter(g->hi, g->lo);
  double t = (x < g->lo) ? g->lo : x;
  x = (hi_open < t) ? hi_open : t;
  if (g->degree == 0) {
    const double n0 = (double)(g->intervals + 2 * g->degree);
    while (x > g->lo && kor_knot_coord(g, x) >= n0) x = nextafter(x, g->lo);
  }
  return x;
}

/* detail::triangle + support_start_at + basis_at_coord, grid.hpp:124-172.
 * Row 0 holds the G+2P indicators plus one zero slot; row d updates entries
 * 0..n0-d with buf[i] = (d1*r)*buf[i] + (d2*r)*buf[i+1] (:130-137). */
int kor_basis_at_coord(const kor_grid* g, double xi, double* out) {
  const int P = g->degree;
  const int n0 = g->intervals + 2 * P;
  const int nb = g->intervals + P;
  double stackbuf[256];
  double* buf = (n0 + 1 <= 256) ? stackbuf : (double*)malloc(sizeof(double) * (size_t)(n0 + 1));
  for (int i = 0; i <= n0; ++i) buf[i] = 0.0;
  const double jf = floor(xi);
  if (jf >= 0.0 && jf < (double)n0) buf[(int)jf] = 1.0;
  for (int d = 1; d <= P; ++d) {
    const double r = 1.0 / d; /* GridSpec::recip, grid.hpp:94 */
    const int top = n0 - d;
    for (int i = 0; i <= top; ++i) {
      const double d1 = xi - i;
      const double d2 = (double)(i + d + 1) - xi;
      buf[i] = (d1 * r) * buf[i] + (d2 * r) * buf[i + 1];
    }
  }
  for (int i = 0; i < nb; ++i) out[i] = buf[i];
  if (buf != stackbuf) free(buf);
  /* support_start_at, grid.hpp:142-147 */
  if (jf < 0.0 || jf >= (double)n0) return 0;
  int j = (int)jf - P;
  if (j < 0) j = 0;
  if (j > nb - 1) j = nb - 1;
  return j;
}

/* ------------------------------------------------------------------------ */
/* quant.hpp                                                                 */
/* ------------------------------------------------------------------------ */

/* compute_quant_params, quant.hpp:33-49 */
int kor_quant_params(double alpha, double beta, int bits, double* scale, int64_t* zero_point,
                     int64_t* q_hi) {
  if (bits < 1 || bits > 8) return -1;
  if (!(beta > alpha)) return -1;
  const int64_t qlo = 0, qhi = ((int64_t)1 << bits) - 1;
  *scale = (beta - alpha) / (double)(qhi - qlo);
  *zero_point = llround((beta * (double)qlo - alpha * (double)qhi) / (beta - alpha));
  *q_hi = qhi;
  return 0;
}

/* quantize_value, quant.hpp:51-54: llround(x/scale + zp), clamped */
int64_t kor_quantize(double x, double scale, int64_t zp, int64_t q_lo, int64_t q_hi) {
  int64_t q = llround(x / scale + (double)zp);
  if (q < q_lo) q = q_lo;
  if (q > q_hi) q = q_hi;
  return q;
}

/* dequantize_value, quant.hpp:56-58 */
double kor_dequantize(int64_t q, double scale, int64_t zp) { return scale * (double)(q - zp); }

/* ------------------------------------------------------------------------ */
/* lut.hpp                                                                   */
/* ------------------------------------------------------------------------ */

/* ActivationLattice::of, lut.hpp:28-38: step = ldexp(delta, -k) */
double kor_lattice_step(const kor_grid* g, int k) { return ldexp(g->delta, -k); }

/* ActivationLattice::max_level, lut.hpp:40-42 */
int64_t kor_lattice_max_level(const kor_grid* g, int k) { return (int64_t)g->intervals << k; }

/* ActivationLattice::quantize, lut.hpp:44-47 */
int64_t kor_lattice_quantize(const kor_grid* g, int k, double x) {
  const double step = kor_lattice_step(g, k);
  int64_t a = llround((x - g->lo) / step);
  const int64_t L = kor_lattice_max_level(g, k);
  if (a < 0) a = 0;
  if (a > L) a = L;
  return a;
}

/* clamp (layers.hpp:111) then quantize (lut.hpp:191) */
int64_t kor_level_of(const kor_grid* g, int k, double x) {
  return kor_lattice_quantize(g, k, kor_clamp(g, x));
}

void kor_levels_f32(const kor_grid* g, int k, const float* x, size_t n, uint16_t* out) {
  for (size_t i = 0; i < n; ++i) out[i] = (uint16_t)kor_level_of(g, k, (double)x[i]);
}

/* next-layer levels of fp64 layer outputs: the consuming layer clamps
 * (layers.hpp:111) and quantizes (lut.hpp:44-47) */
void kor_levels_f64(const kor_grid* g, int k, const double* y, size_t n, uint16_t* out) {
  for (size_t i = 0; i < n; ++i) out[i] = (uint16_t)kor_level_of(g, k, y[i]);
}

/* entries = ceil((P+1)/2) * 2^k + 1 (lut.hpp:118-119) */
size_t kor_lut_size(int P, int k) { return (size_t)((P + 2) / 2) * ((size_t)1 << k) + 1; }

/* build_bspline_lut, lut.hpp:103-131 */
int kor_build_lut(int P, int k, int h, uint8_t* entries, size_t cap) {
  if (P < 1 || k < 1 || k > 8 || h < 2 || h > 8) return -1;
  const size_t stored = kor_lut_size(P, k);
  if (cap < stored) return -1;
  double vs;
  int64_t vz, vhi;
  kor_quant_params(0.0, 1.0, h, &vs, &vz, &vhi);
  kor_grid canon;
  kor_grid_build(1, P, 0.0, 1.0, &canon);
  double basis[64];
  const int64_t fold = (int64_t)(P + 1) << (k - 1);
  for (int64_t m = 0; m < (int64_t)stored; ++m) {
    const int64_t pos = m < fold ? m : fold;
    const double xi = P + ldexp((double)pos, -k);
    kor_basis_at_coord(&canon, xi, basis);
    entries[m] = (uint8_t)kor_quantize(basis[P], vs, vz, 0, vhi);
  }
  entries[0] = 0;
  return (int)stored;
}

/* lut_basis_lookup + BsplineLut::at_offset, lut.hpp:93-96, 136-160 */
int kor_lut_lookup(const kor_grid* g, int k, const uint8_t* entries, int64_t a, uint8_t* vals,
                   int* support_start) {
  const int P = g->degree;
  const int64_t L = (int64_t)g->intervals << k;
  if (a < 0 || a > L) return -1;
  const int64_t jj = a >> k;
  const int64_t frac = a - (jj << k);
  const int64_t fold = (int64_t)(P + 1) << (k - 1);
  const int64_t support = (int64_t)(P + 1) << k;
  const int nb = g->intervals + P;
  int count = 0;
  for (int r = 0; r <= P; ++r) {
    if (jj + r >= nb) break;
    const int64_t m = ((int64_t)(P - r) << k) + frac;
    const int64_t folded = m > fold ? support - m : m;
    vals[r] = entries[folded];
    ++count;
  }
  *support_start = (int)jj;
  return count;
}

/* quantized_basis_reference, lut.hpp:164-180 */
int kor_quantized_basis_reference(const kor_grid* g, int k, int h, int64_t a, uint8_t* vals,
                                  int* support_start) {
  const int nb = g->intervals + g->degree;
  double vs;
  int64_t vz, vhi;
  kor_quant_params(0.0, 1.0, h, &vs, &vz, &vhi);
  double* dense = (double*)malloc(sizeof(double) * (size_t)nb);
  /* ActivationLattice::knot_coord, lut.hpp:53-55 */
  const double xi = g->degree + ldexp((double)a, -k);
  const int start = kor_basis_at_coord(g, xi, dense);
  int count = 0;
  for (int r = 0; r <= g->degree; ++r) {
    const int i = start + r;
    if (i >= nb) break;
    vals[r] = (uint8_t)kor_quantize(dense[i], vs, vz, 0, vhi);
    ++count;
  }
  free(dense);
  *support_start = start;
  return count;
}

/* ------------------------------------------------------------------------ */
/* layers.hpp / matrix.hpp forwards                                          */
/* ------------------------------------------------------------------------ */

/* matmul, matrix.hpp:64-80: k-outer, j-inner fp64 accumulation */
static void matmul_ref(int64_t M, int64_t K, int N, const double* a, const double* b,
                       double* out) {
  for (int64_t m = 0; m < M; ++m) {
    double* orow = out + m * N;
    for (int j = 0; j < N; ++j) orow[j] = 0.0;
    const double* arow = a + m * K;
    for (int64_t kk = 0; kk < K; ++kk) {
      const double av = arow[kk];
      const double* brow = b + kk * N;
      for (int j = 0; j < N; ++j) orow[j] += av * brow[j];
    }
  }
}

/* kan_linear_forward<RecursiveBasis>, layers.hpp:99-121 (dense B, then matmul) */
void kor_linear_forward_fp64(const kor_grid* g, int64_t M, int n_in, int n_out,
                             const double* acts, const double* coeffs, double* out) {
  const int nb = g->intervals + g->degree;
  const int64_t K = (int64_t)n_in * nb;
  /* process in row blocks to bound the dense B footprint */
  const int64_t blk = 64;
  double* bmat = (double*)malloc(sizeof(double) * (size_t)(blk * K));
  for (int64_t m0 = 0; m0 < M; m0 += blk) {
    const int64_t rows = (M - m0) < blk ? (M - m0) : blk;
    memset(bmat, 0, sizeof(double) * (size_t)(rows * K));
    for (int64_t m = 0; m < rows; ++m)
      for (int i = 0; i < n_in; ++i) {
        const double x = kor_clamp(g, acts[(m0 + m) * n_in + i]);
        kor_basis_at_coord(g, kor_knot_coord(g, x), bmat + m * K + (int64_t)i * nb);
      }
    matmul_ref(rows, K, n_out, bmat, coeffs, out + m0 * n_out);
  }
  free(bmat);
}

/* RangeCalibrator(widen) + zero_spanning + compute_quant_params, as used by
 * maybe_fake_quant_weights (eval.hpp:70-76) and tabulated_kan_forward
 * (lut.hpp:222-229); RangeCalibrator::range, quant.hpp:97-107 */
static int wrange(const double* w, size_t n, double* lo, double* hi) {
  if (n == 0) return -1;
  double l = w[0], h = w[0];
  for (size_t i = 1; i < n; ++i) {
    l = (w[i] < l) ? w[i] : l; /* std::min(lo_, v) */
    h = (h < w[i]) ? w[i] : h; /* std::max(hi_, v) */
  }
  if (l == h) {
    const double pad = (fabs(l) > 1.0 ? fabs(l) : 1.0) * 2.220446049250313e-16 * 4.0;
    l = l - pad;
    h = h + pad;
  }
  /* zero_spanning, quant.hpp:123-125 */
  *lo = (0.0 < l) ? 0.0 : l;
  *hi = (h < 0.0) ? 0.0 : h;
  return 0;
}

int kor_wquant_per_tensor(const double* w, size_t n, int bits, uint8_t* q, double* scale,
                          int64_t* zp) {
  double lo, hi;
  if (wrange(w, n, &lo, &hi)) return -1;
  int64_t qhi;
  if (kor_quant_params(lo, hi, bits, scale, zp, &qhi)) return -1;
  for (size_t i = 0; i < n; ++i) q[i] = (uint8_t)kor_quantize(w[i], *scale, *zp, 0, qhi);
  return 0;
}

/* tabulated_kan_forward, lut.hpp:217-231, with LutBasis (lut.hpp:184-196) */
int kor_lut_forward_fp64(const kor_grid* g, int k, int h, int bits_w, int64_t M, int n_in,
                         int n_out, const double* acts, const double* coeffs, double* out) {
  const int nb = g->intervals + g->degree;
  const int64_t K = (int64_t)n_in * nb;
  const size_t nw = (size_t)K * (size_t)n_out;
  uint8_t lut[2048];
  if (kor_build_lut(g->degree, k, h, lut, sizeof lut) < 0) return -1;
  double vs;
  int64_t vz, vhi;
  kor_quant_params(0.0, 1.0, h, &vs, &vz, &vhi);
  double* wq = (double*)malloc(sizeof(double) * nw);
  if (bits_w == 32 || nw == 0) {
    memcpy(wq, coeffs, sizeof(double) * nw);
  } else {
    uint8_t* q = (uint8_t*)malloc(nw);
    double s;
    int64_t z;
    if (kor_wquant_per_tensor(coeffs, nw, bits_w, q, &s, &z)) {
      free(q);
      free(wq);
      return -1;
    }
    for (size_t i = 0; i < nw; ++i) wq[i] = kor_dequantize(q[i], s, z); /* fake_quant, quant.hpp:65-68 */
    free(q);
  }
  const int64_t blk = 64;
  double* bmat = (double*)malloc(sizeof(double) * (size_t)(blk * K));
  for (int64_t m0 = 0; m0 < M; m0 += blk) {
    const int64_t rows = (M - m0) < blk ? (M - m0) : blk;
    memset(bmat, 0, sizeof(double) * (size_t)(rows * K));
    for (int64_t m = 0; m < rows; ++m)
      for (int i = 0; i < n_in; ++i) {
        const double x = kor_clamp(g, acts[(m0 + m) * n_in + i]);
        const int64_t a = kor_lattice_quantize(g, k, x);
        uint8_t vals[16];
        int start;
        const int cnt = kor_lut_lookup(g, k, lut, a, vals, &start);
        double* row = bmat + m * K + (int64_t)i * nb;
        for (int r = 0; r < cnt; ++r) row[start + r] = kor_dequantize(vals[r], vs, vz);
      }
    matmul_ref(rows, K, n_out, bmat, wq, out + m0 * n_out);
  }
  free(bmat);
  free(wq);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Engine extensions (unpinned by the reference; defined here)               */
/* ------------------------------------------------------------------------ */

/* Per-output-channel symmetric quantization.  Rounding reuses the reference's
 * llround(w/s) half-away-from-zero rule (quant.hpp:52).  Q = 2^(b-1)-1,
 * s_j = max_c |w[c,j]| / Q (s_j = 1 for an all-zero column). */
int kor_wquant_per_channel_sym(const double* w, int64_t K, int N, int bits, int8_t* q,
                               double* scale) {
  if (bits < 2 || bits > 8) return -1;
  const int64_t Q = ((int64_t)1 << (bits - 1)) - 1;
  for (int j = 0; j < N; ++j) {
    double mx = 0.0;
    for (int64_t c = 0; c < K; ++c) {
      const double v = fabs(w[c * N + j]);
      mx = (mx < v) ? v : mx;
    }
    const double s = (mx > 0.0) ? mx / (double)Q : 1.0;
    scale[j] = s;
    for (int64_t c = 0; c < K; ++c) {
      int64_t v = llround(w[c * N + j] / s);
      if (v < -Q) v = -Q;
      if (v > Q) v = Q;
      q[c * N + j] = (int8_t)v;
    }
  }
  return 0;
}

/* Joint per-channel symmetric quantization of spline + base weights (see
 * kan_oracle.h).  Rounding is quantize_value's llround (quant.hpp:52). */
int kor_wquant_joint(const double* w, const double* wb, int64_t K, int n_in, int N, int bits,
                     double ratio, int8_t* q, int8_t* qb, double* scale) {
  if (bits < 2 || bits > 8) return -1;
  const int64_t Q = ((int64_t)1 << (bits - 1)) - 1;
  for (int j = 0; j < N; ++j) {
    double mx = 0.0;
    for (int64_t c = 0; c < K; ++c) {
      const double v = fabs(w[c * N + j]);
      mx = (mx < v) ? v : mx;
    }
    for (int i = 0; i < n_in; ++i) {
      const double v = fabs(wb[(int64_t)i * N + j] * ratio);
      mx = (mx < v) ? v : mx;
    }
    const double s = (mx > 0.0) ? mx / (double)Q : 1.0;
    scale[j] = s;
    for (int64_t c = 0; c < K; ++c) {
      int64_t v = llround(w[c * N + j] / s);
      q[c * N + j] = (int8_t)(v < -Q ? -Q : (v > Q ? Q : v));
    }
    for (int i = 0; i < n_in; ++i) {
      int64_t v = llround((wb[(int64_t)i * N + j] * ratio) / s);
      qb[(int64_t)i * N + j] = (int8_t)(v < -Q ? -Q : (v > Q ? Q : v));
    }
  }
  return 0;
}

/* SiLU at every lattice point: v_a = silu(lo + a*step) (ActivationLattice::
 * dequantize, lut.hpp:49), quantized unsigned 8-bit over the zero-spanning
 * range of {v_a} with compute_quant_params / quantize_value (quant.hpp:33-54). */
int kor_silu_table(const kor_grid* g, int k, uint8_t* codes, double* scale, int64_t* zp) {
  const int64_t L = kor_lattice_max_level(g, k);
  const double step = kor_lattice_step(g, k);
  double* v = (double*)malloc(sizeof(double) * (size_t)(L + 1));
  double lo = 0.0, hi = 0.0;
  for (int64_t a = 0; a <= L; ++a) {
    const double t = g->lo + (double)a * step;
    v[a] = t / (1.0 + exp(-t));
    lo = (v[a] < lo) ? v[a] : lo;
    hi = (hi < v[a]) ? v[a] : hi;
  }
  int64_t qhi;
  if (kor_quant_params(lo, hi, 8, scale, zp, &qhi)) {
    free(v);
    return -1;
  }
  for (int64_t a = 0; a <= L; ++a) codes[a] = (uint8_t)kor_quantize(v[a], *scale, *zp, 0, qhi);
  free(v);
  return 0;
}

int kor_int_accumulate(const kor_grid* g, int k, const uint8_t* lut, const kor_int_layer* L,
                       int64_t M, int n_in, int n_out, const uint16_t* levels, int32_t* acc_s,
                       int32_t* acc_b, int64_t* rowsum) {
  const int nb = g->intervals + g->degree;
  for (int64_t m = 0; m < M; ++m) {
    int64_t* as = (int64_t*)calloc((size_t)n_out, sizeof(int64_t));
    int64_t* ab = (int64_t*)calloc((size_t)n_out, sizeof(int64_t));
    int64_t rs = 0;
    for (int i = 0; i < n_in; ++i) {
      const int64_t a = levels[m * n_in + i];
      uint8_t vals[16];
      int start;
      const int cnt = kor_lut_lookup(g, k, lut, a, vals, &start);
      if (cnt < 0) {
        free(as);
        free(ab);
        return -1;
      }
      for (int r = 0; r < cnt; ++r) {
        const int64_t c = (int64_t)i * nb + start + r;
        rs += vals[r];
        for (int j = 0; j < n_out; ++j) {
          const int64_t w = L->wscheme == 0 ? (int64_t)L->qw_u8[c * n_out + j]
                                            : (int64_t)L->qw_s8[c * n_out + j];
          as[j] += (int64_t)vals[r] * w;
        }
      }
      if (L->silu) {
        const int64_t qs = L->silu_codes[a];
        for (int j = 0; j < n_out; ++j) ab[j] += qs * (int64_t)L->qwb[(int64_t)i * n_out + j];
      }
    }
    for (int j = 0; j < n_out; ++j) {
      acc_s[m * n_out + j] = (int32_t)(as[j] + ab[j]); /* single accumulator */
      if (acc_b) acc_b[m * n_out + j] = (int32_t)ab[j];
    }
    if (rowsum) rowsum[m] = rs;
    free(as);
    free(ab);
  }
  return 0;
}

/* Epilogue (fp64, no contraction):
 *   wscheme 0: y = (double)(acc - z_w*rowsum) * (s_b*s_w)
 *   wscheme 1: y = (double)(acc - z_s*colsum_b[j]) * (s_b*s_j)   (acc = spline + base;
 *              colsum_b = 0 without the SiLU term)
 * s_b = value_qp.scale of the table = 1/(2^h-1) (lut.hpp:112). */
double kor_int_epilogue(const kor_grid* g, int h, const kor_int_layer* L, int n_in, int n_out,
                        int j, int32_t acc_s, int32_t acc_b, int64_t rowsum, int64_t colsum_b) {
  (void)g;
  (void)n_in;
  (void)n_out;
  (void)acc_b;
  double sb;
  int64_t zb, hb;
  kor_quant_params(0.0, 1.0, h, &sb, &zb, &hb);
  if (L->wscheme == 0) {
    const double f = sb * L->s_w;
    return (double)((int64_t)acc_s - L->z_w * rowsum) * f;
  }
  const double f = sb * L->s_wc[j];
  const int64_t corr = L->silu ? L->z_s * colsum_b : 0;
  return (double)((int64_t)acc_s - corr) * f;
}

int kor_int_layer_forward(const kor_grid* g, int k, int h, const uint8_t* lut,
                          const kor_int_layer* L, int64_t M, int n_in, int n_out,
                          const uint16_t* levels, double* y) {
  int32_t* as = (int32_t*)malloc(sizeof(int32_t) * (size_t)(M * n_out));
  int32_t* ab = (int32_t*)malloc(sizeof(int32_t) * (size_t)(M * n_out));
  int64_t* rs = (int64_t*)malloc(sizeof(int64_t) * (size_t)(M > 0 ? M : 1));
  int64_t* colsum = (int64_t*)calloc((size_t)n_out, sizeof(int64_t));
  if (L->silu)
    for (int i = 0; i < n_in; ++i)
      for (int j = 0; j < n_out; ++j) colsum[j] += L->qwb[(int64_t)i * n_out + j];
  int rc = kor_int_accumulate(g, k, lut, L, M, n_in, n_out, levels, as, ab, rs);
  if (rc == 0)
    for (int64_t m = 0; m < M; ++m)
      for (int j = 0; j < n_out; ++j)
        y[m * n_out + j] = kor_int_epilogue(g, h, L, n_in, n_out, j, as[m * n_out + j],
                                            ab[m * n_out + j], rs[m], colsum[j]);
  free(as);
  free(ab);
  free(rs);
  free(colsum);
  return rc;
}

/* int8 output requantization: clamp(llround(y/s_out), -127, 127) */
int8_t kor_requant_i8(double y, double s_out) {
  int64_t q = llround(y / s_out);
  if (q < -127) q = -127;
  if (q > 127) q = 127;
  return (int8_t)q;
}

/* im2col, layers.hpp:126-154: zero padding, channel-major columns */
int kor_im2col(const double* in, int C, int H, int W, int kernel, int stride, int padding,
               double* out) {
  if (kernel < 1 || stride < 1 || padding < 0) return -1;
  const int span_h = H + 2 * padding - kernel, span_w = W + 2 * padding - kernel;
  if (span_h < 0 || span_w < 0 || span_h % stride || span_w % stride) return -1;
  const int Ho = span_h / stride + 1, Wo = span_w / stride + 1;
  const int cols = kernel * kernel * C;
  for (int oy = 0; oy < Ho; ++oy)
    for (int ox = 0; ox < Wo; ++ox) {
      double* row = out + ((int64_t)oy * Wo + ox) * cols;
      int col = 0;
      for (int c = 0; c < C; ++c)
        for (int ky = 0; ky < kernel; ++ky)
          for (int kx = 0; kx < kernel; ++kx, ++col) {
            const int y = oy * stride + ky - padding, x = ox * stride + kx - padding;
            row[col] = (y >= 0 && y < H && x >= 0 && x < W)
                           ? in[((int64_t)c * H + y) * W + x]
                           : 0.0;
          }
    }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* spline_table.hpp: spline-table mode                                       */
/* ------------------------------------------------------------------------ */

/* detail::build_tables, spline_table.hpp:38-85.  values [n_in][n_out][2^bits_a]
 * (SplineTableSet::at, :31-33).  Input levels sit on the grid bounds
 * (compute_quant_params(lo, hi, bits_a), :51); each spline is sampled at the
 * dequantized level with basis_at_coord(knot_coord(x)) and the coefficient
 * column dotted in k order (:59-71); one zero-spanning output range over the
 * whole layer (RangeCalibrator + range(true) + zero_spanning, :73-76,
 * quant.hpp:79-123) gives the shared h-bit output quantizer (:77-82). */
int kor_spline_tables_build(const kor_grid* g, const double* coeffs, int n_in, int n_out,
                            int bits_a, int h, uint8_t* values, double* qp_d, int64_t* qp_i) {
  if (bits_a < 1 || bits_a > 8 || h < 2 || h > 8) return -1;
  double in_s, out_s;
  int64_t in_z, in_qhi, out_z, out_qhi;
  if (kor_quant_params(g->lo, g->hi, bits_a, &in_s, &in_z, &in_qhi)) return -1;
  const int64_t levels = (int64_t)1 << bits_a;
  const int nb = g->intervals + g->degree;
  const size_t n_tab = (size_t)n_in * (size_t)n_out;
  double* sampled = (double*)malloc(sizeof(double) * n_tab * (size_t)levels);
  double* basis = (double*)malloc(sizeof(double) * (size_t)nb * (size_t)levels);
  if (!sampled || !basis) {
    free(sampled);
    free(basis);
    return -1;
  }
  for (int64_t m = 0; m < levels; ++m) {
    const double x = kor_dequantize(m, in_s, in_z);
    kor_basis_at_coord(g, kor_knot_coord(g, x), basis + m * nb);
  }
  int seen = 0;
  double lo = 0.0, hi = 0.0;
  for (int i = 0; i < n_in; ++i)
    for (int j = 0; j < n_out; ++j)
      for (int64_t m = 0; m < levels; ++m) {
        double acc = 0.0;
        for (int k = 0; k < nb; ++k)
          acc += basis[m * nb + k] * coeffs[((size_t)i * nb + k) * (size_t)n_out + j];
        sampled[((size_t)i * n_out + j) * (size_t)levels + m] = acc;
      }
  /* RangeCalibrator::observe over sampled.flat() in row-major order */
  for (size_t t = 0; t < n_tab * (size_t)levels; ++t) {
    const double v = sampled[t];
    if (!seen) {
      lo = hi = v;
      seen = 1;
    } else {
      lo = (v < lo) ? v : lo; /* std::min(lo, v) */
      hi = (hi < v) ? v : hi; /* std::max(hi, v) */
    }
  }
  if (!seen) { /* calibrate_range: empty stream */
    free(sampled);
    free(basis);
    return -1;
  }
  if (lo == hi) { /* range(true): symmetric widening, quant.hpp:98-104 */
    const double a = fabs(lo) > 1.0 ? fabs(lo) : 1.0;
    const double pad = a * 2.220446049250313e-16 * 4.0;
    lo = lo - pad;
    hi = hi + pad;
  }
  lo = (0.0 < lo) ? 0.0 : lo; /* zero_spanning, quant.hpp:118-120 */
  hi = (hi < 0.0) ? 0.0 : hi;
  if (kor_quant_params(lo, hi, h, &out_s, &out_z, &out_qhi)) {
    free(sampled);
    free(basis);
    return -1;
  }
  for (size_t t = 0; t < n_tab * (size_t)levels; ++t)
    values[t] = (uint8_t)kor_quantize(sampled[t], out_s, out_z, 0, out_qhi);
  free(sampled);
  free(basis);
  qp_d[0] = in_s;
  qp_d[1] = out_s;
  qp_i[0] = in_z;
  qp_i[1] = in_qhi;
  qp_i[2] = out_z;
  qp_i[3] = out_qhi;
  return 0;
}

/* Input level of one activation: quantize_value(x, in_qp), quant.hpp:51-54
 * (no domain clamp: the level clamps, spline_table.hpp:98). */
int64_t kor_spline_level(double x, double in_s, int64_t in_z, int64_t in_qhi) {
  return kor_quantize(x, in_s, in_z, 0, in_qhi);
}

/* Integer form of spline_table_forward (spline_table.hpp:90-107): levels
 * [M, n_in] -> acc[m, j] = sum_i (table[i][j][level] - z_out), the int64 sum
 * the reference dequantizes once per output (out = s_out * acc). */
int kor_spline_table_accumulate(const uint8_t* values, int n_in, int n_out, int bits_a,
                                int64_t out_z, int64_t M, const uint8_t* levels, int64_t* acc) {
  const int64_t E = (int64_t)1 << bits_a;
  for (int64_t m = 0; m < M; ++m)
    for (int j = 0; j < n_out; ++j) {
      int64_t a = 0;
      for (int i = 0; i < n_in; ++i)
        a += (int64_t)values[((size_t)i * n_out + j) * (size_t)E + levels[m * n_in + i]] - out_z;
      acc[m * n_out + j] = a;
    }
  return 0;
}

/* spline_table_forward, spline_table.hpp:90-107: fp64 activations -> outputs */
int kor_spline_table_forward(const uint8_t* values, int n_in, int n_out, int bits_a,
                             const double* qp_d, const int64_t* qp_i, int64_t M,
                             const double* acts, double* out) {
  uint8_t* lv = (uint8_t*)malloc((size_t)(n_in > 0 ? n_in : 1));
  int64_t* acc = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_out > 0 ? n_out : 1));
  if (!lv || !acc) {
    free(lv);
    free(acc);
    return -1;
  }
  for (int64_t m = 0; m < M; ++m) {
    for (int i = 0; i < n_in; ++i)
      lv[i] = (uint8_t)kor_spline_level(acts[m * n_in + i], qp_d[0], qp_i[0], qp_i[1]);
    kor_spline_table_accumulate(values, n_in, n_out, bits_a, qp_i[2], 1, lv, acc);
    for (int j = 0; j < n_out; ++j) out[m * n_out + j] = qp_d[1] * (double)acc[j];
  }
  free(lv);
  free(acc);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* eval.hpp fake-quant mode (EvalMode::kFakeQuant)                           */
/* ------------------------------------------------------------------------ */

/* forward_linear in fake-quant mode (eval.hpp:135-159): W fake-quantized per
 * tensor (maybe_fake_quant_weights, eval.hpp:70-76), activations fake-quantized
 * on the grid bounds (a_params_for, eval.hpp:55-68; fake_quant, quant.hpp:65-68),
 * then kan_linear_forward (clamp, layers.hpp:111) with RecursiveBasis or
 * FakeQuantBasis over [0, 1] at bits_b (layers.hpp:85-94); 32 = passthrough. */
int kor_fakequant_forward_fp64(const kor_grid* g, int bits_w, int bits_a, int bits_b, int64_t M,
                               int n_in, int n_out, const double* acts, const double* coeffs,
                               double* out) {
  const int nb = g->intervals + g->degree;
  const int64_t K = (int64_t)n_in * nb;
  const size_t nw = (size_t)K * (size_t)n_out;
  double* wq = (double*)malloc(sizeof(double) * (nw ? nw : 1));
  if (bits_w == 32 || nw == 0) {
    memcpy(wq, coeffs, sizeof(double) * nw);
  } else {
    uint8_t* q = (uint8_t*)malloc(nw);
    double s;
    int64_t z;
    if (kor_wquant_per_tensor(coeffs, nw, bits_w, q, &s, &z)) {
      free(q);
      free(wq);
      return -1;
    }
    for (size_t i = 0; i < nw; ++i) wq[i] = kor_dequantize(q[i], s, z);
    free(q);
  }
  double as = 1.0, bs = 1.0;
  int64_t az = 0, ahi = 0, bz = 0, bhi = 0;
  if (bits_a != 32 && kor_quant_params(g->lo, g->hi, bits_a, &as, &az, &ahi)) {
    free(wq);
    return -1;
  }
  if (bits_b != 32 && kor_quant_params(0.0, 1.0, bits_b, &bs, &bz, &bhi)) {
    free(wq);
    return -1;
  }
  const int64_t blk = 64;
  double* bmat = (double*)malloc(sizeof(double) * (size_t)(blk * K));
  for (int64_t m0 = 0; m0 < M; m0 += blk) {
    const int64_t rows = (M - m0) < blk ? (M - m0) : blk;
    for (int64_t m = 0; m < rows; ++m)
      for (int i = 0; i < n_in; ++i) {
        double x = acts[(m0 + m) * n_in + i];
        if (bits_a != 32) x = kor_dequantize(kor_quantize(x, as, az, 0, ahi), as, az);
        double* row = bmat + m * K + (int64_t)i * nb;
        kor_basis_at_coord(g, kor_knot_coord(g, kor_clamp(g, x)), row);
        if (bits_b != 32)
          for (int k = 0; k < nb; ++k) row[k] = kor_dequantize(kor_quantize(row[k], bs, bz, 0, bhi), bs, bz);
      }
    matmul_ref(rows, K, n_out, bmat, wq, out + m0 * n_out);
  }
  free(bmat);
  free(wq);
  return 0;
}
