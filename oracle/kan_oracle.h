/*
 * kan_oracle.h -- CPU restatement of the reference KAN-layer hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the checker the parity tests,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg compare the CUDA
 * engine against.  Nothing in the product path (paper_2603_17230_b200/,
 * include/) links, loads or calls it.
 *
 * Every function restates the algorithm of the reference C++ headers under
 * proj/include/kantize/ (file:line cited per function) in plain C with the
 * same IEEE-754 double operation order, so that the pinned quantities
 * (lattice levels, table entries, quantized basis, fp64 layer outputs) are
 * bit-identical to the reference.  The restatement is pinned against the
 * reference compiled from its own headers (oracle/_ref, see oracle/Makefile)
 * and against the reference's known-answer tests (tests/test_oracle_pins.py).
 *
 * It also DEFINES the engine extensions the reference does not have
 * (per-output-channel symmetric weights, SiLU base term on the lattice,
 * integer accumulators, requantized outputs); those are unpinned by the
 * reference and documented in DESIGN.md section "Integer LUT path".
 */
#ifndef KAN_ORACLE_H
#define KAN_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int intervals; /* G */
  int degree;    /* P */
  double lo, hi, delta;
} kor_grid;

/* ---- grid.hpp ---------------------------------------------------------- */
int kor_grid_build(int G, int P, double lo, double hi, kor_grid* g);
double kor_clamp(const kor_grid* g, double x);
double kor_knot_coord(const kor_grid* g, double x);
/* dense degree-P basis (G+P values) at knot coordinate xi; returns support start */
int kor_basis_at_coord(const kor_grid* g, double xi, double* out);

/* ---- quant.hpp --------------------------------------------------------- */
int kor_quant_params(double alpha, double beta, int bits, double* scale, int64_t* zero_point,
                     int64_t* q_hi);
int64_t kor_quantize(double x, double scale, int64_t zp, int64_t q_lo, int64_t q_hi);
double kor_dequantize(int64_t q, double scale, int64_t zp);

/* ---- lut.hpp ----------------------------------------------------------- */
double kor_lattice_step(const kor_grid* g, int k);
int64_t kor_lattice_max_level(const kor_grid* g, int k);
/* level of an already-clamped activation */
int64_t kor_lattice_quantize(const kor_grid* g, int k, double x);
/* level of a raw activation (clamp_to_domain first, as kan_linear_forward does) */
int64_t kor_level_of(const kor_grid* g, int k, double x);
void kor_levels_f32(const kor_grid* g, int k, const float* x, size_t n, uint16_t* out);
void kor_levels_f64(const kor_grid* g, int k, const double* y, size_t n, uint16_t* out);
size_t kor_lut_size(int P, int k);
int kor_build_lut(int P, int k, int h, uint8_t* entries, size_t cap);
/* returns count (number of values written); -1 when the level is out of range */
int kor_lut_lookup(const kor_grid* g, int k, const uint8_t* entries, int64_t a, uint8_t* vals,
                   int* support_start);
/* quantize the recursion at the exact lattice coordinate (the reference route) */
int kor_quantized_basis_reference(const kor_grid* g, int k, int h, int64_t a, uint8_t* vals,
                                  int* support_start);

/* ---- layers.hpp / matrix.hpp: fp64 forwards ----------------------------- */
/* kan_linear_forward with RecursiveBasis; coeffs [n_in*(G+P), n_out] row-major */
void kor_linear_forward_fp64(const kor_grid* g, int64_t M, int n_in, int n_out,
                             const double* acts, const double* coeffs, double* out);
/* tabulated_kan_forward: lattice + LUT basis, per-tensor asymmetric fake-quant W
 * (bits_w in [1,8], or 32 = passthrough) */
int kor_lut_forward_fp64(const kor_grid* g, int k, int h, int bits_w, int64_t M, int n_in,
                         int n_out, const double* acts, const double* coeffs, double* out);

/* ---- per-tensor asymmetric weight quantization (eval.hpp:70-76) ---------- */
int kor_wquant_per_tensor(const double* w, size_t n, int bits, uint8_t* q, double* scale,
                          int64_t* zp);
/* ---- per-output-channel symmetric weight quantization (engine extension) - */
int kor_wquant_per_channel_sym(const double* w, int64_t K, int N, int bits, int8_t* q,
                               double* scale);
/* Joint per-output-channel symmetric quantization of a layer with a SiLU base
 * term (engine extension): spline rows w [K, N] and base rows wb [n_in, N]
 * share one scale per output channel, in spline-code units:
 *   m_j = max(max_c |w[c,j]|, max_i |wb[i,j]*ratio|), ratio = s_s / s_b,
 *   s_j = m_j / Q (1 for an all-zero column), q = clamp(llround(v / s_j), +-Q)
 * with v = w[c,j] (spline) or wb[i,j]*ratio (base). */
int kor_wquant_joint(const double* w, const double* wb, int64_t K, int n_in, int N, int bits,
                     double ratio, int8_t* q, int8_t* qb, double* scale);
/* SiLU code table on the lattice (engine extension): L+1 u8 codes, scale, zp */
int kor_silu_table(const kor_grid* g, int k, uint8_t* codes, double* scale, int64_t* zp);

/* ---- integer restatement of one LUT layer ------------------------------- */
/* levels [M, n_in] (u16) -> int32 accumulators.
 * Spline part: acc_s[m,j] = sum_c qb[m,c] * qw[c,j]
 *   wscheme 0 (reference, per-tensor asym u8): qw = u8 codes, rowsum[m] = sum_c qb[m,c]
 *   wscheme 1 (per-channel symmetric s8):      qw = s8 codes
 * Base part (silu != 0): acc_b[m,j] = sum_i qs[level[m,i]] * qwb[i,j], and the
 * engine's single accumulator is acc_s + acc_b (joint scale, kor_wquant_joint):
 * acc_s returns that sum, acc_b the base part alone. */
typedef struct {
  int wscheme; /* 0 per-tensor asym (reference), 1 per-channel sym */
  int bits_w;
  int silu;
  /* reference-mode weight quantization */
  const uint8_t* qw_u8; /* [n_in*nb, N] */
  double s_w;
  int64_t z_w;
  /* per-channel */
  const int8_t* qw_s8;   /* [n_in*nb, N] */
  const double* s_wc;    /* [N] */
  /* silu base */
  const uint8_t* silu_codes; /* [L+1] */
  double s_s;
  int64_t z_s;
  const int8_t* qwb;   /* [n_in, N] */
  const double* s_wb;  /* [N] */
} kor_int_layer;

int kor_int_accumulate(const kor_grid* g, int k, const uint8_t* lut, const kor_int_layer* L,
                       int64_t M, int n_in, int n_out, const uint16_t* levels, int32_t* acc_s,
                       int32_t* acc_b, int64_t* rowsum);
/* epilogue: fp64 output value of one element */
double kor_int_epilogue(const kor_grid* g, int h, const kor_int_layer* L, int n_in, int n_out,
                        int j, int32_t acc_s, int32_t acc_b, int64_t rowsum, int64_t colsum_b);
/* full integer layer: levels -> y (fp64) */
int kor_int_layer_forward(const kor_grid* g, int k, int h, const uint8_t* lut,
                          const kor_int_layer* L, int64_t M, int n_in, int n_out,
                          const uint16_t* levels, double* y);

/* requantization helpers */
int8_t kor_requant_i8(double y, double s_out);

/* ---- im2col (layers.hpp:126-154) ---------------------------------------- */
int kor_im2col(const double* in, int C, int H, int W, int kernel, int stride, int padding,
               double* out /* [Ho*Wo, K*K*C] */);


/* ---- spline_table.hpp: spline-table mode -------------------------------- */
/* build_spline_tables (spline_table.hpp:38-85): values [n_in][n_out][2^bits_a];
 * qp_d = {in_scale, out_scale}; qp_i = {in_zp, in_qhi, out_zp, out_qhi}. */
int kor_spline_tables_build(const kor_grid* g, const double* coeffs, int n_in, int n_out,
                            int bits_a, int h, uint8_t* values, double* qp_d, int64_t* qp_i);
/* quantize_value(x, in_qp) (quant.hpp:51-54) */
int64_t kor_spline_level(double x, double in_s, int64_t in_z, int64_t in_qhi);
/* integer sums sum_i (table[i][j][level] - z_out), levels [M, n_in] u8 */
int kor_spline_table_accumulate(const uint8_t* values, int n_in, int n_out, int bits_a,
                                int64_t out_z, int64_t M, const uint8_t* levels, int64_t* acc);
/* spline_table_forward (spline_table.hpp:90-107) */
int kor_spline_table_forward(const uint8_t* values, int n_in, int n_out, int bits_a,
                             const double* qp_d, const int64_t* qp_i, int64_t M,
                             const double* acts, double* out);

/* ---- eval.hpp fake-quant mode: one linear layer (bits 32 = passthrough) --- */
int kor_fakequant_forward_fp64(const kor_grid* g, int bits_w, int bits_a, int bits_b, int64_t M,
                               int n_in, int n_out, const double* acts, const double* coeffs,
                               double* out);

#ifdef __cplusplus
}
#endif
#endif
