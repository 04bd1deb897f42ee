// kan_internal.h -- parameter blocks shared by the host engine and kernels.
#pragma once
#include <cstdint>

namespace kan {

enum EpiKind : int {
  EPI_F32 = 0,    // fp32 values (logits, or hidden activations on the float paths)
  EPI_LEVEL = 1,  // u16 lattice level of the next layer (hidden layers, LUT path)
  EPI_I8 = 2,     // int8 requantized logits
  EPI_RAW = 3,    // raw accumulators (int32 on the LUT path, fp32 bits on bf16)
};

enum XKind : int { X_F32 = 0, X_U16 = 1 };

// One fused gather + tcgen05 GEMM launch (one KAN layer, linear form).
struct GemmParams {
  int M, n_in, N;
  int BN, n_tiles_n;
  int S;  // ring stages
  // stage schedule
  int IPS, GS;
  int n_spline_stages, n_groups, silu;
  int total_stages;  // length of the pre-tiled weight schedule per n-tile
  int x_kind;
  // lattice tables (LUT path), one contiguous blob copied to smem per CTA:
  //   NBP = 8 : ent[g] (16 B) = {thr[g], thr[g+1], row pattern bytes 0-7}
  //   NBP = 16: thr pair[g] (8 B) at off_thr, row pattern[g] (16 B) at off_pat
  //   SiLU codes [L+1] (u8) at off_silu
  // thr[n] = smallest fp32 with level >= n; thr[0] = -inf, thr[L+1] = NaN.
  const uint8_t* tab;
  int tab_bytes, off_thr, off_pat, off_silu;
  int L, k;
  float lo_f, inv_step_f;
  // float basis (bf16 path)
  float flo, fhi_open, finv_delta;
  int G, P;
  // pre-tiled, pre-swizzled weights: [n_tiles_n][total_stages][BN*128] bytes
  const uint8_t* wt;
  int b_signed;
  // split-K: every split writes its partial tile, the last CTA of a tile sums
  // them in split order (int32 sums are exact; fp32 sums are deterministic)
  int splits, groups_per_split;
  int32_t* ws_s;       // [splits][m_tiles*128][n_tiles_n*BN]
  int32_t* ws_b;       // same, SiLU-base accumulator
  int32_t* ws_rowsum;  // [n_tiles_n][splits][m_tiles*128]
  unsigned* counters;  // [m_tiles * n_tiles_n], self-resetting
  // epilogue
  int epi;
  void* out;
  void* out2;
  int ld_out;
  int wscheme, zp;
  double f_tensor;
  long long z_w;
  const double* fs;       // [N]  s_b * s_w[j]
  const double* fb;       // [N]  s_s * s_wb[j]
  const long long* corr_b;  // [N] z_s * colsum(q_wb[:, j])
  double n_lo, n_hi_open, n_step;
  int n_L;
  double out_scale;
  int m_tiles;
};

// fp32 SIMT Cox-de Boor layer (accuracy baseline).
struct Fp32Params {
  int M, n_in, N, NBP, Npad;
  const float* x;
  int ld_x;
  const float* w;   // [n_in*NBP][Npad]
  const float* wb;  // [n_in][Npad] or null
  float* out;
  int ld_out;
  float lo, hi_open, inv_delta;
  int G, P;
};

}  // namespace kan
