// kan_internal.h -- parameter blocks shared by the host engine and kernels.
#pragma once
#include <cstdint>

// Ablation switches (GemmParams::dbg_flags, KAN_OPT_DBG_FLAGS) are compiled
// into the kernels only in a -DKAN_TUNING build; production kernels carry no
// such branches.
#ifdef KAN_TUNING
#define KAN_DBG(p, bit) ((((p).dbg_flags) & (bit)) != 0)
#else
#define KAN_DBG(p, bit) false
#endif

namespace kan {

enum EpiKind : int {
  EPI_F32 = 0,    // fp32 values (logits, or hidden activations on the float paths)
  EPI_LEVEL = 1,  // u16 lattice level of the next layer (hidden layers, LUT path)
  EPI_I8 = 2,     // int8 requantized logits
  EPI_RAW = 3,    // raw accumulators (int32 on the LUT path, fp32 bits on bf16)
};

enum XKind : int { X_F32 = 0, X_U16 = 1 };

// K bytes per pipeline stage of the gather GEMM: eight 32-byte tcgen05.mma
// K-steps; the stage's weight tile is two 128-byte-wide SW128 blocks.
constexpr int KSTAGE = 256;
constexpr int GEMM_PRODUCER_WARPS = 16;
// producers + activation loader + MMA issuer + weight loader + epilogue warps
// (two per TMEM lane quarter, each on every other 16-column group)
constexpr int GEMM_EPI_WARPS = 8;
// per epilogue warp: 32 rows x 16 fp32 columns at an 80-byte pitch (conflict-free 16-byte stores)
constexpr int GEMM_STG_PITCH = 80;
constexpr int GEMM_STG_BYTES = GEMM_EPI_WARPS * 32 * GEMM_STG_PITCH;
constexpr int GEMM_THREADS = 32 * (GEMM_PRODUCER_WARPS + 3 + GEMM_EPI_WARPS);

// One fused gather + tcgen05 GEMM launch (one KAN layer, linear form).
struct GemmParams {
  int M, n_in, N;
  int BN, n_tiles_n;
  int SA;  // A ring stages (released by the MMA)
  int SB;  // weight-tile ring stages (released by the MMA)
  int SX;  // activation ring stages (released by the producers)
  int nacc;  // TMEM accumulators (2: the epilogue overlaps the next tile)
  int mc;    // conv3: CTAs per cluster sharing (multicasting) the weight tiles
  // stage schedule
  int IPS, GS;
  int n_spline_stages, n_groups, silu;
  int total_stages;  // length of the pre-tiled weight schedule per n-tile
  int x_kind;
  // lattice tables (LUT path), one contiguous blob copied to smem per CTA:
  //   vals[2^k] (u32): the P+1 LUT codes of lut_basis_lookup for each in-
  //     interval offset frac, packed little-endian (byte r = basis jj + r)
  //   thr[L+2] (f32) at off_thr: thr[n] = smallest fp32 with level >= n
  //     (thr[0] = -inf, thr[L+1] = NaN), consulted only near rounding ties
  //   SiLU codes [L+1] (u8) at off_silu
  //   NBP = 8: c64[L+1] (u64) at off_c64: the level's full 8-byte code row,
  //     vals[frac] << 8*jj truncated to the row
  // rep = 1 (NBP = 8 where smem allows): lane-private copies instead, so
  //   every table read is one conflict-free wavefront: vals as [2^k][32 lanes]
  //   words, SiLU codes packed 4 per word as [(L+4)/4][32 lanes]; no c64.
  // rep = 2: lane-private vals, shared SiLU codes (fewer instructions)
  const uint8_t* tab;
  int tab_bytes, off_thr, off_silu, off_c64, rep;
  int L, k;
  float lo_f, inv_step_f;  // LUT path: lo_f = -lo/step (fp32), inv_step_f = 1/step
  // float basis (bf16 path)
  float flo, fhi_open, finv_delta;
  int G, P;
  // pre-tiled, pre-swizzled weights: [n_tiles_n][total_stages][BN*KSTAGE] bytes
  const uint8_t* wt;
  int b_signed;
  // split-K over a thread-block cluster of `splits` CTAs along z: partial
  // accumulators are summed through distributed shared memory (int32 sums are
  // exact; fp32 sums run in a fixed order, so they are deterministic)
  int splits, groups_per_split;
  // epilogue
  int epi;
  void* out;
  void* out2;
  int ld_out;
  double f_tensor;
  long long z_w;
  const double* fs;         // [N]  s_b * s_w[j]
  const double* fb;         // [N]  s_s * s_wb[j]
  const long long* corr_b;  // [N] z_s * colsum(q_wb[:, j])
  double n_lo, n_hi_open, n_step, n_inv_step;
  int n_L;
  double out_scale, inv_out_scale;
  int m_tiles;
  // implicit im2col (conv layers; conv == 0 for dense [M, n_in] rows).  K runs
  // tap-major: spline stage sp covers tap sp / cps, channels (sp % cps)*IPS...
  // An M tile is bn_img images x bh output rows x Wo columns (pimg = bh*Wo
  // pixels per image); rows stay contiguous in M = (n, oy, ox).
  int conv, ksz, cstride, pad, cps, H, W, Ho, Wo, bh, bn_img, tpi, pimg;
  int lvl0;    // lattice level of 0.0 (padded taps of u16 level inputs)
  int n_ch;    // valid inputs per row chunk (dense: n_in; conv: c_in)
  // epilogue residual add (engine extension): 2 = stored fp32 values, 0 = none
  int res_kind;
  const void* res;
  int ld_res;
  int out_hw;  // EPI_F32: >0 writes NCHW (H*W per channel), 0 row-major
  // EPI_F32 hidden outputs (LUT path): also the next layer's lattice levels of
  // the stored fp32 values (null when no KAN layer consumes the tensor)
  uint16_t* out_lv;
  int ld_lv;
  // ky-shared 3x3 conv kernel (kan_conv3_kernel): ext_rows = (bh+2)*Wo input
  // pixels expanded once per (kx, channel chunk) "super-stage" and read by the
  // three ky taps through descriptors offset by ky*Wo rows; n_ss super-stages
  // per tile; b_slot = bytes of one tap's weight tile (spline + SiLU parts)
  int ext_rows, n_ss, b_slot;
  int kym;   // kan_convw: ky-merged MMA issue (weight taps per kx in reversed ky order)
  int lock;  // kan_convw: one commit per K block (the window slot's barrier also releases the weight slot)
  int dual;  // kan_convw: two MMA-issuing warps (even / odd accumulators); needs lock, no ky merge, no multicast
  // fused output layer (split-K launches, LUT path): the reduced hidden levels
  // of each CTA's rows stay in smem and feed the next, small KAN layer
  // (N2 <= 16, NBP = 8, per-channel weights) inside this kernel, which writes
  // the model output; f_wq [n_in2][N2] 8 basis weights per (input, output),
  // f_wqb [N2][n_in2] SiLU base weights, both bulk-copied to smem
  int f_on, f_N, f_silu, f_epi, f_ld_out, f_wq_bytes, f_wqb_bytes;
  int stg_on;  // fp32 epilogue staged through smem (the fused-layer region) for row-coalesced stores
  const unsigned long long* f_wq;
  const int8_t* f_wqb;
  const double* f_fs;
  const long long* f_corr;
  void* f_out;
  // optional per-CTA phase timestamps (%globaltimer ns) for tuning:
  // [cta][8] = start, tables ready, first A stage, last A stage, TMEM full,
  // partials exchanged, done
  unsigned long long* dbg;
  int dbg_flags;  // tuning only: bit0 producers write zeros, bit1 skip the MMAs
};

// Small-N LUT layer on CUDA cores (N <= 16, NBP = 8): the per-input 4-code
// dot products as mixed-sign dp4a against the 4 weights selected at byte jj.
struct SmallParams {
  int M, n_in, N, x_kind, ld_x, k, L, mode;  // mode: MODE_PLAIN / MODE_ZP / MODE_SILU
  const void* x;
  const uint8_t* tab;  // standard blob: vals at 0, thr at off_thr, SiLU codes at off_silu
  int tab_bytes, off_thr, off_silu;
  float lo_f, inv_step_f;
  const unsigned long long* wq;  // [n_in][N] 8 basis weights (int8 bytes b = 0..7)
  const int8_t* wqb;             // [N][8][n_in8/8] SiLU base weights (int8) in thread order, n_in8 = roundup(n_in, 64)
  int n_in8;
  int epi;
  void* out;
  int ld_out;
  double f_tensor;
  long long z_w;
  const double* fs;
  const long long* corr_b;
  double n_lo, n_hi_open, n_step, n_inv_step;
  int n_L;
  double out_scale, inv_out_scale;
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

// Spline-table layer (spline_table.hpp:90-123): out = s_out * sum_i (T - z_out).
enum StInKind : int { ST_IN_U8 = 0, ST_IN_F32 = 1 };
struct StParams {
  int64_t rows;  // dense: M; conv: n_img * Ho * Wo (rows ordered (img, oy, ox))
  int n_in, n_out, Np, Lv;
  int lpr, col_tiles, ic;  // lanes per row (16 columns each), column tiles, staged inputs per chunk
  int slices;              // input slices per row (partial sums meet in smem)
  int ft;                  // fp32 tables (fake-quant mode): Np is the row size in bytes
  const uint8_t* T;        // [roundup4(n_in)][Lv][Np]; padded inputs are all-zero slices
  // input: dense rows [rows][ld_x] (u8 levels or fp32 values), or conv u8 NCHW
  int in_kind;
  const void* x;
  int64_t ld_x;
  const float* thr;  // fp32 input: thr[n] = smallest x with level >= n, n = 1..Lv-1
  float inv_s, zf;
  int conv, C, H, W, K, cstride, pad, Ho, Wo, lvl0;
  // epilogue: EPI_F32 (row-major, or NCHW for conv), EPI_LEVEL (u8 levels of
  // the consumer), EPI_RAW (int32 sums minus corr)
  int epi;
  void* out;
  int64_t ld_out;
  long long corr;  // n_in * z_out
  double out_s;
  double in_s, in_zd;  // the consumer's input quantizer (EPI_LEVEL; also the fp32 input's)
  long long in_qhi;
  // EPI_LEVEL: vthr[n] = smallest sum v (minus corr) whose output s_out * v has
  // level >= n (n = 1..in_qhi), ratio_f = s_out / in_s for the fp32 estimate
  const int* vthr;
  float ratio_f;
  // fake-quant EPI_LEVEL: the consuming layer's input quantizer (calibrated
  // ranges give every KAN layer its own): thresholds, 1/s, z, q_hi
  const float* o_thr;
  float o_inv_s, o_zf;
  int o_qhi;
  // fused output layer (dense rows, one warp per row): the hidden levels of
  // each row stay in smem and the next, last layer (n_out <= 16, tables
  // [n_in][Lv][16]) runs in the same warp; f_out gets its fp32 outputs
  int f_on, f_n_in, f_n_out, f_Lv;
  const uint8_t* f_T;
  long long f_corr;
  double f_out_s;
  float* f_out;
  int64_t f_ld_out;
};

}  // namespace kan
