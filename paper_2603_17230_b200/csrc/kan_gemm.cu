// kan_gemm.cu -- fused lattice-gather + tcgen05 GEMM for one KAN layer (sm_100a).
//
// Replaces, at layer granularity, the reference's
//   kan_linear_forward<LutBasis>  (proj/include/kantize/layers.hpp:99-116)
//   = clamp (grid.hpp:49-56) -> ActivationLattice::quantize (lut.hpp:44-47)
//     -> lut_basis_lookup (lut.hpp:136-160) -> dense B row (lut.hpp:189-195)
//     -> matmul (matrix.hpp:64-80)
// and, on the float path, kan_linear_forward<RecursiveBasis> (layers.hpp:118-121).
//
// One CTA computes a 128-row x BN-column output tile over a range of K, in
// KSTAGE (256) byte K stages of eight 32-byte tcgen05.mma steps.
// The dense basis ("A") tile never touches shared memory: producers write it
// straight into tensor memory, where tcgen05.mma reads it (A-from-TMEM form).
// Warp roles (608 threads, one CTA per SM):
//   warps 0..15  producers.  Thread (warp w, lane l) owns row 32*(w%4)+l and
//                K-quarter w/4 of every stage: it reads its row's activations
//                from the TMA-filled (swizzled) smem tile, computes each
//                lattice level (fp32 estimate + exact tie test), expands it
//                into the row of LUT codes (vals[frac] << 8*jj) -- or the fp32
//                Cox-de Boor basis in bf16 on the float path -- and stores its
//                64 bytes into the TMEM A ring with one tcgen05.st.  They also
//                build the SiLU base rows and run the epilogue.
//   warp 16      TMA loader of the activation ring (released by producers).
//   warp 17      TMEM allocation + single-thread tcgen05.mma issuer.
//   warp 18      bulk-copy loader of the lattice tables and the pre-swizzled
//                weight (B) tiles (ring released by the MMA).
// The int32 (LUT) or fp32 (bf16) accumulator lives in TMEM columns [0, BN).
#include <cuda.h>
#include <utility>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "kan_internal.h"
#include "kan_ptx.cuh"

namespace kan {

// exact reference rounding: std::llround (half away from zero)
__device__ __forceinline__ long long llround_ref(double x) {
  const double t = trunc(x);
  double r = t;
  if (fabs(__dsub_rn(x, t)) >= 0.5) r = __dadd_rn(t, copysign(1.0, x));
  return __double2ll_rz(r);
}

// ActivationLattice::quantize(GridSpec::clamp_to_domain(y)) in fp64,
// same operation order as lut.hpp:44-47 / grid.hpp:49-56.
__device__ __forceinline__ int lattice_level_f64(double y, double lo, double hi_open, double step,
                                                 int L) {
  double t = (y < lo) ? lo : y;
  t = (hi_open < t) ? hi_open : t;
  long long a = llround_ref(__ddiv_rn(__dsub_rn(t, lo), step));
  if (a < 0) a = 0;
  if (a > L) a = L;
  return static_cast<int>(a);
}

// float basis (bf16 path): local Cox-de Boor triangle in fp32 (grid.hpp:124-140
// restricted to the P+1 supported functions), knot units.
template <int PMAX>
__device__ __forceinline__ int basis_f32(float x, float lo, float hi_open, float inv_delta, int G,
                                         int P, float (&N)[PMAX + 1]) {
  x = fminf(fmaxf(x, lo), hi_open);
  const float xi = (x - lo) * inv_delta + static_cast<float>(P);
  int j = static_cast<int>(floorf(xi));
  j = min(max(j, P), G + P - 1);
#pragma unroll
  for (int r = 0; r <= PMAX; ++r) N[r] = 0.f;
  N[PMAX] = 1.f;  // N[PMAX - d + r] holds basis (j - d + r) at degree d
#pragma unroll
  for (int d = 1; d <= PMAX; ++d) {
    if (d > P) break;
    const float rd = 1.0f / static_cast<float>(d);
#pragma unroll
    for (int r = 0; r <= d; ++r) {
      const int i = j - d + r;
      const float left = (r == 0) ? 0.f : N[PMAX - d + r];       // B_i^{d-1}
      const float right = (r == d) ? 0.f : N[PMAX - d + r + 1];  // B_{i+1}^{d-1}
      const float d1 = (xi - static_cast<float>(i)) * rd;
      const float d2 = (static_cast<float>(i + d + 1) - xi) * rd;
      N[PMAX - d + r] = d1 * left + d2 * right;
    }
  }
  if (P < PMAX) {
    const int sh = PMAX - P;
#pragma unroll
    for (int r = 0; r <= PMAX; ++r) {
      float v = 0.f;
#pragma unroll
      for (int q = 0; q <= PMAX; ++q) v = (q == r + sh) ? N[q] : v;
      N[r] = v;
    }
  }
  return j - P;
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}

// shift `bits` of new data into the top of a 128-bit little-endian register
__device__ __forceinline__ void shift_in(uint32_t (&w)[4], uint32_t v, int bits) {
  w[0] = __funnelshift_r(w[0], w[1], bits);
  w[1] = __funnelshift_r(w[1], w[2], bits);
  w[2] = __funnelshift_r(w[2], w[3], bits);
  w[3] = __funnelshift_r(w[3], v, bits);
}


// Correctly rounded division, kept out of line: it is only taken for values
// within 1e-7 of a rounding tie, and inlining it per element bloats the
// epilogue that runs once per CTA out of a cold instruction cache.
__device__ __noinline__ double ddiv_rn_slow(double a, double b) { return __ddiv_rn(a, b); }

// Exact ActivationLattice::quantize(clamp_to_domain(y)) without a division on
// the common path: q = (t - lo) * (1/step) is within ~1e-12 of RN((t-lo)/step)
// for every level range the engine supports (L <= 4096), so llround(q) equals
// the reference's llround(RN((t-lo)/step)) unless q lies within 1e-7 of a
// half-integer; only then is the correctly rounded division evaluated.
// Branch-free part of lattice_level_fast: the level from the multiply, plus
// whether q lies in the tie band (then the caller redoes it with
// lattice_level_f64, the division form).  Epilogues evaluate 16 of these with
// no branch in between, so the fp64 chains overlap instead of running one
// after another behind a per-element branch; ties are fixed up afterwards.
__device__ __forceinline__ int level_mul(double y, double lo, double hi_open, double inv_step, int L, bool& tie) {
  double t = (y < lo) ? lo : y;
  t = (hi_open < t) ? hi_open : t;
  const double q = __dmul_rn(__dsub_rn(t, lo), inv_step);  // in [0, L + 1) (or NaN)
  // round q to the nearest integer by the 2^52 shift (no conversion unit):
  // the integer sits in the low word; it is llround(q) unless q is a tie, and
  // ties lie in the band |q - rint(q)| > 0.5 - 1e-7 that is redone exactly.
  // NaN leaves a zero low word: level 0, as llround's INT64_MIN clamps.
  const double m = __dadd_rn(q, 4503599627370496.0);
  const int a = __double2loint(m);
  tie = fabs(__dsub_rn(q, __dsub_rn(m, 4503599627370496.0))) > 0.5 - 1e-7;
  return a > L ? L : a;
}
// Branch-free part of lattice_level_tie: the fp32 estimate rounded to the
// nearest integer by the 1.5 * 2^23 shift, plus whether it lies near a
// rounding tie (then the threshold test decides).
__device__ __forceinline__ int level_tie_est(float x, float inv_step, float nlo_step, int L, bool& tie) {
  float t = fmaf(x, inv_step, nlo_step);
  t = fminf(fmaxf(t, 0.0f), static_cast<float>(L));  // NaN -> 0
  const float m = __fadd_rn(t, 12582912.0f);
  tie = fabsf(fabsf(__fsub_rn(t, __fsub_rn(m, 12582912.0f))) - 0.5f) < 2e-3f;
  return __float_as_int(m) - 0x4B400000;
}
// exact int32 -> fp64 without the conversion unit (2^52 + 2^31 shift)
__device__ __forceinline__ double i32_to_f64(uint32_t v) {
  return __dsub_rn(__hiloint2double(0x43300000, static_cast<int>(v ^ 0x80000000u)), 4503601774854144.0);
}

// out-of-line tie fix-ups (rare; kept out of the epilogues' hot code)
__device__ __noinline__ int level_fixup_f64(double y, double lo, double hi_open, double step, int L) {
  return lattice_level_f64(y, lo, hi_open, step, L);
}
__device__ __noinline__ int level_fixup_f32(float x, float inv_step, float nlo_step, int L, const float* thr) {
  float t = fmaf(x, inv_step, nlo_step);
  t = fminf(fmaxf(t, 0.0f), static_cast<float>(L));
  const int g = static_cast<int>(floorf(t));
  return g + ((x >= thr[g + 1]) ? 1 : 0);
}

// 8 next-layer levels of fp64 values yf(0..7), packed two per word: the
// branch-free estimates first (their fp64 chains overlap), tie fix-ups after
template <class YF>
__device__ __forceinline__ void levels8_f64(YF yf, double lo, double hi_open, double step, double inv_step, int L,
                                            uint32_t* w) {
  int lv[8];
  uint32_t ties = 0;
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    bool t;
    lv[e] = level_mul(yf(e), lo, hi_open, inv_step, L, t);
    ties |= static_cast<uint32_t>(t) << e;
  }
  if (ties) {
#pragma unroll
    for (int e = 0; e < 8; ++e)
      if ((ties >> e) & 1u) lv[e] = level_fixup_f64(yf(e), lo, hi_open, step, L);
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) w[q] = static_cast<uint32_t>(lv[2 * q]) | (static_cast<uint32_t>(lv[2 * q + 1]) << 16);
}
// 8 lattice levels of fp32 values xf(0..7) (lattice_level_tie), same scheme
template <int N = 8, class XF>
__device__ __forceinline__ void levels8_f32(XF xf, float inv_step, float nlo_step, int L, const float* thr, int* lv) {
  uint32_t ties = 0;
#pragma unroll
  for (int e = 0; e < N; ++e) {
    bool t;
    lv[e] = level_tie_est(xf(e), inv_step, nlo_step, L, t);
    ties |= static_cast<uint32_t>(t) << e;
  }
  if (ties) {
#pragma unroll
    for (int e = 0; e < N; ++e)
      if ((ties >> e) & 1u) lv[e] = level_fixup_f32(xf(e), inv_step, nlo_step, L, thr);
  }
}

__device__ __forceinline__ int lattice_level_fast(double y, double lo, double hi_open, double step,
                                                  double inv_step, int L) {
  double t = (y < lo) ? lo : y;
  t = (hi_open < t) ? hi_open : t;
  const double d = __dsub_rn(t, lo);
  // q >= 0 (or NaN), q < L + 1: llround(q) = trunc(q + 0.5), and q + 0.5 is
  // exact below 2^52; f = the fraction of q + 0.5, so q is within 1e-7 of a
  // half-integer exactly when f < 1e-7 or f > 1 - 1e-7 (then divide)
  const double u = __dadd_rn(__dmul_rn(d, inv_step), 0.5);
  int a = __double2int_rz(u);
  const double f = __dsub_rn(u, static_cast<double>(a));
  if (f < 1e-7 || f > 1.0 - 1e-7) a = __double2int_rz(__dadd_rn(ddiv_rn_slow(d, step), 0.5));
  a = a < 0 ? 0 : a;  // NaN converts to INT_MIN: level 0, as llround's INT64_MIN clamps
  return a > L ? L : a;
}

// clamp(llround(y / s), -127, 127) with the same guarded-multiply rule
// (llround = trunc(q +- 0.5), exact for |q| < 2^52)
__device__ __forceinline__ int requant_i8(double y, double s, double inv_s) {
  double q = __dmul_rn(y, inv_s);
  double u = __dadd_rn(q, q < 0.0 ? -0.5 : 0.5);
  long long v = __double2ll_rz(u);
  const double f = fabs(__dsub_rn(u, static_cast<double>(v)));
  if (fabs(q) < 1024.0 && (f < 1e-7 || f > 1.0 - 1e-7)) {
    q = ddiv_rn_slow(y, s);
    v = __double2ll_rz(__dadd_rn(q, q < 0.0 ? -0.5 : 0.5));
  }
  v = v < -127 ? -127 : (v > 127 ? 127 : v);
  return static_cast<int>(v);
}

// ---- distributed shared memory / cluster helpers ---------------------------
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_id_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t n_clusters_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ uint4 ld_cluster_v4(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared::cluster.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(addr)
               : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_cluster_u32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
  return v;
}

// ---------------------------------------------------------------------------
enum { MODE_PLAIN = 0, MODE_ZP = 1, MODE_SILU = 2 };


// ring slot/phase counter without division
struct Ring {
  int slot = 0, n;
  uint32_t phase = 0;
  __device__ explicit Ring(int n_) : n(n_) {}
  __device__ __forceinline__ void next() {
    if (++slot == n) {
      slot = 0;
      phase ^= 1u;
    }
  }
};

template <bool BF16, int NBP>
struct Cfg {
  static constexpr int ESZ = BF16 ? 2 : 1;
  static constexpr int IPS = KSTAGE / (NBP * ESZ);  // inputs per K stage
  static constexpr int Q = IPS / 4;                 // inputs per producer thread per stage
  static constexpr int GS = KSTAGE / ESZ / IPS;     // spline stages per SiLU group
  static constexpr int SW = Q * ESZ / 4;            // SiLU code words per thread per stage
};

// A-from-TMEM MMAs (M = 128, B K-major in smem)
__device__ __forceinline__ void mma_i8_ts(uint32_t d, uint32_t a_tmem, uint64_t bdesc,
                                          uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_f16_ts(uint32_t d, uint32_t a_tmem, uint64_t bdesc,
                                           uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// Byte offset of 16-byte chunk `c` of row `r` in a TMA tile whose rows are
// `row_bytes` wide and written with the matching swizzle (128 / 64 / 32 B rows:
// SWIZZLE_128B / 64B / 32B).  The swizzle makes a warp's row-per-lane 16-byte
// reads bank-conflict free.
__device__ __forceinline__ uint32_t xtile_off(int r, int c, int row_bytes) {
  const int sw = row_bytes == 128 ? (r & 7)
                 : row_bytes == 64 ? ((r >> 1) & 3)
                                   : ((r >> 2) & 1);
  return static_cast<uint32_t>(r * row_bytes + ((c ^ sw) << 4));
}

// This thread's NB activation bytes (NB = 8, 16 or 32) at byte `off` of row r.
template <int NB>
__device__ __forceinline__ void load_x(const uint8_t* xt, int r, int off, int row_bytes,
                                       uint32_t (&d)[NB / 4]) {
  if constexpr (NB == 32) {
    const uint4 a = *reinterpret_cast<const uint4*>(xt + xtile_off(r, off >> 4, row_bytes));
    const uint4 b = *reinterpret_cast<const uint4*>(xt + xtile_off(r, (off >> 4) + 1, row_bytes));
    d[0] = a.x; d[1] = a.y; d[2] = a.z; d[3] = a.w;
    d[4] = b.x; d[5] = b.y; d[6] = b.z; d[7] = b.w;
  } else if constexpr (NB == 16) {
    const uint4 a = *reinterpret_cast<const uint4*>(xt + xtile_off(r, off >> 4, row_bytes));
    d[0] = a.x; d[1] = a.y; d[2] = a.z; d[3] = a.w;
  } else {
    const uint2 a =
        *reinterpret_cast<const uint2*>(xt + xtile_off(r, off >> 4, row_bytes) + (off & 15));
    d[0] = a.x; d[1] = a.y;
  }
}

// Exact lattice level of an fp32 activation.  t = x*(1/step) - lo/step in one
// FFMA is within 7e-4 of the exact quotient (|x| <= 1, L <= 4096), so
// rint(t) is the reference's llround(RN((clamp(x)-lo)/step)) unless t lies
// within 2e-3 of a half-integer; only then (p ~ 4e-3) is the threshold table
// thr[n] = min{x : level(x) >= n} consulted.
__device__ __forceinline__ int lattice_level_tie(float x, float inv_step, float nlo_step, int L,
                                                 const float* thr) {
  float t = fmaf(x, inv_step, nlo_step);  // nlo_step = -lo/step
  t = fminf(fmaxf(t, 0.0f), static_cast<float>(L));
  const float tr = rintf(t);
  int g = static_cast<int>(tr);
  if (fabsf(fabsf(t - tr) - 0.5f) < 2e-3f) {
    g = static_cast<int>(floorf(t));
    g += (x >= thr[g + 1]) ? 1 : 0;
  }
  return g;
}
__device__ __forceinline__ int lattice_level_x(float x, const GemmParams& p, const float* thr) {
  return lattice_level_tie(x, p.inv_step_f, p.lo_f, p.L, thr);  // p.lo_f holds -lo/step
}

// 64 bytes of one A row (this thread's K-quarter of a stage) on the LUT path,
// plus the stage's SiLU code words.  The P+1 codes of lut_basis_lookup
// (lut.hpp:136-160) placed at byte jj = a >> k of the input's NBP-byte row
// segment: for NBP = 8 one 64-bit entry per level (c64[a], built on the host
// from the same lookup); for NBP = 16 vals[frac] (frac = a mod 2^k) shifted
// into place with clamped funnel shifts (branch-free).
template <int NBP, int MODE>
__device__ __forceinline__ void lut_row(const GemmParams& p, const uint32_t* vals,
                                        const uint2* c64, const uint8_t* silu_tab,
                                        const int (&a)[64 / NBP], int i0, uint32_t (&w)[16],
                                        uint32_t& rsum, uint32_t (&nw)[16 / NBP]) {
  constexpr int H = 64 / NBP;  // inputs in this thread's quarter
  const int mask = (1 << p.k) - 1;
  const uint32_t lane = threadIdx.x & 31;
#pragma unroll
  for (int e = 0; e < H; ++e) {
    if constexpr (NBP == 8) {
      if (p.rep) {
        // lane-private copy of vals: conflict-free
        const uint32_t v = vals[((static_cast<uint32_t>(a[e]) & mask) << 5) | lane];
        const unsigned long long pt = static_cast<unsigned long long>(v) << (8 * (a[e] >> p.k));
        w[2 * e] = static_cast<uint32_t>(pt);
        w[2 * e + 1] = static_cast<uint32_t>(pt >> 32);
        if constexpr (MODE == MODE_ZP) {
          // codes shifted past the row end are zero (see lut_basis_lookup)
          if (i0 + e < p.n_ch) rsum = __dp4a(v, 0x01010101u, rsum);
        }
      } else {
        const uint2 c = c64[a[e]];
        w[2 * e] = c.x;
        w[2 * e + 1] = c.y;
        if constexpr (MODE == MODE_ZP) {
          if (i0 + e < p.n_ch) rsum = __dp4a(c.y, 0x01010101u, __dp4a(c.x, 0x01010101u, rsum));
        }
      }
    } else {
      const uint32_t v = vals[a[e] & mask];
      const uint32_t sft = 8u * static_cast<uint32_t>(a[e] >> p.k);
      w[4 * e] = __funnelshift_lc(0u, v, sft);
#pragma unroll
      for (uint32_t q = 1; q < 4; ++q)
        w[4 * e + q] = __funnelshift_lc(0u, v, sft - 32u * q) | __funnelshift_rc(v, 0u, 32u * q - sft);
      if constexpr (MODE == MODE_ZP) {
        if (i0 + e < p.n_ch) rsum = __dp4a(v, 0x01010101u, rsum);
      }
    }
  }
  if constexpr (MODE == MODE_SILU) {
    if (NBP == 8 && p.rep == 1) {
      // lane-private packed codes: word (a >> 2) of this lane, byte a & 3
      const uint32_t* srep = reinterpret_cast<const uint32_t*>(silu_tab);
#pragma unroll
      for (int q = 0; q < H / 4; ++q) {
        uint32_t wd[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) wd[t] = srep[((static_cast<uint32_t>(a[4 * q + t]) >> 2) << 5) | lane];
        const uint32_t lo = __byte_perm(wd[0], wd[1], (a[4 * q] & 3) | ((4 + (a[4 * q + 1] & 3)) << 4));
        const uint32_t hi = __byte_perm(wd[2], wd[3], (a[4 * q + 2] & 3) | ((4 + (a[4 * q + 3] & 3)) << 4));
        nw[q] = __byte_perm(lo, hi, 0x5410);
      }
    } else {
#pragma unroll
      for (int q = 0; q < H / 4; ++q)
        nw[q] = static_cast<uint32_t>(silu_tab[a[4 * q]]) |
                (static_cast<uint32_t>(silu_tab[a[4 * q + 1]]) << 8) |
                (static_cast<uint32_t>(silu_tab[a[4 * q + 2]]) << 16) |
                (static_cast<uint32_t>(silu_tab[a[4 * q + 3]]) << 24);
    }
  }
}

// 64 bytes of one A row on the bf16 path: fp32 Cox-de Boor basis -> bf16.
template <int NBP, int MODE>
__device__ __forceinline__ void bf16_row(const GemmParams& p, const float (&x)[32 / NBP],
                                         uint32_t (&w)[16], uint32_t (&nw)[16 / NBP]) {
  constexpr int H = 32 / NBP;  // inputs in this thread's quarter (bf16: NBP*2 bytes each)
  constexpr int PMAX = 3;
#pragma unroll
  for (int e = 0; e < H; ++e) {
    float Nv[PMAX + 1];
    int jj;
    if (p.P == 3) {
      // uniform cubic: the local Cox-de Boor triangle in closed form (same
      // basis; fp32 rounding differs by ~1e-7, far inside the bf16 bar)
      const float xc = fminf(fmaxf(x[e], p.flo), p.fhi_open);
      const float xi = (xc - p.flo) * p.finv_delta + 3.0f;
      int j = static_cast<int>(floorf(xi));
      j = min(max(j, 3), p.G + 2);
      const float u = xi - static_cast<float>(j), v = 1.0f - u;
      const float u2 = u * u, u3 = u2 * u;
      constexpr float s6 = 1.0f / 6.0f;
      Nv[0] = v * v * v * s6;
      Nv[1] = fmaf(3.0f, u3, fmaf(-6.0f, u2, 4.0f)) * s6;
      Nv[2] = fmaf(-3.0f, u3, fmaf(3.0f, u2, fmaf(3.0f, u, 1.0f))) * s6;
      Nv[3] = u3 * s6;
      jj = j - 3;
    } else {
      jj = basis_f32<PMAX>(x[e], p.flo, p.fhi_open, p.finv_delta, p.G, p.P, Nv);
    }
    // the P+1 values as bf16 at slots jj.. of the NBP-slot row: pack them into
    // up to three words (shifted by half a word when jj is odd), then place
    const uint32_t lo = pack_bf16(Nv[0], Nv[1]), hi = pack_bf16(Nv[2], Nv[3]);
    const bool odd = (jj & 1) != 0;
    const uint32_t A = odd ? (lo << 16) : lo;
    const uint32_t B = odd ? __funnelshift_l(lo, hi, 16) : hi;
    const uint32_t Cw = odd ? (hi >> 16) : 0u;
    const int w0 = jj >> 1;
#pragma unroll
    for (int q = 0; q < NBP / 2; ++q)
      w[e * (NBP / 2) + q] = q == w0 ? A : (q == w0 + 1 ? B : (q == w0 + 2 ? Cw : 0u));
  }
  if constexpr (MODE == MODE_SILU) {
#pragma unroll
    for (int q = 0; q < H / 2; ++q) {
      float s2[2];
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const float xc = fminf(fmaxf(x[2 * q + t], p.flo), p.fhi_open);
        s2[t] = __fdividef(xc, 1.0f + __expf(-xc));
      }
      nw[q] = pack_bf16(s2[0], s2[1]);
    }
  }
}

// u8 x s8 dot product of 4 byte pairs (dp4a.u32.s32): LUT codes x int8 weights
__device__ __forceinline__ int dp4a_us(uint32_t a, uint32_t b, int c) {
  int d;
  asm("dp4a.u32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

// Walk over the conv taps in spline-stage order (tap-major, channel chunk
// minor), without divisions in the loop.
struct TapWalk {
  int cc = 0, kx = 0, ky = 0, tap = 0;
  __device__ TapWalk(const GemmParams& p, int sp0) {
    if (p.conv) {
      tap = sp0 / p.cps;
      cc = sp0 - tap * p.cps;
      ky = tap / p.ksz;
      kx = tap - ky * p.ksz;
    }
  }
  __device__ __forceinline__ void next(const GemmParams& p) {
    if (++cc == p.cps) {
      cc = 0;
      ++tap;
      if (++kx == p.ksz) {
        kx = 0;
        ++ky;
      }
    }
  }
};

// FE: a straight-line epilogue is compiled in -- 1: fp32 row-major output
// (+ levels sidecar), 2: next-layer levels, 3: residual add then levels.  Separate instantiations, so the
// other variants keep their register allocation.
template <bool BF16, int NBP, int MODE, int FE = 0>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    kan_gather_gemm_kernel(const __grid_constant__ CUtensorMap xmap, const GemmParams p) {
  using C = Cfg<BF16, NBP>;
  constexpr int NPW = GEMM_PRODUCER_WARPS, NP = 32 * NPW;
  constexpr int W_X = NPW, W_MMA = NPW + 1, W_B = NPW + 2, W_EPI = NPW + 3;  // + 4 epilogue warps
  constexpr bool SILU = (MODE == MODE_SILU);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);

  const int SA = p.SA, SB = p.SB, SX = p.SX;
  const int BN = p.BN;
  const uint32_t b_bytes = static_cast<uint32_t>(BN) * KSTAGE;
  const uint32_t xesz = (p.x_kind == X_F32) ? 4u : 2u;
  const int x_row_bytes = C::IPS * static_cast<int>(xesz);
  const uint32_t x_bytes = 128u * static_cast<uint32_t>(x_row_bytes);
  uint8_t* sB = smem;
  uint8_t* sX = sB + static_cast<size_t>(SB) * b_bytes;
  uint8_t* sT = sX + static_cast<size_t>(SX) * x_bytes;  // lattice tables (LUT path)
  const int tab_bytes = BF16 ? 0 : p.tab_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sT + tab_bytes);
  int32_t* s_rowsum = reinterpret_cast<int32_t*>(bars + 2 * SA + 2 * SB + 2 * SX + 9);  // [2][4][128]
  // the current tile's column constants: scale fs[j] and SiLU correction (as double)
  double* s_cols = reinterpret_cast<double*>(s_rowsum + 2 * 4 * 128);  // [2][BN]
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(s_cols + 2 * BN);
  // SiLU code staging (MODE_SILU): word wd of K-quarter h of row r at
  // ((h*8 + wd/2)*128 + r)*2 + (wd&1) -- written once per spline stage, read
  // back by the same thread for the group's base stage (conflict-free).
  // Offset arithmetic from smem keeps the compiler on shared-memory accesses.
  const uint32_t sil_off = ((static_cast<uint32_t>(reinterpret_cast<uint8_t*>(s_tmem + 4) - smem)) + 15u) & ~15u;
  uint32_t* s_sil = reinterpret_cast<uint32_t*>(smem + sil_off);
  // fused output layer: its weights and the CTA's hidden-level rows [128][BN]
  const uint32_t f_off = sil_off + (SILU ? 4u * 8u * 128u * 8u : 0u);
  unsigned long long* f_wq = reinterpret_cast<unsigned long long*>(smem + f_off);
  int8_t* f_wqb = reinterpret_cast<int8_t*>(smem + f_off + p.f_wq_bytes);
  uint16_t* f_lv = reinterpret_cast<uint16_t*>(smem + f_off + p.f_wq_bytes + p.f_wqb_bytes);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  unsigned long long* dbg = p.dbg ? p.dbg + 8 * (static_cast<size_t>(blockIdx.z) * gridDim.x + blockIdx.x)
                                  : nullptr;
  auto stamp = [&](int i) {
    if (dbg) dbg[i] = globaltimer();
  };
  if (threadIdx.x == 0) stamp(0);
  pdl_trigger();

  // Tiles: 1D index, N tile fastest (CTAs sharing an activation tile run
  // together).  splits == 1: persistent, this CTA takes tiles blockIdx.x,
  // blockIdx.x + gridDim.x, ...; splits > 1: one tile per CTA, K groups split
  // over the cluster along z.
  const bool persistent = p.splits == 1;
  const int n_tiles = p.m_tiles * p.n_tiles_n;
  const int tile_step = persistent ? static_cast<int>(gridDim.x) : n_tiles;
  const int split = blockIdx.z;
  const int g0 = persistent ? 0 : split * p.groups_per_split;
  const int g1 = persistent ? p.n_groups : min(p.n_groups, g0 + p.groups_per_split);
  const bool has_work = g0 < g1;
  const int spg = C::GS + (SILU ? 1 : 0);
  struct Tile {
    int m0, n_tile, n0, y0;
  };
  auto tile_of = [&](int t) {
    Tile r;
    const int mt = t / p.n_tiles_n;
    r.n_tile = t - mt * p.n_tiles_n;
    r.m0 = mt * 128;
    // conv tiles: first image and first output row of the M tile
    r.n0 = p.conv ? (mt / p.tpi) * p.bn_img : 0;
    r.y0 = p.conv ? (mt % p.tpi) * p.bh : 0;
    return r;
  };

  auto bar_xfull = [&](int s) { return smem_u32(bars + s); };
  auto bar_xempty = [&](int s) { return smem_u32(bars + SX + s); };
  auto bar_afull = [&](int s) { return smem_u32(bars + 2 * SX + s); };
  auto bar_aempty = [&](int s) { return smem_u32(bars + 2 * SX + SA + s); };
  auto bar_bfull = [&](int s) { return smem_u32(bars + 2 * SX + 2 * SA + s); };
  auto bar_bempty = [&](int s) { return smem_u32(bars + 2 * SX + 2 * SA + SB + s); };
  uint64_t* bx = bars + 2 * SX + 2 * SA + 2 * SB;
  auto bar_accfull = [&](int b) { return smem_u32(bx + b); };
  auto bar_accempty = [&](int b) { return smem_u32(bx + 2 + b); };
  auto bar_rsfull = [&](int b) { return smem_u32(bx + 4 + b); };
  auto bar_rsempty = [&](int b) { return smem_u32(bx + 6 + b); };
  const uint32_t bar_tab = smem_u32(bx + 8);

  // TMEM: nacc accumulators of BNa columns (two when they fit, so the epilogue
  // of one tile overlaps the next tile's MMAs), then the A ring of KSTAGE/4-
  // column slots
  constexpr uint32_t tmem_cols = 512;
  constexpr uint32_t acols = KSTAGE / 4;
  const uint32_t BNa = static_cast<uint32_t>((BN + 31) / 32 * 32);
  const int nacc = p.nacc;
  const uint32_t acol0 = static_cast<uint32_t>(nacc) * BNa;

  // ---- setup -------------------------------------------------------------
  if (threadIdx.x == 0) {
    for (int s = 0; s < SX; ++s) {
      mbar_init(bar_xfull(s), 1);
      mbar_init(bar_xempty(s), NPW);
    }
    for (int s = 0; s < SA; ++s) {
      mbar_init(bar_afull(s), NPW);
      mbar_init(bar_aempty(s), 1);
    }
    for (int s = 0; s < SB; ++s) {
      mbar_init(bar_bfull(s), 1);
      mbar_init(bar_bempty(s), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(bar_accfull(b), 1);
      mbar_init(bar_accempty(b), GEMM_EPI_WARPS);
      mbar_init(bar_rsfull(b), NPW);
      mbar_init(bar_rsempty(b), GEMM_EPI_WARPS);
    }
    mbar_init(bar_tab, 1);
    mbar_fence_init();
  }
  if (KAN_DBG(p, 4))  // tuning only (no activation loads): a zero activation ring
    for (uint32_t q = threadIdx.x; q < static_cast<uint32_t>(SX) * x_bytes / 4; q += blockDim.x)
      reinterpret_cast<uint32_t*>(sX)[q] = 0u;
  if (warp == W_X && lane == 0) tma_prefetch(&xmap);
  if (warp == W_MMA) tmem_alloc(smem_u32(s_tmem), tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;

  // Stage tile n_tile's column constants (fs, SiLU correction) in smem: the
  // epilogue reads them per element, and global loads there would serialize
  // one memory latency per column.  Threads [t0, t0 + nt) of the caller.
  auto load_cols = [&](int n_tile, int t0, int nt) {
    if constexpr (!BF16 && MODE != MODE_ZP) {
      for (int i = static_cast<int>(threadIdx.x) - t0; i < BN; i += nt) {
        const int j = min(n_tile * BN + i, p.N - 1);
        s_cols[i] = p.fs[j];
        s_cols[BN + i] = SILU ? static_cast<double>(p.corr_b[j]) : 0.0;
      }
    }
  };
  // Fused output layer (LUT path, N2 <= 16, per-channel weights) over `rows`
  // rows of this CTA's hidden-level buffer f_lv (row pitch BN + 4 levels, so a
  // warp's rows fall in different banks), starting at local row rl0, by `nthr`
  // threads (tid 0 .. nthr-1): TPR = nthr / rows threads per row (a power of
  // two <= 32, so a row's threads share a warp).  Thread sub takes `per`
  // consecutive inputs, four at a time: their 8-byte code rows (vals[frac]
  // shifted to byte jj) and one word of their SiLU codes, then for every output
  // j the four 8-byte weight rows (two mixed-sign dp4a each) and one word of
  // base weights (one dp4a): independent chains over j, every load issued
  // before its use.  Xor-shuffle reduction over the row's threads, then thread
  // j mod TPR finishes output j with the fp64 epilogue.  The same integer sums
  // as kan_small_layer_kernel, so the same outputs.
  auto fused_output = [&](int tid, int nthr, int rl0, int rows, int m0) {
    const int TPR = nthr / rows;
    const int lr = tid / TPR, sub = tid % TPR;
    const int rl = rl0 + lr;
    const int n2 = p.f_N, n_in2 = p.N;
    const int row = m0 + rl;
    const bool valid_row = row < p.M;  // rows past M were never written
    const uint32_t* vals = reinterpret_cast<const uint32_t*>(sT);
    const uint8_t* silu_tab = sT + p.off_silu;
    const uint32_t mask = (1u << p.k) - 1u;
    const uint16_t* lvr = f_lv + rl * (BN + 4);
    const int per = (((n_in2 + TPR - 1) / TPR) + 3) & ~3;
    const int i_beg = sub * per, i_end = min(n_in2, i_beg + per);
    int acc[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[j] = 0;
    if (valid_row) {
#pragma unroll 1
      for (int i0 = i_beg; i0 < i_end; i0 += 4) {
        const uint2 l4 = *reinterpret_cast<const uint2*>(lvr + i0);  // 4 levels (n_in2 % 4 == 0)
        uint32_t clo[4], chi[4], sw = 0u;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const uint32_t a = ((e < 2 ? l4.x : l4.y) >> (16 * (e & 1))) & 0xFFFFu;
          const uint32_t v = p.rep ? vals[((a & mask) << 5) | static_cast<uint32_t>(lane)] : vals[a & mask];
          const unsigned long long pt = static_cast<unsigned long long>(v) << (8u * (a >> p.k));
          clo[e] = static_cast<uint32_t>(pt);
          chi[e] = static_cast<uint32_t>(pt >> 32);
          if (p.f_silu) sw |= static_cast<uint32_t>(silu_tab[a]) << (8 * e);
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          if (j < n2) {
            unsigned long long w[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) w[e] = f_wq[(i0 + e) * n2 + j];
            const uint32_t wb = p.f_silu ? *reinterpret_cast<const uint32_t*>(f_wqb + j * n_in2 + i0) : 0u;
            int t = acc[j];
#pragma unroll
            for (int e = 0; e < 4; ++e)
              t = dp4a_us(chi[e], static_cast<uint32_t>(w[e] >> 32), dp4a_us(clo[e], static_cast<uint32_t>(w[e]), t));
            acc[j] = dp4a_us(sw, wb, t);
          }
        }
      }
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1)
      if (off < TPR)
#pragma unroll
        for (int j = 0; j < 16; ++j) acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], off);
    if (valid_row) {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        if (j < n2 && (j & (TPR - 1)) == sub) {  // output j belongs to thread j mod TPR of the row
          const size_t o = static_cast<size_t>(row) * p.f_ld_out + j;
          const long long corr_j = p.f_silu ? p.f_corr[j] : 0ll;
          const double y = __dmul_rn(static_cast<double>(static_cast<long long>(acc[j]) - corr_j), p.f_fs[j]);
          if (p.f_epi == EPI_F32)
            static_cast<float*>(p.f_out)[o] = __double2float_rn(y);
          else
            static_cast<int8_t*>(p.f_out)[o] = static_cast<int8_t>(requant_i8(y, p.out_scale, p.inv_out_scale));
        }
      }
    }
  };

  // Epilogue of 4 accumulator columns of one output row (fp64, then the
  // requested output: raw, fp32, next-layer level, int8), shared by the
  // persistent epilogue warps and the split-K reduction.
  auto finish4 = [&](int row, int col0, const uint32_t(&ra)[4], int32_t rs, const float* rpre = nullptr) {
    if (row >= p.M) return;
    const size_t base = static_cast<size_t>(row) * p.ld_out + col0;
    const int nvalid = min(4, p.N - col0);
    if (p.epi == EPI_RAW) {
      uint32_t* o = reinterpret_cast<uint32_t*>(p.out) + base;
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (e < nvalid) o[e] = ra[e];
      return;
    }
    double y[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int j = min(col0 + e, p.N - 1);
      if constexpr (BF16) {
        y[e] = static_cast<double>(__uint_as_float(ra[e]));
      } else if constexpr (MODE == MODE_ZP) {
        const long long v =
            static_cast<long long>(static_cast<int32_t>(ra[e])) - p.z_w * static_cast<long long>(rs);
        y[e] = __dmul_rn(static_cast<double>(v), p.f_tensor);
      } else {
        // column constants staged in smem for the tile (load_cols)
        const int jl = j - (j / BN) * BN;
        const long long v = static_cast<long long>(static_cast<int32_t>(ra[e])) -
                            (SILU ? static_cast<long long>(s_cols[BN + jl]) : 0ll);
        y[e] = __dmul_rn(static_cast<double>(v), s_cols[jl]);
      }
    }
    if (p.res_kind) {
      // residual add of a stored fp32 tensor (engine extension, GemmParams::res_kind);
      // rpre: values the persistent epilogue prefetched
      const float* rr = rpre ? rpre : reinterpret_cast<const float*>(p.res) + static_cast<size_t>(row) * p.ld_res + col0;
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (e < nvalid) y[e] = __dadd_rn(y[e], static_cast<double>(rr[e]));
    }
    if (p.epi == EPI_F32 && p.out_hw > 0) {
      // NCHW model output (convkan_forward reshapes rows to [c_out, H, W], layers.hpp:179-184)
      const int hw = p.out_hw;
      const int img = row / hw;
      float* o = reinterpret_cast<float*>(p.out) + static_cast<size_t>(img) * p.N * hw +
                 static_cast<size_t>(col0) * hw + (row - img * hw);
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (e < nvalid) o[static_cast<size_t>(e) * hw] = __double2float_rn(y[e]);
    } else if (p.epi == EPI_F32) {
      float* o = reinterpret_cast<float*>(p.out) + base;
      if (nvalid == 4 && (reinterpret_cast<uintptr_t>(o) & 15) == 0) {
        *reinterpret_cast<float4*>(o) = make_float4(__double2float_rn(y[0]), __double2float_rn(y[1]),
                                                    __double2float_rn(y[2]), __double2float_rn(y[3]));
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (e < nvalid) o[e] = __double2float_rn(y[e]);
      }
      if constexpr (!BF16) {
        if (p.out_lv) {
          // levels sidecar: what the consuming KAN layer would compute from these values
          const float* thr = reinterpret_cast<const float*>(sT + p.off_thr);
          uint32_t a[4];
#pragma unroll
          for (int e = 0; e < 4; ++e)
            a[e] = static_cast<uint32_t>(lattice_level_tie(__double2float_rn(y[e]), p.inv_step_f, p.lo_f, p.L, thr));
          uint16_t* ol = p.out_lv + static_cast<size_t>(row) * p.ld_lv + col0;
          if (nvalid == 4 && (reinterpret_cast<uintptr_t>(ol) & 7) == 0) {
            *reinterpret_cast<uint2*>(ol) = make_uint2(a[0] | (a[1] << 16), a[2] | (a[3] << 16));
          } else {
#pragma unroll
            for (int e = 0; e < 4; ++e)
              if (e < nvalid) ol[e] = static_cast<uint16_t>(a[e]);
          }
        }
      }
    } else if (p.epi == EPI_LEVEL) {
      // fused output layer: the levels stay in this CTA's smem row buffer
      uint16_t* o = p.f_on ? f_lv + (row & 127) * (BN + 4) + (col0 % BN) : reinterpret_cast<uint16_t*>(p.out) + base;
      uint32_t a[4];
#pragma unroll
      for (int e = 0; e < 4; ++e)
        a[e] = static_cast<uint32_t>(lattice_level_fast(y[e], p.n_lo, p.n_hi_open, p.n_step, p.n_inv_step, p.n_L));
      if (nvalid == 4 && (reinterpret_cast<uintptr_t>(o) & 7) == 0) {
        *reinterpret_cast<uint2*>(o) = make_uint2(a[0] | (a[1] << 16), a[2] | (a[3] << 16));  // one 8-byte store
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (e < nvalid) o[e] = static_cast<uint16_t>(a[e]);
      }
    } else {  // EPI_I8
      int8_t* o = reinterpret_cast<int8_t*>(p.out) + base;
      uint32_t q[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) q[e] = static_cast<uint32_t>(requant_i8(y[e], p.out_scale, p.inv_out_scale)) & 0xFFu;
      if (nvalid == 4 && (reinterpret_cast<uintptr_t>(o) & 3) == 0) {
        *reinterpret_cast<uint32_t*>(o) = q[0] | (q[1] << 8) | (q[2] << 16) | (q[3] << 24);
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (e < nvalid) o[e] = static_cast<int8_t>(q[e]);
      }
    }
  };
  // Role loops run on whole warps (all lanes wait, lane 0 issues) so the warps
  // stay converged for the aligned barriers and tcgen05 ops that follow.
  if (warp == W_X) {
    // ========================= activation loader ==========================
    // the activations are the previous kernel's output: everything the other
    // roles read before the first x tile lands is constant (tables, weights)
    pdl_wait();
    Ring rx(SX);
    for (int t = blockIdx.x; t < n_tiles; t += tile_step) {
      const Tile tl = tile_of(t);
      TapWalk tw(p, g0 * C::GS);
      for (int g = g0; g < g1; ++g) {
        const int nsp = min(C::GS, p.n_spline_stages - g * C::GS);
        for (int s = 0; s < nsp; ++s, rx.next(), tw.next(p)) {
          mbar_wait(bar_xempty(rx.slot), rx.phase ^ 1);
          if (lane == 0) {
            const uint32_t dst = smem_u32(sX + static_cast<size_t>(rx.slot) * x_bytes);
            if (KAN_DBG(p, 4)) {  // tuning only: no activation load (stale tile)
              mbar_arrive(bar_xfull(rx.slot));
            } else {
            mbar_arrive_tx(bar_xfull(rx.slot), x_bytes);
            if (!p.conv) {
              tma_load_2d(dst, &xmap, (g * C::GS + s) * C::IPS, tl.m0, bar_xfull(rx.slot));
            } else {
              // the tap's input window: rows y0*stride + ky - pad.., columns kx - pad..
              // (element strides in the tensor map step by the conv stride)
              const int iy = tl.y0 * p.cstride + tw.ky - p.pad, ix = tw.kx - p.pad;
              tma_load_4d(dst, &xmap, tw.cc * C::IPS, ix, iy, tl.n0, bar_xfull(rx.slot));
            }
            }
          }
          __syncwarp();
        }
      }
    }
  } else if (warp == W_B) {
    // ===================== table + weight-tile loader =====================
    if (lane == 0 && tab_bytes > 0) {
      const uint32_t fb = p.f_on ? static_cast<uint32_t>(p.f_wq_bytes + p.f_wqb_bytes) : 0u;
      mbar_arrive_tx(bar_tab, static_cast<uint32_t>(tab_bytes) + fb);
      bulk_load(smem_u32(sT), p.tab, static_cast<uint32_t>(tab_bytes), bar_tab);
      if (p.f_on) {
        bulk_load(smem_u32(f_wq), p.f_wq, static_cast<uint32_t>(p.f_wq_bytes), bar_tab);
        bulk_load(smem_u32(f_wqb), p.f_wqb, static_cast<uint32_t>(p.f_wqb_bytes), bar_tab);
      }
    }
    __syncwarp();
    Ring rb(SB);
    for (int t = blockIdx.x; t < n_tiles; t += tile_step) {
      const Tile tl = tile_of(t);
      for (int g = g0; g < g1; ++g) {
        const int nsp = min(C::GS, p.n_spline_stages - g * C::GS);
        for (int s = 0; s < nsp + (SILU ? 1 : 0); ++s, rb.next()) {
          mbar_wait(bar_bempty(rb.slot), rb.phase ^ 1);
          if (lane == 0) {
            const size_t wt = static_cast<size_t>(tl.n_tile) * p.total_stages + g * spg + s;
            mbar_arrive_tx(bar_bfull(rb.slot), b_bytes);
            bulk_load(smem_u32(sB + static_cast<size_t>(rb.slot) * b_bytes), p.wt + wt * b_bytes,
                      b_bytes, bar_bfull(rb.slot));
          }
          __syncwarp();
        }
      }
    }
  } else if (warp == W_MMA) {
    // ============================ MMA issuer ==============================
    // Warp-uniform waits and operands, one elected lane issues (operands stay
    // in uniform registers: no per-MMA R2UR waterfall; it matters at small N).
    const uint32_t idesc = BF16 ? idesc_bf16(BN) : idesc_i8(BN, p.b_signed != 0);
    const bool no_mma = KAN_DBG(p, 2) != 0;
    const uint32_t b_kstep = static_cast<uint32_t>(BN) * 8u;  // next 128-byte K block (x16 B)
    Ring ra(SA), rb(SB);
    int lt = 0;
    for (int t = blockIdx.x; t < n_tiles; t += tile_step, ++lt) {
      const int ab = nacc == 2 ? (lt & 1) : 0;
      const int use = nacc == 2 ? (lt >> 1) : lt;
      // the accumulator must have been drained by the epilogue of its last tile
      mbar_wait_warp(bar_accempty(ab), (use & 1) ^ 1);
      tc_fence_after();
      const uint32_t dacc = tmem + static_cast<uint32_t>(ab) * BNa;
      uint32_t acc = 0u;
      for (int g = g0; g < g1; ++g) {
        const int nsp = min(C::GS, p.n_spline_stages - g * C::GS);
        for (int s = 0; s < nsp + (SILU ? 1 : 0); ++s, ra.next(), rb.next()) {
          mbar_wait_warp(bar_afull(ra.slot), ra.phase);
          mbar_wait_warp(bar_bfull(rb.slot), rb.phase);
          tc_fence_after();
          const uint32_t a_tmem = tmem + acol0 + acols * static_cast<uint32_t>(ra.slot);
          const uint64_t bd0 = umma_desc_sw128(smem_u32(sB + static_cast<size_t>(rb.slot) * b_bytes));
          if (elect_one()) {
            if (!no_mma) {
#pragma unroll
              for (int kk = 0; kk < KSTAGE / 32; ++kk) {
                // K step kk: SW128 block kk/4 of the stage's weight tile, 32 bytes in
                const uint64_t bd = bd0 + (kk >> 2) * b_kstep + 2 * (kk & 3);
                const uint32_t a = kk == 0 ? acc : 1u;
                if (BF16)
                  mma_f16_ts(dacc, a_tmem + 8 * kk, bd, idesc, a);
                else
                  mma_i8_ts(dacc, a_tmem + 8 * kk, bd, idesc, a);
              }
            }
            tc_commit(bar_aempty(ra.slot));
            tc_commit(bar_bempty(rb.slot));
          }
          __syncwarp();
          acc = 1u;
        }
      }
      if (elect_one()) tc_commit(bar_accfull(ab));
      __syncwarp();
    }
  } else if (warp < NPW) {
    // ============================ producers ===============================
    const int quarter = warp & 3;
    const int h = warp >> 2;  // K-quarter of each stage this thread fills
    const int r = quarter * 32 + lane;
    const uint32_t t_lane = static_cast<uint32_t>(quarter * 32) << 16;
    if (tab_bytes > 0) mbar_wait(bar_tab, 0);
    if (threadIdx.x == 0) stamp(1);
    const uint32_t* vals = reinterpret_cast<const uint32_t*>(sT);
    const float* thr = reinterpret_cast<const float*>(sT + p.off_thr);
    const uint8_t* silu_tab = sT + p.off_silu;
    const uint2* c64 = reinterpret_cast<const uint2*>(sT + p.off_c64);
    constexpr int H = C::Q;
    const int xoff = h * H * static_cast<int>(xesz);  // this thread's bytes in the x row
    uint32_t* sil_row = s_sil + (h * 8 * 128 + r) * 2;  // + wp*256 words: word pair wp
    // conv: this row's position within its M tile
    int yy = 0, ox = 0;
    if (p.conv) {
      const int pix = r % p.pimg;
      yy = pix / p.Wo;
      ox = pix - yy * p.Wo;
    }
    Ring ra(SA), rx(SX);
    int idx = 0, lt = 0;
    for (int t = blockIdx.x; t < n_tiles; t += tile_step, ++lt) {
      const Tile tl = tile_of(t);
      const int oy = tl.y0 + yy;
      TapWalk tw(p, g0 * C::GS);
      // conv: bit (ky*K + kx) set when that tap of this row's pixel is padding
      uint32_t padmask = 0;
      if (p.conv) {
        for (int ky = 0; ky < p.ksz; ++ky)
          for (int kx = 0; kx < p.ksz; ++kx) {
            const int iy = oy * p.cstride + ky - p.pad, ix = ox * p.cstride + kx - p.pad;
            if (static_cast<unsigned>(iy) >= static_cast<unsigned>(p.H) ||
                static_cast<unsigned>(ix) >= static_cast<unsigned>(p.W))
              padmask |= 1u << (ky * p.ksz + kx);
          }
      }
      uint32_t rsum = 0;
      for (int g = g0; g < g1; ++g) {
        const int nsp = min(C::GS, p.n_spline_stages - g * C::GS);
        for (int s = 0; s < nsp + (SILU ? 1 : 0); ++s, ++idx, ra.next()) {
          uint32_t w[16];
          if (s < nsp) {
            // 1. this thread's activations of the stage -> registers; free the slot
            mbar_wait(bar_xfull(rx.slot), rx.phase);
            const uint8_t* xt = sX + static_cast<size_t>(rx.slot) * x_bytes;
            const int i0 = (p.conv ? tw.cc * C::IPS : (g * C::GS + s) * C::IPS) + h * H;
            // padded conv taps read level(0.0) (layers.hpp:146-147 leaves them 0.0)
            const bool padtap = (padmask >> tw.tap) & 1u;
            tw.next(p);
            uint32_t nw[C::SW];
            if constexpr (BF16) {
              uint32_t xr[H];
              load_x<4 * H>(xt, r, xoff, x_row_bytes, xr);
              __syncwarp();
              if (lane == 0) mbar_arrive(bar_xempty(rx.slot));
              rx.next();
              float x[H];
#pragma unroll
              for (int e = 0; e < H; ++e) x[e] = __uint_as_float(xr[e]);
              bf16_row<NBP, MODE>(p, x, w, nw);
            } else {
              int a[H];
              if (p.x_kind == X_F32) {
                uint32_t xr[H];
                load_x<4 * H>(xt, r, xoff, x_row_bytes, xr);
                __syncwarp();
                if (lane == 0) mbar_arrive(bar_xempty(rx.slot));
                levels8_f32<H>([&](int e) { return __uint_as_float(xr[e]); }, p.inv_step_f, p.lo_f, p.L, thr, a);
              } else {
                uint32_t xr[H / 2];
                load_x<2 * H>(xt, r, xoff, x_row_bytes, xr);
                __syncwarp();
                if (lane == 0) mbar_arrive(bar_xempty(rx.slot));
#pragma unroll
                for (int q = 0; q < H / 2; ++q) {
                  a[2 * q] = padtap ? p.lvl0 : static_cast<int>(xr[q] & 0xFFFF);
                  a[2 * q + 1] = padtap ? p.lvl0 : static_cast<int>(xr[q] >> 16);
                }
              }
              rx.next();
              lut_row<NBP, MODE>(p, vals, c64, silu_tab, a, i0, w, rsum, nw);
            }
            if constexpr (SILU) {
              // stage s's SiLU words are words s*SW.. of this thread's 64-byte base row
              if constexpr (C::SW == 2) {
                *reinterpret_cast<uint2*>(sil_row + s * 256) = make_uint2(nw[0], nw[1]);
              } else {
                sil_row[(s >> 1) * 256 + (s & 1)] = nw[0];
              }
            }
          } else {
            // base (SiLU) stage: this thread's 64 bytes of codes staged above;
            // words of stages a short last group lacks are zeroed (stale bf16
            // words could be NaN, and NaN * 0 is not 0)
            const int valid = nsp * C::SW;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const uint2 v = *reinterpret_cast<const uint2*>(sil_row + q * 256);
              w[2 * q] = 2 * q < valid ? v.x : 0u;
              w[2 * q + 1] = 2 * q + 1 < valid ? v.y : 0u;
            }
          }
          // 2. the A slot must be free (its previous MMAs retired), then store
          mbar_wait(bar_aempty(ra.slot), ra.phase ^ 1);
          tc_fence_after();
          tmem_st16(tmem + t_lane + acol0 + acols * static_cast<uint32_t>(ra.slot) + 16u * h, w);
          tmem_wait_st();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(bar_afull(ra.slot));
          if (threadIdx.x == 0 && idx == 0) stamp(2);
        }
      }
      if constexpr (MODE == MODE_ZP) {
        // this K-quarter's row sums of the tile's codes, for the zero-point term
        const int rb2 = lt & 1;
        mbar_wait(bar_rsempty(rb2), ((lt >> 1) & 1) ^ 1);
        s_rowsum[(rb2 * 4 + h) * 128 + r] = static_cast<int32_t>(rsum);
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_rsfull(rb2));
      }
    }
    if (threadIdx.x == 0) stamp(3);
    if (!persistent) {
      // split-K: dump this CTA's partial accumulators into its smem (the B/x
      // rings are idle once the accumulator is complete); reduced below
      const int rstride = BN + 4;  // words per row (+4 breaks bank conflicts)
      uint32_t* red = reinterpret_cast<uint32_t*>(sB);
      const uint32_t t_row = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
      if (has_work) {
        mbar_wait(bar_accfull(0), 0);
        tc_fence_after();
      }
      if (threadIdx.x == 0) stamp(4);
#pragma unroll 1
      for (int gq = h; gq < BN / 4; gq += 4) {
        uint32_t ra[4] = {0, 0, 0, 0};
        if (has_work) {
          tmem_ld4(t_row + gq * 4, ra);
          tmem_wait_ld();
        }
        *reinterpret_cast<uint4*>(red + r * rstride + gq * 4) = make_uint4(ra[0], ra[1], ra[2], ra[3]);
      }
    }
  } else {
    // ============================ epilogue ================================
    // One warp per TMEM lane quarter; each thread finishes its row of the
    // tile, 4 columns at a time (rolled: the epilogue code stays small).
    if (tab_bytes > 0) mbar_wait(bar_tab, 0);  // the levels sidecar reads the thresholds
    const int wq = warp & 3;
    const int rloc = wq * 32 + lane;
    const uint32_t t_row = tmem + (static_cast<uint32_t>(wq * 32) << 16);
    const int ngroups = BN / 4;
    auto row_sum = [&](int b) {
      int32_t rs = 0;
      if constexpr (MODE == MODE_ZP) {
#pragma unroll
        for (int q = 0; q < 4; ++q) rs += s_rowsum[(b * 4 + q) * 128 + rloc];
      }
      return rs;
    };

    if (persistent) {
      int lt = 0;
      int cur_n = -1;
      for (int t = blockIdx.x; t < n_tiles; t += tile_step, ++lt) {
        const Tile tl = tile_of(t);
        const int ab = nacc == 2 ? (lt & 1) : 0;
        const int use = nacc == 2 ? (lt >> 1) : lt;
        mbar_wait(bar_accfull(ab), use & 1);
        tc_fence_after();
        if (threadIdx.x == 32 * W_EPI && lt == 0) stamp(4);
        // all epilogue warps are past the previous tile: restage the columns
        // (only when the column tile changes; every epilogue warp walks the
        // same tiles, so the branch is uniform)
        if (tl.n_tile != cur_n) {
          asm volatile("bar.sync 4, %0;" ::"r"(32 * GEMM_EPI_WARPS) : "memory");
          load_cols(tl.n_tile, 32 * W_EPI, 32 * GEMM_EPI_WARPS);
          asm volatile("bar.sync 4, %0;" ::"r"(32 * GEMM_EPI_WARPS) : "memory");
          cur_n = tl.n_tile;
        }
        int32_t rs = 0;
        if constexpr (MODE == MODE_ZP) {
          const int rb2 = lt & 1;
          mbar_wait(bar_rsfull(rb2), (lt >> 1) & 1);
          rs = row_sum(rb2);
          __syncwarp();
          if (lane == 0) mbar_arrive(bar_rsempty(rb2));
        }
        const uint32_t tacc = t_row + static_cast<uint32_t>(ab) * BNa;
        const int row = tl.m0 + rloc;
        // the straight-line paths' fp64 value of accumulator r of tile column c:
        // (acc - corr_c) * fs_c, or with the reference's zero point (acc - z_w *
        // rowsum) * f -- finish4's arithmetic (the subtractions are exact in fp64)
        const double zc_row = MODE == MODE_ZP ? static_cast<double>(p.z_w * static_cast<long long>(rs)) : 0.0;
        auto ycol = [&](uint32_t r, int c) -> double {
          if constexpr (MODE == MODE_ZP)
            return __dmul_rn(__dsub_rn(i32_to_f64(r), zc_row), p.f_tensor);
          else
            return __dmul_rn(__dsub_rn(i32_to_f64(r), s_cols[BN + c]), s_cols[c]);
        };
        float rv[32];  // residual prefetch: 32 columns in flight per thread
        const int ng = KAN_DBG(p, 8) ? 0 : ngroups;  // tuning only: skip the epilogue math
        // 16 columns per TMEM load (BN is a multiple of 16); the two warps of
        // a lane quarter take alternate 16-column groups
        const int half = (warp - W_EPI) >> 2;
        if constexpr (FE == 2 || FE == 3) {
          // next-layer levels of full-width tiles, 16 columns per TMEM load:
          // finish4's fp64 (acc - corr) * fs (exact subtraction, as below) and
          // lattice_level_fast, two 16-byte stores per row block
          const int n0 = tl.n_tile * BN;
          if (p.epi == EPI_LEVEL && !p.f_on && (FE == 3) == (p.res_kind != 0) &&
              (FE == 2 || ((p.ld_res & 3) == 0 && (reinterpret_cast<uintptr_t>(p.res) & 15) == 0)) &&
              n0 + BN <= p.N && (p.ld_out & 7) == 0 &&
              (reinterpret_cast<uintptr_t>(p.out) & 15) == 0 && !KAN_DBG(p, 8)) {
#pragma unroll 1
            for (int g16 = half; g16 < ngroups / 4; g16 += 2) {
              float4 rv4[4] = {};
              if (FE == 3 && row < p.M) {  // residual row segment, loaded before the TMEM read
                const float4* rp = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(p.res) +
                                                                   static_cast<size_t>(row) * p.ld_res + n0 + g16 * 16);
#pragma unroll
                for (int q = 0; q < 4; ++q) rv4[q] = rp[q];
              }
              uint32_t r16[16];
              tmem_ld16(tacc + g16 * 16, r16);
              tmem_wait_ld();
              if (row < p.M) {
                const int cl = g16 * 16;
                uint32_t w[8];
#pragma unroll
                for (int hh = 0; hh < 2; ++hh)
                  levels8_f64(
                      [&](int e8) {
                        const int e = 8 * hh + e8;
                        double y = ycol(r16[e], cl + e);
                        if constexpr (FE == 3) y = __dadd_rn(y, static_cast<double>((&rv4[e >> 2].x)[e & 3]));
                        return y;
                      },
                      p.n_lo, p.n_hi_open, p.n_step, p.n_inv_step, p.n_L, w + 4 * hh);
                uint4* o = reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(p.out) +
                                                    static_cast<size_t>(row) * p.ld_out + n0 + cl);
                o[0] = make_uint4(w[0], w[1], w[2], w[3]);
                o[1] = make_uint4(w[4], w[5], w[6], w[7]);
              }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(bar_accempty(ab));
            continue;
          }
        }
        if constexpr (FE == 1) {
          // Straight-line epilogue for the common fp32 row-major output
          // (+ levels sidecar) of a full-width tile: the same fp64 arithmetic
          // as finish4 with the per-group checks hoisted.  (int32 acc - corr)
          // is an integer below 2^53, so the fp64 subtraction is exact.
          const int n0 = tl.n_tile * BN;
          const bool fast = p.epi == EPI_F32 && p.out_hw == 0 && !p.res_kind && n0 + BN <= p.N &&
                            (p.ld_out & 3) == 0 && (reinterpret_cast<uintptr_t>(p.out) & 15) == 0 &&
                            (p.out_lv == nullptr ||
                             ((p.ld_lv & 7) == 0 && (reinterpret_cast<uintptr_t>(p.out_lv) & 15) == 0)) &&
                            !KAN_DBG(p, 8);
          if (fast) {
            const float* thr = reinterpret_cast<const float*>(sT + p.off_thr);
#pragma unroll 1
            for (int g16 = half; g16 < ngroups / 4; g16 += 2) {
              uint32_t r16[16];
              tmem_ld16(tacc + g16 * 16, r16);
              tmem_wait_ld();
              if (p.stg_on) {
                // this warp's 32 rows x 16 columns through smem: each store
                // instruction then writes 8 whole 64-byte row segments (levels:
                // 16 whole 32-byte segments) instead of 32 half sectors
                const int cl = g16 * 16;
                uint8_t* sg = smem + f_off + static_cast<uint32_t>(warp - W_EPI) * (32u * GEMM_STG_PITCH);
                float f[16];
#pragma unroll
                for (int e = 0; e < 16; ++e) f[e] = __double2float_rn(ycol(r16[e], cl + e));
#pragma unroll
                for (int q = 0; q < 4; ++q)
                  *reinterpret_cast<float4*>(sg + lane * GEMM_STG_PITCH + q * 16) =
                      make_float4(f[4 * q], f[4 * q + 1], f[4 * q + 2], f[4 * q + 3]);
                __syncwarp();
                const int rb = tl.m0 + wq * 32;
#pragma unroll
                for (int s = 0; s < 4; ++s) {
                  const int rl = s * 8 + (lane >> 2);
                  const float4 v = *reinterpret_cast<const float4*>(sg + rl * GEMM_STG_PITCH + (lane & 3) * 16);
                  if (rb + rl < p.M)
                    *reinterpret_cast<float4*>(reinterpret_cast<float*>(p.out) + static_cast<size_t>(rb + rl) * p.ld_out +
                                               n0 + cl + (lane & 3) * 4) = v;
                }
                if (p.out_lv) {
                  uint32_t w[8];
#pragma unroll
                  for (int hh = 0; hh < 2; ++hh) {
                    int lv[8];
                    levels8_f32([&](int e8) { return f[8 * hh + e8]; }, p.inv_step_f, p.lo_f, p.L, thr, lv);
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                      w[4 * hh + q] = static_cast<uint32_t>(lv[2 * q]) | (static_cast<uint32_t>(lv[2 * q + 1]) << 16);
                  }
                  __syncwarp();
                  // 48-byte pitch: conflict-free 16-byte stores
                  *reinterpret_cast<uint4*>(sg + lane * 48) = make_uint4(w[0], w[1], w[2], w[3]);
                  *reinterpret_cast<uint4*>(sg + lane * 48 + 16) = make_uint4(w[4], w[5], w[6], w[7]);
                  __syncwarp();
#pragma unroll
                  for (int s = 0; s < 2; ++s) {
                    const int rl = s * 16 + (lane >> 1);
                    const uint4 v = *reinterpret_cast<const uint4*>(sg + rl * 48 + (lane & 1) * 16);
                    if (rb + rl < p.M)
                      *reinterpret_cast<uint4*>(p.out_lv + static_cast<size_t>(rb + rl) * p.ld_lv + n0 + cl +
                                                (lane & 1) * 8) = v;
                  }
                }
                __syncwarp();
              } else if (row < p.M) {
                const int cl = g16 * 16;
                float f[16];
#pragma unroll
                for (int e = 0; e < 16; ++e) f[e] = __double2float_rn(ycol(r16[e], cl + e));
                float4* o = reinterpret_cast<float4*>(reinterpret_cast<float*>(p.out) +
                                                      static_cast<size_t>(row) * p.ld_out + n0 + cl);
#pragma unroll
                for (int q = 0; q < 4; ++q) o[q] = make_float4(f[4 * q], f[4 * q + 1], f[4 * q + 2], f[4 * q + 3]);
                if (p.out_lv) {
                  uint32_t w[8];
#pragma unroll
                  for (int hh = 0; hh < 2; ++hh) {
                    int lv[8];
                    levels8_f32([&](int e8) { return f[8 * hh + e8]; }, p.inv_step_f, p.lo_f, p.L, thr, lv);
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                      w[4 * hh + q] = static_cast<uint32_t>(lv[2 * q]) | (static_cast<uint32_t>(lv[2 * q + 1]) << 16);
                  }
                  uint4* ol = reinterpret_cast<uint4*>(p.out_lv + static_cast<size_t>(row) * p.ld_lv + n0 + cl);
                  ol[0] = make_uint4(w[0], w[1], w[2], w[3]);
                  ol[1] = make_uint4(w[4], w[5], w[6], w[7]);
                }
              }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(bar_accempty(ab));
            continue;
          }
        }
#pragma unroll 1
        for (int g16 = half; g16 < ng / 4; g16 += 2) {
          if (p.res_kind && (g16 & 3) == half) {
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              // this warp's next two 16-column groups: g16 and g16 + 2
              const int gg = 4 * (g16 + 2 * (q >> 2)) + (q & 3);
              const int c = tl.n_tile * BN + gg * 4;
#pragma unroll
              for (int e = 0; e < 4; ++e)
                rv[4 * q + e] = (row < p.M && gg < ngroups && c + e < p.N)
                                    ? reinterpret_cast<const float*>(p.res)[static_cast<size_t>(row) * p.ld_res + c + e]
                                    : 0.f;
            }
          }
          uint32_t r16[16];
          tmem_ld16(tacc + g16 * 16, r16);
          tmem_wait_ld();
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const uint32_t ra[4] = {r16[4 * q], r16[4 * q + 1], r16[4 * q + 2], r16[4 * q + 3]};
            finish4(row, tl.n_tile * BN + (4 * g16 + q) * 4, ra, rs,
                    p.res_kind ? rv + (((g16 >> 1) & 1) * 4 + q) * 4 : nullptr);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_accempty(ab));
        if (p.f_on) {
          // fused output layer (persistent launches): the tile's 128 rows of
          // hidden levels are in f_lv; the epilogue warps run the small layer
          // while the next tile's MMAs proceed
          asm volatile("bar.sync 4, %0;" ::"r"(32 * GEMM_EPI_WARPS) : "memory");
          fused_output(static_cast<int>(threadIdx.x) - 32 * W_EPI, 32 * GEMM_EPI_WARPS, 0, 128, tl.m0);
          asm volatile("bar.sync 4, %0;" ::"r"(32 * GEMM_EPI_WARPS) : "memory");  // f_lv free for the next tile
        }
      }
    } else if constexpr (MODE == MODE_ZP) {
      // split-K: this CTA's row sums for the reduction below
      int32_t rs = 0;
      if (has_work) {
        mbar_wait(bar_rsfull(0), 0);
        rs = row_sum(0);
      }
      __syncwarp();
      asm volatile("bar.sync 2, %0;" ::"r"(32 * GEMM_EPI_WARPS) : "memory");  // all epilogue warps read slot 0 first
      s_rowsum[rloc] = rs;
    }
  }

  if (!persistent) {
    // split-K across the cluster: every CTA reduces a slice of the tile's rows
    // over all peers through distributed shared memory
    cluster_sync_all();
    if (threadIdx.x == 0) stamp(5);
    if (warp < NPW) {
      const Tile tl = tile_of(blockIdx.x);
      load_cols(tl.n_tile, 0, NP);
      asm volatile("bar.sync 3, %0;" ::"r"(NP) : "memory");
      const int rstride = BN + 4;
      const uint32_t* red = reinterpret_cast<const uint32_t*>(sB);
      const int ngroups = BN / 4;
      const int S = p.splits;
      const uint32_t rank = cluster_rank();
      const int rows_per = 128 / S;
      const int items = rows_per * ngroups;
      const uint32_t red_addr = smem_u32(red);
      const uint32_t rs_addr = smem_u32(s_rowsum);
#pragma unroll 1
      for (int it = threadIdx.x; it < items; it += NP) {
        const int rl = static_cast<int>(rank) * rows_per + it / ngroups;
        const int gq = it % ngroups;
        uint32_t ra[4] = {0, 0, 0, 0};
        int32_t rs = 0;
        const uint32_t off = red_addr + static_cast<uint32_t>((rl * rstride + gq * 4) * 4);
        // all S remote loads first (cluster <= 8 CTAs), then the sums
        uint4 wq8[8];
        int32_t rq8[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          if (q < S) {
            wq8[q] = ld_cluster_v4(mapa(off, q));
            if constexpr (MODE == MODE_ZP) rq8[q] = static_cast<int32_t>(ld_cluster_u32(mapa(rs_addr + rl * 4, q)));
          }
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          if (q >= S) break;
          const uint4 wa = wq8[q];
          if constexpr (MODE == MODE_ZP) rs += rq8[q];
          if constexpr (BF16) {
            ra[0] = __float_as_uint(__uint_as_float(ra[0]) + __uint_as_float(wa.x));
            ra[1] = __float_as_uint(__uint_as_float(ra[1]) + __uint_as_float(wa.y));
            ra[2] = __float_as_uint(__uint_as_float(ra[2]) + __uint_as_float(wa.z));
            ra[3] = __float_as_uint(__uint_as_float(ra[3]) + __uint_as_float(wa.w));
          } else {
            ra[0] += wa.x;
            ra[1] += wa.y;
            ra[2] += wa.z;
            ra[3] += wa.w;
          }
        }
        finish4(tl.m0 + rl, tl.n_tile * BN + gq * 4, ra, rs);
      }
      if (p.f_on) {
        asm volatile("bar.sync 3, %0;" ::"r"(NP) : "memory");  // the CTA's reduced rows are in f_lv
        fused_output(static_cast<int>(threadIdx.x), NP, static_cast<int>(rank) * rows_per, rows_per, tl.m0);
      }
    }
    if (threadIdx.x == 0) stamp(7);
    cluster_sync_all();  // peers' smem must outlive every remote read
  }
  if (threadIdx.x == 0) stamp(6);

  tc_fence_before();
  __syncthreads();
  if (warp == W_MMA) {
    tc_fence_after();
    tmem_dealloc(tmem, tmem_cols);
  }
}

// ---------------------------------------------------------------------------
// host-side launch helpers (called from kan_engine.cpp)

// cudaLaunchKernelEx with programmatic stream serialization (PDL), so the
// kernel's prologue overlaps its predecessor's tail (see pdl_wait/pdl_trigger).
template <class... KArgs, class... Args>
static cudaError_t launch_pdl(void (*kfn)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
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
template <bool BF16, int NBP, int MODE, int FE = 0>
static cudaError_t launch_impl(const CUtensorMap& xmap, const GemmParams& p, size_t smem,
                               cudaStream_t st) {
  auto kfn = kan_gather_gemm_kernel<BF16, NBP, MODE, FE>;
  static std::atomic<unsigned long long> optin{0};  // per instantiation, per device
  (void)smem;
  if (cudaError_t e = smem_optin(kfn, optin); e != cudaSuccess) return e;
  const int n_sm = device_sm_count();
  const int tiles = p.n_tiles_n * p.m_tiles;
  cudaLaunchConfig_t cfg{};
  // splits == 1: persistent CTAs (one per SM) loop over the tiles
  cfg.gridDim = dim3(static_cast<unsigned>(p.splits == 1 ? (tiles < n_sm ? tiles : n_sm) : tiles), 1,
                     p.splits);
  cfg.blockDim = dim3(GEMM_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = 1;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = p.splits;
  cfg.attrs = attr;
  cfg.numAttrs = p.splits > 1 ? 2 : 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kfn, xmap, p);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

#include "kan_conv3.cuh"
#include "kan_convw.cuh"

int gemm_ips(bool bf16, int nbp) { return KSTAGE / (nbp * (bf16 ? 2 : 1)); }
int gemm_gs(bool bf16, int nbp) { return KSTAGE / (bf16 ? 2 : 1) / gemm_ips(bf16, nbp); }
int gemm_threads() { return GEMM_THREADS; }
// TMEM accumulators: two (double-buffered across persistent tiles) when they
// leave room for at least two A-ring slots
int gemm_tmem_accs(int BN, int splits) {
  const int bna = (BN + 31) / 32 * 32;
  return (splits == 1 && 2 * bna + 2 * (KSTAGE / 4) <= 512) ? 2 : 1;
}
// TMEM A-ring depth: KSTAGE/4-column slots after the accumulator columns
int gemm_tmem_slots(int BN, int nacc) {
  const int acol0 = nacc * ((BN + 31) / 32 * 32);
  const int n = (512 - acol0) / (KSTAGE / 4);
  return n < 8 ? n : 8;
}

size_t gemm_smem_bytes(bool bf16, int nbp, int BN, int SA, int SB, int SX, int x_kind,
                       int tab_bytes, bool silu, int fused_bytes) {
  const size_t b = static_cast<size_t>(BN) * KSTAGE;
  const size_t x = 128u * gemm_ips(bf16, nbp) * (x_kind == X_F32 ? 4 : 2);
  const size_t t = (bf16 ? 0 : static_cast<size_t>(tab_bytes)) +
                   (2 * SA + 2 * SB + 2 * SX + 9) * 8 + 2 * 4 * 128 * 4 + 2 * BN * 8 + 16 + 16 +
                   (silu ? 4 * 8 * 128 * 8 : 0) +  // SiLU code staging
                   static_cast<size_t>(fused_bytes);
  return 1024 + SB * b + SX * x + t;
}

cudaError_t launch_gather_gemm(bool bf16, int nbp, int mode, const CUtensorMap& xmap,
                               const GemmParams& p, size_t smem, cudaStream_t st) {
  if (bf16) {
    if (mode == MODE_SILU)
      return nbp == 8 ? launch_impl<true, 8, MODE_SILU>(xmap, p, smem, st)
                      : launch_impl<true, 16, MODE_SILU>(xmap, p, smem, st);
    return nbp == 8 ? launch_impl<true, 8, MODE_PLAIN>(xmap, p, smem, st)
                    : launch_impl<true, 16, MODE_PLAIN>(xmap, p, smem, st);
  }
  // fp32 row-major outputs take the instantiation with the fast epilogue
  const int fe = p.splits != 1                                      ? 0
                 : (p.epi == EPI_F32 && p.out_hw == 0 && !p.res_kind) ? 1
                 : (p.epi == EPI_LEVEL && !p.f_on)                    ? (p.res_kind ? 3 : 2)
                                                                      : 0;
  switch (mode) {
    case MODE_ZP:
      if (fe == 1)
        return nbp == 8 ? launch_impl<false, 8, MODE_ZP, 1>(xmap, p, smem, st)
                        : launch_impl<false, 16, MODE_ZP, 1>(xmap, p, smem, st);
      if (fe == 2)
        return nbp == 8 ? launch_impl<false, 8, MODE_ZP, 2>(xmap, p, smem, st)
                        : launch_impl<false, 16, MODE_ZP, 2>(xmap, p, smem, st);
      if (fe == 3)
        return nbp == 8 ? launch_impl<false, 8, MODE_ZP, 3>(xmap, p, smem, st)
                        : launch_impl<false, 16, MODE_ZP, 3>(xmap, p, smem, st);
      return nbp == 8 ? launch_impl<false, 8, MODE_ZP>(xmap, p, smem, st)
                      : launch_impl<false, 16, MODE_ZP>(xmap, p, smem, st);
    case MODE_SILU:
      if (fe == 1)
        return nbp == 8 ? launch_impl<false, 8, MODE_SILU, 1>(xmap, p, smem, st)
                        : launch_impl<false, 16, MODE_SILU, 1>(xmap, p, smem, st);
      if (fe == 2)
        return nbp == 8 ? launch_impl<false, 8, MODE_SILU, 2>(xmap, p, smem, st)
                        : launch_impl<false, 16, MODE_SILU, 2>(xmap, p, smem, st);
      if (fe == 3)
        return nbp == 8 ? launch_impl<false, 8, MODE_SILU, 3>(xmap, p, smem, st)
                        : launch_impl<false, 16, MODE_SILU, 3>(xmap, p, smem, st);
      return nbp == 8 ? launch_impl<false, 8, MODE_SILU>(xmap, p, smem, st)
                      : launch_impl<false, 16, MODE_SILU>(xmap, p, smem, st);
    default:
      if (fe == 1)
        return nbp == 8 ? launch_impl<false, 8, MODE_PLAIN, 1>(xmap, p, smem, st)
                        : launch_impl<false, 16, MODE_PLAIN, 1>(xmap, p, smem, st);
      if (fe == 2)
        return nbp == 8 ? launch_impl<false, 8, MODE_PLAIN, 2>(xmap, p, smem, st)
                        : launch_impl<false, 16, MODE_PLAIN, 2>(xmap, p, smem, st);
      if (fe == 3)
        return nbp == 8 ? launch_impl<false, 8, MODE_PLAIN, 3>(xmap, p, smem, st)
                        : launch_impl<false, 16, MODE_PLAIN, 3>(xmap, p, smem, st);
      return nbp == 8 ? launch_impl<false, 8, MODE_PLAIN>(xmap, p, smem, st)
                      : launch_impl<false, 16, MODE_PLAIN>(xmap, p, smem, st);
  }
}

// ---------------------------------------------------------------------------
// Lattice levels of an fp32 tensor (parity probe for the quantized indices).
// Runs lattice_level_tie, the function every hot-path producer uses, so the
// threshold / +-inf / NaN edge cases of the parity tests exercise it directly.
__global__ void kan_levels_kernel(const float* __restrict__ x, int64_t n,
                                  const float* __restrict__ thr, float nlo_step, float inv_step, int L,
                                  uint16_t* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ float s_thr[];
  for (int i = threadIdx.x; i < L + 2; i += blockDim.x) s_thr[i] = thr[i];
  __syncthreads();
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = static_cast<uint16_t>(lattice_level_tie(x[i], inv_step, nlo_step, L, s_thr));
}

cudaError_t launch_levels(const float* x, int64_t n, const float* thr, float nlo_step, float inv_step,
                          int L, uint16_t* out, cudaStream_t st) {
  const int64_t nb = (n + 255) / 256;
  int blocks = static_cast<int>(nb < 148 * 8 ? nb : 148 * 8);
  if (blocks < 1) blocks = 1;
  return launch_pdl(kan_levels_kernel, dim3(blocks), dim3(256), (L + 2) * sizeof(float), st, x, n, thr,
                    nlo_step, inv_step, L, out);
}

// ---------------------------------------------------------------------------
// Small-N LUT layer on CUDA cores (engine's choice for N <= 16, NBP = 8, e.g.
// the 64 -> 10 classifier of C1/C2).  Same integer restatement as the GEMM:
// acc[j] = sum_i sum_r code_r(a_i) * q[i, jj_i + r, j] (+ SiLU codes * q_b),
// here as one mixed-sign dp4a per (input, output) -- the 4 codes against the
// 4 weights at bytes jj..jj+3 of the input's 8 basis weights -- so results
// are identical to the tensor-core path.  TPR threads share a row (8
// consecutive inputs each) and reduce by shuffles (integer sums: exact).

template <int NMAX, int TPR, bool SILU>
__global__ void __launch_bounds__(256) kan_small_layer_kernel(const SmallParams p) {
  extern __shared__ __align__(16) uint8_t sm[];
  const int n_in = p.n_in, N = p.N;
  const int per = p.n_in8 / TPR;  // inputs per thread (multiple of 8)
  const int tabb = (p.tab_bytes + 15) & ~15;
  const int wqb_bytes = SILU ? N * p.n_in8 : 0;
  const int wq_bytes = (n_in * N * 8 + 15) & ~15;
  unsigned long long* s_wq = reinterpret_cast<unsigned long long*>(sm + tabb);
  int8_t* s_wqb = reinterpret_cast<int8_t*>(sm + tabb + wq_bytes);
  __shared__ uint64_t fill_bar;
  // tables + weights: three bulk copies on one mbarrier (one memory round trip)
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&fill_bar), 1);
    mbar_fence_init();
    mbar_arrive_tx(smem_u32(&fill_bar), static_cast<uint32_t>(tabb + wq_bytes + wqb_bytes));
    bulk_load(smem_u32(sm), p.tab, static_cast<uint32_t>(tabb), smem_u32(&fill_bar));
    bulk_load(smem_u32(s_wq), p.wq, static_cast<uint32_t>(wq_bytes), smem_u32(&fill_bar));
    if (wqb_bytes > 0)
      bulk_load(smem_u32(s_wqb), p.wqb, static_cast<uint32_t>(wqb_bytes), smem_u32(&fill_bar));
  }
  pdl_trigger();
  __syncthreads();
  mbar_wait(smem_u32(&fill_bar), 0);
  pdl_wait();  // the activations are the previous kernel's output
  const uint32_t* vals = reinterpret_cast<const uint32_t*>(sm);
  const float* thr = reinterpret_cast<const float*>(sm + p.off_thr);
  const uint8_t* silu_tab = sm + p.off_silu;
  const uint32_t mask = (1u << p.k) - 1u;

  const int64_t gt = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t row = gt / TPR;
  const int t = static_cast<int>(gt % TPR);
  int acc[NMAX];
#pragma unroll
  for (int j = 0; j < NMAX; ++j) acc[j] = 0;
  if (row < p.M) {
    // this thread's inputs: i = t + TPR*e (the row's threads read neighbouring
    // inputs, so their weight rows fall in distinct banks; rows broadcast)
    for (int e0 = 0; e0 < per; e0 += 8) {
      uint32_t sw[2] = {0u, 0u};
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int i = t + TPR * (e0 + e);
        if (i < n_in) {
          int a;
          if (p.x_kind == X_U16)
            a = static_cast<const uint16_t*>(p.x)[row * p.ld_x + i];
          else
            a = lattice_level_tie(static_cast<const float*>(p.x)[row * p.ld_x + i], p.inv_step_f,
                                  p.lo_f, p.L, thr);
          const uint32_t v = vals[static_cast<uint32_t>(a) & mask];
          const uint32_t sft = 8u * static_cast<uint32_t>(a >> p.k);
          const unsigned long long* wrow = s_wq + i * N;
#pragma unroll
          for (int j = 0; j < NMAX; ++j)
            if (j < N) acc[j] = dp4a_us(v, static_cast<uint32_t>(wrow[j] >> sft), acc[j]);
          if constexpr (SILU) sw[e >> 2] |= static_cast<uint32_t>(silu_tab[a]) << (8 * (e & 3));
        }
      }
      if constexpr (SILU) {
#pragma unroll
        for (int j = 0; j < NMAX; ++j) {
          if (j < N) {
            // SiLU weights of this thread's inputs, in its order: [j][t][e]
            const uint2 wb = *reinterpret_cast<const uint2*>(s_wqb + (j * TPR + t) * per + e0);
            acc[j] = dp4a_us(sw[1], wb.y, dp4a_us(sw[0], wb.x, acc[j]));
          }
        }
      }
    }
  }
#pragma unroll
  for (int j = 0; j < NMAX; ++j)
#pragma unroll
    for (int off = TPR / 2; off > 0; off >>= 1) acc[j] += __shfl_down_sync(0xffffffffu, acc[j], off, TPR);
  if (t != 0 || row >= p.M) return;
#pragma unroll
  for (int j = 0; j < NMAX; ++j) {
    if (j >= N) break;
    const size_t o = static_cast<size_t>(row) * p.ld_out + j;
    if (p.epi == EPI_RAW) {
      static_cast<int32_t*>(p.out)[o] = acc[j];
      continue;
    }
    const long long v = static_cast<long long>(acc[j]) - (SILU ? p.corr_b[j] : 0ll);
    const double y = __dmul_rn(static_cast<double>(v), p.fs[j]);
    if (p.epi == EPI_F32)
      static_cast<float*>(p.out)[o] = __double2float_rn(y);
    else if (p.epi == EPI_LEVEL)
      static_cast<uint16_t*>(p.out)[o] =
          static_cast<uint16_t>(lattice_level_fast(y, p.n_lo, p.n_hi_open, p.n_step, p.n_inv_step, p.n_L));
    else
      static_cast<int8_t*>(p.out)[o] = static_cast<int8_t>(requant_i8(y, p.out_scale, p.inv_out_scale));
  }
}

size_t small_smem_bytes(const SmallParams& p) {
  return static_cast<size_t>((p.tab_bytes + 15) & ~15) +
         static_cast<size_t>((p.n_in * p.N * 8 + 15) & ~15) +
         static_cast<size_t>(p.mode == MODE_SILU ? p.N * p.n_in8 : 0) + 16;
}

cudaError_t launch_small_layer(const SmallParams& p, cudaStream_t st) {
  if (p.M == 0) return cudaSuccess;
  constexpr int TPR = 8, THREADS = 256;
  const size_t smem = small_smem_bytes(p);
  const unsigned blocks = static_cast<unsigned>((static_cast<int64_t>(p.M) * TPR + THREADS - 1) / THREADS);
  static std::atomic<unsigned long long> optin[2];  // per kernel variant, per device
  auto go = [&](auto kfn, int v) -> cudaError_t {
    if (cudaError_t e = smem_optin(kfn, optin[v]); e != cudaSuccess) return e;
    return launch_pdl(kfn, dim3(blocks), dim3(THREADS), smem, st, p);
  };
  if (p.mode == MODE_SILU) return go(kan_small_layer_kernel<16, TPR, true>, 1);
  return go(kan_small_layer_kernel<16, TPR, false>, 0);
}

// ---------------------------------------------------------------------------
// Pooling over stored activations (NHWC; u16 lattice levels on the LUT path,
// fp32 on the float paths).
//
// maxpool2 (layers.hpp:193-210): max over window x window, stride = window.
// The lattice level is monotone in x, so the max of levels is the level of
// the max the reference feeds the next layer.
template <class T>
__global__ void kan_maxpool_kernel(const T* __restrict__ in, int64_t n_img, int H, int W, int C,
                                   int ld_in, int win, T* __restrict__ out, int ld_out) {
  pdl_wait();
  pdl_trigger();
  const int Ho = H / win, Wo = W / win;
  const int64_t total = n_img * Ho * Wo * C;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(i % C);
    const int64_t q = i / C;
    const int ox = static_cast<int>(q % Wo);
    const int oy = static_cast<int>((q / Wo) % Ho);
    const int64_t n = q / (static_cast<int64_t>(Wo) * Ho);
    T best = in[((n * H + oy * win) * W + ox * win) * ld_in + c];
    for (int dy = 0; dy < win; ++dy)
      for (int dx = 0; dx < win; ++dx) {
        const T v = in[((n * H + oy * win + dy) * W + ox * win + dx) * ld_in + c];
        best = v > best ? v : best;
      }
    out[((n * Ho + oy) * Wo + ox) * ld_out + c] = best;
  }
}

// Global average pool (engine extension for ResKAN18): mean over the H*W
// positions of each channel of stored fp32 values, summed in position order
// in fp64, rounded to fp32.
__global__ void kan_avgpool_f32_kernel(const float* __restrict__ in, int64_t n_img, int HW, int C,
                                       int ld_in, float* __restrict__ out, int ld_out) {
  pdl_wait();
  pdl_trigger();
  const int64_t total = n_img * C;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(i % C);
    const int64_t n = i / C;
    const float* src = in + n * HW * ld_in + c;
    double acc = 0.0;
    for (int q = 0; q < HW; ++q) acc = __dadd_rn(acc, static_cast<double>(src[q * ld_in]));
    out[n * ld_out + c] = __double2float_rn(__ddiv_rn(acc, static_cast<double>(HW)));
  }
}

static int pool_blocks(int64_t total) {
  const int64_t nb = (total + 255) / 256;
  return static_cast<int>(nb < 148 * 16 ? (nb < 1 ? 1 : nb) : 148 * 16);
}

cudaError_t launch_maxpool(bool levels, const void* in, int64_t n_img, int H, int W, int C,
                           int ld_in, int win, void* out, int ld_out, cudaStream_t st) {
  const int64_t total = n_img * (H / win) * (W / win) * C;
  if (total == 0) return cudaSuccess;
  if (levels)
    return launch_pdl(kan_maxpool_kernel<uint16_t>, dim3(pool_blocks(total)), dim3(256), 0, st,
                      static_cast<const uint16_t*>(in), n_img, H, W, C, ld_in, win, static_cast<uint16_t*>(out),
                      ld_out);
  return launch_pdl(kan_maxpool_kernel<float>, dim3(pool_blocks(total)), dim3(256), 0, st,
                    static_cast<const float*>(in), n_img, H, W, C, ld_in, win, static_cast<float*>(out), ld_out);
}

cudaError_t launch_avgpool(const void* in, int64_t n_img, int HW, int C, int ld_in, void* out,
                           int ld_out, cudaStream_t st) {
  const int64_t total = n_img * C;
  if (total == 0) return cudaSuccess;
  return launch_pdl(kan_avgpool_f32_kernel, dim3(pool_blocks(total)), dim3(256), 0, st,
                    static_cast<const float*>(in), n_img, HW, C, ld_in, static_cast<float*>(out), ld_out);
}

// NCHW fp32 model input -> NHWC (lattice levels on the LUT path, fp32 on the
// float paths) for the conv layers' TMA, which needs the innermost (channel)
// box start 16-byte aligned.  32x32 (pixel x channel) tiles through smem;
// levels as lattice_level_tie (exact ActivationLattice::quantize of clamp(x));
// `lo` here is -lo/step.
template <bool LEVELS>
__global__ void __launch_bounds__(256) kan_nchw_to_nhwc_kernel(const float* __restrict__ in, int C, int HW,
                                                                void* __restrict__ out, int ldc,
                                                                const float* __restrict__ thr, float lo,
                                                                float inv_step, int L) {
  pdl_wait();
  pdl_trigger();
  // tile: 64 channels x 32 pixels; loads coalesced along pixels, stores of a
  // pixel's 64 channels as one 128-byte (levels) / 256-byte (fp32) warp row
  __shared__ float tile[64][33];
  const int64_t n = blockIdx.z;
  const int p0 = blockIdx.x * 32, c0 = blockIdx.y * 64;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 8 warps
  const float* src = in + n * C * HW;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int cy = ty + 8 * k, c = c0 + cy, q = p0 + tx;
    tile[cy][tx] = (c < C && q < HW) ? src[static_cast<int64_t>(c) * HW + q] : 0.f;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int py = ty + 8 * k, q = p0 + py;
    const int c = c0 + 2 * tx;  // lane -> channel pair
    if (q >= HW || c >= C) continue;
    const float v0 = tile[2 * tx][py];
    const float v1 = tile[2 * tx + 1][py];
    const int64_t o = (n * HW + q) * ldc + c;
    if constexpr (LEVELS) {
      const uint32_t a0 = static_cast<uint32_t>(lattice_level_tie(v0, inv_step, lo, L, thr));
      const uint32_t a1 = static_cast<uint32_t>(lattice_level_tie(v1, inv_step, lo, L, thr));
      if (c + 1 < C)
        *reinterpret_cast<uint32_t*>(static_cast<uint16_t*>(out) + o) = a0 | (a1 << 16);
      else
        static_cast<uint16_t*>(out)[o] = static_cast<uint16_t>(a0);
    } else {
      if (c + 1 < C)
        *reinterpret_cast<float2*>(static_cast<float*>(out) + o) = make_float2(v0, v1);
      else
        static_cast<float*>(out)[o] = v0;
    }
  }
}

cudaError_t launch_nchw_to_nhwc(bool levels, const float* in, int64_t n_img, int C, int HW,
                                void* out, int ldc, const float* thr, float lo, float inv_step,
                                int L, cudaStream_t st) {
  if (n_img == 0) return cudaSuccess;
  const dim3 grid((HW + 31) / 32, (C + 63) / 64, static_cast<unsigned>(n_img));
  if (levels)
    return launch_pdl(kan_nchw_to_nhwc_kernel<true>, grid, dim3(256), 0, st, in, C, HW, out, ldc, thr, lo,
                      inv_step, L);
  return launch_pdl(kan_nchw_to_nhwc_kernel<false>, grid, dim3(256), 0, st, in, C, HW, out, ldc, thr, lo,
                    inv_step, L);
}

// Lattice levels of fp32 activation rows [M, n] (pitch ld_x) into u16 rows
// (pitch ld_o): the level prepass of large fp32-input layers, so their GEMM
// reads 2-byte levels and its producers skip the level arithmetic.
__global__ void __launch_bounds__(256) kan_rows_to_levels_kernel(const float* __restrict__ x, int64_t M, int n,
                                                                 int ld_x, uint16_t* __restrict__ out, int ld_o,
                                                                 const float* __restrict__ thr, float nlo_step,
                                                                 float inv_step, int L) {
  pdl_wait();
  pdl_trigger();
  const int q4 = (n + 3) / 4;  // float4 groups per row
  const int64_t total = M * q4;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / q4;
    const int c = static_cast<int>(i - r * q4) * 4;
    const float* src = x + r * ld_x + c;
    float v[4];
    if (c + 3 < n && (ld_x & 3) == 0) {
      const float4 f = *reinterpret_cast<const float4*>(src);
      v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) v[e] = c + e < n ? src[e] : 0.f;
    }
    uint32_t a[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) a[e] = static_cast<uint32_t>(lattice_level_tie(v[e], inv_step, nlo_step, L, thr));
    uint16_t* dst = out + r * ld_o + c;
    if (c + 3 < n) {
      *reinterpret_cast<uint2*>(dst) = make_uint2(a[0] | (a[1] << 16), a[2] | (a[3] << 16));
    } else {
      for (int e = 0; e < 4; ++e)
        if (c + e < n) dst[e] = static_cast<uint16_t>(a[e]);
    }
  }
}

cudaError_t launch_rows_to_levels(const float* x, int64_t M, int n, int ld_x, uint16_t* out, int ld_o,
                                  const float* thr, float nlo_step, float inv_step, int L, cudaStream_t st) {
  const int64_t total = M * ((n + 3) / 4);
  if (total == 0) return cudaSuccess;
  const int64_t nb = (total + 255) / 256;
  const unsigned blocks = static_cast<unsigned>(nb < 148 * 32 ? nb : 148 * 32);
  return launch_pdl(kan_rows_to_levels_kernel, dim3(blocks), dim3(256), 0, st, x, M, n, ld_x, out, ld_o, thr,
                    nlo_step, inv_step, L);
}

// Explicit im2col over the NCHW fp32 model input into lattice levels, for convs
// whose c_in is far below one channel chunk (the ResKAN stem, c_in = 3): one
// row per output pixel (n, oy, ox), columns in the reference's channel-major
// order c*K*K + ky*K + kx (layers.hpp:140-149), padded taps at level(0.0).
// The layer then runs as a dense (c_in*K*K)-input GEMM.
// One thread per output pixel: its whole patch row (channel-major, then ky,
// kx: im2col's column order, layers.hpp:140-149) as lattice levels, written
// as 16-byte chunks of the pitch-ld_o row; columns past the patch hold level 0
// (their weights are zero and the zero-point row sums skip them).  Index math
// per row, not per element (the earlier per-element 64-bit divisions made
// this 1.8 ms on C5's stem).
__global__ void __launch_bounds__(256) kan_im2col_levels_kernel(const float* __restrict__ x, int64_t n_img, int C,
                                                                int H, int W, int K, int stride, int pad, int Ho,
                                                                int Wo, uint16_t* __restrict__ out, int ld_o,
                                                                const float* __restrict__ thr, float nlo_step,
                                                                float inv_step, int L, int lvl0) {
  pdl_wait();
  pdl_trigger();
  const int ncol = C * K * K;
  const int hw_o = Ho * Wo;
  const int64_t rows = n_img * hw_o;
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < rows;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t n = r / hw_o;
    const int pix = static_cast<int>(r - n * hw_o);
    const int oy = pix / Wo, ox = pix - (pix / Wo) * Wo;
    const float* xn = x + n * C * H * W;
    uint16_t* o = out + r * ld_o;
    int c = 0, ky = 0, kx = 0;
    for (int col0 = 0; col0 < ld_o; col0 += 8) {
      uint32_t w[4];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        int a = 0;
        if (col0 + q < ncol) {
          const int iy = oy * stride + ky - pad, ix = ox * stride + kx - pad;
          a = lvl0;
          if (static_cast<unsigned>(iy) < static_cast<unsigned>(H) && static_cast<unsigned>(ix) < static_cast<unsigned>(W))
            a = lattice_level_tie(xn[(c * H + iy) * W + ix], inv_step, nlo_step, L, thr);
          if (++kx == K) {
            kx = 0;
            if (++ky == K) {
              ky = 0;
              ++c;
            }
          }
        }
        if (q & 1)
          w[q >> 1] |= static_cast<uint32_t>(a) << 16;
        else
          w[q >> 1] = static_cast<uint32_t>(a);
      }
      *reinterpret_cast<uint4*>(o + col0) = make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
}

cudaError_t launch_im2col_levels(const float* x, int64_t n_img, int C, int H, int W, int K, int stride, int pad,
                                 int Ho, int Wo, uint16_t* out, int ld_o, const float* thr, float nlo_step,
                                 float inv_step, int L, int lvl0, cudaStream_t st) {
  const int64_t rows = n_img * Ho * Wo;
  if (rows == 0) return cudaSuccess;
  if (ld_o % 8 != 0) return cudaErrorInvalidValue;  // 16-byte row chunks (pitch16 rows)
  const int64_t nb = (rows + 255) / 256;
  const unsigned blocks = static_cast<unsigned>(nb < 148 * 32 ? nb : 148 * 32);
  return launch_pdl(kan_im2col_levels_kernel, dim3(blocks), dim3(256), 0, st, x, n_img, C, H, W, K, stride, pad, Ho,
                    Wo, out, ld_o, thr, nlo_step, inv_step, L, lvl0);
}

// argmax over logits rows (predict, eval.hpp:268-272: first maximum wins)
__global__ void kan_argmax_kernel(const float* __restrict__ logits, int64_t M, int N, int ld,
                                  int32_t* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const int64_t m = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (m >= M) return;
  const float* r = logits + m * ld;
  int best = 0;
  for (int j = 1; j < N; ++j)
    if (r[j] > r[best]) best = j;
  out[m] = best;
}

cudaError_t launch_argmax(const float* logits, int64_t M, int N, int ld, int32_t* out,
                          cudaStream_t st) {
  if (M == 0) return cudaSuccess;
  return launch_pdl(kan_argmax_kernel, dim3(static_cast<unsigned>((M + 255) / 256)), dim3(256), 0, st, logits,
                    M, N, ld, out);
}

}  // namespace kan
