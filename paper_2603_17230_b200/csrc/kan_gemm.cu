// kan_gemm.cu -- fused lattice-gather + tcgen05 GEMM for one KAN layer (sm_100a).
//
// Replaces, at layer granularity, the reference's
//   kan_linear_forward<LutBasis>  (proj/include/kantize/layers.hpp:99-116)
//   = clamp (grid.hpp:49-56) -> ActivationLattice::quantize (lut.hpp:44-47)
//     -> lut_basis_lookup (lut.hpp:136-160) -> dense B row (lut.hpp:189-195)
//     -> matmul (matrix.hpp:64-80)
// and, on the float path, kan_linear_forward<RecursiveBasis> (layers.hpp:118-121).
//
// One CTA computes a 128-row x BN-column output tile over a range of K.
// Warp roles:
//   warps 0..NPW-1  producers: read the activation tile TMA put in smem,
//                   quantize each activation to its lattice level (exact: an
//                   fp32 guess corrected against host-computed thresholds),
//                   fetch the level's precomputed basis-row pattern (u8 LUT
//                   codes at the support offset) and write the A tile straight
//                   into smem in the UMMA K-major 128B-swizzle layout; the
//                   bf16 path evaluates the basis in fp32 instead.  Afterwards
//                   they run the epilogue (TMEM -> regs -> global).
//   warp NPW        loader: one bulk copy for the lattice tables, then per stage
//                   a TMA 2D load of the activation tile and a bulk copy of the
//                   pre-swizzled weight tile.
//   warp NPW+1      TMEM allocation and the single-thread tcgen05.mma issuer.
// Accumulators live in TMEM (int32 on the LUT path, fp32 on bf16); the K loop
// is a ring of S stages of 128 bytes of K each (4 MMAs of K = 32 bytes).
#include <cuda.h>
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

// fp32 guess of the lattice level (exact after one threshold correction)
__device__ __forceinline__ int level_guess(float x, float lo, float inv_step, float Lf) {
  float t = (x - lo) * inv_step;
  t = fminf(fmaxf(t, 0.0f), Lf);  // NaN -> 0 (fmaxf returns the non-NaN operand)
  return __float2int_rn(t);
}

// Level of an fp32 activation against thr[n] = min{x : level(x) >= n}.
__device__ __forceinline__ int lattice_level_f32(float x, const float* thr, float lo,
                                                 float inv_step, int L) {
  int g = level_guess(x, lo, inv_step, static_cast<float>(L));
  g += (x >= thr[g + 1]) ? 1 : 0;
  g -= (x < thr[g]) ? 1 : 0;
  return g;
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
__device__ __forceinline__ int lattice_level_fast(double y, double lo, double hi_open, double step,
                                                  double inv_step, int L) {
  double t = (y < lo) ? lo : y;
  t = (hi_open < t) ? hi_open : t;
  const double d = __dsub_rn(t, lo);
  double q = __dmul_rn(d, inv_step);
  if (fabs(__dsub_rn(__dsub_rn(q, floor(q)), 0.5)) < 1e-7) q = ddiv_rn_slow(d, step);
  long long a = llround_ref(q);
  if (a < 0) a = 0;
  if (a > L) a = L;
  return static_cast<int>(a);
}

// clamp(llround(y / s), -127, 127) with the same guarded-multiply rule
__device__ __forceinline__ int requant_i8(double y, double s, double inv_s) {
  double q = __dmul_rn(y, inv_s);
  if (fabs(q) < 1024.0 && fabs(__dsub_rn(__dsub_rn(q, floor(q)), 0.5)) < 1e-7) q = ddiv_rn_slow(y, s);
  long long v = llround_ref(q);
  v = v < -127 ? -127 : (v > 127 ? 127 : v);
  return static_cast<int>(v);
}

// ---- distributed shared memory / cluster helpers ---------------------------
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
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

template <bool BF16, int NBP, int NPW>
struct Cfg {
  static constexpr int NP = NPW * 32;
  static constexpr int ESZ = BF16 ? 2 : 1;
  static constexpr int IPS = 128 / (NBP * ESZ);       // inputs per 128-byte K stage
  static constexpr int GS = (BF16 ? 64 : 128) / IPS;  // spline stages per base group
  static constexpr int RPT = 1024 / NP;               // rows per producer thread per stage
  static constexpr int ROW_STEP = NP / 8;
  // inputs of one 16-byte A chunk: u8 NBP=8 -> 2, u8 NBP=16 -> 1, bf16 -> 1
  static constexpr int IPC = BF16 ? 1 : ((NBP == 8) ? 2 : 1);
};

// Activation values of one thread for one stage (RPT rows x IPC inputs).
template <int RPT, int IPC>
struct XRegs {
  float f[RPT][IPC];
  int lv[RPT][IPC];
};

// Exact lattice level of an fp32 activation.  t = x*(1/step) - lo/step in one
// FFMA is within 7e-4 of the exact quotient (|x| <= 1, L <= 4096), so
// rint(t) is the reference's llround(RN((clamp(x)-lo)/step)) unless t lies
// within 2e-3 of a half-integer; only then (p ~ 4e-3) is the threshold table
// thr[n] = min{x : level(x) >= n} consulted.
__device__ __forceinline__ int lattice_level_x(float x, const GemmParams& p, const float* thr) {
  float t = fmaf(x, p.inv_step_f, p.lo_f);  // p.lo_f holds -lo/step on this path
  t = fminf(fmaxf(t, 0.0f), static_cast<float>(p.L));
  const float tr = rintf(t);
  int g = static_cast<int>(tr);
  if (fabsf(fabsf(t - tr) - 0.5f) < 2e-3f) {
    g = static_cast<int>(floorf(t));
    g += (x >= thr[g + 1]) ? 1 : 0;
  }
  return g;
}

// One A chunk (16 bytes) of the LUT path.  The P+1 codes of lut_basis_lookup
// depend only on frac = a mod 2^k (lut.hpp:145-157), so vals[frac] (2^k u32)
// holds them packed and the chunk is vals[frac] shifted to byte jj = a >> k.
template <int NBP, int MODE, int XK>
__device__ __forceinline__ uint4 lut_chunk(const GemmParams& p, const uint32_t* vals,
                                           const float* thr, const uint8_t* silu_tab,
                                           const float* xf, const int* xl, int i0, uint32_t& rsum,
                                           uint32_t (&silu)[4]) {
  constexpr int IPC = (NBP == 8) ? 2 : 1;
  const int mask = (1 << p.k) - 1;
  int a[IPC];
  uint32_t v[IPC];
#pragma unroll
  for (int e = 0; e < IPC; ++e) {
    a[e] = (XK == X_F32) ? lattice_level_x(xf[e], p, thr) : xl[e];
    v[e] = vals[a[e] & mask];
  }
  uint4 out;
  if constexpr (NBP == 8) {
    const unsigned long long p0 = static_cast<unsigned long long>(v[0]) << (8 * (a[0] >> p.k));
    const unsigned long long p1 = static_cast<unsigned long long>(v[1]) << (8 * (a[1] >> p.k));
    out = make_uint4(static_cast<uint32_t>(p0), static_cast<uint32_t>(p0 >> 32),
                     static_cast<uint32_t>(p1), static_cast<uint32_t>(p1 >> 32));
    if constexpr (MODE == MODE_ZP) {
      // bytes shifted past the 8-byte row are zero codes (see lut_basis_lookup)
      if (i0 < p.n_in) rsum = __dp4a(v[0], 0x01010101u, rsum);
      if (i0 + 1 < p.n_in) rsum = __dp4a(v[1], 0x01010101u, rsum);
    }
    if constexpr (MODE == MODE_SILU)
      shift_in(silu, static_cast<uint32_t>(silu_tab[a[0]]) | (static_cast<uint32_t>(silu_tab[a[1]]) << 8), 16);
  } else {
    const int jj = a[0] >> p.k;
    const int wi = jj >> 2, sh = (jj & 3) * 8;
    const uint32_t lo = __funnelshift_l(0u, v[0], sh);
    const uint32_t hi = __funnelshift_l(v[0], 0u, sh);
    out.x = (wi == 0) ? lo : 0u;
    out.y = (wi == 1) ? lo : ((wi == 0) ? hi : 0u);
    out.z = (wi == 2) ? lo : ((wi == 1) ? hi : 0u);
    out.w = (wi == 3) ? lo : ((wi == 2) ? hi : 0u);
    if constexpr (MODE == MODE_ZP) {
      if (i0 < p.n_in) rsum = __dp4a(v[0], 0x01010101u, rsum);
    }
    if constexpr (MODE == MODE_SILU) shift_in(silu, static_cast<uint32_t>(silu_tab[a[0]]), 8);
  }
  return out;
}

// One A chunk of the bf16 path: fp32 Cox-de Boor basis, 8 bf16 values.
template <int NBP, int MODE>
__device__ __forceinline__ uint4 bf16_chunk(const GemmParams& p, float x, int c, int s,
                                            uint32_t (&silu)[4]) {
  constexpr int PMAX = 3;
  const int half = (NBP == 8) ? 0 : (c & 1);
  float Nv[PMAX + 1];
  const int jj = basis_f32<PMAX>(x, p.flo, p.fhi_open, p.finv_delta, p.G, p.P, Nv);
  float v[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const int rr = 8 * half + e - jj;
    float val = 0.f;
#pragma unroll
    for (int q = 0; q <= PMAX; ++q) val = (rr == q) ? Nv[q] : val;
    v[e] = val;
  }
  if constexpr (MODE == MODE_SILU) {
    if (NBP == 8 || (s & 1) == half) {
      const float xc = fminf(fmaxf(x, p.flo), p.fhi_open);
      const float sv = xc / (1.0f + __expf(-xc));
      const __nv_bfloat16 b = __float2bfloat16_rn(sv);
      shift_in(silu, static_cast<uint32_t>(*reinterpret_cast<const uint16_t*>(&b)), 16);
    }
  }
  return make_uint4(pack_bf16(v[0], v[1]), pack_bf16(v[2], v[3]), pack_bf16(v[4], v[5]),
                    pack_bf16(v[6], v[7]));
}

template <bool BF16, int NBP, int NPW, int MODE>
__global__ void __launch_bounds__(NPW * 32 + 96, 1)
    kan_gather_gemm_kernel(const __grid_constant__ CUtensorMap xmap, const GemmParams p) {
  using C = Cfg<BF16, NBP, NPW>;
  constexpr bool SILU = (MODE == MODE_SILU);
  constexpr bool HAS_B = SILU && !BF16;  // separate base accumulator (LUT path)
  constexpr int NACC = HAS_B ? 2 : 1;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-align the dynamic smem base (SW128 atoms); pointer arithmetic on the
  // __shared__ array keeps the shared address space visible to the compiler.
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);

  const int SA = p.SA, SB = p.SB, SX = p.SX;
  const int BN = p.BN;
  constexpr uint32_t a_bytes = 16384;
  const uint32_t b_bytes = static_cast<uint32_t>(BN) * 128u;
  const uint32_t xesz = (p.x_kind == X_F32) ? 4u : 2u;
  const uint32_t x_bytes = 128u * C::IPS * xesz;
  uint8_t* sA = smem;
  uint8_t* sB = sA + static_cast<size_t>(SA) * a_bytes;
  uint8_t* sX = sB + static_cast<size_t>(SB) * b_bytes;
  uint8_t* sT = sX + static_cast<size_t>(SX) * x_bytes;  // lattice tables (LUT path)
  const int tab_bytes = BF16 ? 0 : p.tab_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sT + tab_bytes);
  int32_t* s_rowsum = reinterpret_cast<int32_t*>(bars + 2 * SA + 2 * SB + 2 * SX + 2);
  double* s_cols = reinterpret_cast<double*>(s_rowsum + 128);  // [3][BN] fs, fb, corr
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(s_cols + 3 * BN);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  unsigned long long* dbg =
      p.dbg ? p.dbg + 8 * ((static_cast<size_t>(blockIdx.z) * gridDim.y + blockIdx.y) * gridDim.x +
                           blockIdx.x)
            : nullptr;
  auto stamp = [&](int i) {
    if (dbg) dbg[i] = globaltimer();
  };
  if (threadIdx.x == 0) stamp(0);
  const int m_tile = blockIdx.y;
  const int n_tile = blockIdx.x;
  const int split = blockIdx.z;
  const int m0 = m_tile * 128;

  // groups of K stages handled by this CTA (may be empty for the last split)
  const int g0 = split * p.groups_per_split;
  const int g1 = min(p.n_groups, g0 + p.groups_per_split);
  const bool has_work = g0 < g1;
  const int spg = C::GS + (SILU ? 1 : 0);  // schedule stages per full group

  auto bar_xfull = [&](int s) { return smem_u32(bars + s); };
  auto bar_xempty = [&](int s) { return smem_u32(bars + SX + s); };
  auto bar_afull = [&](int s) { return smem_u32(bars + 2 * SX + s); };
  auto bar_aempty = [&](int s) { return smem_u32(bars + 2 * SX + SA + s); };
  auto bar_bfull = [&](int s) { return smem_u32(bars + 2 * SX + 2 * SA + s); };
  auto bar_bempty = [&](int s) { return smem_u32(bars + 2 * SX + 2 * SA + SB + s); };
  const uint32_t bar_tmem_full = smem_u32(bars + 2 * SX + 2 * SA + 2 * SB);
  const uint32_t bar_tab = smem_u32(bars + 2 * SX + 2 * SA + 2 * SB + 1);

  uint32_t tmem_cols = 32;
  while (tmem_cols < static_cast<uint32_t>(BN) * NACC) tmem_cols <<= 1;

  // ---- setup: barriers, TMEM ----------------------------------------------
  if (threadIdx.x < 128) s_rowsum[threadIdx.x] = 0;
  if constexpr (!BF16 && MODE != MODE_ZP) {
    for (int i = threadIdx.x; i < BN; i += blockDim.x) {
      const int j = min(n_tile * BN + i, p.N - 1);
      s_cols[i] = p.fs[j];
      s_cols[BN + i] = HAS_B ? p.fb[j] : 0.0;
      s_cols[2 * BN + i] = HAS_B ? static_cast<double>(p.corr_b[j]) : 0.0;
    }
  }
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
    mbar_init(bar_tmem_full, 1);
    mbar_init(bar_tab, 1);
    mbar_fence_init();
  }
  if (warp == NPW && lane == 0) tma_prefetch(&xmap);
  if (warp == NPW + 1) tmem_alloc(smem_u32(s_tmem), tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;

  // Role loops run on whole warps (all lanes wait, lane 0 issues) so the warps
  // stay converged for the aligned barriers and tcgen05 ops that follow.
  if (warp == NPW) {
    // ========================= activation loader ==========================
    Ring rx(SX);
    for (int g = g0; g < g1; ++g) {
      const int nsp = min(C::GS, p.n_spline_stages - g * C::GS);
      for (int s = 0; s < nsp; ++s, rx.next()) {
        const int xs = rx.slot;
        mbar_wait(bar_xempty(xs), rx.phase ^ 1);
        if (lane == 0) {
          if (p.dbg_flags & 8) {
            mbar_arrive(bar_xfull(xs));
          } else {
            mbar_arrive_tx(bar_xfull(xs), x_bytes);
            tma_load_2d(smem_u32(sX + static_cast<size_t>(xs) * x_bytes), &xmap,
                        (g * C::GS + s) * C::IPS, m0, bar_xfull(xs));
          }
        }
        __syncwarp();
      }
    }
  } else if (warp == NPW + 2) {
    // ===================== table + weight-tile loader =====================
    if (lane == 0 && tab_bytes > 0) {
      mbar_arrive_tx(bar_tab, static_cast<uint32_t>(tab_bytes));
      bulk_load(smem_u32(sT), p.tab, static_cast<uint32_t>(tab_bytes), bar_tab);
    }
    __syncwarp();
    Ring rb(SB);
    for (int g = g0; g < g1; ++g) {
      const int nsp = min(C::GS, p.n_spline_stages - g * C::GS);
      for (int s = 0; s < nsp + (SILU ? 1 : 0); ++s, rb.next()) {
        const int bs = rb.slot;
        mbar_wait(bar_bempty(bs), rb.phase ^ 1);
        if (lane == 0) {
          const size_t tile = static_cast<size_t>(n_tile) * p.total_stages + g * spg + s;
          if (p.dbg_flags & 16) {
            mbar_arrive(bar_bfull(bs));
          } else {
            mbar_arrive_tx(bar_bfull(bs), b_bytes);
            bulk_load(smem_u32(sB + static_cast<size_t>(bs) * b_bytes), p.wt + tile * b_bytes,
                      b_bytes, bar_bfull(bs));
          }
        }
        __syncwarp();
      }
    }
  } else if (warp == NPW + 1) {
    // ============================ MMA issuer ==============================
    const uint32_t idesc = BF16 ? idesc_bf16(BN) : idesc_i8(BN, p.b_signed != 0);
    const int nk = (p.dbg_flags & 2) ? 0 : 4;
    Ring ra(SA), rb(SB);
    bool first_s = true, first_b = true;
    for (int g = g0; g < g1; ++g) {
      const int nsp = min(C::GS, p.n_spline_stages - g * C::GS);
      for (int s = 0; s < nsp + (SILU ? 1 : 0); ++s, ra.next(), rb.next()) {
        const int as = ra.slot, bs = rb.slot;
        mbar_wait(bar_afull(as), ra.phase);
        mbar_wait(bar_bfull(bs), rb.phase);
        tc_fence_after();
        const bool is_base = HAS_B && (s >= nsp);
        if (lane == 0) {
          const uint32_t d = tmem + (is_base ? static_cast<uint32_t>(BN) : 0u);
          const bool first = is_base ? first_b : first_s;
          const uint32_t a_addr = smem_u32(sA + static_cast<size_t>(as) * a_bytes);
          const uint32_t b_addr = smem_u32(sB + static_cast<size_t>(bs) * b_bytes);
          for (int kk = 0; kk < nk; ++kk) {
            const uint64_t ad = umma_desc_sw128(a_addr + 32 * kk);
            const uint64_t bd = umma_desc_sw128(b_addr + 32 * kk);
            const uint32_t acc = (first && kk == 0) ? 0u : 1u;
            if (BF16)
              mma_f16(d, ad, bd, idesc, acc);
            else
              mma_i8(d, ad, bd, idesc, acc);
          }
          if (p.dbg_flags & 64) {
            mbar_arrive(bar_aempty(as));
            mbar_arrive(bar_bempty(bs));
          } else {
            tc_commit(bar_aempty(as));
            tc_commit(bar_bempty(bs));
          }
        }
        __syncwarp();
        if (is_base)
          first_b = false;
        else
          first_s = false;
      }
    }
    if (lane == 0) tc_commit(bar_tmem_full);
    __syncwarp();
  } else {
    // ============================ producers ===============================
    const int pt = threadIdx.x;
    const int c = pt & 7;
    const int r0 = pt >> 3;
    uint32_t silu_w[C::RPT][4];
    uint32_t rsum[C::RPT];
#pragma unroll
    for (int j = 0; j < C::RPT; ++j) {
      rsum[j] = 0;
#pragma unroll
      for (int w = 0; w < 4; ++w) silu_w[j][w] = 0;
    }
    if (tab_bytes > 0) mbar_wait(bar_tab, 0);
    if (pt == 0) stamp(1);
    const uint32_t* vals = reinterpret_cast<const uint32_t*>(sT);
    const float* thr = reinterpret_cast<const float*>(sT + p.off_thr);
    const uint8_t* silu_tab = sT + p.off_silu;

    // loop-invariant smem offsets of this thread's chunks
    const int in_c = BF16 ? ((NBP == 8) ? c : (c >> 1)) : c * C::IPC;
    uint32_t a_off[C::RPT], x_off[C::RPT];
#pragma unroll
    for (int j = 0; j < C::RPT; ++j) {
      a_off[j] = sw128_off(r0 + j * C::ROW_STEP, c);
      x_off[j] = static_cast<uint32_t>((r0 + j * C::ROW_STEP) * C::IPS + in_c) * xesz;
    }
    Ring ra(SA), rx(SX);
    int idx = 0;
    for (int g = g0; g < g1; ++g) {
      const int nsp = min(C::GS, p.n_spline_stages - g * C::GS);
      for (int s = 0; s < nsp + (SILU ? 1 : 0); ++s, ++idx, ra.next()) {
        const int as = ra.slot;
        const uint32_t aph = ra.phase;
        uint8_t* a_tile = sA + static_cast<size_t>(as) * a_bytes;
        if (s < nsp) {
          // 1. activations of this stage -> registers, release the x slot
          const int xs = rx.slot;
          mbar_wait(bar_xfull(xs), rx.phase);
          rx.next();
          const uint8_t* xt = sX + static_cast<size_t>(xs) * x_bytes;
          XRegs<C::RPT, C::IPC> xr;
          if (BF16 || p.x_kind == X_F32) {
#pragma unroll
            for (int j = 0; j < C::RPT; ++j) {
              const float* xp = reinterpret_cast<const float*>(xt + x_off[j]);
              if constexpr (C::IPC == 2) {
                const float2 v = *reinterpret_cast<const float2*>(xp);
                xr.f[j][0] = v.x;
                xr.f[j][1] = v.y;
              } else {
                xr.f[j][0] = xp[0];
              }
            }
          } else {
#pragma unroll
            for (int j = 0; j < C::RPT; ++j) {
              const uint16_t* xp = reinterpret_cast<const uint16_t*>(xt + x_off[j]);
              if constexpr (C::IPC == 2) {
                const uint32_t v = *reinterpret_cast<const uint32_t*>(xp);
                xr.lv[j][0] = static_cast<int>(v & 0xFFFF);
                xr.lv[j][1] = static_cast<int>(v >> 16);
              } else {
                xr.lv[j][0] = xp[0];
              }
            }
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(bar_xempty(xs));
          // 2. wait for the A slot, expand levels into basis rows
          mbar_wait(bar_aempty(as), aph ^ 1);
          const int i0 = (g * C::GS + s) * C::IPS + in_c;
          uint4 out[C::RPT];
          if (p.dbg_flags & 1) {
#pragma unroll
            for (int j = 0; j < C::RPT; ++j) out[j] = make_uint4(0, 0, 0, 0);
          } else if constexpr (BF16) {
#pragma unroll
            for (int j = 0; j < C::RPT; ++j) out[j] = bf16_chunk<NBP, MODE>(p, xr.f[j][0], c, s, silu_w[j]);
          } else {
            if (p.x_kind == X_F32) {
#pragma unroll
              for (int j = 0; j < C::RPT; ++j)
                out[j] = lut_chunk<NBP, MODE, X_F32>(p, vals, thr, silu_tab, xr.f[j], xr.lv[j], i0, rsum[j], silu_w[j]);
            } else {
#pragma unroll
              for (int j = 0; j < C::RPT; ++j)
                out[j] = lut_chunk<NBP, MODE, X_U16>(p, vals, thr, silu_tab, xr.f[j], xr.lv[j], i0, rsum[j], silu_w[j]);
            }
          }
#pragma unroll
          for (int j = 0; j < C::RPT; ++j) *reinterpret_cast<uint4*>(a_tile + a_off[j]) = out[j];
        } else if constexpr (SILU) {
          // base (SiLU) stage: flush the per-thread 16-byte chunk of each row,
          // first padding the shift register for stages the last group lacks.
          // (bf16 with NBP=16: a thread contributes on stages of parity c&1.)
          mbar_wait(bar_aempty(as), aph ^ 1);
          const int bits = BF16 ? 16 : ((NBP == 8) ? 16 : 8);
          int pad = C::GS - nsp;
          if (BF16 && NBP == 16) {
            pad = 0;
            for (int t = nsp; t < C::GS; ++t) pad += ((t & 1) == (c & 1)) ? 1 : 0;
          }
#pragma unroll
          for (int j = 0; j < C::RPT; ++j) {
            for (int t = 0; t < pad; ++t) shift_in(silu_w[j], 0u, bits);
            *reinterpret_cast<uint4*>(a_tile + a_off[j]) =
                make_uint4(silu_w[j][0], silu_w[j][1], silu_w[j][2], silu_w[j][3]);
#pragma unroll
            for (int w = 0; w < 4; ++w) silu_w[j][w] = 0;
          }
        }
        if (!(p.dbg_flags & 32)) fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_afull(as));
        if (pt == 0 && idx == 0) stamp(2);
      }
    }
    if (pt == 0) stamp(3);

    // ---- row sums of the basis codes (per-tensor zero-point correction) ----
    if constexpr (MODE == MODE_ZP) {
#pragma unroll
      for (int j = 0; j < C::RPT; ++j) {
        int v = static_cast<int>(rsum[j]);
        v += __shfl_xor_sync(0xffffffffu, v, 1);
        v += __shfl_xor_sync(0xffffffffu, v, 2);
        v += __shfl_xor_sync(0xffffffffu, v, 4);
        if (c == 0) s_rowsum[r0 + j * C::ROW_STEP] = v;
      }
    }
    asm volatile("bar.sync 1, %0;" ::"r"(C::NP) : "memory");
  }

  // ============================ epilogue ==================================
  const int wq = warp & 3;
  const int wh = warp >> 2;
  const int rloc = wq * 32 + lane;
  const uint32_t t_row = tmem + (static_cast<uint32_t>(wq * 32) << 16);
  const int nchunks = BN / 16;

  // The epilogue runs once per CTA out of a cold instruction cache, so it
  // works on 4-column groups in rolled loops to keep its code small.
  auto finish4 = [&](int row, int col0, const uint32_t(&ra)[4], const uint32_t(&rb)[4],
                     int32_t rs) {
    if (row >= p.M) return;
    const size_t base = static_cast<size_t>(row) * p.ld_out + col0;
    const int nvalid = min(4, p.N - col0);
    if (p.epi == EPI_RAW) {
      uint32_t* o = reinterpret_cast<uint32_t*>(p.out) + base;
      uint32_t* o2 = reinterpret_cast<uint32_t*>(p.out2) + base;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if (e < nvalid) {
          o[e] = ra[e];
          if (HAS_B && p.out2) o2[e] = rb[e];
        }
      }
      return;
    }
    double y[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int jl = col0 - n_tile * BN + e;  // column within this CTA's tile
      if constexpr (BF16) {
        y[e] = static_cast<double>(__uint_as_float(ra[e]));
      } else if constexpr (MODE == MODE_ZP) {
        const long long v =
            static_cast<long long>(static_cast<int32_t>(ra[e])) - p.z_w * static_cast<long long>(rs);
        y[e] = __dmul_rn(static_cast<double>(v), p.f_tensor);
      } else {
        double v = __dmul_rn(static_cast<double>(static_cast<int32_t>(ra[e])), s_cols[jl]);
        if constexpr (HAS_B) {
          const long long vb = static_cast<long long>(static_cast<int32_t>(rb[e])) -
                               static_cast<long long>(s_cols[2 * BN + jl]);
          v = __dadd_rn(v, __dmul_rn(static_cast<double>(vb), s_cols[BN + jl]));
        }
        y[e] = v;
      }
    }
    if (p.epi == EPI_F32) {
      float* o = reinterpret_cast<float*>(p.out) + base;
      if (nvalid == 4 && (reinterpret_cast<uintptr_t>(o) & 15) == 0) {
        *reinterpret_cast<float4*>(o) = make_float4(__double2float_rn(y[0]), __double2float_rn(y[1]),
                                                    __double2float_rn(y[2]), __double2float_rn(y[3]));
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (e < nvalid) o[e] = __double2float_rn(y[e]);
      }
    } else if (p.epi == EPI_LEVEL) {
      uint16_t* o = reinterpret_cast<uint16_t*>(p.out) + base;
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (e < nvalid)
          o[e] = static_cast<uint16_t>(
              lattice_level_fast(y[e], p.n_lo, p.n_hi_open, p.n_step, p.n_inv_step, p.n_L));
    } else {  // EPI_I8
      int8_t* o = reinterpret_cast<int8_t*>(p.out) + base;
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (e < nvalid) o[e] = static_cast<int8_t>(requant_i8(y[e], p.out_scale, p.inv_out_scale));
    }
  };
  const int ngroups = BN / 4;

  if (p.splits == 1) {
    if (warp < NPW) {
      mbar_wait(bar_tmem_full, 0);
      tc_fence_after();
      if (threadIdx.x == 0) stamp(4);
      const int32_t rowsum = s_rowsum[rloc];
#pragma unroll 1
      for (int gq = wh; gq < ngroups; gq += NPW / 4) {
        uint32_t ra[4], rb[4] = {0, 0, 0, 0};
        tmem_ld4(t_row + gq * 4, ra);
        if constexpr (HAS_B) tmem_ld4(t_row + BN + gq * 4, rb);
        tmem_wait_ld();
        finish4(m0 + rloc, n_tile * BN + gq * 4, ra, rb, rowsum);
      }
    }
  } else {
    // split-K across the cluster: dump the partial accumulators into this
    // CTA's smem (the A/B rings are idle now), then every CTA reduces a slice
    // of rows over all peers through distributed shared memory.
    const int rstride = NACC * BN + 4;  // words per row (+4 breaks bank conflicts)
    uint32_t* red = reinterpret_cast<uint32_t*>(sA);
    if (warp < NPW) {
      if (has_work) {
        mbar_wait(bar_tmem_full, 0);
        tc_fence_after();
      }
      if (threadIdx.x == 0) stamp(4);
#pragma unroll 1
      for (int gq = wh; gq < ngroups; gq += NPW / 4) {
        uint32_t ra[4] = {0, 0, 0, 0}, rb[4] = {0, 0, 0, 0};
        if (has_work) {
          tmem_ld4(t_row + gq * 4, ra);
          if constexpr (HAS_B) tmem_ld4(t_row + BN + gq * 4, rb);
          tmem_wait_ld();
        }
        *reinterpret_cast<uint4*>(red + rloc * rstride + gq * 4) = make_uint4(ra[0], ra[1], ra[2], ra[3]);
        if constexpr (HAS_B)
          *reinterpret_cast<uint4*>(red + rloc * rstride + BN + gq * 4) = make_uint4(rb[0], rb[1], rb[2], rb[3]);
      }
    }
    cluster_sync_all();
    if (threadIdx.x == 0) stamp(5);
    if (warp < NPW) {
      const int S = p.splits;
      const uint32_t rank = cluster_rank();
      const int rows_per = 128 / S;
      const int items = rows_per * ngroups;
      const uint32_t red_addr = smem_u32(red);
      const uint32_t rs_addr = smem_u32(s_rowsum);
#pragma unroll 1
      for (int it = threadIdx.x; it < items; it += C::NP) {
        const int rl = static_cast<int>(rank) * rows_per + it / ngroups;
        const int gq = it % ngroups;
        uint32_t ra[4] = {0, 0, 0, 0}, rb[4] = {0, 0, 0, 0};
        int32_t rs = 0;
        const uint32_t off = red_addr + static_cast<uint32_t>((rl * rstride + gq * 4) * 4);
#pragma unroll 1
        for (int q = 0; q < S; ++q) {
          const uint32_t ad = mapa(off, q);
          const uint4 wa = ld_cluster_v4(ad);
          uint4 wb = make_uint4(0, 0, 0, 0);
          if constexpr (HAS_B) wb = ld_cluster_v4(ad + BN * 4);
          if constexpr (MODE == MODE_ZP) rs += static_cast<int32_t>(ld_cluster_u32(mapa(rs_addr + rl * 4, q)));
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
          rb[0] += wb.x;
          rb[1] += wb.y;
          rb[2] += wb.z;
          rb[3] += wb.w;
        }
        finish4(m0 + rl, n_tile * BN + gq * 4, ra, rb, rs);
      }
    }
    if (threadIdx.x == 0) stamp(7);
    cluster_sync_all();  // peers' smem must outlive every remote read
  }
  if (threadIdx.x == 0) stamp(6);

  tc_fence_before();
  __syncthreads();
  if (warp == NPW + 1) {
    tc_fence_after();
    tmem_dealloc(tmem, tmem_cols);
  }
}

// ---------------------------------------------------------------------------
// host-side launch helpers (called from kan_engine.cpp)
constexpr int kNPW = 8;

template <bool BF16, int NBP, int MODE>
static cudaError_t launch_impl(const CUtensorMap& xmap, const GemmParams& p, size_t smem,
                               cudaStream_t st) {
  auto kfn = kan_gather_gemm_kernel<BF16, NBP, kNPW, MODE>;
  cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(p.n_tiles_n, p.m_tiles, p.splits);
  cfg.blockDim = dim3(kNPW * 32 + 96);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = p.splits;
  cfg.attrs = attr;
  cfg.numAttrs = p.splits > 1 ? 1 : 0;
  e = cudaLaunchKernelEx(&cfg, kfn, xmap, p);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

int gemm_ips(bool bf16, int nbp) { return 128 / (nbp * (bf16 ? 2 : 1)); }
int gemm_gs(bool bf16, int nbp) { return (bf16 ? 64 : 128) / gemm_ips(bf16, nbp); }
int gemm_threads() { return kNPW * 32 + 96; }

size_t gemm_smem_bytes(bool bf16, int nbp, int BN, int SA, int SB, int SX, int x_kind,
                       int tab_bytes) {
  const size_t a = 16384, b = static_cast<size_t>(BN) * 128;
  const size_t x = 128u * gemm_ips(bf16, nbp) * (x_kind == X_F32 ? 4 : 2);
  const size_t t = (bf16 ? 0 : static_cast<size_t>(tab_bytes)) +
                   (2 * SA + 2 * SB + 2 * SX + 2) * 8 + 128 * 4 + 3 * BN * 8 + 16;
  return 1024 + SA * a + SB * b + SX * x + t;
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
  switch (mode) {
    case MODE_ZP:
      return nbp == 8 ? launch_impl<false, 8, MODE_ZP>(xmap, p, smem, st)
                      : launch_impl<false, 16, MODE_ZP>(xmap, p, smem, st);
    case MODE_SILU:
      return nbp == 8 ? launch_impl<false, 8, MODE_SILU>(xmap, p, smem, st)
                      : launch_impl<false, 16, MODE_SILU>(xmap, p, smem, st);
    default:
      return nbp == 8 ? launch_impl<false, 8, MODE_PLAIN>(xmap, p, smem, st)
                      : launch_impl<false, 16, MODE_PLAIN>(xmap, p, smem, st);
  }
}

// ---------------------------------------------------------------------------
// Lattice levels of an fp32 tensor (parity probe for the quantized indices).
__global__ void kan_levels_kernel(const float* __restrict__ x, int64_t n,
                                  const float* __restrict__ thr, float lo, float inv_step, int L,
                                  uint16_t* __restrict__ out) {
  extern __shared__ float s_thr[];
  for (int i = threadIdx.x; i < L + 2; i += blockDim.x) s_thr[i] = thr[i];
  __syncthreads();
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = static_cast<uint16_t>(lattice_level_f32(x[i], s_thr, lo, inv_step, L));
}

cudaError_t launch_levels(const float* x, int64_t n, const float* thr, float lo, float inv_step,
                          int L, uint16_t* out, cudaStream_t st) {
  const int64_t nb = (n + 255) / 256;
  int blocks = static_cast<int>(nb < 148 * 8 ? nb : 148 * 8);
  if (blocks < 1) blocks = 1;
  kan_levels_kernel<<<blocks, 256, (L + 2) * sizeof(float), st>>>(x, n, thr, lo, inv_step, L,
                                                                   out);
  return cudaGetLastError();
}

// argmax over logits rows (predict, eval.hpp:268-272: first maximum wins)
__global__ void kan_argmax_kernel(const float* __restrict__ logits, int64_t M, int N, int ld,
                                  int32_t* __restrict__ out) {
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
  kan_argmax_kernel<<<static_cast<unsigned>((M + 255) / 256), 256, 0, st>>>(logits, M, N, ld,
                                                                            out);
  return cudaGetLastError();
}

}  // namespace kan
