// kan_gemm.cu -- fused lattice-gather + tcgen05 GEMM for one KAN layer (sm_100a).
//
// Replaces, at layer granularity, the reference's
//   kan_linear_forward<LutBasis>  (proj/include/kantize/layers.hpp:99-116)
//   = clamp (grid.hpp:49-56) -> ActivationLattice::quantize (lut.hpp:44-47)
//     -> lut_basis_lookup (lut.hpp:136-160) -> dense B row (lut.hpp:189-195)
//     -> matmul (matrix.hpp:64-80)
// and, on the float path, kan_linear_forward<RecursiveBasis> (layers.hpp:118-121).
//
// One CTA computes a 128-row x BN-column output tile.  Warp roles:
//   warps 0..NPW-1  producers: read the activation tile TMA put in smem,
//                   quantize each activation to its lattice level (exact, via
//                   a threshold table), expand the level into its basis row
//                   (u8 LUT codes, or bf16 basis values) and write the A tile
//                   straight into smem in the UMMA K-major 128B-swizzle layout;
//                   afterwards they run the epilogue (TMEM -> regs -> global).
//   warp NPW        loader: TMA for the activation tile, one bulk copy per
//                   stage for the pre-swizzled weight tile.
//   warp NPW+1      TMEM allocation and the single-thread tcgen05.mma issuer.
// The int32 accumulators live in TMEM; the K loop is a ring of S stages, each
// 128 bytes of K (4 MMAs of K=32 bytes).
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

// Level of an fp32 activation: fp32 guess, then exact correction against the
// host-computed thresholds thr[n] = min{x : level(x) >= n}.
__device__ __forceinline__ int lattice_level_f32(float x, const float* thr, float lo,
                                                 float inv_step, int L) {
  float t = (x - lo) * inv_step;
  t = fminf(fmaxf(t, 0.0f), static_cast<float>(L));
  int g = __float2int_rn(t);
  g += (x >= thr[g + 1]) ? 1 : 0;
  g -= (x < thr[g]) ? 1 : 0;
  return g;
}

// ---------------------------------------------------------------------------
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
      const int i = j - d + r;  // basis index at degree d
      const float left = (r == 0) ? 0.f : N[PMAX - d + r];        // B_i^{d-1}
      const float right = (r == d) ? 0.f : N[PMAX - d + r + 1];   // B_{i+1}^{d-1}
      const float d1 = (xi - static_cast<float>(i)) * rd;
      const float d2 = (static_cast<float>(i + d + 1) - xi) * rd;
      N[PMAX - d + r] = d1 * left + d2 * right;
    }
  }
  // shift so that N[r] = basis (j - P + r)
  if (P < PMAX) {
#pragma unroll
    for (int r = 0; r <= PMAX; ++r) N[r] = (r + PMAX - P <= PMAX) ? N[r + PMAX - P] : 0.f;
  }
  return j - P;  // support start
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}

// ---------------------------------------------------------------------------
template <bool BF16, int NBP, int NPW>
struct Cfg {
  static constexpr int NP = NPW * 32;
  static constexpr int ESZ = BF16 ? 2 : 1;
  static constexpr int IPS = 128 / (NBP * ESZ);   // inputs per 128-byte K stage
  static constexpr int GS = (BF16 ? 64 : 128) / IPS;  // spline stages per silu group
  static constexpr int RPT = 1024 / NP;           // rows per producer thread per stage
  static constexpr int ROW_STEP = NP / 8;
};

template <bool BF16, int NBP, int NPW>
__global__ void __launch_bounds__(NPW * 32 + 64, 1)
    kan_gather_gemm_kernel(const __grid_constant__ CUtensorMap xmap, const GemmParams p) {
  using C = Cfg<BF16, NBP, NPW>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-align the dynamic smem base (SW128 atoms)
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));

  const int S = p.S;
  const int BN = p.BN;
  const uint32_t a_bytes = 16384;
  const uint32_t b_bytes = static_cast<uint32_t>(BN) * 128u;
  const uint32_t xesz = (p.x_kind == X_F32) ? 4u : 2u;
  const uint32_t x_bytes = 128u * C::IPS * xesz;
  uint8_t* sA = smem;
  uint8_t* sB = sA + static_cast<size_t>(S) * a_bytes;
  uint8_t* sX = sB + static_cast<size_t>(S) * b_bytes;
  uint8_t* sT = sX + static_cast<size_t>(S) * x_bytes;  // tables
  float* t_thr = reinterpret_cast<float*>(sT);
  const int L = p.L;
  const int nthr = BF16 ? 0 : ((p.x_kind == X_F32) ? L + 2 : 0);
  uint32_t* t_vals = reinterpret_cast<uint32_t*>(t_thr + ((nthr + 3) & ~3));
  const int nvals = BF16 ? 0 : L + 1;
  uint8_t* t_silu = reinterpret_cast<uint8_t*>(t_vals + ((nvals + 3) & ~3));
  const int nsilu = (!BF16 && p.silu) ? L + 1 : 0;
  uint64_t* bars = reinterpret_cast<uint64_t*>(t_silu + ((nsilu + 15) & ~15));
  int32_t* s_rowsum = reinterpret_cast<int32_t*>(bars + 4 * S + 2);
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(s_rowsum + 128);
  uint32_t* s_flag = s_tmem + 1;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int m_tile = blockIdx.y;
  const int n_tile = blockIdx.x;
  const int split = blockIdx.z;
  const int m0 = m_tile * 128;

  // groups handled by this CTA
  const int g0 = split * p.groups_per_split;
  const int g1 = min(p.n_groups, g0 + p.groups_per_split);
  const int spg = C::GS + p.silu;  // schedule stages per full group
  auto bar_full_x = [&](int s) { return smem_u32(bars + s); };
  auto bar_full_b = [&](int s) { return smem_u32(bars + S + s); };
  auto bar_full_a = [&](int s) { return smem_u32(bars + 2 * S + s); };
  auto bar_empty = [&](int s) { return smem_u32(bars + 3 * S + s); };
  const uint32_t bar_tmem_full = smem_u32(bars + 4 * S);

  const uint32_t tmem_cols = [&] {
    uint32_t need = static_cast<uint32_t>(BN) * ((!BF16 && p.silu) ? 2u : 1u);
    uint32_t c = 32;
    while (c < need) c <<= 1;
    return c;
  }();

  // ---- setup: tables, barriers, TMEM -------------------------------------
  for (int i = threadIdx.x; i < nthr; i += blockDim.x) t_thr[i] = p.thr[i];
  for (int i = threadIdx.x; i < nvals; i += blockDim.x) t_vals[i] = p.vals[i];
  for (int i = threadIdx.x; i < nsilu; i += blockDim.x) t_silu[i] = p.silu_codes[i];
  if (threadIdx.x < 128) s_rowsum[threadIdx.x] = 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(bar_full_x(s), 1);
      mbar_init(bar_full_b(s), 1);
      mbar_init(bar_full_a(s), NPW);
      mbar_init(bar_empty(s), 1);
    }
    mbar_init(bar_tmem_full, 1);
    mbar_fence_init();
  }
  if (warp == NPW && lane == 0) tma_prefetch(&xmap);
  if (warp == NPW + 1) tmem_alloc(smem_u32(s_tmem), tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;

  if (warp == NPW) {
    // ============================ loader ==================================
    if (lane == 0) {
      int idx = 0;
      for (int g = g0; g < g1; ++g) {
        const int nsp = min(C::GS, p.n_spline_stages - g * C::GS);
        for (int s = 0; s < nsp + p.silu; ++s, ++idx) {
          const int slot = idx % S;
          const uint32_t ph = (idx / S) & 1;
          mbar_wait(bar_empty(slot), ph ^ 1);
          if (s < nsp) {
            mbar_arrive_tx(bar_full_x(slot), x_bytes);
            tma_load_2d(smem_u32(sX + static_cast<size_t>(slot) * x_bytes), &xmap,
                        (g * C::GS + s) * C::IPS, m0, bar_full_x(slot));
          } else {
            mbar_arrive(bar_full_x(slot));
          }
          const size_t tile = static_cast<size_t>(n_tile) * p.total_stages + g * spg + s;
          mbar_arrive_tx(bar_full_b(slot), b_bytes);
          bulk_load(smem_u32(sB + static_cast<size_t>(slot) * b_bytes), p.wt + tile * b_bytes,
                    b_bytes, bar_full_b(slot));
        }
      }
    }
  } else if (warp == NPW + 1) {
    // ============================ MMA issuer ==============================
    if (lane == 0) {
      const uint32_t idesc = BF16 ? idesc_bf16(BN) : idesc_i8(BN, p.b_signed != 0);
      int idx = 0;
      bool first_s = true, first_b = true;
      for (int g = g0; g < g1; ++g) {
        const int nsp = min(C::GS, p.n_spline_stages - g * C::GS);
        for (int s = 0; s < nsp + p.silu; ++s, ++idx) {
          const int slot = idx % S;
          const uint32_t ph = (idx / S) & 1;
          mbar_wait(bar_full_a(slot), ph);
          mbar_wait(bar_full_b(slot), ph);
          tc_fence_after();
          const bool is_base = (s >= nsp);
          const uint32_t d = tmem + ((is_base && !BF16) ? static_cast<uint32_t>(BN) : 0u);
          bool& first = (is_base && !BF16) ? first_b : first_s;
          const uint32_t a_addr = smem_u32(sA + static_cast<size_t>(slot) * a_bytes);
          const uint32_t b_addr = smem_u32(sB + static_cast<size_t>(slot) * b_bytes);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint64_t ad = umma_desc_sw128(a_addr + 32 * kk);
            const uint64_t bd = umma_desc_sw128(b_addr + 32 * kk);
            const uint32_t acc = (first && kk == 0) ? 0u : 1u;
            if (BF16)
              mma_f16(d, ad, bd, idesc, acc);
            else
              mma_i8(d, ad, bd, idesc, acc);
          }
          first = false;
          tc_commit(bar_empty(slot));
        }
      }
      tc_commit(bar_tmem_full);
    }
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
    // shift `bits` of new data into the top of a 128-bit little-endian register
    auto shift_in = [](uint32_t(&w)[4], uint32_t v, int bits) {
      w[0] = __funnelshift_r(w[0], w[1], bits);
      w[1] = __funnelshift_r(w[1], w[2], bits);
      w[2] = __funnelshift_r(w[2], w[3], bits);
      w[3] = __funnelshift_r(w[3], v, bits);
    };

    int idx = 0;
    for (int g = g0; g < g1; ++g) {
      const int nsp = min(C::GS, p.n_spline_stages - g * C::GS);
      for (int s = 0; s < nsp + p.silu; ++s, ++idx) {
        const int slot = idx % S;
        const uint32_t ph = (idx / S) & 1;
        mbar_wait(bar_full_x(slot), ph);
        uint8_t* a_tile = sA + static_cast<size_t>(slot) * a_bytes;
        if (s < nsp) {
          const uint8_t* xt = sX + static_cast<size_t>(slot) * x_bytes;
          const int i_base = (g * C::GS + s) * C::IPS;
#pragma unroll
          for (int j = 0; j < C::RPT; ++j) {
            const int r = r0 + j * C::ROW_STEP;
            uint4 out;
            if constexpr (!BF16) {
              constexpr int IPC = (NBP == 8) ? 2 : 1;
              int a[IPC];
              if (p.x_kind == X_F32) {
                const float* xr = reinterpret_cast<const float*>(xt) + r * C::IPS + c * IPC;
                if constexpr (IPC == 2) {
                  const float2 xv = *reinterpret_cast<const float2*>(xr);
                  a[0] = lattice_level_f32(xv.x, t_thr, p.lo_f, p.inv_step_f, L);
                  a[1] = lattice_level_f32(xv.y, t_thr, p.lo_f, p.inv_step_f, L);
                } else {
                  a[0] = lattice_level_f32(xr[0], t_thr, p.lo_f, p.inv_step_f, L);
                }
              } else {
                const uint16_t* xr =
                    reinterpret_cast<const uint16_t*>(xt) + r * C::IPS + c * IPC;
                if constexpr (IPC == 2) {
                  const uint32_t v2 = *reinterpret_cast<const uint32_t*>(xr);
                  a[0] = static_cast<int>(v2 & 0xFFFF);
                  a[1] = static_cast<int>(v2 >> 16);
                } else {
                  a[0] = xr[0];
                }
              }
              if constexpr (NBP == 8) {
                const uint32_t v0 = t_vals[a[0]], v1 = t_vals[a[1]];
                const unsigned long long p0 = static_cast<unsigned long long>(v0)
                                              << (8 * (a[0] >> p.k));
                const unsigned long long p1 = static_cast<unsigned long long>(v1)
                                              << (8 * (a[1] >> p.k));
                out = make_uint4(static_cast<uint32_t>(p0), static_cast<uint32_t>(p0 >> 32),
                                 static_cast<uint32_t>(p1), static_cast<uint32_t>(p1 >> 32));
                if (p.zp) {
                  const int i0 = i_base + 2 * c;
                  if (i0 < p.n_in) rsum[j] = __dp4a(v0, 0x01010101u, rsum[j]);
                  if (i0 + 1 < p.n_in) rsum[j] = __dp4a(v1, 0x01010101u, rsum[j]);
                }
                if (p.silu) {
                  const uint32_t sc = static_cast<uint32_t>(t_silu[a[0]]) |
                                      (static_cast<uint32_t>(t_silu[a[1]]) << 8);
                  shift_in(silu_w[j], sc, 16);
                }
              } else {
                const uint32_t v0 = t_vals[a[0]];
                const int jj = a[0] >> p.k;
                const int wi = jj >> 2, sh = (jj & 3) * 8;
                const uint32_t lo = v0 << sh;
                const uint32_t hi = sh ? (v0 >> (32 - sh)) : 0u;
                out.x = (wi == 0) ? lo : 0u;
                out.y = (wi == 1) ? lo : ((wi == 0) ? hi : 0u);
                out.z = (wi == 2) ? lo : ((wi == 1) ? hi : 0u);
                out.w = (wi == 3) ? lo : ((wi == 2) ? hi : 0u);
                if (p.zp && i_base + c < p.n_in) rsum[j] = __dp4a(v0, 0x01010101u, rsum[j]);
                if (p.silu) shift_in(silu_w[j], static_cast<uint32_t>(t_silu[a[0]]), 8);
              }
            } else {
              // bf16 basis values
              constexpr int PMAX = 3;
              const int in_idx = (NBP == 8) ? c : (c >> 1);
              const int half = (NBP == 8) ? 0 : (c & 1);
              const float x = reinterpret_cast<const float*>(xt)[r * C::IPS + in_idx];
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
              out = make_uint4(pack_bf16(v[0], v[1]), pack_bf16(v[2], v[3]), pack_bf16(v[4], v[5]),
                               pack_bf16(v[6], v[7]));
              if (p.silu && (NBP == 8 || (s & 1) == half)) {
                const float xc = fminf(fmaxf(x, p.flo), p.fhi_open);
                const float sv = xc / (1.0f + __expf(-xc));
                const __nv_bfloat16 b = __float2bfloat16_rn(sv);
                const uint32_t bits = *reinterpret_cast<const uint16_t*>(&b);
                shift_in(silu_w[j], bits, 16);
              }
            }
            *reinterpret_cast<uint4*>(a_tile + sw128_off(r, c)) = out;
          }
        } else {
          // base (SiLU) stage: flush the per-thread 16-byte chunk of each row,
          // first padding the shift register for stages the last group lacks.
          // (bf16 with NBP=16: a thread contributes on stages of parity c&1.)
          const int bits = BF16 ? 16 : ((NBP == 8) ? 16 : 8);
          int pad = C::GS - nsp;
          if (BF16 && NBP == 16) {
            pad = 0;
            for (int t = nsp; t < C::GS; ++t) pad += ((t & 1) == (c & 1)) ? 1 : 0;
          }
#pragma unroll
          for (int j = 0; j < C::RPT; ++j) {
            for (int t = 0; t < pad; ++t) shift_in(silu_w[j], 0u, bits);
            const int r = r0 + j * C::ROW_STEP;
            *reinterpret_cast<uint4*>(a_tile + sw128_off(r, c)) =
                make_uint4(silu_w[j][0], silu_w[j][1], silu_w[j][2], silu_w[j][3]);
#pragma unroll
            for (int w = 0; w < 4; ++w) silu_w[j][w] = 0;
          }
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_full_a(slot));
      }
    }

    // ---- row sums of the basis codes (per-tensor zero-point correction) ----
    if (p.zp) {
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

    // ============================ epilogue ================================
    mbar_wait(bar_tmem_full, 0);
    tc_fence_after();
    const int wq = warp & 3;
    const int wh = warp >> 2;
    const int rloc = wq * 32 + lane;
    const int row = m0 + rloc;
    const uint32_t t_row = tmem + (static_cast<uint32_t>(wq * 32) << 16);
    const int nchunks = BN / 16;
    const bool has_b = (!BF16 && p.silu);
    int32_t rowsum = s_rowsum[rloc];
    const size_t tile_id = static_cast<size_t>(m_tile) * p.n_tiles_n + n_tile;

    auto finish = [&](int col0, const uint32_t(&ra)[16], const uint32_t(&rb)[16], int32_t rs) {
      if (row >= p.M) return;
      if (p.epi == EPI_RAW) {
        for (int e = 0; e < 16; ++e) {
          const int j = col0 + e;
          if (j >= p.N) break;
          reinterpret_cast<uint32_t*>(p.out)[static_cast<size_t>(row) * p.ld_out + j] = ra[e];
          if (has_b && p.out2)
            reinterpret_cast<uint32_t*>(p.out2)[static_cast<size_t>(row) * p.ld_out + j] = rb[e];
        }
        return;
      }
      double y[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const int j = min(col0 + e, p.N - 1);
        if (BF16) {
          y[e] = static_cast<double>(__uint_as_float(ra[e]));
        } else if (p.wscheme == 0) {
          const long long v = static_cast<long long>(static_cast<int32_t>(ra[e])) -
                              p.z_w * static_cast<long long>(rs);
          y[e] = __dmul_rn(static_cast<double>(v), p.f_tensor);
        } else {
          double v = __dmul_rn(static_cast<double>(static_cast<int32_t>(ra[e])), p.fs[j]);
          if (has_b) {
            const long long vb =
                static_cast<long long>(static_cast<int32_t>(rb[e])) - p.corr_b[j];
            v = __dadd_rn(v, __dmul_rn(static_cast<double>(vb), p.fb[j]));
          }
          y[e] = v;
        }
      }
      const size_t base = static_cast<size_t>(row) * p.ld_out + col0;
      const int nvalid = min(16, p.N - col0);
      if (p.epi == EPI_F32) {
        float* o = reinterpret_cast<float*>(p.out) + base;
        if (nvalid == 16 && (reinterpret_cast<uintptr_t>(o) & 15) == 0) {
#pragma unroll
          for (int e = 0; e < 16; e += 4)
            *reinterpret_cast<float4*>(o + e) =
                make_float4(__double2float_rn(y[e]), __double2float_rn(y[e + 1]),
                            __double2float_rn(y[e + 2]), __double2float_rn(y[e + 3]));
        } else {
          for (int e = 0; e < nvalid; ++e) o[e] = __double2float_rn(y[e]);
        }
      } else if (p.epi == EPI_LEVEL) {
        uint16_t* o = reinterpret_cast<uint16_t*>(p.out) + base;
        uint32_t lv[8];
#pragma unroll
        for (int e = 0; e < 16; e += 2) {
          const uint32_t l0 = lattice_level_f64(y[e], p.n_lo, p.n_hi_open, p.n_step, p.n_L);
          const uint32_t l1 = lattice_level_f64(y[e + 1], p.n_lo, p.n_hi_open, p.n_step, p.n_L);
          lv[e / 2] = l0 | (l1 << 16);
        }
        if (nvalid == 16 && (reinterpret_cast<uintptr_t>(o) & 15) == 0) {
          *reinterpret_cast<uint4*>(o) = make_uint4(lv[0], lv[1], lv[2], lv[3]);
          *reinterpret_cast<uint4*>(o + 8) = make_uint4(lv[4], lv[5], lv[6], lv[7]);
        } else {
          for (int e = 0; e < nvalid; ++e) o[e] = static_cast<uint16_t>(lv[e / 2] >> (16 * (e & 1)));
        }
      } else {  // EPI_I8
        int8_t* o = reinterpret_cast<int8_t*>(p.out) + base;
        for (int e = 0; e < nvalid; ++e) {
          long long q = llround_ref(__ddiv_rn(y[e], p.out_scale));
          q = q < -127 ? -127 : (q > 127 ? 127 : q);
          o[e] = static_cast<int8_t>(q);
        }
      }
    };

    if (p.splits == 1) {
      for (int cc = wh; cc < nchunks; cc += NPW / 4) {
        uint32_t ra[16], rb[16];
        tmem_ld16(t_row + cc * 16, ra);
        if (has_b) tmem_ld16(t_row + BN + cc * 16, rb);
        tmem_wait_ld();
        finish(n_tile * BN + cc * 16, ra, rb, rowsum);
      }
    } else {
      // split-K: integer partial sums are exact and associative -> bit-exact
      for (int cc = wh; cc < nchunks; cc += NPW / 4) {
        uint32_t ra[16], rb[16];
        tmem_ld16(t_row + cc * 16, ra);
        if (has_b) tmem_ld16(t_row + BN + cc * 16, rb);
        tmem_wait_ld();
        if (row < p.M) {
          const int col0 = n_tile * BN + cc * 16;
          for (int e = 0; e < 16; ++e) {
            const int j = col0 + e;
            if (j >= p.N) break;
            const size_t o = static_cast<size_t>(row) * p.N + j;
            if (BF16)
              atomicAdd(reinterpret_cast<float*>(p.ws_s) + o, __uint_as_float(ra[e]));
            else
              atomicAdd(p.ws_s + o, static_cast<int32_t>(ra[e]));
            if (has_b) atomicAdd(p.ws_b + o, static_cast<int32_t>(rb[e]));
          }
        }
      }
      if (p.zp && wh == 0 && row < p.M)
        atomicAdd(p.ws_rowsum + static_cast<size_t>(n_tile) * p.M + row, rowsum);
      __threadfence();
      asm volatile("bar.sync 1, %0;" ::"r"(C::NP) : "memory");
      if (threadIdx.x == 0) {
        const unsigned prev = atomicAdd(p.counters + tile_id, 1u);
        *s_flag = (prev == static_cast<unsigned>(p.splits - 1)) ? 1u : 0u;
      }
      asm volatile("bar.sync 1, %0;" ::"r"(C::NP) : "memory");
      if (*s_flag) {
        __threadfence();
        if (p.zp && row < p.M)
          rowsum = *reinterpret_cast<volatile int32_t*>(p.ws_rowsum +
                                                        static_cast<size_t>(n_tile) * p.M + row);
        asm volatile("bar.sync 1, %0;" ::"r"(C::NP) : "memory");
        if (p.zp && wh == 0 && row < p.M) p.ws_rowsum[static_cast<size_t>(n_tile) * p.M + row] = 0;
        for (int cc = wh; cc < nchunks; cc += NPW / 4) {
          uint32_t ra[16], rb[16];
          const int col0 = n_tile * BN + cc * 16;
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            ra[e] = 0;
            rb[e] = 0;
            const int j = col0 + e;
            if (row < p.M && j < p.N) {
              const size_t o = static_cast<size_t>(row) * p.N + j;
              ra[e] = static_cast<uint32_t>(atomicExch(p.ws_s + o, 0));
              if (has_b) rb[e] = static_cast<uint32_t>(atomicExch(p.ws_b + o, 0));
            }
          }
          finish(col0, ra, rb, rowsum);
        }
        if (threadIdx.x == 0) p.counters[tile_id] = 0u;
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == NPW + 1) {
    tc_fence_after();
    tmem_dealloc(tmem, tmem_cols);
  }
}

// ---------------------------------------------------------------------------
// host-side launch helpers (called from kan_engine.cpp)
template <bool BF16, int NBP, int NPW>
static cudaError_t launch_impl(const CUtensorMap& xmap, const GemmParams& p, size_t smem,
                               cudaStream_t st) {
  auto kfn = kan_gather_gemm_kernel<BF16, NBP, NPW>;
  cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  dim3 grid(p.n_tiles_n, p.m_tiles, p.splits);
  kfn<<<grid, NPW * 32 + 64, smem, st>>>(xmap, p);
  return cudaGetLastError();
}

int gemm_ips(bool bf16, int nbp) { return 128 / (nbp * (bf16 ? 2 : 1)); }
int gemm_gs(bool bf16, int nbp) { return (bf16 ? 64 : 128) / gemm_ips(bf16, nbp); }
constexpr int kNPW = 8;
int gemm_threads() { return kNPW * 32 + 64; }

size_t gemm_smem_bytes(bool bf16, int nbp, int BN, int S, int x_kind, int L, int silu) {
  const size_t a = 16384, b = static_cast<size_t>(BN) * 128;
  const size_t x = 128u * gemm_ips(bf16, nbp) * (x_kind == X_F32 ? 4 : 2);
  size_t t = 0;
  if (!bf16) {
    const size_t nthr = (x_kind == X_F32) ? L + 2 : 0;
    t += ((nthr + 3) & ~size_t(3)) * 4;
    t += ((L + 1 + 3) & ~size_t(3)) * 4;
    if (silu) t += (L + 1 + 15) & ~size_t(15);
  }
  t += (4 * S + 2) * 8 + 128 * 4 + 16;
  return 1024 + S * (a + b + x) + t;
}

cudaError_t launch_gather_gemm(bool bf16, int nbp, const CUtensorMap& xmap, const GemmParams& p,
                               size_t smem, cudaStream_t st) {
  if (bf16) {
    if (nbp == 8) return launch_impl<true, 8, kNPW>(xmap, p, smem, st);
    return launch_impl<true, 16, kNPW>(xmap, p, smem, st);
  }
  if (nbp == 8) return launch_impl<false, 8, kNPW>(xmap, p, smem, st);
  return launch_impl<false, 16, kNPW>(xmap, p, smem, st);
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
  int64_t nb_ = (n + 255) / 256;
  int blocks = static_cast<int>(nb_ < 148 * 8 ? nb_ : 148 * 8);
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
