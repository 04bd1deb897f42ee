// kan_conv3.cuh -- ky-shared 3x3 / stride-1 / pad-1 KAN conv on the LUT path
// (included by kan_gemm.cu, which provides the level, table and epilogue
// helpers).  Same result as kan_gather_gemm_kernel on the same layer: the
// int32 accumulator is the same sum of products, in another order.
//
// Replaces, for these layers, convkan_forward (layers.hpp:162-190) =
// im2col (layers.hpp:126-154) + kan_linear_forward<LutBasis>.
//
// Why a second kernel: an output tile is bh rows x Wo columns of one image.
// Its three ky taps read the same input pixels shifted by whole rows of Wo
// pixels.  So the producers expand the (bh+2)-row input window of one (kx,
// channel chunk) "super-stage" once -- codes into a K-major SW128 tile in
// shared memory, SiLU codes into a 32-byte-row SW32 tile -- and the MMA warp
// issues the three taps as SS-mode tcgen05.mma whose A descriptors start
// ky*Wo rows in (Wo % 8 == 0 keeps every start on an 8-row swizzle atom).
// The SiLU base term of a tap is one extra K=32 MMA against the SiLU tile.
// This halves the producer work per tap, the bound of these layers.
//
// Warp roles as in kan_gather_gemm_kernel (persistent tiles, 16 producers,
// activation TMA, MMA, weight loader, 4 epilogue warps, double-buffered TMEM
// accumulators).

// LF: a straight-line epilogue is compiled in -- 1: next-layer levels,
// 2: fp32 row-major output (+ residual add, + levels sidecar).  Each is its
// own instantiation: adding the level path to the residual variant cost that
// one registers and measured 25 % on C5's residual convs.
template <int MODE, int LF = 0>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    kan_conv3_kernel(const __grid_constant__ CUtensorMap xmap, const GemmParams p) {
  constexpr int NBP = 8;
  constexpr int IPS = KSTAGE / NBP;  // 32 channels per super-stage
  constexpr int H = IPS / 4;         // inputs per producer thread quarter
  constexpr int NPW = GEMM_PRODUCER_WARPS;
  constexpr int W_X = NPW, W_MMA = NPW + 1, W_B = NPW + 2, W_EPI = NPW + 3;
  constexpr bool SILU = (MODE == MODE_SILU);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);

  const int SA = p.SA, SB = p.SB, SX = p.SX;
  const int BN = p.BN;
  const int R = p.ext_rows;  // expanded rows per super-stage
  const uint32_t b_slot = static_cast<uint32_t>(p.b_slot);
  const uint32_t xesz = (p.x_kind == X_F32) ? 4u : 2u;
  const int x_row_bytes = IPS * static_cast<int>(xesz);
  const uint32_t x_bytes = static_cast<uint32_t>(R) * x_row_bytes;
  const uint32_t a_code_bytes = static_cast<uint32_t>(R) * KSTAGE;  // [2 kblocks][R][128 B]
  const uint32_t a_bytes = a_code_bytes + (SILU ? static_cast<uint32_t>(R) * 32u : 0u);
  uint8_t* sB = smem;
  uint8_t* sA = sB + static_cast<size_t>(SB) * b_slot;
  uint8_t* sX = sA + static_cast<size_t>(SA) * a_bytes;
  uint8_t* sT = sX + static_cast<size_t>(SX) * x_bytes;
  const int tab_bytes = p.tab_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sT + tab_bytes);
  double* s_cols = reinterpret_cast<double*>(bars + 2 * SA + 2 * SB + 2 * SX + 9);  // [2][BN] per tile
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(s_cols + 2 * BN);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  pdl_trigger();

  // Work units: with p.mc == 2 the two CTAs of a cluster take the two M tiles
  // of a unit (same N tile) and each issues half of the unit's weight-tile
  // loads, multicast into both CTAs' rings -- half the L2 weight traffic.
  // Every CTA walks every unit of its cluster (an odd last M tile leaves the
  // second CTA a unit without a tile: it only releases its weight slots).
  const int MC = p.mc > 1 ? p.mc : 1;
  const uint32_t crank = MC > 1 ? cluster_rank() : 0u;
  const int unit0 = MC > 1 ? static_cast<int>(cluster_id_x()) : static_cast<int>(blockIdx.x);
  const int unit_step = MC > 1 ? static_cast<int>(n_clusters_x()) : static_cast<int>(gridDim.x);
  const int n_units = (p.m_tiles + MC - 1) / MC * p.n_tiles_n;
  const uint16_t mc_mask = static_cast<uint16_t>((1u << MC) - 1u);
  struct Tile {
    int m0, n_tile, n0, y0;
    bool valid;
  };
  auto tile_of = [&](int u) {
    Tile r;
    const int mu = u / p.n_tiles_n;
    r.n_tile = u - mu * p.n_tiles_n;
    const int mt = mu * MC + static_cast<int>(crank);
    r.valid = mt < p.m_tiles;
    r.m0 = mt * 128;
    r.n0 = mt / p.tpi;
    r.y0 = (mt % p.tpi) * p.bh;
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
  const uint32_t bar_tab = smem_u32(bx + 8);

  constexpr uint32_t tmem_cols = 512;
  const uint32_t BNa = static_cast<uint32_t>((BN + 31) / 32 * 32);
  const int nacc = p.nacc;

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
      mbar_init(bar_bempty(s), MC);  // every CTA of the cluster releases the slot
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(bar_accfull(b), 1);
      mbar_init(bar_accempty(b), GEMM_EPI_WARPS);
    }
    mbar_init(bar_tab, 1);
    mbar_fence_init();
  }
  if (warp == W_X && lane == 0) tma_prefetch(&xmap);
  if (warp == W_MMA) tmem_alloc(smem_u32(s_tmem), tmem_cols);
  tc_fence_before();
  __syncthreads();
  if (MC > 1) cluster_sync_all();  // peers' barriers initialised before any multicast
  tc_fence_after();
  const uint32_t tmem = *s_tmem;

  if (warp == W_X) {
    // ================= activation loader: one window per super-stage ========
    pdl_wait();
    Ring rx(SX);
    for (int u = unit0; u < n_units; u += unit_step) {
      const Tile tl = tile_of(u);
      if (!tl.valid) continue;
      for (int ss = 0; ss < p.n_ss; ++ss, rx.next()) {
        const int kx = ss / p.cps, cc = ss - kx * p.cps;
        mbar_wait(bar_xempty(rx.slot), rx.phase ^ 1);
        if (lane == 0 && KAN_DBG(p, 4)) {  // tuning only: no activation load (stale window)
          mbar_arrive(bar_xfull(rx.slot));
        } else if (lane == 0) {
          mbar_arrive_tx(bar_xfull(rx.slot), x_bytes);
          // rows y0-1 .. y0+bh, columns kx-1 .. kx-1+Wo-1 (zero outside)
          tma_load_4d(smem_u32(sX + static_cast<size_t>(rx.slot) * x_bytes), &xmap, cc * IPS, kx - 1,
                      tl.y0 - 1, tl.n0, bar_xfull(rx.slot));
        }
        __syncwarp();
      }
    }
  } else if (warp == W_B) {
    // ============== table + weight-tile loader: 3 taps per super-stage ======
    if (lane == 0 && tab_bytes > 0) {
      mbar_arrive_tx(bar_tab, static_cast<uint32_t>(tab_bytes));
      bulk_load(smem_u32(sT), p.tab, static_cast<uint32_t>(tab_bytes), bar_tab);
    }
    __syncwarp();
    Ring rb(SB);
    uint32_t fill = 0;
    for (int u = unit0; u < n_units; u += unit_step) {
      const Tile tl = tile_of(u);
      for (int q = 0; q < 3 * p.n_ss; ++q, rb.next(), ++fill) {
        // released by every CTA of the cluster: safe to refill everywhere
        mbar_wait(bar_bempty(rb.slot), rb.phase ^ 1);
        if (lane == 0) {
          const size_t wt = static_cast<size_t>(tl.n_tile) * 3 * p.n_ss + q;
          const uint32_t dst = smem_u32(sB + static_cast<size_t>(rb.slot) * b_slot);
          if (KAN_DBG(p, 32))  // tuning only: no weight loads (stale slots)
            mbar_arrive(bar_bfull(rb.slot));
          else
            mbar_arrive_tx(bar_bfull(rb.slot), b_slot);
          if (KAN_DBG(p, 32)) {
          } else if (MC == 1)
            bulk_load(dst, p.wt + wt * b_slot, b_slot, bar_bfull(rb.slot));
          else if (fill % MC == crank)
            bulk_load_mc(dst, p.wt + wt * b_slot, b_slot, bar_bfull(rb.slot), mc_mask);
        }
        __syncwarp();
      }
    }
    // drain: every peer's release of our slots has landed before the CTA exits
    for (int s = 0; s < SB; ++s, rb.next()) mbar_wait(bar_bempty(rb.slot), rb.phase ^ 1);
  } else if (warp == W_MMA) {
    // ============ MMA issuer: SS-mode, three row-shifted taps per stage ====
    // Warp-uniform waits and descriptors, one elected lane issues: at N = 64
    // a tap is only ~300 tensor cycles, so the issue path must stay short.
    const uint32_t idesc = idesc_i8(BN, true);
    const uint32_t a_kstep = static_cast<uint32_t>(R) * 8u;   // next 128-byte K block of A (x16 B)
    const uint32_t b_kstep = static_cast<uint32_t>(BN) * 8u;  // next 128-byte K block of B (x16 B)
    Ring ra(SA), rb(SB);
    int lt = 0;
    auto release_b = [&](uint32_t bar) {
      if (MC == 1)
        tc_commit(bar);
      else
        tc_commit_mc(bar, mc_mask);
    };
    for (int u = unit0; u < n_units; u += unit_step) {
      if (!tile_of(u).valid) {  // no tile here: release the unit's weight slots
        for (int q = 0; q < 3 * p.n_ss; ++q, rb.next()) {
          mbar_wait_warp(bar_bfull(rb.slot), rb.phase);
          if (elect_one()) release_b(bar_bempty(rb.slot));
          __syncwarp();
        }
        continue;
      }
      const int ab = nacc == 2 ? (lt & 1) : 0;
      const int use = nacc == 2 ? (lt >> 1) : lt;
      mbar_wait_warp(bar_accempty(ab), (use & 1) ^ 1);
      tc_fence_after();
      const uint32_t dacc = tmem + static_cast<uint32_t>(ab) * BNa;
      uint32_t acc = 0u;
      for (int ss = 0; ss < p.n_ss; ++ss, ra.next()) {
        mbar_wait_warp(bar_afull(ra.slot), ra.phase);
        tc_fence_after();
        const uint32_t a_addr = smem_u32(sA + static_cast<size_t>(ra.slot) * a_bytes);
        for (int ky = 0; ky < 3; ++ky, rb.next()) {
          mbar_wait_warp(bar_bfull(rb.slot), rb.phase);
          tc_fence_after();
          const uint32_t b_addr = smem_u32(sB + static_cast<size_t>(rb.slot) * b_slot);
          const uint32_t row_off = static_cast<uint32_t>(ky * p.Wo / 8) * 1024u;  // whole SW128 atoms
          const uint64_t ad0 = umma_desc_sw128(a_addr + row_off);
          const uint64_t bd0 = umma_desc_sw128(b_addr);
          const uint64_t sd_a = umma_desc_sw32(a_addr + a_code_bytes + static_cast<uint32_t>(ky * p.Wo / 8) * 256u);
          const uint64_t sd_b = umma_desc_sw32(b_addr + BN * KSTAGE);
          if (elect_one()) {
            if (!KAN_DBG(p, 2)) {  // (tuning only: flag 2 skips the MMAs)
#pragma unroll
              for (int kk = 0; kk < KSTAGE / 32; ++kk) {
                // descriptor start addresses advance in 16-byte units (no carry: smem < 256 KB)
                const uint64_t ad = ad0 + (kk >> 2) * a_kstep + 2 * (kk & 3);
                const uint64_t bd = bd0 + (kk >> 2) * b_kstep + 2 * (kk & 3);
                mma_i8(dacc, ad, bd, idesc, kk == 0 ? acc : 1u);
              }
              // the tap's SiLU base term: K = 32 codes against the SW32 SiLU weights
              if (SILU) mma_i8(dacc, sd_a, sd_b, idesc, 1u);
            }
            release_b(bar_bempty(rb.slot));
          }
          __syncwarp();
          acc = 1u;
        }
        if (elect_one()) tc_commit(bar_aempty(ra.slot));
        __syncwarp();
      }
      if (elect_one()) tc_commit(bar_accfull(ab));
      __syncwarp();
      ++lt;
    }
  } else if (warp < NPW) {
    // ==================== producers: expand each window once ================
    if (tab_bytes > 0) mbar_wait(bar_tab, 0);
    const uint32_t* vals = reinterpret_cast<const uint32_t*>(sT);
    const float* thr = reinterpret_cast<const float*>(sT + p.off_thr);
    const uint8_t* silu_tab = sT + p.off_silu;
    const uint2* c64 = reinterpret_cast<const uint2*>(sT + p.off_c64);
    const int units = (R / 32) * 4;  // (32-row group, K quarter) pairs
    Ring ra(SA), rx(SX);
    for (int u = unit0; u < n_units; u += unit_step) {
      const Tile tl = tile_of(u);
      if (!tl.valid) continue;
      uint32_t rsum = 0;
      for (int ss = 0; ss < p.n_ss; ++ss, ra.next(), rx.next()) {
        const int kx = ss / p.cps;
        mbar_wait(bar_xfull(rx.slot), rx.phase);
        mbar_wait(bar_aempty(ra.slot), ra.phase ^ 1);
        const uint8_t* xt = sX + static_cast<size_t>(rx.slot) * x_bytes;
        uint8_t* at = sA + static_cast<size_t>(ra.slot) * a_bytes;
        for (int u = KAN_DBG(p, 16) ? units : warp; u < units; u += NPW) {  // (flag 16: no expansion)
          const int g = u >> 2, h = u & 3;
          const int rr = 32 * g + lane;  // expanded row = input pixel of the window
          const int wy = rr / p.Wo, wx = rr - wy * p.Wo;
          const int iy = tl.y0 - 1 + wy, ix = wx + kx - 1;
          const bool pad = static_cast<unsigned>(iy) >= static_cast<unsigned>(p.H) ||
                           static_cast<unsigned>(ix) >= static_cast<unsigned>(p.W);
          int a[H];
          const int xoff = h * H * static_cast<int>(xesz);
          if (p.x_kind == X_F32) {
            uint32_t xr[H];
            load_x<4 * H>(xt, rr, xoff, x_row_bytes, xr);
            levels8_f32<H>([&](int e) { return __uint_as_float(xr[e]); }, p.inv_step_f, p.lo_f, p.L, thr, a);
            if (pad)
#pragma unroll
              for (int e = 0; e < H; ++e) a[e] = p.lvl0;
          } else {
            uint32_t xr[H / 2];
            load_x<2 * H>(xt, rr, xoff, x_row_bytes, xr);
#pragma unroll
            for (int q = 0; q < H / 2; ++q) {
              a[2 * q] = pad ? p.lvl0 : static_cast<int>(xr[q] & 0xFFFF);
              a[2 * q + 1] = pad ? p.lvl0 : static_cast<int>(xr[q] >> 16);
            }
          }
          uint32_t w[16], nw[2];
          lut_row<NBP, MODE>(p, vals, c64, silu_tab, a, 0, w, rsum, nw);
          // codes: row rr, K bytes [64h, 64h+64) of the SW128 tile
          uint8_t* ab = at + (h >> 1) * R * 128 + (rr >> 3) * 1024 + (rr & 7) * 128;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const int ch = (h & 1) * 4 + c;
            *reinterpret_cast<uint4*>(ab + ((ch ^ (rr & 7)) << 4)) =
                make_uint4(w[4 * c], w[4 * c + 1], w[4 * c + 2], w[4 * c + 3]);
          }
          if constexpr (SILU) {
            // SiLU codes: row rr, bytes [8h, 8h+8) of the SW32 tile
            uint8_t* sb = at + a_code_bytes + (rr >> 3) * 256 + (rr & 7) * 32 +
                          ((((h >> 1) ^ ((rr >> 2) & 1))) << 4) + (h & 1) * 8;
            *reinterpret_cast<uint2*>(sb) = make_uint2(nw[0], nw[1]);
          }
        }
        // generic-proxy smem writes -> visible to the tensor core (async proxy)
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(bar_xempty(rx.slot));
          mbar_arrive(bar_afull(ra.slot));
        }
      }
    }
  } else {
    // ============================ epilogue ================================
    if (tab_bytes > 0) mbar_wait(bar_tab, 0);
    const int wq = warp & 3;
    const int rloc = wq * 32 + lane;
    const uint32_t t_row = tmem + (static_cast<uint32_t>(wq * 32) << 16);
    int lt = 0;
    for (int u = unit0; u < n_units; u += unit_step) {
      const Tile tl = tile_of(u);
      if (!tl.valid) continue;
      const int ab = nacc == 2 ? (lt & 1) : 0;
      const int use = nacc == 2 ? (lt >> 1) : lt;
      ++lt;
      mbar_wait(bar_accfull(ab), use & 1);
      tc_fence_after();
      // the tile's column constants, staged in smem (see kan_gather_gemm_kernel)
      asm volatile("bar.sync 4, %0;" ::"r"(32 * GEMM_EPI_WARPS) : "memory");
      for (int i = static_cast<int>(threadIdx.x) - 32 * W_EPI; i < BN; i += 32 * GEMM_EPI_WARPS) {
        const int j = min(tl.n_tile * BN + i, p.N - 1);
        s_cols[i] = p.fs[j];
        s_cols[BN + i] = SILU ? static_cast<double>(p.corr_b[j]) : 0.0;
      }
      asm volatile("bar.sync 4, %0;" ::"r"(32 * GEMM_EPI_WARPS) : "memory");
      const uint32_t tacc = t_row + static_cast<uint32_t>(ab) * BNa;
      const int row = tl.m0 + rloc;
      float rv[32];  // residual prefetch: 32 columns in flight per thread
      const int half = (warp - W_EPI) >> 2;  // the two warps of a lane quarter take alternate 32-column blocks
      const bool lvl_fast = LF == 1 && p.epi == EPI_LEVEL && !p.res_kind && tl.n_tile * BN + BN <= p.N &&
                            (p.ld_out & 7) == 0 && (reinterpret_cast<uintptr_t>(p.out) & 15) == 0;
      // 32-column blocks (the two warps of a lane quarter alternate), read as
      // two 16-column TMEM loads: 2 round trips per block instead of 8
      if constexpr (LF == 2) {
        const int n0 = tl.n_tile * BN;
        if (p.epi == EPI_F32 && p.out_hw == 0 && n0 + BN <= p.N && (p.ld_out & 3) == 0 &&
            (reinterpret_cast<uintptr_t>(p.out) & 15) == 0 &&
            (!p.res_kind || ((p.ld_res & 3) == 0 && (reinterpret_cast<uintptr_t>(p.res) & 15) == 0)) &&
            (p.out_lv == nullptr || ((p.ld_lv & 7) == 0 && (reinterpret_cast<uintptr_t>(p.out_lv) & 15) == 0)) &&
            !KAN_DBG(p, 8)) {
          // 16 columns per step: residual loads issued before the TMEM load,
          // then finish4's fp64 (acc - corr) * fs [+ residual] (exact
          // subtraction), the fp32 row and its levels sidecar
          const float* thr = reinterpret_cast<const float*>(sT + p.off_thr);
#pragma unroll 1
          for (int cl = half * 16; cl < BN; cl += 32) {
            float4 rv4[4] = {};
            if (p.res_kind && row < p.M) {
              const float4* rp = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(p.res) +
                                                                 static_cast<size_t>(row) * p.ld_res + n0 + cl);
#pragma unroll
              for (int q = 0; q < 4; ++q) rv4[q] = rp[q];
            }
            uint32_t r16[16];
            tmem_ld16(tacc + cl, r16);
            tmem_wait_ld();
            if (row < p.M) {
              float f[16];
#pragma unroll
              for (int e = 0; e < 16; ++e) {
                double y = __dmul_rn(__dsub_rn(i32_to_f64(r16[e]), s_cols[BN + cl + e]),
                                     s_cols[cl + e]);
                if (p.res_kind) y = __dadd_rn(y, static_cast<double>((&rv4[e >> 2].x)[e & 3]));
                f[e] = __double2float_rn(y);
              }
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
      for (int blk = half; blk < (KAN_DBG(p, 8) ? 0 : (BN + 31) / 32); blk += 2) {
        const int gq0 = blk * 8;
        if (p.res_kind) {
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int c = tl.n_tile * BN + (gq0 + q) * 4;
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (row < p.M && c + 3 < p.N && gq0 + q < BN / 4)
              v = *reinterpret_cast<const float4*>(reinterpret_cast<const float*>(p.res) +
                                                   static_cast<size_t>(row) * p.ld_res + c);
            else if (row < p.M && gq0 + q < BN / 4)
              for (int e = 0; e < 4; ++e)
                if (c + e < p.N)
                  (&v.x)[e] = reinterpret_cast<const float*>(p.res)[static_cast<size_t>(row) * p.ld_res + c + e];
            rv[4 * q] = v.x;
            rv[4 * q + 1] = v.y;
            rv[4 * q + 2] = v.z;
            rv[4 * q + 3] = v.w;
          }
        }
#pragma unroll 1
        for (int sub = 0; sub < 2; ++sub) {
        uint32_t r16[16];
        tmem_ld16(tacc + blk * 32 + sub * 16, r16);
        tmem_wait_ld();
        if (LF == 1 && lvl_fast) {
          // next-layer levels of 16 full columns, straight-line: the same fp64
          // (acc - corr) * fs (the subtraction is exact in fp64: an integer
          // below 2^53) and lattice_level_fast, then two 16-byte stores
          const int cl = blk * 32 + sub * 16;
          if (row < p.M && cl < BN) {
            uint32_t w[8];
#pragma unroll
            for (int hh = 0; hh < 2; ++hh)
              levels8_f64(
                  [&](int e8) {
                    const int e = 8 * hh + e8;
                    return __dmul_rn(__dsub_rn(i32_to_f64(r16[e]), s_cols[BN + cl + e]),
                                     s_cols[cl + e]);
                  },
                  p.n_lo, p.n_hi_open, p.n_step, p.n_inv_step, p.n_L, w + 4 * hh);
            uint4* o = reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(p.out) + static_cast<size_t>(row) * p.ld_out +
                                                tl.n_tile * BN + cl);
            o[0] = make_uint4(w[0], w[1], w[2], w[3]);
            o[1] = make_uint4(w[4], w[5], w[6], w[7]);
          }
          continue;
        }
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
        const int q = sub * 4 + q4;
        const int gq = gq0 + q;
        if (gq >= BN / 4) break;
        const uint32_t ra[4] = {r16[4 * q4], r16[4 * q4 + 1], r16[4 * q4 + 2], r16[4 * q4 + 3]};
        const int col0 = tl.n_tile * BN + gq * 4;
        if (row >= p.M) continue;
        const size_t base = static_cast<size_t>(row) * p.ld_out + col0;
        const int nvalid = min(4, p.N - col0);
        if (p.epi == EPI_RAW) {
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if (e < nvalid) reinterpret_cast<uint32_t*>(p.out)[base + e] = ra[e];
          continue;
        }
        double y[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int jl = gq * 4 + e;
          const long long v = static_cast<long long>(static_cast<int32_t>(ra[e])) -
                              (SILU ? static_cast<long long>(s_cols[BN + jl]) : 0ll);
          y[e] = __dmul_rn(static_cast<double>(v), s_cols[jl]);
          if (p.res_kind && e < nvalid) y[e] = __dadd_rn(y[e], static_cast<double>(rv[(gq & 7) * 4 + e]));
        }
        if (p.epi == EPI_F32 && p.out_hw > 0) {
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
          if (p.out_lv) {  // levels sidecar (see kan_gather_gemm_kernel), one 8-byte store
            const float* thr = reinterpret_cast<const float*>(sT + p.off_thr);
            uint16_t* ol = p.out_lv + static_cast<size_t>(row) * p.ld_lv + col0;
            uint32_t a[4];
#pragma unroll
            for (int e = 0; e < 4; ++e)
              a[e] = static_cast<uint32_t>(lattice_level_tie(__double2float_rn(y[e]), p.inv_step_f, p.lo_f, p.L, thr));
            if (nvalid == 4 && (reinterpret_cast<uintptr_t>(ol) & 7) == 0) {
              *reinterpret_cast<uint2*>(ol) = make_uint2(a[0] | (a[1] << 16), a[2] | (a[3] << 16));
            } else {
#pragma unroll
              for (int e = 0; e < 4; ++e)
                if (e < nvalid) ol[e] = static_cast<uint16_t>(a[e]);
            }
          }
        } else {  // EPI_LEVEL
          uint16_t* o = reinterpret_cast<uint16_t*>(p.out) + base;
          uint32_t a[4];
#pragma unroll
          for (int e = 0; e < 4; ++e)
            a[e] = static_cast<uint32_t>(lattice_level_fast(y[e], p.n_lo, p.n_hi_open, p.n_step, p.n_inv_step, p.n_L));
          if (nvalid == 4 && (reinterpret_cast<uintptr_t>(o) & 7) == 0) {
            *reinterpret_cast<uint2*>(o) = make_uint2(a[0] | (a[1] << 16), a[2] | (a[3] << 16));
          } else {
#pragma unroll
            for (int e = 0; e < 4; ++e)
              if (e < nvalid) o[e] = static_cast<uint16_t>(a[e]);
          }
        }
        }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_accempty(ab));
    }
  }

  tc_fence_before();
  __syncthreads();
  if (MC > 1) cluster_sync_all();  // no multicast into / release of an exited CTA
  if (warp == W_MMA) {
    tc_fence_after();
    tmem_dealloc(tmem, tmem_cols);
  }
}

size_t conv3_smem_bytes(int BN, int R, int SA, int SB, int SX, int x_kind, int tab_bytes, bool silu) {
  const size_t b_slot = (static_cast<size_t>(BN) * (KSTAGE + (silu ? 32 : 0)) + 1023) / 1024 * 1024;
  const size_t a = static_cast<size_t>(R) * (KSTAGE + (silu ? 32 : 0));
  const size_t x = static_cast<size_t>(R) * (KSTAGE / 8) * (x_kind == X_F32 ? 4 : 2);
  return 1024 + SB * b_slot + SA * a + SX * x + static_cast<size_t>(tab_bytes) + (2 * SA + 2 * SB + 2 * SX + 9) * 8 +
         2 * static_cast<size_t>(BN) * 8 + 16;
}

cudaError_t launch_conv3(int mode, const CUtensorMap& xmap, const GemmParams& p, size_t smem, cudaStream_t st) {
  static std::atomic<unsigned long long> optin[9];  // per kernel variant, per device
  const int lf = (p.epi == EPI_LEVEL && !p.res_kind) ? 1 : (p.epi == EPI_F32 && p.out_hw == 0) ? 2 : 0;
  const int var = mode * 3 + lf;
  auto go = [&](auto kfn) -> cudaError_t {
    if (cudaError_t e = smem_optin(kfn, optin[var]); e != cudaSuccess) return e;
    const int n_sm = device_sm_count();
    const int mc = p.mc > 1 ? p.mc : 1;
    const int units = (p.m_tiles + mc - 1) / mc * p.n_tiles_n;
    const int clusters = units < n_sm / mc ? units : n_sm / mc;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(clusters * mc));
    cfg.blockDim = dim3(GEMM_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = static_cast<unsigned>(mc);
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    return cudaLaunchKernelEx(&cfg, kfn, xmap, p);
  };
  if (mode == MODE_SILU)
    return lf == 1 ? go(kan_conv3_kernel<MODE_SILU, 1>)
                   : (lf == 2 ? go(kan_conv3_kernel<MODE_SILU, 2>) : go(kan_conv3_kernel<MODE_SILU>));
  return lf == 1 ? go(kan_conv3_kernel<MODE_PLAIN, 1>)
                 : (lf == 2 ? go(kan_conv3_kernel<MODE_PLAIN, 2>) : go(kan_conv3_kernel<MODE_PLAIN>));
}
