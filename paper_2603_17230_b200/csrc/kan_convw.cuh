// kan_convw.cuh -- window-shared 3x3 / stride-1 / pad-1 KAN conv on the LUT
// path, all nine taps from one expanded input window (included by
// kan_gemm.cu, which provides the level, table, ring and PTX helpers).  Same
// int32 accumulators as kan_gather_gemm_kernel on the same layer (the same
// sum of products in another order), so the same outputs, bit for bit.
//
// Replaces, for these layers, convkan_forward (layers.hpp:162-190) = im2col
// (layers.hpp:126-154) + kan_linear_forward<LutBasis> (layers.hpp:99-121).
//
// Why: on the N = 64 / 128 convs of ResKAN18 stages 1-2 the im2col kernels
// are bound by the producers' code expansion (every input pixel is expanded
// once per tap, 9x; kan_conv3 shares the three ky taps, 4.5x).  Here an M
// tile's rows are (output pixel, image) with EIGHT images of the batch
// innermost, read straight from the NHWC tensor by one 4D TMA box whose image
// dimension is the second fastest.  A one-pixel shift is then exactly one
// 8-row core-matrix group, so every tap (ky, kx) of an accumulator's 16
// consecutive output pixels is the SAME expanded window addressed 8*((ky *
// (W+2)) + kx) rows further on: one SW32 K-major window per 4-channel K block
// serves 9 taps x NACC accumulators of SS-mode tcgen05.mma (expansion ~2x per
// output instead of 9x).  Outputs go back to NHWC row by row (each thread one
// row of BN channels), so neighbouring layers are unaffected.
//
// Tile: 8 images x TR output rows x W columns (W = 16 or 32); NACC = TR*W/16
// accumulators of 128 rows x BN columns, double-buffered in TMEM
// (NACC * BN <= 256).  K: C_in / 4 blocks of 32 bytes (4 channels x NBP = 8
// basis bytes); an activation load (8 channels, u16 levels) feeds two blocks,
// expanded one per producer step so the A ring runs SA - 1 blocks ahead.
// MODE_ZP (the reference's per-tensor asymmetric weights): the producers sum
// each window row's codes over all channels (wsum), and the epilogue forms
// each output row's code sum from the 9 window rows it read.
//
// Warp roles as in kan_gather_gemm_kernel (12 producers here), activation TMA,
// MMA issuer, weight loader, 8 epilogue warps (two per TMEM lane quarter).

// 12 producer warps (the window expansion is cheap here), so the epilogue's
// 16-column fp64 chains get more registers than the 27-warp gather kernel's
constexpr int CONVW_PRODUCER_WARPS = 12;
constexpr int CONVW_THREADS = 32 * (CONVW_PRODUCER_WARPS + 3 + GEMM_EPI_WARPS);
constexpr int CONVW_MAX_ROWS = 3 * 32 * CONVW_PRODUCER_WARPS;  // window rows: RPT rows per producer thread

template <int MODE>
__global__ void __launch_bounds__(CONVW_THREADS, 1)
    kan_convw_kernel(const __grid_constant__ CUtensorMap xmap, const GemmParams p) {
  constexpr int NPW = CONVW_PRODUCER_WARPS, NP = 32 * NPW;
  constexpr int W_X = NPW, W_MMA = NPW + 1, W_B = NPW + 2, W_EPI = NPW + 3;
  constexpr bool ZP = (MODE == MODE_ZP);
  constexpr int RPT = CONVW_MAX_ROWS / NP;  // window rows per producer thread (max)
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);

  const int SA = p.SA, SB = p.SB, SX = p.SX;
  const int BN = p.BN;
  const int W = p.W, H = p.H, TR = p.bh;
  const int WP = W + 2;                // window pitch in pixels
  const int WR = p.ext_rows;           // window rows = (TR + 2) * WP * 8
  const int NACC = p.nacc;             // accumulators per tile
  const int n_kb = p.n_ss;             // 32-byte K blocks (4 channels each)
  const uint32_t a_bytes = static_cast<uint32_t>(WR) * 32u;
  const uint32_t x_bytes = static_cast<uint32_t>(WR) * 16u;  // 8 channels of u16 levels per row
  const uint32_t b_slot = static_cast<uint32_t>(p.b_slot);  // 9 taps x BN rows x 32 B
  uint8_t* sB = smem;
  uint8_t* sA = sB + static_cast<size_t>(SB) * b_slot;
  uint8_t* sX = sA + static_cast<size_t>(SA) * a_bytes;
  uint8_t* sT = sX + static_cast<size_t>(SX) * x_bytes;
  const int tab_bytes = p.tab_bytes;
  int32_t* s_wsum = reinterpret_cast<int32_t*>(sT + ((tab_bytes + 15) & ~15));  // [2][WR] (ZP)
  uint64_t* bars = reinterpret_cast<uint64_t*>(s_wsum + (ZP ? 2 * WR : 0));
  double* s_cols = reinterpret_cast<double*>(bars + 2 * SA + 2 * SB + 2 * SX + 13);  // [BN]
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(s_cols + BN);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  pdl_trigger();

  // tiles: (image group of 8, band of TR output rows, N tile), N tile fastest
  const int bands = H / TR;
  const int n_groups = (p.M + 7) / 8;  // p.M = images
  const int n_tiles = n_groups * bands * p.n_tiles_n;
  struct Tile {
    int g, oy0, nt;
  };
  auto tile_of = [&](int t) {
    Tile r;
    r.nt = t % p.n_tiles_n;
    const int gb = t / p.n_tiles_n;
    r.g = gb / bands;
    r.oy0 = (gb - r.g * bands) * TR;
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
  auto bar_wsfull = [&](int b) { return smem_u32(bx + 4 + b); };
  auto bar_wsempty = [&](int b) { return smem_u32(bx + 6 + b); };
  const uint32_t bar_tab = smem_u32(bx + 8);

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
      mbar_init(bar_wsfull(b), NPW);
      mbar_init(bar_wsempty(b), GEMM_EPI_WARPS);
    }
    mbar_init(bar_tab, 1);
    mbar_fence_init();
  }
  if (warp == W_X && lane == 0) tma_prefetch(&xmap);
  if (warp == W_MMA) tmem_alloc(smem_u32(s_tmem), 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;

  if (warp == W_X) {
    // ============ activation loader: the tile's window, 8 channels per load ======
    pdl_wait();
    Ring rx(SX);
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
      const Tile tl = tile_of(t);
      for (int kp = 0; kp < n_kb / 2; ++kp, rx.next()) {
        mbar_wait(bar_xempty(rx.slot), rx.phase ^ 1);
        if (lane == 0) {
          mbar_arrive_tx(bar_xfull(rx.slot), x_bytes);
          // box (8 channels, 8 images, W+2 columns, TR+2 rows) from (c, img, -1, oy0-1)
          tma_load_4d(smem_u32(sX + static_cast<size_t>(rx.slot) * x_bytes), &xmap, kp * 8, tl.g * 8, -1,
                      tl.oy0 - 1, bar_xfull(rx.slot));
        }
        __syncwarp();
      }
    }
  } else if (warp == W_B) {
    // ============ table + weight loader: 9 taps x BN x 32 B per K block ==========
    if (lane == 0 && tab_bytes > 0) {
      mbar_arrive_tx(bar_tab, static_cast<uint32_t>(tab_bytes));
      bulk_load(smem_u32(sT), p.tab, static_cast<uint32_t>(tab_bytes), bar_tab);
    }
    __syncwarp();
    Ring rb(SB);
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
      const Tile tl = tile_of(t);
      for (int kb = 0; kb < n_kb; ++kb, rb.next()) {
        mbar_wait(bar_bempty(rb.slot), rb.phase ^ 1);
        if (lane == 0) {
          mbar_arrive_tx(bar_bfull(rb.slot), b_slot);
          bulk_load(smem_u32(sB + static_cast<size_t>(rb.slot) * b_slot),
                    p.wt + (static_cast<size_t>(tl.nt) * n_kb + kb) * b_slot, b_slot, bar_bfull(rb.slot));
        }
        __syncwarp();
      }
    }
  } else if (warp == W_MMA) {
    // ============ MMA issuer: 9 taps x NACC accumulators per K block ============
    const uint32_t idesc = idesc_i8(BN, p.b_signed != 0);
    // descriptor start addresses advance in 16-byte units: one window row
    // (32 B) is 2 units.  Row offsets of each accumulator's first pixel and of
    // each tap, computed once (no divisions in the issue loop: at N = 64 a
    // K block is 36 MMAs of ~34 tensor cycles each, so the loop must be short)
    uint32_t acc_row[8], tap_row[9];
#pragma unroll
    for (int a = 0; a < 8; ++a) {
      const int py = (a * 16) / W, px = a * 16 - py * W;
      acc_row[a] = static_cast<uint32_t>((py * WP + px) * 8 * 2);
    }
#pragma unroll
    for (int tap = 0; tap < 9; ++tap) tap_row[tap] = static_cast<uint32_t>(((tap / 3) * WP + tap % 3) * 8 * 2);
    const uint64_t b_tap = static_cast<uint64_t>(BN) * 2u;  // one tap's weight tile (BN x 32 B) in 16-byte units
    Ring ra(SA), rb(SB);
    int lt = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++lt) {
      const int ab = lt & 1;
      mbar_wait_warp(bar_accempty(ab), ((lt >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t dacc = tmem + static_cast<uint32_t>(ab) * 256u;
      for (int kb = 0; kb < n_kb; ++kb, ra.next(), rb.next()) {
        mbar_wait_warp(bar_afull(ra.slot), ra.phase);
        mbar_wait_warp(bar_bfull(rb.slot), rb.phase);
        tc_fence_after();
        const uint64_t ad0 = umma_desc_sw32(smem_u32(sA + static_cast<size_t>(ra.slot) * a_bytes));
        const uint64_t bd0 = umma_desc_sw32(smem_u32(sB + static_cast<size_t>(rb.slot) * b_slot));
        if (elect_one()) {
#pragma unroll
          for (int tap = 0; tap < 9; ++tap) {
            const uint64_t bd = bd0 + static_cast<uint64_t>(tap) * b_tap;
            const uint32_t acc = (kb | tap) != 0 ? 1u : 0u;
#pragma unroll
            for (int a = 0; a < 8; ++a)
              if (a < NACC && !KAN_DBG(p, 2))  // (tuning only: flag 2 skips the MMAs)
                mma_i8(dacc + static_cast<uint32_t>(a * BN), ad0 + (acc_row[a] + tap_row[tap]), bd, idesc, acc);
          }
          tc_commit(bar_aempty(ra.slot));
          tc_commit(bar_bempty(rb.slot));
        }
        __syncwarp();
      }
      if (elect_one()) tc_commit(bar_accfull(ab));
      __syncwarp();
    }
  } else if (warp < NPW) {
    // ============ producers: expand the window once per K block =================
    if (tab_bytes > 0) mbar_wait(bar_tab, 0);
    const uint2* c64 = reinterpret_cast<const uint2*>(sT + p.off_c64);
    const int tid = threadIdx.x;  // 0 .. NP-1
    Ring ra(SA), rx(SX);
    int lt = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++lt) {
      const Tile tl = tile_of(t);
      // this thread's window rows r = tid + q*NP: spatial padding flags (taps
      // outside the map read level(0.0), as im2col's zero taps do)
      bool pad[RPT];
      uint32_t rs[RPT];
#pragma unroll
      for (int q = 0; q < RPT; ++q) {
        const int r = tid + q * NP;
        const int pix = r >> 3, wy = pix / WP, wx = pix - wy * WP;
        const int iy = tl.oy0 - 1 + wy, ix = wx - 1;
        pad[q] = static_cast<unsigned>(iy) >= static_cast<unsigned>(H) || static_cast<unsigned>(ix) >= static_cast<unsigned>(W);
        rs[q] = 0u;
      }
      for (int kb = 0; kb < n_kb; ++kb, ra.next()) {
        // one K block (4 channels) per step; an activation load covers two
        const int xh = kb & 1;
        if (xh == 0) mbar_wait(bar_xfull(rx.slot), rx.phase);
        mbar_wait(bar_aempty(ra.slot), ra.phase ^ 1);
        const uint8_t* xt = sX + static_cast<size_t>(rx.slot) * x_bytes + xh * 8;
        uint8_t* at = sA + static_cast<size_t>(ra.slot) * a_bytes;
#pragma unroll
        for (int q = 0; q < RPT; ++q) {
          const int r = tid + q * NP;
          if (r < WR) {
            const uint2 lv = *reinterpret_cast<const uint2*>(xt + static_cast<size_t>(r) * 16);
            const uint32_t lw[2] = {lv.x, lv.y};
            uint32_t w[8];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const uint32_t a = pad[q] ? static_cast<uint32_t>(p.lvl0) : ((lw[e >> 1] >> (16 * (e & 1))) & 0xFFFFu);
              const uint2 c = c64[KAN_DBG(p, 64) ? lane : a];  // (tuning only: flag 64 = conflict-free fake lookups)
              w[2 * e] = c.x;
              w[2 * e + 1] = c.y;
              if constexpr (ZP) rs[q] = __dp4a(c.y, 0x01010101u, __dp4a(c.x, 0x01010101u, rs[q]));
            }
            // row r of the SW32 K-major window: 16-byte chunk c at c ^ row bit 2
            const uint32_t sw = (static_cast<uint32_t>(r) >> 2) & 1u;
            uint8_t* d = at + static_cast<size_t>(r) * 32;
            *reinterpret_cast<uint4*>(d + (sw << 4)) = make_uint4(w[0], w[1], w[2], w[3]);
            *reinterpret_cast<uint4*>(d + ((sw ^ 1u) << 4)) = make_uint4(w[4], w[5], w[6], w[7]);
          }
        }
        fence_proxy_async_smem();  // generic-proxy writes -> visible to the tensor core
        __syncwarp();
        if (lane == 0) {
          if (xh == 1) mbar_arrive(bar_xempty(rx.slot));
          mbar_arrive(bar_afull(ra.slot));
        }
        if (xh == 1) rx.next();
      }
      if constexpr (ZP) {
        // the window rows' code sums for the epilogue's zero-point term
        const int wb = lt & 1;
        mbar_wait(bar_wsempty(wb), ((lt >> 1) & 1) ^ 1);
#pragma unroll
        for (int q = 0; q < RPT; ++q) {
          const int r = tid + q * NP;
          if (r < WR) s_wsum[wb * WR + r] = static_cast<int32_t>(rs[q]);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_wsfull(wb));
      }
    }
  } else {
    // ============ epilogue: NACC accumulators x BN columns -> NHWC rows ==========
    if (tab_bytes > 0) mbar_wait(bar_tab, 0);
    const float* thr = reinterpret_cast<const float*>(sT + p.off_thr);
    const int wq = warp & 3;             // TMEM lane quarter
    const int half = (warp - W_EPI) >> 2;  // alternate 16-column groups
    const int rloc = wq * 32 + lane;     // row within an accumulator
    const int img_l = rloc & 7, pl_ = rloc >> 3;
    const uint32_t t_row = tmem + (static_cast<uint32_t>(wq * 32) << 16);
    const int et = static_cast<int>(threadIdx.x) - 32 * W_EPI;
    int lt = 0;
    int staged_nt = -1;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++lt) {
      const Tile tl = tile_of(t);
      const int ab = lt & 1;
      if (!ZP && tl.nt != staged_nt) {  // per-column scales (restaged when the N tile changes)
        asm volatile("bar.sync 5, %0;" ::"r"(32 * GEMM_EPI_WARPS) : "memory");
        for (int i = et; i < BN; i += 32 * GEMM_EPI_WARPS) s_cols[i] = p.fs[min(tl.nt * BN + i, p.N - 1)];
        asm volatile("bar.sync 5, %0;" ::"r"(32 * GEMM_EPI_WARPS) : "memory");
        staged_nt = tl.nt;
      }
      mbar_wait(bar_accfull(ab), (lt >> 1) & 1);
      tc_fence_after();
      const int32_t* ws = s_wsum + (lt & 1) * WR;
      if constexpr (ZP) mbar_wait(bar_wsfull(lt & 1), (lt >> 1) & 1);
      const int img = tl.g * 8 + img_l;
      const bool valid = img < p.M;
      const int n0 = tl.nt * BN;
#pragma unroll 1
      for (int a = 0; a < NACC; ++a) {
        const int pix = a * 16 + pl_;
        const int py = pix / W, px = pix - py * W;
        const int oy = tl.oy0 + py;
        const size_t orow = (static_cast<size_t>(img) * H + oy) * W + px;  // NHWC row
        long long zc = 0;
        if constexpr (ZP) {
          // the row's code sum: the 9 window rows its taps read (zero-point term)
          int s_ = 0;
#pragma unroll
          for (int tap = 0; tap < 9; ++tap) s_ += ws[(((py + tap / 3) * WP + px + tap % 3) << 3) + img_l];
          zc = p.z_w * static_cast<long long>(s_);
        }
        const uint32_t tacc = t_row + static_cast<uint32_t>(ab) * 256u + static_cast<uint32_t>(a * BN);
#pragma unroll 1
        for (int cl = half * 16; cl < (KAN_DBG(p, 8) ? 0 : BN); cl += 32) {  // (tuning: flag 8 skips the epilogue)
          const bool full = n0 + cl + 16 <= p.N;
          if (p.res_kind && valid) {
            // pull the NEXT group's residual segment into L1 while this one is processed
            size_t nrow = orow;
            int ncl = cl + 32;
            if (ncl >= BN && a + 1 < NACC) {
              const int npix = (a + 1) * 16 + pl_;
              const int npy = npix / W;
              nrow = (static_cast<size_t>(img) * H + tl.oy0 + npy) * W + (npix - npy * W);
              ncl = half * 16;
            }
            if (ncl < BN && n0 + ncl < p.N)
              asm volatile("prefetch.global.L1 [%0];" ::"l"(reinterpret_cast<const float*>(p.res) + nrow * p.ld_res + n0 + ncl));
          }
          float4 rv4[4] = {};
          if (p.res_kind && valid && full) {
            const float4* rp =
                reinterpret_cast<const float4*>(reinterpret_cast<const float*>(p.res) + orow * p.ld_res + n0 + cl);
#pragma unroll
            for (int q = 0; q < 4; ++q) rv4[q] = rp[q];
          }
          uint32_t r16[16];
          tmem_ld16(tacc + cl, r16);
          tmem_wait_ld();
          if (!valid) continue;
          // y = (acc - z_w * rowsum) * f (ZP) or acc * fs[j]; + residual (fp64)
          auto yval = [&](int e) -> double {
            double y;
            if constexpr (ZP)
              y = __dmul_rn(static_cast<double>(static_cast<long long>(static_cast<int32_t>(r16[e])) - zc), p.f_tensor);
            else
              y = __dmul_rn(static_cast<double>(static_cast<int32_t>(r16[e])), s_cols[cl + e]);
            if (p.res_kind) y = __dadd_rn(y, static_cast<double>((&rv4[e >> 2].x)[e & 3]));
            return y;
          };
          if (full) {
            if (p.epi == EPI_LEVEL) {
              // branch-free level estimates 8 at a time, then the (rare) tie fix-ups
              uint32_t w[8];
#pragma unroll
              for (int hh = 0; hh < 2; ++hh)
                levels8_f64([&](int e8) { return yval(8 * hh + e8); }, p.n_lo, p.n_hi_open, p.n_step, p.n_inv_step,
                            p.n_L, w + 4 * hh);
              uint4* o = reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(p.out) + orow * p.ld_out + n0 + cl);
              o[0] = make_uint4(w[0], w[1], w[2], w[3]);
              o[1] = make_uint4(w[4], w[5], w[6], w[7]);
            } else {  // EPI_F32 row-major (+ levels sidecar)
              float f[16];
#pragma unroll
              for (int e = 0; e < 16; ++e) f[e] = __double2float_rn(yval(e));
              float4* o = reinterpret_cast<float4*>(reinterpret_cast<float*>(p.out) + orow * p.ld_out + n0 + cl);
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
                uint4* ol = reinterpret_cast<uint4*>(p.out_lv + orow * p.ld_lv + n0 + cl);
                ol[0] = make_uint4(w[0], w[1], w[2], w[3]);
                ol[1] = make_uint4(w[4], w[5], w[6], w[7]);
              }
            }
          } else {
            // ragged last column group: element-wise (the residual read here)
            for (int e = 0; e < 16; ++e) {
              const int j = n0 + cl + e;
              if (j >= p.N) break;
              double v;
              if constexpr (ZP)
                v = __dmul_rn(static_cast<double>(static_cast<long long>(static_cast<int32_t>(r16[e])) - zc), p.f_tensor);
              else
                v = __dmul_rn(static_cast<double>(static_cast<int32_t>(r16[e])), s_cols[cl + e]);
              if (p.res_kind) v = __dadd_rn(v, static_cast<double>(reinterpret_cast<const float*>(p.res)[orow * p.ld_res + j]));
              if (p.epi == EPI_LEVEL) {
                reinterpret_cast<uint16_t*>(p.out)[orow * p.ld_out + j] =
                    static_cast<uint16_t>(lattice_level_fast(v, p.n_lo, p.n_hi_open, p.n_step, p.n_inv_step, p.n_L));
              } else {
                const float f = __double2float_rn(v);
                reinterpret_cast<float*>(p.out)[orow * p.ld_out + j] = f;
                if (p.out_lv)
                  p.out_lv[orow * p.ld_lv + j] = static_cast<uint16_t>(lattice_level_tie(f, p.inv_step_f, p.lo_f, p.L, thr));
              }
            }
          }
        }
      }
      if constexpr (ZP) {
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_wsempty(lt & 1));
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_accempty(ab));
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == W_MMA) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

size_t convw_smem_bytes(int BN, int WR, int SA, int SB, int SX, int tab_bytes, bool zp) {
  const size_t b = static_cast<size_t>(9) * BN * 32;
  return 1024 + SB * b + SA * static_cast<size_t>(WR) * 32 + SX * static_cast<size_t>(WR) * 16 +
         ((static_cast<size_t>(tab_bytes) + 15) & ~static_cast<size_t>(15)) + (zp ? 2 * static_cast<size_t>(WR) * 4 : 0) +
         (2 * SA + 2 * SB + 2 * SX + 13) * 8 + static_cast<size_t>(BN) * 8 + 16;
}

cudaError_t launch_convw(int mode, const CUtensorMap& xmap, const GemmParams& p, size_t smem, cudaStream_t st) {
  static std::atomic<unsigned long long> optin[2];
  auto go = [&](auto kfn, int v) -> cudaError_t {
    if (cudaError_t e = smem_optin(kfn, optin[v]); e != cudaSuccess) return e;
    const int n_sm = device_sm_count();
    const int tiles = (p.M + 7) / 8 * (p.H / p.bh) * p.n_tiles_n;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(tiles < n_sm ? tiles : n_sm));
    cfg.blockDim = dim3(CONVW_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kfn, xmap, p);
  };
  if (mode == MODE_ZP) return go(kan_convw_kernel<MODE_ZP>, 1);
  return go(kan_convw_kernel<MODE_PLAIN>, 0);
}
