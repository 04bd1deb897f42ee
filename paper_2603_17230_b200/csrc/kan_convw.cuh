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
// Tile: G images x TR output rows x TW columns, TW = min(W, 16) and G = 128 /
// TW (8 images for maps 16 or 32 wide, 16 for 8-wide, 32 for 4-wide maps);
// NACC = TR accumulators of 128 rows (one output row of TW pixels x G images)
// x BN columns, double-buffered in TMEM (NACC * BN <= 256).  The window is
// (TR+2) rows x (TW+2) columns x G images; a one-pixel shift is G/8 core-matrix
// groups.  K: C_in / 4 blocks of 32 bytes (4
// channels x NBP = 8 basis bytes), expanded one per producer step; an
// activation load brings CX = 8 / 16 / 32 channels of every window row (16 /
// 32 / 64-byte rows, TMA swizzle none / 32B / 64B, so the producers' 8-byte
// reads stay conflict-free) and feeds CX / 4 blocks.
// MODE_ZP (the reference's per-tensor asymmetric weights): the producers sum
// each window row's codes over all channels (wsum), and the epilogue forms
// each output row's code sum from the 9 window rows it read.
//
// Warp roles as in kan_gather_gemm_kernel (12 producers here), activation TMA,
// MMA issuer, weight loader, a second MMA issuer (p.dual: the odd accumulators;
// idle otherwise), 8 epilogue warps (two per TMEM lane quarter).
// One tcgen05.commit per K block where p.lock is set: the window slot's
// barrier also releases the weight slot (the weight loader waits for the
// commit of the K block that last read its slot; weight ring <= window ring).

// Warp counts per output kind: the level epilogue (branch-free fp64 chains,
// no fp32 staging) runs on 16 warps next to 8 producers; the fp32 + sidecar
// epilogue needs more registers per thread, so it keeps 8 warps and 12
// producers (measured: 16 epilogue warps make the levels layers 5-13 % faster
// and the fp32 ones 4-14 % slower).  Window rows per producer thread (RPT)
// bound the window at CONVW_MAX_ROWS rows either way.
// MODE_SILU (per-channel weights + the SiLU base term): the producers also
// carry each window row's SiLU codes in registers (8 words per row), so those
// instantiations keep 12 producer warps x 3 rows for both output kinds.
// The stride-2 form expands a (2 TR + 1)-row window per TR output rows, so it
// is producer-heavy: 12 + 8 there too (measured: the stage-2 entry conv -14 %).
template <int OUT, bool SILU = false, int S = 1, int LG = 3>
struct ConvwWarps {
  static constexpr bool WIDE_EPI = OUT == EPI_LEVEL && !SILU && S == 1;
  static constexpr int PW = WIDE_EPI ? 8 : 12;
  static constexpr int EW = WIDE_EPI ? 16 : 8;  // a multiple of 4 (TMEM lane quarters)
  static constexpr int RPT = WIDE_EPI ? 4 : 3;
  // MODE_SILU level outputs split the register file by role (setmaxnreg works
  // on aligned groups of 4 warps: 12 producers, 4 utility warps, 8 epilogue
  // warps): the launch allocates 80 registers per thread (768 threads); the
  // 12 producer warps give back 16 each and the 8 epilogue warps run their
  // fp64 level chains at 104 without spilling (ResKAN18 per-channel + SiLU:
  // stage-1 level layers -8...-17 %, the whole forward -4.7 %).  Measured
  // neutral or slower on the other instantiations, which keep one budget.
  static constexpr bool REGSPLIT = SILU && OUT == EPI_LEVEL;
  // Utility warps: activation loader, MMA issuer, weight loader and, except in
  // the SiLU fp32-output form of 8-image tiles (C4's conv: measured 4 % faster
  // without it), a second MMA issuer (p.dual; see convw_dual_capable).
  static constexpr bool DUAL_OK = !(SILU && OUT == EPI_F32 && LG == 3);
  static constexpr int UW = DUAL_OK ? 4 : 3;
  static constexpr int THREADS = 32 * (PW + UW + EW);
  static constexpr int R_LAUNCH = 80, R_PROD = 64, R_EPI = 104;
  static_assert(!REGSPLIT || (PW * R_PROD + UW * R_LAUNCH + EW * R_EPI <= (PW + UW + EW) * R_LAUNCH &&
                              R_LAUNCH * THREADS <= 65536 && PW % 4 == 0 && EW % 4 == 0),
                "register pool");
};
constexpr int CONVW_MAX_ROWS = 1024;  // <= RPT * 32 * PW for both kinds

// S: conv stride (1, or 2 for 16-wide outputs with G = 8: consecutive output
// pixels are then every other window pixel, a core-matrix stride of 512 B).
template <int MODE, int OUT, int LG, int S>
__global__ void __launch_bounds__(ConvwWarps<OUT, MODE == MODE_SILU, S, LG>::THREADS, 1)
    kan_convw_kernel(const __grid_constant__ CUtensorMap xmap, const GemmParams p) {
  constexpr bool SILU = (MODE == MODE_SILU);
  using WarpsT = ConvwWarps<OUT, SILU, S, LG>;
  constexpr int CONVW_EPI_WARPS = WarpsT::EW;
  constexpr int NPW = WarpsT::PW, NP = 32 * NPW;
  constexpr int W_X = NPW, W_MMA = NPW + 1, W_B = NPW + 2, W_MMA2 = NPW + 3, W_EPI = NPW + WarpsT::UW;
  constexpr bool ZP = (MODE == MODE_ZP);
  const bool dual = WarpsT::DUAL_OK && p.dual != 0;  // two MMA-issuing warps
  constexpr int RPT = WarpsT::RPT;  // window rows per producer thread (max)
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);

  const int SA = p.SA, SB = p.SB, SX = p.SX;
  const int BN = p.BN;
  // input map H x W, output map Ho x Wo (= H x W at stride 1)
  const int W = p.W, H = p.H, Ho = p.Ho, Wo = p.pimg, TR = p.bh;
  constexpr int G = 1 << LG;           // images per tile (8, 16, 32)
  constexpr int TW = 128 / G;          // output columns per tile
  constexpr int WP = (TW - 1) * S + 3;  // window pitch in input pixels
  constexpr int lg = LG;
  const int CX = p.cps;                // channels per activation load
  const int KPX = CX / 4;              // K blocks per activation load
  const int WR = p.ext_rows;           // window rows = (TR + 2) * WP * G
  const int NACC = p.nacc;             // accumulators per tile
  const int n_kb = p.n_ss;             // 32-byte K blocks (4 channels each)
  // MODE_SILU: after every 8 K blocks (32 channels) one more 32-byte block of
  // those channels' SiLU codes, against the base weights (n_kb % 8 == 0)
  const int n_blk = SILU ? n_kb + (n_kb >> 3) : n_kb;
  const uint32_t a_bytes = (static_cast<uint32_t>(WR) * 32u + 1023u) & ~1023u;  // 1 KB-aligned slots
  const uint32_t x_row = static_cast<uint32_t>(CX) * 2u;      // bytes per window row of one load
  const uint32_t x_bytes = ((static_cast<uint32_t>(WR) * x_row + 1023u) & ~1023u);
  const uint32_t b_slot = static_cast<uint32_t>(p.b_slot);  // 9 taps x BN rows x 32 B
  uint8_t* sB = smem;
  uint8_t* sA = sB + static_cast<size_t>(SB) * b_slot;
  uint8_t* sX = sA + static_cast<size_t>(SA) * a_bytes;
  uint8_t* sT = sX + static_cast<size_t>(SX) * x_bytes;
  const int tab_bytes = p.tab_bytes;
  int32_t* s_wsum = reinterpret_cast<int32_t*>(sT + ((tab_bytes + 15) & ~15));  // [2][WR] (ZP)
  uint64_t* bars = reinterpret_cast<uint64_t*>(s_wsum + (ZP ? 2 * WR : 0));
  double* s_cols = reinterpret_cast<double*>(bars + 2 * SA + 2 * SB + 2 * SX + 13);  // [BN] (+ [BN] SiLU corrections)
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(s_cols + (SILU ? 2 * BN : BN));

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  pdl_trigger();

  // Work units: (block of MC image groups, band of TR output rows, TW-column
  // block, N tile), N tile fastest.  With p.mc = MC > 1 the MC CTAs of a
  // cluster take the MC image groups of a unit and share its weight slots:
  // each slot is fetched once (by one CTA, in turn) and multicast into every
  // CTA's ring, so L2 serves the weights once per cluster; a CTA whose image
  // group is past the batch only releases the unit's weight slots.
  const int MC = p.mc > 1 ? p.mc : 1;
  const uint32_t crank = MC > 1 ? cluster_rank() : 0u;
  const int unit0 = MC > 1 ? static_cast<int>(cluster_id_x()) : static_cast<int>(blockIdx.x);
  const int unit_step = MC > 1 ? static_cast<int>(n_clusters_x()) : static_cast<int>(gridDim.x);
  const uint16_t mc_mask = static_cast<uint16_t>((1u << MC) - 1u);
  const int bands = Ho / TR, cblocks = Wo / TW;
  const int n_groups = (p.M + G - 1) / G;  // p.M = images
  const int n_units = (n_groups + MC - 1) / MC * bands * cblocks * p.n_tiles_n;
  struct Tile {
    int g, oy0, x0, nt;
    bool valid;
  };
  auto tile_of = [&](int u) {
    Tile r;
    r.nt = u % p.n_tiles_n;
    int q = u / p.n_tiles_n;
    const int cb = q % cblocks;
    q /= cblocks;
    const int gb = q / bands;
    r.oy0 = (q - gb * bands) * TR;
    r.x0 = cb * TW;
    r.g = gb * MC + static_cast<int>(crank);
    r.valid = r.g < n_groups;
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
      mbar_init(bar_aempty(s), dual ? 2 : 1);  // every MMA issuer commits its share of a K block
    }
    for (int s = 0; s < SB; ++s) {
      mbar_init(bar_bfull(s), 1);
      mbar_init(bar_bempty(s), MC);  // every CTA of the cluster releases the slot
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(bar_accfull(b), dual ? 2 : 1);
      mbar_init(bar_accempty(b), CONVW_EPI_WARPS);
      mbar_init(bar_wsfull(b), NPW);
      mbar_init(bar_wsempty(b), CONVW_EPI_WARPS);
    }
    mbar_init(bar_tab, 1);
    mbar_fence_init();
  }
  if (warp == W_X && lane == 0) tma_prefetch(&xmap);
  if (warp == W_MMA) tmem_alloc(smem_u32(s_tmem), 512);
  tc_fence_before();
  __syncthreads();
  if (MC > 1) cluster_sync_all();  // peers' barriers initialised before any multicast
  tc_fence_after();
  const uint32_t tmem = *s_tmem;

  if (warp == W_X) {
    // ============ activation loader: the tile's window, CX channels per load ====
    pdl_wait();
    Ring rx(SX);
    for (int u = unit0; u < n_units; u += unit_step) {
      const Tile tl = tile_of(u);
      if (!tl.valid) continue;
      if (p.res_kind && !KAN_DBG(p, 4096)) {
        // the tile's residual rows into L2 now, so the epilogue (a whole tile
        // of MMAs later) reads them from L2 instead of HBM: one contiguous TW-
        // pixel NHWC segment per (image, output row)
        for (int i = lane; i < G * TR; i += 32) {
          const int img = tl.g * G + i % G, oy = tl.oy0 + i / G;
          if (img < p.M)
            bulk_prefetch_l2(
                reinterpret_cast<const float*>(p.res) + ((static_cast<size_t>(img) * Ho + oy) * Wo + tl.x0) * p.ld_res,
                static_cast<uint32_t>(TW * p.ld_res * 4));
        }
      }
      for (int kp = 0; kp < n_kb / KPX; ++kp, rx.next()) {
        mbar_wait(bar_xempty(rx.slot), rx.phase ^ 1);
        if (lane == 0 && KAN_DBG(p, 128)) {  // tuning only (flag 128): no activation loads (stale window)
          mbar_arrive(bar_xfull(rx.slot));
        } else if (lane == 0) {
          mbar_arrive_tx(bar_xfull(rx.slot), static_cast<uint32_t>(WR) * x_row);
          // box (CX channels, G images, WP columns, (TR-1)*S+3 rows) from
          // (c, img, x0*S-1, oy0*S-1): every input pixel the tile's taps read
          tma_load_4d(smem_u32(sX + static_cast<size_t>(rx.slot) * x_bytes), &xmap, kp * CX, tl.g * G, tl.x0 * S - 1,
                      tl.oy0 * S - 1, bar_xfull(rx.slot));
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
    uint32_t fill = 0;
    for (int u = unit0; u < n_units; u += unit_step) {
      const Tile tl = tile_of(u);
      for (int kb = 0; kb < n_blk; ++kb, rb.next(), ++fill) {
        // released by every CTA of the cluster: safe to refill everywhere.
        // One commit per K block (p.lock, SB <= SA): block g = fill - SB, the
        // last reader of this weight slot, released window slot g % SA with
        // its commit, in that barrier's phase g / SA
        if (p.lock) {
          if (fill >= static_cast<uint32_t>(SB)) {
            const uint32_t g = fill - static_cast<uint32_t>(SB);
            mbar_wait(bar_aempty(static_cast<int>(g % static_cast<uint32_t>(SA))), (g / static_cast<uint32_t>(SA)) & 1u);
          }
        } else {
          mbar_wait(bar_bempty(rb.slot), rb.phase ^ 1);
        }
        if (lane == 0) {
          const uint32_t dst = smem_u32(sB + static_cast<size_t>(rb.slot) * b_slot);
          const uint8_t* src = p.wt + (static_cast<size_t>(tl.nt) * n_blk + kb) * b_slot;
          if (KAN_DBG(p, 32)) {  // tuning only: no weight loads (stale slots)
            mbar_arrive(bar_bfull(rb.slot));
          } else {
          mbar_arrive_tx(bar_bfull(rb.slot), b_slot);
          if (MC == 1)
            bulk_load(dst, src, b_slot, bar_bfull(rb.slot));
          else if (fill % MC == crank)
            bulk_load_mc(dst, src, b_slot, bar_bfull(rb.slot), mc_mask);
          }
        }
        __syncwarp();
      }
    }
    // drain: every peer's release of our slots has landed before the CTA exits
    if (!p.lock)
      for (int s = 0; s < SB; ++s, rb.next()) mbar_wait(bar_bempty(rb.slot), rb.phase ^ 1);
  } else if (warp == W_MMA || (dual && warp == W_MMA2)) {
    // ============ MMA issuer: 9 taps x NACC accumulators per K block ============
    // p.dual (one commit per K block, no ky merge, no multicast): two issuing
    // warps, the even accumulators on one and the odd ones on the other.  A
    // single thread sustains one MMA per ~55-60 cycles and pays for the
    // commits and barrier waits of every K block (scripts/mma_commit.cu), which
    // leaves no slack against the 64 tensor cycles of an N = 128 MMA.
    const int a_first = dual && warp == W_MMA2 ? 1 : 0, a_step = dual ? 2 : 1;
    const uint32_t idesc = idesc_i8(BN, p.b_signed != 0);
    const uint32_t idesc2 = idesc_i8(2 * BN, p.b_signed != 0), idesc3 = idesc_i8(3 * BN, p.b_signed != 0);
    // Descriptor start addresses advance in 16-byte units: one window row
    // (32 B) is 2 units, and a start address below 256 KB never carries out of
    // the low word, so the issue loop moves 32-bit low words only.  Per K
    // block: NACC accumulators (runtime loop) x 9 taps (unrolled, the taps'
    // row offsets are compile-time constants).
    const uint32_t d_hi = static_cast<uint32_t>(umma_desc_sw32(0u) >> 32);
    const uint32_t acc_step = static_cast<uint32_t>(S * WP * G * 2);  // next accumulator = next band row
    const uint32_t a_hi = d_hi + static_cast<uint32_t>((S - 1) * (256 >> 4));  // A's core-matrix stride: S x 256 B
    const uint32_t b_tap = static_cast<uint32_t>(BN) * 2u;        // one tap's weight tile (BN x 32 B)
    Ring ra(SA), rb(SB);
    auto release_b = [&](uint32_t bar) {
      if (MC == 1)
        tc_commit(bar);
      else
        tc_commit_mc(bar, mc_mask);
    };
    int lt = 0;
    for (int u = unit0; u < n_units; u += unit_step) {
      if (!tile_of(u).valid) {  // no tile here: release the unit's weight slots
        for (int kb = 0; kb < n_blk; ++kb, rb.next()) {
          mbar_wait_warp(bar_bfull(rb.slot), rb.phase);
          if (elect_one()) release_b(bar_bempty(rb.slot));
          __syncwarp();
        }
        continue;
      }
      const int ab = lt & 1;
      mbar_wait_warp(bar_accempty(ab), ((lt >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t dacc = tmem + static_cast<uint32_t>(ab) * 256u;
      for (int kb = 0; kb < n_blk; ++kb, ra.next(), rb.next()) {
        mbar_wait_warp(bar_afull(ra.slot), ra.phase);
        mbar_wait_warp(bar_bfull(rb.slot), rb.phase);
        tc_fence_after();
        const uint32_t a_lo = static_cast<uint32_t>(umma_desc_sw32(smem_u32(sA + static_cast<size_t>(ra.slot) * a_bytes)));
        const uint32_t b_lo = static_cast<uint32_t>(umma_desc_sw32(smem_u32(sB + static_cast<size_t>(rb.slot) * b_slot)));
        if (elect_one()) {
          if (S == 1 && p.kym && !KAN_DBG(p, 2)) {
            // ky-merged issue (3 * BN <= 256): the tile's accumulators are
            // adjacent TMEM column blocks out[0 .. NACC-1], and the weight slot
            // holds, per kx, the taps in REVERSED ky order [B(2,kx) | B(1,kx) |
            // B(0,kx)].  Window row w feeds out[w - ky] for every valid ky, so
            // ONE MMA of N = nky * BN columns starting at out[w - ky_hi] adds
            // all of them: 3 * (NACC + 2) MMAs of up to 3 BN columns per K block
            // instead of 9 * NACC of BN columns (an N = 64 MMA costs 55 cycles,
            // N = 192 costs 96).  The accumulate flag is per MMA, so the first
            // (kb, kx) of a tile initialises each out[a] with its ky = 0 tap alone.
            for (int w = 0; w < NACC + 2; ++w) {
              const int ky_lo = max(0, w - (NACC - 1)), ky_hi = min(2, w);
              const uint32_t arow = a_lo + static_cast<uint32_t>(w) * acc_step;
#pragma unroll
              for (int kx = 0; kx < 3; ++kx) {
                const uint32_t ak = arow + static_cast<uint32_t>(kx * G * 2);
                const uint32_t bk = b_lo + static_cast<uint32_t>(kx * 3) * b_tap;
                int hi = ky_hi;
                if (kb == 0 && kx == 0) {
                  if (ky_lo == 0) {  // out[w] starts with its ky = 0 tap
                    mma_i8_lh(dacc + static_cast<uint32_t>(w * BN), ak, a_hi, bk + 2u * b_tap, d_hi, idesc, 0u);
                    if (hi == 0) continue;
                  }
                }
                const int lo = (kb == 0 && kx == 0) ? max(ky_lo, 1) : ky_lo;
                if (lo > hi) continue;
                const int nky = hi - lo + 1;
                mma_i8_lh(dacc + static_cast<uint32_t>((w - hi) * BN), ak, a_hi, bk + static_cast<uint32_t>(2 - hi) * b_tap,
                          d_hi, nky == 3 ? idesc3 : (nky == 2 ? idesc2 : idesc), 1u);
              }
            }
          } else if (!KAN_DBG(p, 2)) {  // (tuning only: flag 2 skips the MMAs)
            for (int a = a_first; a < NACC; a += a_step) {
              const uint32_t arow = a_lo + static_cast<uint32_t>(a) * acc_step;
              const uint32_t d = dacc + static_cast<uint32_t>(a * BN);
#pragma unroll
              for (int tap = 0; tap < 9; ++tap) {
                constexpr int TR9[9] = {0, 1, 2, WP, WP + 1, WP + 2, 2 * WP, 2 * WP + 1, 2 * WP + 2};
                mma_i8_lh(d, arow + static_cast<uint32_t>(TR9[tap] * G * 2), a_hi, b_lo + static_cast<uint32_t>(tap) * b_tap,
                          d_hi, idesc, (kb | tap) != 0 ? 1u : 0u);
              }
            }
          }
          if (KAN_DBG(p, 512)) {  // (tuning only: plain arrivals instead of commits, no MMAs in flight)
            mbar_arrive(bar_aempty(ra.slot));
            mbar_arrive(bar_bempty(rb.slot));
          } else {
            // one commit per K block when the rings run in lockstep (each
            // commit costs the issuing thread a few hundred cycles)
            tc_commit(bar_aempty(ra.slot));
            if (!p.lock) release_b(bar_bempty(rb.slot));
          }
        }
        __syncwarp();
      }
      if (elect_one()) tc_commit(bar_accfull(ab));
      __syncwarp();
      ++lt;
    }
  } else if (warp < NPW) {
    // ============ producers: expand the window once per K block =================
    if constexpr (WarpsT::REGSPLIT) reg_dealloc<WarpsT::R_PROD>();
    if (tab_bytes > 0) mbar_wait(bar_tab, 0);
    const uint2* c64 = reinterpret_cast<const uint2*>(sT + p.off_c64);
    const uint8_t* silu_tab = sT + p.off_silu;  // SiLU code per lattice level (MODE_SILU)
    const int tid = threadIdx.x;  // 0 .. NP-1
    Ring ra(SA), rx(SX);
    int lt = 0;
    for (int u = unit0; u < n_units; u += unit_step) {
      const Tile tl = tile_of(u);
      if (!tl.valid) continue;
      // this thread's window rows r = tid + q*NP: spatial padding flags (taps
      // outside the map read level(0.0), as im2col's zero taps do)
      bool pad[RPT];
      uint32_t rs[RPT];
      uint32_t sl[SILU ? RPT : 1][8];  // MODE_SILU: the rows' SiLU codes of the current 32 channels
#pragma unroll
      for (int q = 0; q < RPT; ++q) {
        const int r = tid + q * NP;
        const int pix = r >> lg, wy = pix / WP, wx = pix - wy * WP;
        const int iy = tl.oy0 * S - 1 + wy, ix = tl.x0 * S - 1 + wx;
        pad[q] = static_cast<unsigned>(iy) >= static_cast<unsigned>(H) || static_cast<unsigned>(ix) >= static_cast<unsigned>(W);
        rs[q] = 0u;
      }
      for (int kb = 0; kb < n_kb; ++kb, ra.next()) {
        // one K block (4 channels) per step; an activation load covers KPX
        const int xh = kb & (KPX - 1);  // KPX = 2, 4 or 8
        if (xh == 0) mbar_wait(bar_xfull(rx.slot), rx.phase);
        mbar_wait(bar_aempty(ra.slot), ra.phase ^ 1);
        const uint8_t* xt = sX + static_cast<size_t>(rx.slot) * x_bytes;
        uint8_t* at = sA + static_cast<size_t>(ra.slot) * a_bytes;
        // this block's 8 bytes of a window row: 16-byte chunk xh/2 (swizzled
        // with the row as the TMA wrote it), half xh&1
        const uint32_t chunk = static_cast<uint32_t>(xh >> 1), off8 = static_cast<uint32_t>(xh & 1) * 8u;
#pragma unroll
        for (int q = 0; q < RPT; ++q) {
          const int r = tid + q * NP;
          if (r < WR && !KAN_DBG(p, 256)) {  // (tuning only: flag 256 skips the expansion)
            const uint32_t ur = static_cast<uint32_t>(r);
            const uint32_t sw = CX == 32 ? ((ur >> 1) & 3u) : (CX == 16 ? ((ur >> 2) & 1u) : 0u);
            const uint2 lv = *reinterpret_cast<const uint2*>(xt + ur * x_row + ((chunk ^ sw) << 4) + off8);
            const uint32_t lw[2] = {lv.x, lv.y};
            uint32_t w[8];
            uint32_t sw4 = 0u;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              uint32_t a = pad[q] ? static_cast<uint32_t>(p.lvl0) : ((lw[e >> 1] >> (16 * (e & 1))) & 0xFFFFu);
              if (KAN_DBG(p, 128)) a &= 1023u;  // (tuning only: stale windows hold garbage levels)
              const uint2 c = c64[KAN_DBG(p, 64) ? lane : a];  // (tuning only: flag 64 = conflict-free fake lookups)
              w[2 * e] = c.x;
              w[2 * e + 1] = c.y;
              if constexpr (ZP) rs[q] = __dp4a(c.y, 0x01010101u, __dp4a(c.x, 0x01010101u, rs[q]));
              if constexpr (SILU) sw4 |= static_cast<uint32_t>(silu_tab[a]) << (8 * e);
            }
            if constexpr (SILU) {
              // word kb % 8 of the row's SiLU block (channels 4*(kb % 8) ...)
#pragma unroll
              for (int j = 0; j < 8; ++j)
                if ((kb & 7) == j) sl[q][j] = sw4;
            }
            // row r of the SW32 K-major window: 16-byte chunk c at c ^ row bit 2
            const uint32_t sa = (ur >> 2) & 1u;
            uint8_t* d = at + static_cast<size_t>(r) * 32;
            *reinterpret_cast<uint4*>(d + (sa << 4)) = make_uint4(w[0], w[1], w[2], w[3]);
            *reinterpret_cast<uint4*>(d + ((sa ^ 1u) << 4)) = make_uint4(w[4], w[5], w[6], w[7]);
          }
        }
        if (!KAN_DBG(p, 1024)) fence_proxy_async_smem();  // generic-proxy writes -> visible to the tensor core
        __syncwarp();
        if (lane == 0) {
          if (xh == KPX - 1) mbar_arrive(bar_xempty(rx.slot));
          mbar_arrive(bar_afull(ra.slot));
        }
        if (xh == KPX - 1) rx.next();
        if constexpr (SILU) {
          if ((kb & 7) == 7) {
            // the SiLU block of these 32 channels: one more window in the A ring
            ra.next();
            mbar_wait(bar_aempty(ra.slot), ra.phase ^ 1);
            uint8_t* as = sA + static_cast<size_t>(ra.slot) * a_bytes;
#pragma unroll
            for (int q = 0; q < RPT; ++q) {
              const int r = tid + q * NP;
              if (r < WR) {
                const uint32_t sa = (static_cast<uint32_t>(r) >> 2) & 1u;
                uint8_t* d = as + static_cast<size_t>(r) * 32;
                *reinterpret_cast<uint4*>(d + (sa << 4)) = make_uint4(sl[q][0], sl[q][1], sl[q][2], sl[q][3]);
                *reinterpret_cast<uint4*>(d + ((sa ^ 1u) << 4)) = make_uint4(sl[q][4], sl[q][5], sl[q][6], sl[q][7]);
              }
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(bar_afull(ra.slot));
          }
        }
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
      ++lt;
    }
  } else if (warp >= W_EPI) {
    // ============ epilogue: NACC accumulators x BN columns -> NHWC rows ==========
    if constexpr (WarpsT::REGSPLIT) reg_alloc<WarpsT::R_EPI>();
    if (tab_bytes > 0) mbar_wait(bar_tab, 0);
    const float* thr = reinterpret_cast<const float*>(sT + p.off_thr);
    const int wq = warp & 3;             // TMEM lane quarter
    constexpr int EQ = CONVW_EPI_WARPS / 4;  // warps per TMEM lane quarter
    const int half = (warp - W_EPI) >> 2;  // this warp's 16-column groups: half, half + EQ, ...
    const int rloc = wq * 32 + lane;     // row within an accumulator
    const int img_l = rloc & (G - 1), pl_ = rloc >> lg;
    const uint32_t t_row = tmem + (static_cast<uint32_t>(wq * 32) << 16);
    const int et = static_cast<int>(threadIdx.x) - 32 * W_EPI;
    int lt = 0;
    int staged_nt = -1;
    for (int u = unit0; u < n_units; u += unit_step) {
      const Tile tl = tile_of(u);
      if (!tl.valid) continue;
      const int ab = lt & 1;
      if (!ZP && tl.nt != staged_nt) {  // per-column scales (restaged when the N tile changes)
        asm volatile("bar.sync 5, %0;" ::"r"(32 * CONVW_EPI_WARPS) : "memory");
        for (int i = et; i < BN; i += 32 * CONVW_EPI_WARPS) {
          const int j = min(tl.nt * BN + i, p.N - 1);
          s_cols[i] = p.fs[j];
          if constexpr (SILU) s_cols[BN + i] = static_cast<double>(p.corr_b[j]);
        }
        asm volatile("bar.sync 5, %0;" ::"r"(32 * CONVW_EPI_WARPS) : "memory");
        staged_nt = tl.nt;
      }
      mbar_wait(bar_accfull(ab), (lt >> 1) & 1);
      tc_fence_after();
      const int32_t* ws = s_wsum + (lt & 1) * WR;
      if constexpr (ZP) mbar_wait(bar_wsfull(lt & 1), (lt >> 1) & 1);
      const int img = tl.g * G + img_l;
      const bool valid = img < p.M;
      const int n0 = tl.nt * BN;
#pragma unroll 1
      for (int a = 0; a < NACC; ++a) {
        const int py = a, px = pl_;  // accumulator a = band row a; its rows = TW pixels x G images
        const int oy = tl.oy0 + py;
        const size_t orow = (static_cast<size_t>(img) * Ho + oy) * Wo + tl.x0 + px;  // NHWC row
        double zc = 0.0;
        if constexpr (ZP) {
          // the row's code sum: the 9 window rows its taps read (zero-point term)
          int s_ = 0;
#pragma unroll
          for (int tap = 0; tap < 9; ++tap) s_ += ws[(((S * py + tap / 3) * WP + S * px + tap % 3) << lg) + img_l];
          zc = static_cast<double>(p.z_w * static_cast<long long>(s_));  // exact below 2^53
        }
        const uint32_t tacc = t_row + static_cast<uint32_t>(ab) * 256u + static_cast<uint32_t>(a * BN);
#pragma unroll 1
        for (int cl = half * 16; cl < (KAN_DBG(p, 8) ? 0 : BN); cl += 16 * EQ) {  // (tuning: flag 8 skips the epilogue)
          const bool full = n0 + cl + 16 <= p.N;
          if (p.res_kind && valid && !KAN_DBG(p, 4096)) {  // (tuning only: flag 4096 drops the residual reads)
            // pull the NEXT group's residual segment into L1 while this one is processed
            size_t nrow = orow;
            int ncl = cl + 16 * EQ;
            if (ncl >= BN && a + 1 < NACC) {
              nrow = orow + static_cast<size_t>(Wo);  // the next band row, same pixel
              ncl = half * 16;
            }
            if (ncl < BN && n0 + ncl < p.N)
              asm volatile("prefetch.global.L1 [%0];" ::"l"(reinterpret_cast<const float*>(p.res) + nrow * p.ld_res + n0 + ncl));
          }
          float4 rv4[4] = {};
          if (p.res_kind && valid && full && !KAN_DBG(p, 4096)) {
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
          // (acc - z_w * rowsum) is exact in fp64, so converting first changes nothing
          auto yval = [&](int e) -> double {
            double y;
            if constexpr (ZP)
              y = __dmul_rn(__dsub_rn(i32_to_f64(r16[e]), zc), p.f_tensor);
            else if constexpr (SILU)  // minus z_s * colsum(base weight codes)
              y = __dmul_rn(__dsub_rn(i32_to_f64(r16[e]), s_cols[BN + cl + e]), s_cols[cl + e]);
            else
              y = __dmul_rn(i32_to_f64(r16[e]), s_cols[cl + e]);
            if (p.res_kind) y = __dadd_rn(y, static_cast<double>((&rv4[e >> 2].x)[e & 3]));
            return y;
          };
          if (full) {
            if constexpr (OUT == EPI_LEVEL) {
              // branch-free level estimates 8 at a time, then the (rare) tie fix-ups
              uint32_t w[8];
#pragma unroll
              for (int hh = 0; hh < 2; ++hh)
                levels8_f64([&](int e8) { return yval(8 * hh + e8); }, p.n_lo, p.n_hi_open, p.n_step, p.n_inv_step,
                            p.n_L, w + 4 * hh);
              uint4* o = reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(p.out) + orow * p.ld_out + n0 + cl);
              o[0] = make_uint4(w[0], w[1], w[2], w[3]);
              o[1] = make_uint4(w[4], w[5], w[6], w[7]);
            } else if (p.out_hw > 0) {  // EPI_F32, NCHW (a model output): lanes = 4 pixels x 8 images
              float* o = reinterpret_cast<float*>(p.out) +
                         (static_cast<size_t>(img) * p.N + n0 + cl) * p.out_hw + static_cast<size_t>(oy) * Wo + tl.x0 + px;
#pragma unroll
              for (int e = 0; e < 16; ++e) o[static_cast<size_t>(e) * p.out_hw] = __double2float_rn(yval(e));
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
                v = __dmul_rn(__dsub_rn(i32_to_f64(r16[e]), zc), p.f_tensor);
              else if constexpr (SILU)
                v = __dmul_rn(__dsub_rn(i32_to_f64(r16[e]), s_cols[BN + cl + e]), s_cols[cl + e]);
              else
                v = __dmul_rn(i32_to_f64(r16[e]), s_cols[cl + e]);
              if (p.res_kind) v = __dadd_rn(v, static_cast<double>(reinterpret_cast<const float*>(p.res)[orow * p.ld_res + j]));
              if constexpr (OUT == EPI_LEVEL) {
                reinterpret_cast<uint16_t*>(p.out)[orow * p.ld_out + j] =
                    static_cast<uint16_t>(lattice_level_fast(v, p.n_lo, p.n_hi_open, p.n_step, p.n_inv_step, p.n_L));
              } else {
                const float f = __double2float_rn(v);
                if (p.out_hw > 0) {
                  reinterpret_cast<float*>(p.out)[(static_cast<size_t>(img) * p.N + j) * p.out_hw +
                                                  static_cast<size_t>(oy) * Wo + tl.x0 + px] = f;
                  continue;
                }
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
      ++lt;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (MC > 1) cluster_sync_all();  // no multicast into / release of an exited CTA
  if (warp == W_MMA) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

int convw_max_rows() { return CONVW_MAX_ROWS; }

// whether the instantiation that launch_convw picks has the second MMA-issuing warp
bool convw_dual_capable(int mode, int epi, int g_img) { return !(mode == MODE_SILU && epi == EPI_F32 && g_img == 8); }

size_t convw_smem_bytes(int BN, int WR, int CX, int SA, int SB, int SX, int tab_bytes, bool zp, bool silu) {
  const size_t b = static_cast<size_t>(9) * BN * 32;
  const size_t x = (static_cast<size_t>(WR) * CX * 2 + 1023) / 1024 * 1024;
  return 1024 + SB * b + SA * ((static_cast<size_t>(WR) * 32 + 1023) / 1024 * 1024) + SX * x +
         ((static_cast<size_t>(tab_bytes) + 15) & ~static_cast<size_t>(15)) + (zp ? 2 * static_cast<size_t>(WR) * 4 : 0) +
         (2 * SA + 2 * SB + 2 * SX + 13) * 8 + static_cast<size_t>(BN) * (silu ? 16 : 8) + 16;
}

cudaError_t launch_convw(int mode, const CUtensorMap& xmap, const GemmParams& p, size_t smem, cudaStream_t st) {
  static std::atomic<unsigned long long> optin[24];
  auto go = [&](auto kfn, int v, int threads) -> cudaError_t {
    if (cudaError_t e = smem_optin(kfn, optin[v]); e != cudaSuccess) return e;
    const int n_sm = device_sm_count();
    const int mc = p.mc > 1 ? p.mc : 1;
    const int units = ((p.M + p.bn_img - 1) / p.bn_img + mc - 1) / mc * (p.Ho / p.bh) * (p.pimg / p.Wo) * p.n_tiles_n;
    const int clusters = units < n_sm / mc ? units : n_sm / mc;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(clusters * mc));
    cfg.blockDim = dim3(static_cast<unsigned>(threads));
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
    cfg.numAttrs = mc > 1 ? 2 : 1;  // a cluster launch only when the weights are multicast
    return cudaLaunchKernelEx(&cfg, kfn, xmap, p);
  };
  const bool lvl = p.epi == EPI_LEVEL;
  auto pick = [&](auto lgc, auto sc) -> cudaError_t {
    constexpr int LG = decltype(lgc)::value, S = decltype(sc)::value;
    const int v = 4 * (LG - 3) + (S == 2 ? 12 : 0);
    constexpr int TL = ConvwWarps<EPI_LEVEL, false, S, LG>::THREADS, TF = ConvwWarps<EPI_F32, false, S, LG>::THREADS;
    constexpr int TS = ConvwWarps<EPI_F32, true, S, LG>::THREADS, TSL = ConvwWarps<EPI_LEVEL, true, S, LG>::THREADS;
    if (mode == MODE_SILU)
      return lvl ? go(kan_convw_kernel<MODE_SILU, EPI_LEVEL, LG, S>, 16 + v / 2 + 1, TSL)
                 : go(kan_convw_kernel<MODE_SILU, EPI_F32, LG, S>, 16 + v / 2, TS);
    if (mode == MODE_ZP)
      return lvl ? go(kan_convw_kernel<MODE_ZP, EPI_LEVEL, LG, S>, v + 3, TL)
                 : go(kan_convw_kernel<MODE_ZP, EPI_F32, LG, S>, v + 2, TF);
    return lvl ? go(kan_convw_kernel<MODE_PLAIN, EPI_LEVEL, LG, S>, v + 1, TL)
               : go(kan_convw_kernel<MODE_PLAIN, EPI_F32, LG, S>, v, TF);
  };
  using I3 = std::integral_constant<int, 3>;
  using S1 = std::integral_constant<int, 1>;
  if (p.cstride == 2) return pick(I3{}, std::integral_constant<int, 2>{});  // 16-wide outputs, 8 images
  if (p.bn_img == 8) return pick(I3{}, S1{});
  if (p.bn_img == 16) return pick(std::integral_constant<int, 4>{}, S1{});
  return pick(std::integral_constant<int, 5>{}, S1{});
}
