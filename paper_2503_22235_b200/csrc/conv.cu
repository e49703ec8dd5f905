// K6/K7: implicit-GEMM convolutions of the encoder/decoder pyramids on tcgen05.
//
// Reference geometry (model.py:296-325, autodiff.py:585-764): 3x3 convs with rows zero-padded by 1 and
// columns periodic (centred taps), stride 1 or 2; 4x4 stride-2 transposed convs, the exact adjoint (rows
// padded (1,1), columns wrapped with c = 1).  All depth planes share the pyramid weights, so the planes are
// batched as images of one launch.
//
// Activation layout: bf16 NHWC with a 1-pixel halo, [img][H + 2][W + 2][Cp]: halo rows are zero (row pad),
// halo columns hold the opposite edge (longitude wrap), Cp = channels rounded up to 64.  Every tap of every
// conv is then a plain rectangular TMA box:
//   3x3 s1      out (r, c) tap (kh, kw) reads padded (r + kh, c + kw)               3D box {64, 128, 1}
//   3x3 s2      reads padded (2r + kh, 2c + kw): columns viewed as (pair, parity)    4D box {64, 1, 128, 1}
//   convT s2    output parity class (a, b), taps (tr, tc) in {0,1}^2: out (2r + a, 2c + b) reads padded
//               (r + a + tr, c + b + tc) with kernel tap (3 - a - 2 tr, 3 - b - 2 tc)
// GEMM view: M = output pixels of one row (128-pixel tiles), N = Cout, K = taps x Cp (weights pre-arranged
// [class][Cout_pad][tap][Cp], K-major).  Warp roles as in gemm.cu; the epilogue (one pixel per thread) applies
// bias, optional GELU and the optional residual (res-block skip) and writes the next padded NHWC activation
// through a per-warp shared-memory tile — residual chunk in and output chunk out by TMA (32 pixels x 32
// channels, 64-byte swizzle; the two wrap-column copies per row by their owning threads) — or, straight from
// registers, fp32 tokens or fp32 NCHW fields.
#include "common.cuh"
#include "launch.h"
#include "../../include/wm3.h"

namespace wm3 {

constexpr int CV_BM = 128;
constexpr int CV_BK = 64;
constexpr int CV_THREADS = 384;

struct ConvParams {
  int mode;            // WM3_CONV_S1 / S2 / T2
  int imgs;
  int hin, win, cinp;  // input extents (unpadded) and padded channel count
  int hout, wout;      // output extents
  int rows_t, cols_t;  // GEMM output sub-grid per class: rows x cols (cols tiled by 128)
  int nclass, ntap, ncb;
  int cout, cout_pad;  // real output channels, per-class padded N
  int tiles_per_row, tiles_per_class;
  int tile_rows, tile_cols;  // a 128-pixel tile = tile_rows output rows x tile_cols columns (1 x 128 or 2 x 64)
  // epilogue
  const float* bias;
  int act_gelu;
  const elem_t* resid;  // padded NHWC with the output's spatial extents, or null
  int resid_cp;
  int out_kind;
  void* out;
  int out_cp;                  // NHWC: padded channel pitch of the output
  long long img_stride;        // FIELD: elements between images;   TOKENS: unused
  long long a_stride, p_stride;  // FIELD: channel c -> (c / chan_div) * a_stride + (c % chan_div) * p_stride
  int chan_div;
  int tma_out;  // NHWC output: TMA-staged epilogue stores (tmO), residual chunks via tmR
};

// CG = 2: CTA pairs (cluster of 2 on a TPC, tcgen05.mma.cta_group::2, M = 256): each CTA stages its own 128
// output pixels and half of the BN weight rows, the leader issues the pair's MMAs, so per-SM operand traffic
// from L2 drops from (16 KB A + BN x 128 B) to (16 KB A + BN x 64 B) per 64-deep k-block and the freed shared
// memory deepens the ring.  (The Cout = 192 convs at 720 x 1440 were bound by that L2 -> SM operand stream.)
// STRIP (stride-1 convs): a stage holds one strip of 130 input pixels of a kernel row (kh, channel block) and
// the three column taps' weight boxes; the MMAs of tap kw read the strip from row kw (descriptor start + kw x
// 128 B), so the A operand crosses L2 -> SM once per kernel row instead of once per tap.
constexpr int CV_STRIP_ROWS = CV_BM + 2;
#ifndef WM3_CONV_TMA_EPI
#define WM3_CONV_TMA_EPI 1
#endif
#if !defined(WM3_OPERAND_BF16) && WM3_GELU_VARIANT == 2
#define CONV_GELU_H2 true
#else
#define CONV_GELU_H2 false
#endif
template <int BN, int CG = 1, bool STRIP = false>
struct ConvCfg {
  static constexpr int TAPS = STRIP ? 3 : 1;  // weight boxes per stage
  static constexpr uint32_t A_BYTES = STRIP ? 17408u : CV_BM * CV_BK * 2;  // 130 rows x 128 B, 1 KB aligned
  static constexpr uint32_t B1_BYTES = (BN / CG) * CV_BK * 2;
  static constexpr uint32_t B_BYTES = TAPS * B1_BYTES;
  static constexpr uint32_t A_TX = STRIP ? CV_STRIP_ROWS * 128u : A_BYTES;  // bytes TMA writes
  static constexpr int STAGES_FIT = static_cast<int>((224u * 1024u - 1280u) / (A_BYTES + B_BYTES));
  static constexpr int STAGES_NT = (CG == 1 && !STRIP) ? ((BN == 256) ? 4 : (BN == 64 ? 8 : 5))
                                                       : (STAGES_FIT < 8 ? STAGES_FIT : 8);
  // TMA-staged epilogue: each epilogue warp owns a 2 KB staging tile (32 pixels x 32 channels, 64-byte swizzle)
  // that takes its residual chunk by TMA and sends its output chunk back by TMA, instead of per-thread 16-byte
  // global accesses one pixel (384-512 B) apart; WM3_CONV_TMA_EPI=2 keeps it only where no ring stage is lost
  static constexpr uint32_t EPI_STAGING = 8u * 2048u;
  static constexpr int FIT_T = static_cast<int>((224u * 1024u - 1280u - EPI_STAGING) / (A_BYTES + B_BYTES));
  static constexpr bool TMA_EPI = (WM3_CONV_TMA_EPI == 1 && FIT_T >= 3) || (WM3_CONV_TMA_EPI == 2 && FIT_T >= STAGES_NT);
  static constexpr int STAGES = TMA_EPI ? (FIT_T < STAGES_NT ? FIT_T : STAGES_NT) : STAGES_NT;
  static constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr uint32_t TX_BYTES = A_TX + B_BYTES;
  static constexpr uint32_t SMEM = STAGES * STAGE_BYTES + (TMA_EPI ? EPI_STAGING : 0u) + 1024 + 256;
  static constexpr uint32_t TMEM_COLS = (2 * BN <= 256) ? 256 : 512;
};

// m-tile -> image, class, output sub-grid row, first column.  With CTA pairs an m-tile is a pair of
// consecutive 128-pixel tiles of one (image, class) (the two halves of an M = 256 MMA share the class's
// weights, not their pixels); rank r takes the r-th; a missing second tile (odd count) is a dummy (`valid`
// false: its loads stay in bounds and nothing is stored).
template <int CG>
DEVI void conv_tile(const ConvParams& p, int mt, int rank, int& img, int& cls, int& r, int& c0, bool& valid) {
  const int per_class = (p.tiles_per_class + CG - 1) / CG;
  const int per_img = p.nclass * per_class;
  img = mt / per_img;
  int rest = mt - img * per_img;
  cls = rest / per_class;
  int t = (rest - cls * per_class) * CG + rank;
  valid = t < p.tiles_per_class;
  if (!valid) t = p.tiles_per_class - 1;
  const int tr = t / p.tiles_per_row;
  r = tr * p.tile_rows;
  c0 = (t - tr * p.tiles_per_row) * p.tile_cols;
}

template <int BN, int CG, bool STRIP>
__global__ void __launch_bounds__(CV_THREADS, 1)
    conv_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmO, const __grid_constant__ CUtensorMap tmR, ConvParams p) {
  griddep_launch_dependents();  // PDL: the next kernel may start its prologue
  using Cfg = ConvCfg<BN, CG, STRIP>;
  constexpr int STAGES = Cfg::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = smem_u32(smem);
  const uint32_t staging0 = sbase + STAGES * Cfg::STAGE_BYTES;  // TMA_EPI: 8 x 2 KB, one per epilogue warp
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::STAGE_BYTES + (Cfg::TMA_EPI ? Cfg::EPI_STAGING : 0u));
  const uint32_t bar0 = smem_u32(bars);
  auto full_bar = [&](int s) { return bar0 + 8u * s; };
  auto empty_bar = [&](int s) { return bar0 + 8u * (STAGES + s); };
  auto tfull_bar = [&](int a) { return bar0 + 8u * (2 * STAGES + a); };
  auto tempty_bar = [&](int a) { return bar0 + 8u * (2 * STAGES + 2 + a); };
  auto res_bar = [&](int w) { return bar0 + 8u * (2 * STAGES + 4 + w); };  // TMA_EPI: residual chunk landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 4 + 8);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int nn = p.cout_pad / BN;
  const int ntiles = p.imgs * p.nclass * ((p.tiles_per_class + CG - 1) / CG) * nn;
  // strip stages: one per (kernel row, channel block); a stride-1 strip serves 3 column taps, a transposed
  // conv's (parity class) strip its 2
  const int strip_taps = (p.mode == WM3_CONV_T2) ? 2 : 3;
  const int nk = (STRIP ? (p.mode == WM3_CONV_T2 ? 2 : 3) : p.ntap) * p.ncb;  // stages per tile
  // CTA pairs: cluster = (2k, 2k + 1) walks the pair tiles together
  const int rank = (CG == 2) ? static_cast<int>(cluster_ctarank()) : 0;
  const int tile0 = (CG == 2) ? static_cast<int>(blockIdx.x >> 1) : static_cast<int>(blockIdx.x);
  const int tstep = (CG == 2) ? static_cast<int>(gridDim.x >> 1) : static_cast<int>(gridDim.x);

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    if (Cfg::TMA_EPI && p.tma_out) {
      tma_prefetch(&tmO);
      if (p.resid != nullptr) tma_prefetch(&tmR);
    }
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(empty_bar(s), 1);
    }
    for (int w = 0; w < 8; ++w) mbar_init(res_bar(w), 1);
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull_bar(a), 1);
      mbar_init(tempty_bar(a), 8 * CG);  // every epilogue warp of the pair arrives on the leader's barrier
    }
    fence_barrier_init();
  }
  if (warp == 2) {
    if (CG == 2) {
      tmem_alloc_cg2(smem_u32(tmem_slot), Cfg::TMEM_COLS);
      tmem_relinquish_cg2();
    } else {
      tmem_alloc(smem_u32(tmem_slot), Cfg::TMEM_COLS);
      tmem_relinquish();
    }
  }
  tc_fence_before();
  if (CG == 2)
    cluster_sync();  // both CTAs' barriers exist before any cross-CTA arrive / TMA completion
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  griddep_wait();  // PDL: inputs are complete from here on

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      const int hp = p.hin + 2;
      for (int tile = tile0; tile < ntiles; tile += tstep) {
        int img, cls, r, c0;
        bool valid;
        conv_tile<CG>(p, tile / nn, rank, img, cls, r, c0, valid);
        const int n0 = (tile % nn) * BN + rank * (BN / CG);
        const int a = cls >> 1, b = cls & 1;
        for (int kb = 0; kb < nk; ++kb) {
          const int tap = kb / p.ncb, cb = kb - tap * p.ncb;  // STRIP: `tap` is the kernel row kh
          mbar_wait(empty_bar(stage), phase ^ 1);
          const uint32_t sa = sbase + stage * Cfg::STAGE_BYTES;
          const uint32_t sb = sa + Cfg::A_BYTES;
          // pairs: both CTAs' bytes complete on the leader's full barrier; only the leader arms it
          const uint32_t fb = (CG == 2) ? mapa_shared(full_bar(stage), 0) : full_bar(stage);
          if (rank == 0)
            mbar_arrive_expect_tx(full_bar(stage),
                                  CG * (STRIP ? Cfg::A_TX + strip_taps * Cfg::B1_BYTES : Cfg::TX_BYTES));
          if (STRIP) {
            // stride 1: strip of padded columns [c0, c0 + 130) of input row r + kh, weights of taps (kh, 0..2);
            // transposed (class (a, b)): strip of columns [c0 + b, +130) of input row r + a + tr, weights of
            // taps (tr, 0..1) — its two column taps read input columns one apart
            const bool t2 = p.mode == WM3_CONV_T2;
            const int scol = t2 ? c0 + b : c0, srow = img * hp + r + (t2 ? a : 0) + tap;
            if (CG == 2) tma_load_3d_cg2(sa, &tmA, fb, cb * CV_BK, scol, srow);
            else tma_load_3d(sa, &tmA, fb, cb * CV_BK, scol, srow);
#pragma unroll
            for (int kw = 0; kw < 3; ++kw) {
              if (kw >= strip_taps) break;
              const int kcol = ((strip_taps * tap + kw) * p.ncb + cb) * CV_BK;
              if (CG == 2) tma_load_2d_cg2(sb + kw * Cfg::B1_BYTES, &tmB, fb, kcol, cls * p.cout_pad + n0);
              else tma_load_2d(sb + kw * Cfg::B1_BYTES, &tmB, fb, kcol, cls * p.cout_pad + n0);
            }
          } else if (p.mode == WM3_CONV_S2) {
            const int kh = tap / 3, kw = tap - 3 * (tap / 3);
            if (CG == 2) tma_load_4d_cg2(sa, &tmA, fb, cb * CV_BK, kw & 1, c0 + (kw >> 1), img * hp + 2 * r + kh);
            else tma_load_4d(sa, &tmA, fb, cb * CV_BK, kw & 1, c0 + (kw >> 1), img * hp + 2 * r + kh);
          } else if (p.mode == WM3_CONV_S1) {
            const int kh = tap / 3, kw = tap - 3 * (tap / 3);
            if (CG == 2) tma_load_3d_cg2(sa, &tmA, fb, cb * CV_BK, c0 + kw, img * hp + r + kh);
            else tma_load_3d(sa, &tmA, fb, cb * CV_BK, c0 + kw, img * hp + r + kh);
          } else {  // transposed, parity class (a, b), tap (tr, tc)
            const int tr = tap >> 1, tc = tap & 1;
            if (CG == 2) tma_load_3d_cg2(sa, &tmA, fb, cb * CV_BK, c0 + b + tc, img * hp + r + a + tr);
            else tma_load_3d(sa, &tmA, fb, cb * CV_BK, c0 + b + tc, img * hp + r + a + tr);
          }
          if (!STRIP) {
            if (CG == 2) tma_load_2d_cg2(sb, &tmB, fb, kb * CV_BK, cls * p.cout_pad + n0);
            else tma_load_2d(sb, &tmB, fb, kb * CV_BK, cls * p.cout_pad + n0);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // The whole warp walks the k-blocks (warp-wide waits, warp-uniform descriptors in uniform registers);
    // one elected lane issues the MMAs and commits.  Pairs: the leader issues M = 256 MMAs for both CTAs and
    // its commits arrive on both CTAs' barriers.
    if (rank == 0) {
      constexpr uint32_t idesc = make_idesc(CV_BM * CG, BN, 0, 0);
      const uint64_t d0 = make_sdesc_sw128(sbase, 16, 1024);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t aphase = 0;
      for (int tile = tile0; tile < ntiles; tile += tstep) {
        mbar_wait(tempty_bar(acc), aphase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(full_bar(stage), phase);
          tc_fence_after();
          const uint64_t da = d0 + ((stage * Cfg::STAGE_BYTES) >> 4), db = da + (Cfg::A_BYTES >> 4);
          if (elect_one()) {
#pragma unroll
            for (int kw = 0; kw < Cfg::TAPS; ++kw) {
              if (STRIP && kw >= strip_taps) break;
              // tap kw reads strip rows [kw, kw + 128): start address + kw x 128 B.  The MMA unit swizzles on
              // the absolute shared-memory address (as TMA wrote it), so the descriptor's base-offset field
              // stays 0 (setting it to kw broke parity, measured).
              const uint64_t dak = da + 8u * kw;
              const uint64_t dbk = db + kw * (Cfg::B1_BYTES >> 4);
#pragma unroll
              for (int k = 0; k < CV_BK / 16; ++k) {
                const uint32_t acc_on = (kb | kw | k) != 0 ? 1u : 0u;
                if (CG == 2) umma_ss_cg2(d_tmem, dak + 2 * k, dbk + 2 * k, idesc, acc_on);
                else umma_bf16_ss(d_tmem, dak + 2 * k, dbk + 2 * k, idesc, acc_on);
              }
            }
            if (CG == 2) umma_commit_mc(empty_bar(stage), 0x3);  // frees the stage in both CTAs
            else umma_commit(empty_bar(stage));
          }
          __syncwarp();
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        if (elect_one()) {
          if (CG == 2) umma_commit_mc(tfull_bar(acc), 0x3);
          else umma_commit(tfull_bar(acc));
        }
        __syncwarp();
        acc ^= 1;
        if (acc == 0) aphase ^= 1;
      }
    }
  } else if (warp >= 4) {
    const int g = (warp - 4) >> 2;
    const int q = warp & 3;
    const int i = 32 * q + lane;  // pixel within the tile
    int acc = 0;
    uint32_t aphase = 0;
    const uint32_t tempty_leader0 = (CG == 2) ? mapa_shared(tempty_bar(0), 0) : 0u;
    const uint32_t stg = staging0 + (warp - 4) * 2048u;  // TMA_EPI: this warp's 32 x 32 staging tile
    const uint32_t rbar = res_bar(warp - 4);
    uint32_t rph = 0;
    // 64-byte swizzle of the staging tile (rows = pixels, 4 x 16-byte chunks of 8 channels)
    const uint32_t srow = stg + 64u * lane, sxor = (lane >> 1) & 3;
    for (int tile = tile0; tile < ntiles; tile += tstep) {
      int img, cls, r, c0;
      bool valid;
      conv_tile<CG>(p, tile / nn, rank, img, cls, r, c0, valid);
      const int n0 = (tile % nn) * BN;
      // this thread's pixel of the tile (tile_rows x tile_cols) and the first pixel of this warp's 32
      const int di = i / p.tile_cols, row = r + di, col = c0 + i - di * p.tile_cols;
      const int dw = (32 * q) / p.tile_cols, roww = r + dw, colw = c0 + 32 * q - dw * p.tile_cols;
      const bool ok = valid && col < p.cols_t && row < p.rows_t;
      // output pixel
      int orow = row, ocol = col;
      if (p.mode == WM3_CONV_T2) { orow = 2 * row + (cls >> 1); ocol = 2 * col + (cls & 1); }
      const bool tma_tile = Cfg::TMA_EPI && p.tma_out && valid;  // uniform over the CTA
      if (p.resid != nullptr && ok && !tma_tile) {
        // pull this pixel's residual channels toward L2 while the accumulator is still being computed
        const size_t rpix = (static_cast<size_t>(img) * (p.hout + 2) + orow + 1) * (p.wout + 2) + ocol + 1;
        const char* rb = reinterpret_cast<const char*>(p.resid + rpix * p.resid_cp + n0);
        for (int off = 64 * g; off < BN * 2; off += 128)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(rb + off));
      }
      mbar_wait(tfull_bar(acc), aphase);
      tc_fence_after();
      const uint32_t taddr = tmem_base + acc * BN + (static_cast<uint32_t>(32 * q) << 16);
      for (int u = g; u < BN / 32; u += 2) {
        const int n = n0 + 32 * u;
        const bool tma = tma_tile && n < p.cout;  // uniform over the warp
        if (tma && p.resid != nullptr && lane == 0) {
          // this warp's residual chunk (its 32 pixels x 32 channels) into its staging tile, under the TMEM load
          bulk_wait_read<0>();  // the previous output chunk has left the staging tile
          mbar_arrive_expect_tx(rbar, 2048u);
          tma_load_4d(stg, &tmR, rbar, n, colw + 1, roww + 1, img);  // (residual convs are stride 1)
        }
        uint32_t rr[32];
        tmem_ld32(taddr + 32 * u, rr);
        tmem_ld_wait();
        if (!tma && (!ok || n >= p.cout)) continue;
        const int nvalid = min(32, p.cout - n);
        float v[32];
        if (nvalid == 32 && (p.cout & 3) == 0) {  // bias as 8 16-byte loads (the same 128 B for every lane)
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float4 b = __ldg(reinterpret_cast<const float4*>(p.bias + n) + j);
            v[4 * j + 0] = __uint_as_float(rr[4 * j + 0]) + b.x;
            v[4 * j + 1] = __uint_as_float(rr[4 * j + 1]) + b.y;
            v[4 * j + 2] = __uint_as_float(rr[4 * j + 2]) + b.z;
            v[4 * j + 3] = __uint_as_float(rr[4 * j + 3]) + b.w;
          }
        } else {
#pragma unroll
          for (int e = 0; e < 32; ++e) v[e] = __uint_as_float(rr[e]) + (e < nvalid ? __ldg(p.bias + n + e) : 0.f);
        }
        // GELU (res-block conv1, NHWC 16-bit out): packed f16x2 straight to the output pairs, as the W1 GEMM
        // epilogue (gemm.cu); the fp32 form for the other outputs
        uint32_t gpk[16];
        const bool gelu_h2 = p.act_gelu && p.out_kind == WM3_CONV_OUT_NHWC && p.resid == nullptr && CONV_GELU_H2;
        if (gelu_h2) {
#pragma unroll
          for (int e = 0; e < 16; ++e) gpk[e] = gelu_tanh_h2(v[2 * e], v[2 * e + 1]);
        } else if (p.act_gelu) {
#pragma unroll
          for (int e = 0; e < 32; ++e) v[e] = gelu_epi(v[e]);
        }
        const size_t pix = (static_cast<size_t>(img) * (p.hout + 2) + orow + 1) * (p.wout + 2) + ocol + 1;
        if (tma) {
          // residual from the staging tile (the TMA landed it), output back into it, one TMA store per warp;
          // pixels past the row end are clipped by the output map (its column extent stops at the last pixel)
          if (p.resid != nullptr) {
            mbar_wait(rbar, rph & 1);
            ++rph;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              uint32_t w0, w1, w2, w3;
              asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                           : "=r"(w0), "=r"(w1), "=r"(w2), "=r"(w3) : "r"(srow + ((j ^ sxor) << 4)));
              const uint32_t ws[4] = {w0, w1, w2, w3};
#pragma unroll
              for (int t = 0; t < 4; ++t) {
                const float2 h2 = unpack_elem2(ws[t]);
                v[8 * j + 2 * t] += h2.x;
                v[8 * j + 2 * t + 1] += h2.y;
              }
            }
          } else {
            if (lane == 0) bulk_wait_read<0>();  // the previous output chunk has left the staging tile
            __syncwarp();
          }
          uint4 pk[4];
          if (gelu_h2) {
#pragma unroll
            for (int j = 0; j < 4; ++j) pk[j] = make_uint4(gpk[4 * j], gpk[4 * j + 1], gpk[4 * j + 2], gpk[4 * j + 3]);
          } else {
#pragma unroll
            for (int j = 0; j < 4; ++j)
              pk[j] = make_uint4(pack_elem(v[8 * j], v[8 * j + 1]), pack_elem(v[8 * j + 2], v[8 * j + 3]),
                                 pack_elem(v[8 * j + 4], v[8 * j + 5]), pack_elem(v[8 * j + 6], v[8 * j + 7]));
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) st_shared_v4(srow + ((j ^ sxor) << 4), pk[j].x, pk[j].y, pk[j].z, pk[j].w);
          fence_proxy_async();
          __syncwarp();
          if (lane == 0) {
            // first padded column of the warp's 32 pixels (transposed convs: every other column of the class)
            const bool t2 = p.mode == WM3_CONV_T2;
            const int pc = t2 ? 2 * colw + (cls & 1) + 1 : colw + 1;
            const int pr = t2 ? 2 * roww + (cls >> 1) + 1 : roww + 1;
            tma_store_4d(&tmO, stg, n, pc, pr, img);
            bulk_commit();
          }
          if (ok && (ocol == 0 || ocol == p.wout - 1)) {  // longitude wrap columns of the padded output
            const size_t hp = pix + (ocol == 0 ? p.wout : -static_cast<long long>(p.wout));
            uint4* d2 = reinterpret_cast<uint4*>(reinterpret_cast<elem_t*>(p.out) + hp * p.out_cp + n);
#pragma unroll
            for (int j = 0; j < 4; ++j) d2[j] = pk[j];
          }
          continue;
        }
        if (p.resid != nullptr) {
          const uint4* rs = reinterpret_cast<const uint4*>(p.resid + pix * p.resid_cp + n);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint4 w4 = __ldg(rs + j);
            const uint32_t ws[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              const float2 h2 = unpack_elem2(ws[t]);
              v[8 * j + 2 * t] += h2.x;
              v[8 * j + 2 * t + 1] += h2.y;
            }
          }
        }
        if (p.out_kind == WM3_CONV_OUT_NHWC) {
          uint4 pk[4];
          if (gelu_h2) {
#pragma unroll
            for (int j = 0; j < 4; ++j) pk[j] = make_uint4(gpk[4 * j], gpk[4 * j + 1], gpk[4 * j + 2], gpk[4 * j + 3]);
          } else {
#pragma unroll
            for (int j = 0; j < 4; ++j)
              pk[j] = make_uint4(pack_elem(v[8 * j], v[8 * j + 1]), pack_elem(v[8 * j + 2], v[8 * j + 3]),
                                 pack_elem(v[8 * j + 4], v[8 * j + 5]), pack_elem(v[8 * j + 6], v[8 * j + 7]));
          }
          elem_t* ob = reinterpret_cast<elem_t*>(p.out);
          uint4* d = reinterpret_cast<uint4*>(ob + pix * p.out_cp + n);
#pragma unroll
          for (int j = 0; j < 4; ++j) d[j] = pk[j];
          // longitude wrap columns of the padded output
          if (ocol == 0 || ocol == p.wout - 1) {
            const size_t hp = pix + (ocol == 0 ? p.wout : -static_cast<long long>(p.wout));
            uint4* d2 = reinterpret_cast<uint4*>(ob + hp * p.out_cp + n);
#pragma unroll
            for (int j = 0; j < 4; ++j) d2[j] = pk[j];
          }
        } else if (p.out_kind == WM3_CONV_OUT_TOKENS) {
          // fp32 tokens [img][hout][wout][cout]
          float* ot = reinterpret_cast<float*>(p.out) +
                      ((static_cast<size_t>(img) * p.hout + orow) * p.wout + ocol) * p.cout + n;
          if (nvalid == 32 && (p.cout % 4) == 0) {
            float4* d4 = reinterpret_cast<float4*>(ot);
#pragma unroll
            for (int j = 0; j < 8; ++j) d4[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
          } else {
#pragma unroll
            for (int e = 0; e < 32; ++e)
              if (e < nvalid) ot[e] = v[e];
          }
        } else {  // fp32 NCHW fields with channel remap (model.py:340-347 level unfold)
          float* of = reinterpret_cast<float*>(p.out) + static_cast<size_t>(img) * p.img_stride +
                      static_cast<size_t>(orow) * p.wout + ocol;
          // channel c -> (c / chan_div, c % chan_div), stepped from n (no division per element; the unrolled
          // loop keeps v[] in registers)
          int cq = n / p.chan_div, cr = n - cq * p.chan_div;
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            if (e < nvalid) of[cq * p.a_stride + cr * p.p_stride] = v[e];
            if (++cr == p.chan_div) { cr = 0; ++cq; }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (CG == 2) mbar_arrive_cluster_relaxed(tempty_leader0 + 8u * acc);  // the leader's MMA warp reuses it
        else mbar_arrive(tempty_bar(acc));
      }
      acc ^= 1;
      if (acc == 0) aphase ^= 1;
    }
    if (Cfg::TMA_EPI && lane == 0) bulk_wait<0>();  // output chunks written before the CTA (and its smem) retires
  }
  tc_fence_before();
  if (CG == 2)
    cluster_sync();  // the pair's MMAs read this CTA's smem and write its TMEM until the last tile
  else
    __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    if (CG == 2) tmem_dealloc_cg2(tmem_base, Cfg::TMEM_COLS);
    else tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
  }
}

// ---------------------------------------------------------------------------------------------
// layout kernels: fp32 NCHW / tokens -> padded bf16 NHWC (zero halo rows, wrapped halo columns)
// ---------------------------------------------------------------------------------------------
// dst[img][h + 1][w + 1][c] = src[img * img_stride + (c / cdiv) * a_stride + (c % cdiv) * p_stride + h * W + w],
// channels >= C zero; halo columns copied from the opposite edge, halo rows zero.
// Tiled transpose: a block owns one padded row of one image and 32 padded columns; it reads each channel's 32
// columns as one coalesced 128-byte run of the NCHW plane into shared memory, then writes the 32 NHWC pixels
// (32 x cp contiguous operand elements) with consecutive threads on consecutive element pairs.  Values outside
// the operand's finite range (|x| > 65504 for fp16, or non-finite) set *overflow (when non-null), so the host
// can refuse the input instead of silently convolving infinities.
constexpr int F2N_W = 32, F2N_THREADS = 256;
__global__ void __launch_bounds__(F2N_THREADS) fields_to_nhwc_kernel(
    const float* __restrict__ src, long long img_stride, long long a_stride, long long p_stride, int cdiv, int imgs,
    int C, int H, int W, int cp, elem_t* __restrict__ dst, int* __restrict__ overflow) {
  griddep_launch_dependents();  // PDL: the next kernel may start its prologue
  griddep_wait();
  __shared__ float tile[F2N_W][64 + 1];
  __shared__ long long coff[64];  // source offset of each channel of the current 64-channel chunk (-1: pad)
  const int ntw = (W + 2 + F2N_W - 1) / F2N_W;
  const int pw0 = (blockIdx.x % ntw) * F2N_W;
  const int ph = (blockIdx.x / ntw) % (H + 2);
  const int img = blockIdx.x / (ntw * (H + 2));
  const int tid = threadIdx.x, lane = tid & 31, ty = tid >> 5;
  const int npix = min(F2N_W, W + 2 - pw0);
  uint32_t* out = reinterpret_cast<uint32_t*>(dst + ((static_cast<size_t>(img) * (H + 2) + ph) * (W + 2) + pw0) * cp);
  if (ph == 0 || ph == H + 1) {  // zero halo row
    for (int e = tid; e < npix * cp / 2; e += F2N_THREADS) out[e] = 0u;
    return;
  }
  const int h = ph - 1;
  const int pw = pw0 + lane;
  const int wsrc = pw == 0 ? W - 1 : (pw == W + 1 ? 0 : pw - 1);
  const float maxf = (kElemFmt == 0) ? 65504.f : 3.0e38f;
  bool bad = false;
  const float* base = src + img * img_stride + static_cast<long long>(h) * W + wsrc;
  for (int cc = 0; cc < cp; cc += 64) {
    if (tid < 64) {
      const int c = cc + tid;
      coff[tid] = c < C ? (c / cdiv) * a_stride + (c % cdiv) * p_stride : -1;
    }
    __syncthreads();
#pragma unroll 4
    for (int cl = ty; cl < 64; cl += F2N_THREADS / 32) {
      const long long off = coff[cl];
      float v = 0.f;
      if (off >= 0 && lane < npix) {
        v = __ldg(base + off);
        bad |= !(fabsf(v) <= maxf);
      }
      tile[lane][cl] = v;
    }
    __syncthreads();
    for (int e = tid; e < npix * 32; e += F2N_THREADS) {
      const int wl = e >> 5, c2 = (e & 31) * 2;
      out[(wl * cp + cc + c2) >> 1] = pack_elem(tile[wl][c2], tile[wl][c2 + 1]);
    }
    __syncthreads();
  }
  if (overflow != nullptr && __any_sync(0xffffffffu, bad) && lane == 0) atomicOr(overflow, 1);
}

// tokens fp32 [img][H][W][C] (C = hidden) -> padded bf16 NHWC with cp channels
__global__ void tokens_to_nhwc_kernel(const float* __restrict__ tok, int imgs, int H, int W, int C, int cp,
                                      elem_t* __restrict__ dst) {
  griddep_launch_dependents();  // PDL: the next kernel may start its prologue
  griddep_wait();
  const long long total = static_cast<long long>(imgs) * (H + 2) * (W + 2) * (cp / 2);
  for (long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int c2 = static_cast<int>(idx % (cp / 2)) * 2;
    long long rest = idx / (cp / 2);
    const int pw = static_cast<int>(rest % (W + 2));
    rest /= (W + 2);
    const int ph = static_cast<int>(rest % (H + 2));
    const int img = static_cast<int>(rest / (H + 2));
    float a = 0.f, b = 0.f;
    if (ph >= 1 && ph <= H) {
      const int h = ph - 1;
      const int w = pw == 0 ? W - 1 : (pw == W + 1 ? 0 : pw - 1);
      const float* s = tok + ((static_cast<size_t>(img) * H + h) * W + w) * C;
      if (c2 < C) a = s[c2];
      if (c2 + 1 < C) b = s[c2 + 1];
    }
    reinterpret_cast<uint32_t*>(dst)[idx] = pack_elem(a, b);
  }
}

template <int BN, int CG, bool STRIP>
static int launch_conv(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& to, const CUtensorMap& tr,
                       ConvParams p, cudaStream_t s) {
  if (!ConvCfg<BN, CG, STRIP>::TMA_EPI) p.tma_out = 0;
  using Cfg = ConvCfg<BN, CG, STRIP>;
  auto kern = conv_tc_kernel<BN, CG, STRIP>;
  if (ensure_smem_attr(reinterpret_cast<const void*>(kern), Cfg::SMEM, "conv")) return -1;
  const long long ntiles =
      static_cast<long long>(p.imgs) * p.nclass * ((p.tiles_per_class + CG - 1) / CG) * (p.cout_pad / BN);
  if (CG == 1) {
    const int grid = static_cast<int>(ntiles < sm_count() ? ntiles : sm_count());
    if (launch_pdl(kern, dim3(grid), dim3(CV_THREADS), Cfg::SMEM, s, ta, tb, to, tr, p)) return -1;
    return check_launch("conv_tc_kernel");
  }
  const int pairs = sm_count() / 2;
  const int grid = 2 * static_cast<int>(ntiles < pairs ? ntiles : pairs);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(CV_THREADS);
  cfg.dynamicSmemBytes = Cfg::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelEx(&cfg, kern, ta, tb, to, tr, p) != cudaSuccess)
    return set_error("conv_tc_kernel (pairs): launch failed: %s", cudaGetErrorString(cudaGetLastError()));
  return check_launch("conv_tc_kernel");
}

template <int BN, int CG>
static int launch_conv_mode(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& to, const CUtensorMap& tr,
                            const ConvParams& p, cudaStream_t s, bool strip) {
  // the strip stage (A strip + three weight boxes) must still leave a 3-deep ring
  if (strip && ConvCfg<BN, CG, true>::STAGES_FIT >= 3) return launch_conv<BN, CG, true>(ta, tb, to, tr, p, s);
  return launch_conv<BN, CG, false>(ta, tb, to, tr, p, s);
}

}  // namespace wm3

using namespace wm3;

// two-row conv tiles for rows that 128-pixel tiles would mostly pad (WM3_CONV_TWOROW=0 turns them off, A/B aid)
static bool conv_two_row_enabled() {
  static const bool on = [] {
    const char* e = getenv("WM3_CONV_TWOROW");
    return !(e && e[0] == '0');
  }();
  return on;
}

// transposed convs on A strips (WM3_CONV_T2STRIP=0 turns it off, A/B aid)
static bool conv_t2_strip_enabled() {
  static const bool on = [] {
    const char* e = getenv("WM3_CONV_T2STRIP");
    return !(e && e[0] == '0');
  }();
  return on;
}

// TMA-staged conv epilogue (WM3_CONV_TMA=0 turns it off, A/B aid)
static bool conv_tma_epi_enabled() {
  static const bool on = [] {
    const char* e = getenv("WM3_CONV_TMA");
    return !(e && e[0] == '0');
  }();
  return on;
}

// CTA pairs (WM3_CONV_PAIRS=0 turns them off, A/B aid): each CTA's weight box is half of the BN rows.
// Measured (full-scale encode + decode, one B200): the 3x3 / transposed convs with Cout >= 128 run 7-12 %
// faster (encode 27.3 -> 25.4 ms device time); the BN = 64 heads 20-25 % slower, so they stay single-CTA.
static bool conv_pairs_enabled() {
  static const bool on = [] {
    const char* e = getenv("WM3_CONV_PAIRS");
    return !(e && e[0] == '0');
  }();
  return on;
}
static bool conv_strip_fits(int bn, int cg) {
  switch (bn * 4 + cg) {
    case 64 * 4 + 1: return ConvCfg<64, 1, true>::STAGES_FIT >= 3;
    case 128 * 4 + 1: return ConvCfg<128, 1, true>::STAGES_FIT >= 3;
    case 192 * 4 + 1: return ConvCfg<192, 1, true>::STAGES_FIT >= 3;
    case 256 * 4 + 1: return ConvCfg<256, 1, true>::STAGES_FIT >= 3;
    case 128 * 4 + 2: return ConvCfg<128, 2, true>::STAGES_FIT >= 3;
    case 192 * 4 + 2: return ConvCfg<192, 2, true>::STAGES_FIT >= 3;
    case 256 * 4 + 2: return ConvCfg<256, 2, true>::STAGES_FIT >= 3;
    default: return false;
  }
}

extern "C" int wm3_conv_bn(int cout) {
  if (cout <= 64) return 64;  // decoder heads (17 / 35 channels): half the MMA columns of a 128 tile
  if (cout <= 128) return 128;
  if (cout <= 192) return 192;
  return 256;
}

extern "C" int wm3_conv(int mode, const void* in, int imgs, int hin, int win, int cinp, const void* w, int cout,
                        const float* bias, int act_gelu, const void* resid, int resid_cp, int out_kind, void* out,
                        int out_cp,
                        long long img_stride, long long a_stride, long long p_stride, int chan_div, void* stream) {
  if (mode != WM3_CONV_S1 && mode != WM3_CONV_S2 && mode != WM3_CONV_T2) return set_error("wm3_conv: bad mode");
  if (cinp % 64) return set_error("wm3_conv: padded input channels %d not a multiple of 64", cinp);
  if ((mode == WM3_CONV_S2 && win % 2) || hin < 1 || win < 1)
    return set_error("wm3_conv: bad input extents %dx%d", hin, win);
  ConvParams p{};
  p.mode = mode;
  p.imgs = imgs;
  p.hin = hin; p.win = win; p.cinp = cinp;
  if (mode == WM3_CONV_S1) { p.hout = hin; p.wout = win; p.nclass = 1; p.ntap = 9; }
  else if (mode == WM3_CONV_S2) { p.hout = (hin - 1) / 2 + 1; p.wout = win / 2; p.nclass = 1; p.ntap = 9; }
  else { p.hout = 2 * hin; p.wout = 2 * win; p.nclass = 4; p.ntap = 4; }
  p.rows_t = (mode == WM3_CONV_T2) ? hin : p.hout;
  p.cols_t = (mode == WM3_CONV_T2) ? win : p.wout;
  p.ncb = cinp / 64;
  p.cout = cout;
  const int bn = wm3_conv_bn(cout);
  p.cout_pad = ((cout + bn - 1) / bn) * bn;
  p.tile_rows = 1;
  p.tile_cols = CV_BM;
  p.bias = bias;
  p.act_gelu = act_gelu;
  p.resid = reinterpret_cast<const elem_t*>(resid);
  p.resid_cp = resid_cp;
  if (resid && (resid_cp % 64 || resid_cp < cout)) return set_error("wm3_conv: bad resid_cp");
  p.out_kind = out_kind;
  p.out = out;
  p.out_cp = out_cp;
  p.img_stride = img_stride; p.a_stride = a_stride; p.p_stride = p_stride; p.chan_div = chan_div > 0 ? chan_div : 1;
  if (out_kind == WM3_CONV_OUT_NHWC && (out_cp % 64 || out_cp < cout)) return set_error("wm3_conv: bad out_cp");
  // stride-1 convs stage one 130-pixel strip per kernel row for its three column taps (WM3_CONV_STRIP=0: per tap)
  static const bool strip_env = [] {
    const char* e = getenv("WM3_CONV_STRIP");
    return !(e && e[0] == '0');
  }();
  const int bn_ = wm3_conv_bn(cout);
  const bool pairs_ = conv_pairs_enabled() && bn_ >= 128;
  bool strip = strip_env && (mode == WM3_CONV_S1 || (mode == WM3_CONV_T2 && conv_t2_strip_enabled())) &&
               conv_strip_fits(bn_, pairs_ ? 2 : 1);
  // two-row tiles (2 x 64 pixels) where a row's 128-pixel tiles would be mostly padding (a 180-pixel row: 128 +
  // 52 valid of 256 computed; 2 x 64: 180 of 192); they take one A box per tap (no strip)
  if (conv_two_row_enabled()) {
    const double w1 = ((p.cols_t + 127) / 128) * 128.0 / p.cols_t, w2 = ((p.cols_t + 63) / 64) * 64.0 / p.cols_t;
    if (w2 < 0.85 * w1) {
      p.tile_rows = 2;
      p.tile_cols = 64;
      strip = false;
    }
  }
  p.tiles_per_row = (p.cols_t + p.tile_cols - 1) / p.tile_cols;
  p.tiles_per_class = ((p.rows_t + p.tile_rows - 1) / p.tile_rows) * p.tiles_per_row;
  // A: padded NHWC input, images stacked along rows
  CUtensorMap ta, tb;
  const uint64_t wp = win + 2;
  const uint64_t rows = static_cast<uint64_t>(imgs) * (hin + 2);
  if (mode == WM3_CONV_S2) {
    const uint64_t dims[4] = {static_cast<uint64_t>(cinp), 2, wp / 2, rows};
    const uint64_t strides[3] = {static_cast<uint64_t>(cinp), 2ull * cinp, wp * cinp};
    // two-row tiles: output rows r, r + 1 read input rows 2r + kh, 2r + 2 + kh (a row box of 4 at stride 2)
    const bool two = p.tile_rows == 2;
    const uint32_t box[4] = {64, 1, static_cast<uint32_t>(p.tile_cols), two ? 4u : 1u};
    const uint32_t es[4] = {1, 1, 1, two ? 2u : 1u};
    if (make_tmap(&ta, in, TMAP_BF16, 4, dims, strides, box, es)) return -1;
  } else {
    const uint64_t dims[3] = {static_cast<uint64_t>(cinp), wp, rows};
    const uint64_t strides[2] = {static_cast<uint64_t>(cinp), wp * cinp};
    const uint32_t box[3] = {64, static_cast<uint32_t>(strip ? CV_STRIP_ROWS : p.tile_cols),
                             static_cast<uint32_t>(p.tile_rows)};
    if (make_tmap(&ta, in, TMAP_BF16, 3, dims, strides, box, nullptr)) return -1;
  }
  // B: weights [class][cout_pad][ntap * cinp], K-major
  const int kdim = p.ntap * cinp;
  const int cg = pairs_ ? 2 : 1;
  if (make_tmap_2d_bf16(&tb, w, kdim, static_cast<uint64_t>(p.nclass) * p.cout_pad, kdim, CV_BK, bn / cg)) return -1;
  // output / residual maps for the TMA-staged epilogue (NHWC output: a warp's 32 pixels are consecutive columns
  // of one output row, or every other column for a transposed conv): boxes of 32 channels x 32 pixels, 64-byte
  // swizzle; the
  // output map's column extent ends at the last real pixel (padded column W + 1 is the wrap copy of pixel 0,
  // written by the thread that owns pixel 0), so a tile's overhang past the row end is clipped
  CUtensorMap to{}, tr{};
  p.tma_out = 0;
  if (out_kind == WM3_CONV_OUT_NHWC && conv_tma_epi_enabled() && !(mode == WM3_CONV_T2 && resid)) {
    const uint64_t wpo = static_cast<uint64_t>(p.wout) + 2, hpo = static_cast<uint64_t>(p.hout) + 2;
    const uint32_t box[4] = {32, 32, 1, 1};
    // transposed convs: a warp's 32 pixels are every other output column (one parity class), so the store box
    // spans 64 columns with traversal stride 2 (32 rows in shared memory)
    const uint32_t tbox[4] = {32, 64, 1, 1}, tstr[4] = {1, 2, 1, 1};
    const bool t2 = mode == WM3_CONV_T2;
    // column extent ends at the last real pixel (pad column W + 1 is the wrap copy), row extent at the last
    // real row (the bottom pad row stays zero): a tile's overhang past either edge is clipped
    const uint64_t od[4] = {static_cast<uint64_t>(out_cp), wpo - 1, hpo - 1, static_cast<uint64_t>(imgs)};
    const uint64_t os[3] = {static_cast<uint64_t>(out_cp), wpo * out_cp, hpo * wpo * out_cp};
    if (make_tmap_swz(&to, out, TMAP_BF16, 4, od, os, t2 ? tbox : box, t2 ? tstr : nullptr, 64)) return -1;
    if (resid) {
      const uint64_t rd[4] = {static_cast<uint64_t>(resid_cp), wpo, hpo, static_cast<uint64_t>(imgs)};
      const uint64_t rs[3] = {static_cast<uint64_t>(resid_cp), wpo * resid_cp, hpo * wpo * resid_cp};
      if (make_tmap_swz(&tr, resid, TMAP_BF16, 4, rd, rs, box, nullptr, 64)) return -1;
    }
    p.tma_out = 1;
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (cg == 2) {
    if (bn == 128) return launch_conv_mode<128, 2>(ta, tb, to, tr, p, s, strip);
    if (bn == 192) return launch_conv_mode<192, 2>(ta, tb, to, tr, p, s, strip);
    return launch_conv_mode<256, 2>(ta, tb, to, tr, p, s, strip);
  }
  if (bn == 64) return launch_conv_mode<64, 1>(ta, tb, to, tr, p, s, strip);
  if (bn == 128) return launch_conv_mode<128, 1>(ta, tb, to, tr, p, s, strip);
  if (bn == 192) return launch_conv_mode<192, 1>(ta, tb, to, tr, p, s, strip);
  return launch_conv_mode<256, 1>(ta, tb, to, tr, p, s, strip);
}

extern "C" int wm3_fields_to_nhwc(const float* src, long long img_stride, long long a_stride, long long p_stride,
                                  int chan_div, int imgs, int channels, int h, int w, int cp, void* dst,
                                  int* overflow, void* stream) {
  if (channels > cp || cp % 64) return set_error("wm3_fields_to_nhwc: bad channel padding");
  const long long blocks = static_cast<long long>(imgs) * (h + 2) * ((w + 2 + F2N_W - 1) / F2N_W);
  if (blocks > 0x7fffffffLL) return set_error("wm3_fields_to_nhwc: too many images");
  if (launch_pdl(fields_to_nhwc_kernel, dim3(static_cast<int>(blocks)), dim3(F2N_THREADS), 0,
                 reinterpret_cast<cudaStream_t>(stream), src, img_stride, a_stride, p_stride,
                 chan_div > 0 ? chan_div : 1, imgs, channels, h, w, cp, reinterpret_cast<elem_t*>(dst), overflow))
    return -1;
  return check_launch("fields_to_nhwc_kernel");
}

extern "C" int wm3_tokens_to_nhwc(const float* tokens, int imgs, int h, int w, int channels, int cp, void* dst,
                                  void* stream) {
  if (channels > cp || cp % 64) return set_error("wm3_tokens_to_nhwc: bad channel padding");
  const long long total = static_cast<long long>(imgs) * (h + 2) * (w + 2) * (cp / 2);
  long long blocks = (total + 255) / 256;
  if (blocks > 148LL * 64) blocks = 148LL * 64;
  if (launch_pdl(tokens_to_nhwc_kernel, dim3(static_cast<int>(blocks)), dim3(256), 0,
                 reinterpret_cast<cudaStream_t>(stream), tokens, imgs, h, w, channels, cp,
                 reinterpret_cast<elem_t*>(dst)))
    return -1;
  return check_launch("tokens_to_nhwc_kernel");
}
