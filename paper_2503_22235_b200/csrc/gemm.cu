// Persistent warp-specialised tcgen05 GEMM with fused epilogues (K2-K5 of DESIGN.md).
//
//   C[M, N] = A[M, K] * B[N, K]^T     A: activations bf16 (K-major), B: weights bf16 pre-transposed
//                                     to (out, in) so both operands are K-major SWIZZLE_128B tiles.
// CG = 2 (default for N >= 256): CTA pairs (cluster of 2 on one TPC) issue tcgen05.mma.cta_group::2 with
// M = 256: each CTA loads its own 128 A rows and half of the B tile (BN / 2 rows) into its smem, the leader's
// MMA reads B from both SMs, and each CTA's TMEM receives its 128 x BN accumulator; per-SM smem operand
// traffic halves (A 16 KB + B/2 16 KB per k-block instead of 16 + 32 KB), freeing smem for a 6-deep ring.
// Roles (one CTA per SM, 384 threads):
//   warp 0       TMA producer: A/B k-blocks into a STAGES-deep smem ring (mbarrier full/empty)
//   warp 1       MMA issuer: one thread issues tcgen05.mma 128xBNx16, accumulator in TMEM,
//                double-buffered (2 x BN columns) so the epilogue of tile i overlaps the MMAs of tile i+1
//   warp 2       TMEM allocator
//   warps 4..11  epilogue, two groups of 4 warps (each group covers the 128 TMEM lanes) working on
//                alternating column chunks: tcgen05.ld -> bias / GELU / rotary / residual in registers ->
//                SWIZZLE_128B smem staging -> TMA store (coalesced, asynchronous, clipped at the edges).
// Reference semantics: attention.py:142-143 (_linear), :167-171 (q,k,v + rotary), :179 and :183
// (residual adds), :182 (erf-form GELU, autodiff.py:372-382; common.cuh gelu_tanh, |err| <= 2.5e-5).
#include <cstdlib>

#include "common.cuh"
#include "launch.h"
#include "../../include/wm3.h"

namespace wm3 {

struct EpiParams {
  const float* resid;  // fp32 residual stream (read), same buffer the output map writes
  int ld_resid;
  int resid_v8;  // residual base and pitch 32 B aligned: 256-bit loads
  const float* bias;
  int n_valid;
  // GEMM rows form `planes` planes of `plane_rows` rows; M-tiles never straddle a plane, so every tile
  // is one clipped TMA box store at (n, r0, plane) of the (n, row, plane) output map.
  int plane_rows, planes, tiles_per_plane;
  wm3_rope_t rope;
  wm3_halo_t halo;  // QKV epilogue: boundary rows also stored into the neighbours' K/V grids (peer memory)
  int has_halo;
  wm3_ln_fold_t fold;  // LayerNorm fold (include/wm3.h): producer (residual epilogue) / consumer (next GEMM)
  int ln_prod, ln_cons;
  int mn;  // operands MN-major (wm3_linear_tn: C = A^T B with A [K][M], B [K][N] row-major, 64 x 64 boxes)
  const unsigned* gscale;  // WM3_EPI_GELU_GRAD_F32: amax bits of the output gradient's operand scale
  int ksplit;  // > 1: split-K — output plane p = the partial product over k-block range p (A rows = plane rows)
  unsigned* amax_out;  // WM3_EPI_GELU_GRAD_F32: atomicMax of max |out| (float bits), NULL = none
};

// epilogues that read the fp32 output buffer before overwriting it (the residual stream, or the stored GELU
// pre-activation of the in-place GELU backward)
__host__ __device__ constexpr bool epi_reads_out(int e) {
  return e == WM3_EPI_BIAS_RESID_F32 || e == WM3_EPI_GELU_GRAD_F32;
}

constexpr int GEMM_BM = 128;
constexpr int GEMM_BK = 64;
constexpr int GEMM_THREADS = 384;
constexpr int EPI_WARP0 = 4;

#ifndef WM3_PAIR_STAGING
#define WM3_PAIR_STAGING 1
#endif
#ifndef WM3_RESID_TMA
#define WM3_RESID_TMA 1
#endif
#ifndef WM3_RSLOTS
#define WM3_RSLOTS 2  // residual slots (even); each pair of slots costs one mainloop stage
#endif
template <int BN, int CG = 1, int EPI = 0>
struct GemmCfg {
  // Residual epilogue: the fp32 residual chunks stream into RSLOTS smem slots by TMA (warp 3), ahead of the
  // epilogue, instead of per-thread global loads (the O-proj epilogue was HBM-latency bound); one mainloop
  // stage gives up its smem for them.
  static constexpr bool RESID_TMA = epi_reads_out(EPI) && WM3_RESID_TMA;
  // Two slots: with an even slot count and even units per tile, slot c % RSLOTS has the parity of the unit, so
  // each slot is consumed by one epilogue group only, in order (an odd count interleaves the groups on a slot
  // and a fast group can then pass a parity wait one phase early).
  static constexpr int RSLOTS = RESID_TMA ? WM3_RSLOTS : 0;
  // CTA pairs free 16 KB per stage: 6 stages, or 5 stages with double-buffered epilogue staging
  static constexpr int STAGES = (CG == 2) ? ((WM3_PAIR_STAGING == 2 || RESID_TMA) ? (RESID_TMA ? 6 - WM3_RSLOTS / 2 : 5)
                                                                                  : 6)
                                          : (RESID_TMA ? 3 : 4);
  static constexpr int STAGING_PER_GROUP = (BN == 256) ? ((CG == 2) ? WM3_PAIR_STAGING : 1) : 2;
  static constexpr uint32_t A_BYTES = GEMM_BM * GEMM_BK * 2;
  static constexpr uint32_t B_BYTES = (BN / CG) * GEMM_BK * 2;  // this CTA's share of the B tile
  static constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr uint32_t STAGING_BYTES = 16384;  // 128 rows x 128 B
  static constexpr uint32_t RSLOT_BYTES = 16384;    // 128 rows x 32 fp32
  static constexpr uint32_t SMEM = STAGES * STAGE_BYTES + 2 * STAGING_PER_GROUP * STAGING_BYTES +
                                   RSLOTS * RSLOT_BYTES + 1024 /*align*/ + 256 /*barriers*/;
  static constexpr uint32_t TMEM_COLS = 2 * BN;
};

template <int EPI>
struct EpiTraits {
  static constexpr bool F32 = (EPI == WM3_EPI_F32 || epi_reads_out(EPI));
  static constexpr int CW = F32 ? 32 : 64;  // columns per staged chunk (128 B rows)
};

// 32 residual floats of one row at column n: 256-bit loads when the residual base and pitch are 32 B
// aligned (else 128-bit), scalar tail at n_valid.
template <class EP>
DEVI void load_resid(const EP& ep, int row, bool row_ok, int n, float (&x)[32]) {
  const float* src = ep.resid + static_cast<size_t>(row) * ep.ld_resid + n;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    float t[8];
    if (row_ok && n + 8 * j + 8 <= ep.n_valid) {
      if (ep.resid_v8) {
        ldg256(src + 8 * j, t);
      } else {
        const float4 lo = *reinterpret_cast<const float4*>(src + 8 * j);
        const float4 hi = *reinterpret_cast<const float4*>(src + 8 * j + 4);
        t[0] = lo.x; t[1] = lo.y; t[2] = lo.z; t[3] = lo.w; t[4] = hi.x; t[5] = hi.y; t[6] = hi.z; t[7] = hi.w;
      }
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) t[e] = (row_ok && n + 8 * j + e < ep.n_valid) ? src[8 * j + e] : 0.f;
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) x[8 * j + e] = t[e];
  }
}

// Rotary on interleaved pairs: columns (2i, 2i+1) of a q/k head hold the reference pair (i, i + dh/2).
// Token `row` -> (depth plane d, band row h, column w).  Depth / row pairs come from the dr table row of (d, h),
// which the 32 tokens of a warp (consecutive columns) share: 256-bit broadcast loads.  Column pair k (k = 1,
// 2, ... from `split`) has phase k * alpha_w (attention.py:76-78: integer wavenumbers), so its (cos, sin) is
// e^{i alpha_w} raised step by step from the first column pair of the chunk: two coalesced loads per chunk
// instead of one per pair (|error| <= ~1e-6, far below the fp16 output rounding).  (A per-token table made
// every lane read its own 512 B row: 32 sectors per load, 0.07 ms of the QKV GEMM.)
DEVI void rope_chunk(const wm3_rope_t& rp, int row, int M, int col0_in_head, float (&v)[64]) {
  int t = row < M ? row : 0;
  if (rp.period > 0) t %= rp.period;  // ensemble members share the tables
  const int rc = rp.rows * rp.cols;
  const int d = t / rc;
  const int rem = t - d * rc;
  const int h = rem / rp.cols;
  const int w = rem - h * rp.cols;
  const int p0 = col0_in_head >> 1;  // first pair of this 64-column chunk
  const float* dr = rp.dr + static_cast<size_t>(d * rp.rows + h) * 128 + p0;
  const float* col_c = rp.col + w;
  const float* col_s = rp.col + static_cast<size_t>(64) * rp.cols + w;
  float cr = 1.f, ci = 0.f, er = 1.f, ei = 0.f;  // current e^{i k alpha}, step e^{i alpha}
  if (p0 + 32 > rp.split) {
    const int pc0 = max(p0, rp.split);
    cr = __ldg(col_c + static_cast<size_t>(pc0) * rp.cols);
    ci = __ldg(col_s + static_cast<size_t>(pc0) * rp.cols);
    er = __ldg(col_c + static_cast<size_t>(rp.split) * rp.cols);
    ei = __ldg(col_s + static_cast<size_t>(rp.split) * rp.cols);
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int pa = p0 + 8 * q;  // first pair of this vector (warp-uniform branches)
    float cs[8], sn[8];
    if (pa < rp.split) {
      ldg256(dr + 8 * q, cs);
      ldg256(dr + 64 + 8 * q, sn);
    }
    if (pa + 8 > rp.split) {
#pragma unroll
      for (int e = 0; e < 8; ++e)
        if (pa + e >= rp.split) {
          cs[e] = cr;
          sn[e] = ci;
          const float nr = cr * er - ci * ei;
          ci = fmaf(cr, ei, ci * er);
          cr = nr;
        }
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int k = 8 * q + e;
      const float x1 = v[2 * k], x2 = v[2 * k + 1];
      v[2 * k] = x1 * cs[e] - x2 * sn[e];
      v[2 * k + 1] = x1 * sn[e] + x2 * cs[e];
    }
  }
}

template <int BN, int EPI, int CG>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmOut, int M, int N, int K, EpiParams ep) {
  griddep_launch_dependents();  // PDL: the next kernel may start its prologue
  using Cfg = GemmCfg<BN, CG, EPI>;
  using Tr = EpiTraits<EPI>;
  constexpr int STAGES = Cfg::STAGES;
  constexpr int RSLOTS = Cfg::RSLOTS;
  constexpr int CW = Tr::CW;
  constexpr int NUNITS = BN / CW;
  static_assert(!Cfg::RESID_TMA || (NUNITS % 2 == 0 && Cfg::RSLOTS % 2 == 0),
                "residual slots must map onto one epilogue group each");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = smem_u32(smem);
  const uint32_t staging0 = sbase + STAGES * Cfg::STAGE_BYTES;
  const uint32_t rslot0 = staging0 + 2 * Cfg::STAGING_PER_GROUP * Cfg::STAGING_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::STAGE_BYTES +
                                               2 * Cfg::STAGING_PER_GROUP * Cfg::STAGING_BYTES +
                                               RSLOTS * Cfg::RSLOT_BYTES);
  const uint32_t bar0 = smem_u32(bars);
  auto full_bar = [&](int s) { return bar0 + 8u * s; };
  auto empty_bar = [&](int s) { return bar0 + 8u * (STAGES + s); };
  auto tfull_bar = [&](int a) { return bar0 + 8u * (2 * STAGES + a); };
  auto tempty_bar = [&](int a) { return bar0 + 8u * (2 * STAGES + 2 + a); };
  auto rfull_bar = [&](int r) { return bar0 + 8u * (2 * STAGES + 4 + r); };
  auto rempty_bar = [&](int r) { return bar0 + 8u * (2 * STAGES + 4 + RSLOTS + r); };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 4 + 2 * RSLOTS);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  // CTA pairs: cluster = (2k, 2k+1); the pair walks the tile list together, rank r owns rows [128 r, +128)
  const uint32_t rank = (CG == 2) ? cluster_ctarank() : 0u;
  const int tile0 = (CG == 2) ? static_cast<int>(blockIdx.x >> 1) : static_cast<int>(blockIdx.x);
  const int tstep = (CG == 2) ? static_cast<int>(gridDim.x >> 1) : static_cast<int>(gridDim.x);
  const int nm = ep.planes * ep.tiles_per_plane;
  const int nn = (N + BN - 1) / BN;
  const int ntiles = nm * nn;
  const int nk = (K + GEMM_BK - 1) / GEMM_BK;
  // tile -> (plane, this CTA's first row in the plane, its first GEMM row); a tile is CG x 128 rows
  auto tile_rows = [&](int tile, int& plane, int& r0) {
    const int mt = tile / nn;
    plane = mt / ep.tiles_per_plane;
    r0 = (mt - plane * ep.tiles_per_plane) * (GEMM_BM * CG) + static_cast<int>(rank) * GEMM_BM;
    return plane * ep.plane_rows + r0;
  };

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    tma_prefetch(&tmOut);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(empty_bar(s), 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull_bar(a), 1);
      mbar_init(tempty_bar(a), 8 * CG);  // every epilogue warp of the pair arrives on the leader's barrier
    }
    for (int r = 0; r < RSLOTS; ++r) {
      mbar_init(rfull_bar(r), 1);
      mbar_init(rempty_bar(r), 4);  // the 4 warps of the epilogue group that consumes the chunk
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
  griddep_wait();  // PDL: inputs (A, residual) are complete from here on

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = tile0; tile < ntiles; tile += tstep) {
        int plane, r0;
        const int mrow = tile_rows(tile, plane, r0);
        const int m0 = ep.ksplit > 1 ? r0 : mrow;  // split-K: every plane reads the same A rows
        const int n0 = (tile % nn) * BN + static_cast<int>(rank) * (BN / CG);
        const int kb0 = ep.ksplit > 1 ? plane * nk / ep.ksplit : 0;
        const int kb1 = ep.ksplit > 1 ? (plane + 1) * nk / ep.ksplit : nk;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(empty_bar(stage), phase ^ 1);
          const uint32_t sa = sbase + stage * Cfg::STAGE_BYTES;
          const uint32_t sb = sa + Cfg::A_BYTES;
          if (ep.mn) {
            // MN-major operands: 64 (M or N) x 64 (K) boxes, each 64 K-rows of 128 B
            const uint32_t fb = (CG == 2) ? mapa_shared(full_bar(stage), 0) : full_bar(stage);
            if (rank == 0) mbar_arrive_expect_tx(full_bar(stage), CG * Cfg::STAGE_BYTES);
            for (int i = 0; i < GEMM_BM / 64; ++i) {
              if (CG == 2) tma_load_2d_cg2(sa + i * 8192u, &tmA, fb, m0 + 64 * i, kb * GEMM_BK);
              else tma_load_2d(sa + i * 8192u, &tmA, fb, m0 + 64 * i, kb * GEMM_BK);
            }
            for (int i = 0; i < BN / CG / 64; ++i) {
              if (CG == 2) tma_load_2d_cg2(sb + i * 8192u, &tmB, fb, n0 + 64 * i, kb * GEMM_BK);
              else tma_load_2d(sb + i * 8192u, &tmB, fb, n0 + 64 * i, kb * GEMM_BK);
            }
          } else if (CG == 2) {
            // both CTAs' bytes complete on the leader's full barrier; only the leader arms it
            const uint32_t fb = mapa_shared(full_bar(stage), 0);
            if (rank == 0) mbar_arrive_expect_tx(full_bar(stage), 2 * Cfg::STAGE_BYTES);
            tma_load_2d_cg2(sa, &tmA, fb, kb * GEMM_BK, m0);
            tma_load_2d_cg2(sb, &tmB, fb, kb * GEMM_BK, n0);
          } else {
            mbar_arrive_expect_tx(full_bar(stage), Cfg::STAGE_BYTES);
            tma_load_2d(sa, &tmA, full_bar(stage), kb * GEMM_BK, m0);
            tma_load_2d(sb, &tmB, full_bar(stage), kb * GEMM_BK, n0);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {  // the leader issues the pair's MMAs
      // The whole warp walks the k-blocks (warp-wide waits, warp-uniform descriptors in uniform registers);
      // one elected lane issues the MMAs and commits.
      const uint32_t idesc = make_idesc(GEMM_BM * CG, BN, ep.mn, ep.mn);
      // K-major: k-steps of 16 elements are 32 B apart in a row; MN-major: 16 K-rows (2 KB), 64-wide M / N
      // chunks 8 KB apart (LBO)
      const uint64_t d0 = make_sdesc_sw128(sbase, ep.mn ? 8192u : 16u, 1024);
      const uint32_t kstep = ep.mn ? 128u : 2u;
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t aphase = 0;
      for (int tile = tile0; tile < ntiles; tile += tstep) {
        mbar_wait(tempty_bar(acc), aphase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        int kb0 = 0, kb1 = nk;
        if (ep.ksplit > 1) {
          int plane, r0;
          tile_rows(tile, plane, r0);
          kb0 = plane * nk / ep.ksplit;
          kb1 = (plane + 1) * nk / ep.ksplit;
        }
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(full_bar(stage), phase);
          tc_fence_after();
          const uint64_t ad = d0 + ((stage * Cfg::STAGE_BYTES) >> 4), bd = ad + (Cfg::A_BYTES >> 4);
          if (elect_one()) {
#pragma unroll
            for (int k = 0; k < GEMM_BK / 16; ++k) {
              if (CG == 2)
                umma_ss_cg2(d_tmem, ad + kstep * k, bd + kstep * k, idesc, ((kb - kb0) | k) != 0 ? 1u : 0u);
              else
                umma_bf16_ss(d_tmem, ad + kstep * k, bd + kstep * k, idesc, ((kb - kb0) | k) != 0 ? 1u : 0u);
            }
            if (CG == 2)
              umma_commit_mc(empty_bar(stage), 0x3);  // frees the stage in both CTAs
            else
              umma_commit(empty_bar(stage));
          }
          __syncwarp();
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        if (elect_one()) {
          if (CG == 2)
            umma_commit_mc(tfull_bar(acc), 0x3);
          else
            umma_commit(tfull_bar(acc));
        }
        __syncwarp();
        acc ^= 1;
        if (acc == 0) aphase ^= 1;
      }
    }
  } else if (Cfg::RESID_TMA && warp == 3) {
    // residual producer: chunk c of this CTA (tile-major, column units in order) -> slot c % RSLOTS
    if (lane == 0) {
      int c = 0;
      for (int tile = tile0; tile < ntiles; tile += tstep) {
        int plane, r0;
        tile_rows(tile, plane, r0);
        const int n0 = (tile % nn) * BN;
        for (int u = 0; u < NUNITS; ++u, ++c) {
          constexpr int RS = RSLOTS > 0 ? RSLOTS : 1;
          const int slot = c % RS;
          mbar_wait(rempty_bar(slot), ((c / RS) & 1) ^ 1);
          mbar_arrive_expect_tx(rfull_bar(slot), Cfg::RSLOT_BYTES);
          tma_load_3d(rslot0 + slot * Cfg::RSLOT_BYTES, &tmOut, rfull_bar(slot), n0 + u * CW, r0, plane);
        }
      }
    }
  } else if (warp >= EPI_WARP0) {
    const int g = (warp - EPI_WARP0) >> 2;  // epilogue group
    const int q = warp & 3;                  // TMEM lane quarter
    const int r_in_tile = 32 * q + lane;
    const bool elected = (warp == EPI_WARP0 + 4 * g) && lane == 0;
    const int bar_id = 1 + g;
    int acc = 0;
    uint32_t aphase = 0;
    int sbuf = 0;
    const uint32_t tempty_leader0 = (CG == 2) ? mapa_shared(tempty_bar(0), 0) : 0u;
    int tile_it = 0;
    // LayerNorm fold, consumer side: the row's (rstd, rstd * mean), loaded one tile ahead so its latency never
    // sits between the accumulator and the epilogue.
    constexpr bool kCons = (!epi_reads_out(EPI) && EPI != WM3_EPI_F32);
    const bool cons = kCons && ep.ln_cons;
    auto stats_load = [&](int t) {
      int pl, rr;
      const int rw = (t < ntiles) ? tile_rows(t, pl, rr) + r_in_tile : 0;
      return __ldg(reinterpret_cast<const float2*>(ep.fold.row_stats) + (rw < M ? rw : 0));
    };
    float2 ln_next = cons ? stats_load(tile0) : make_float2(0.f, 0.f);
    const float ginv = (EPI == WM3_EPI_GELU_GRAD_F32) ? 1.f / grad_scale(ep.gscale) : 1.f;
    float gmax = 0.f;  // WM3_EPI_GELU_GRAD_F32: this thread's max |out| (the next operand scale, no extra pass)
    for (int tile = tile0; tile < ntiles; tile += tstep, ++tile_it) {
      int plane, r0;
      const int m0 = tile_rows(tile, plane, r0);
      const int n0 = (tile % nn) * BN;
      const int row = m0 + r_in_tile;
      const int prow = r0 + r_in_tile;  // row within the plane
      const bool row_ok = (prow < ep.plane_rows) && row < M;
      const float ln_rstd = ln_next.x, ln_rmu = ln_next.y;
      if (cons) ln_next = stats_load(tile + tstep);  // consumed by the next tile
      // LayerNorm fold, producer side: partial (sum, sum of squares) of this group's columns of the row
      float ln_s1 = 0.f, ln_s2 = 0.f;
      // residual prefetch, RESID_DEPTH chunks of this group ahead: the first ones overlap the mainloop wait
      // (the residual epilogue is HBM-latency bound: more bytes in flight per thread)
#ifndef WM3_RESID_DEPTH
#define WM3_RESID_DEPTH 1  // deeper prefetch spills registers and measured slower (A/B: depth 1 0.25 ms, 2 0.28 ms O-proj)
#endif
      constexpr int RESID_DEPTH = WM3_RESID_DEPTH;
      float xr[RESID_DEPTH + 1][32];
      if (epi_reads_out(EPI) && !Cfg::RESID_TMA) {
#pragma unroll
        for (int i = 0; i < RESID_DEPTH; ++i)
          if (g + 2 * i < NUNITS) load_resid(ep, row, row_ok, n0 + (g + 2 * i) * CW, xr[i]);
      }
      mbar_wait(tfull_bar(acc), aphase);
      tc_fence_after();
      const uint32_t taddr = tmem_base + acc * BN + (static_cast<uint32_t>(32 * q) << 16);
#pragma unroll
      for (int u = g; u < NUNITS; u += 2) {
        const int n = n0 + u * CW;
        const int it = (u - g) >> 1;  // compile-time after unrolling
        const float* xa = Cfg::RESID_TMA ? nullptr : xr[it % (RESID_DEPTH + 1)];
        if (epi_reads_out(EPI) && !Cfg::RESID_TMA && u + 2 * RESID_DEPTH < NUNITS)
          load_resid(ep, row, row_ok, n + 2 * RESID_DEPTH * CW, xr[(it + RESID_DEPTH) % (RESID_DEPTH + 1)]);
        if (Tr::F32) {
          uint32_t r[32];
          tmem_ld32(taddr + u * CW, r);
          tmem_ld_wait();
          float* v = reinterpret_cast<float*>(r);  // accumulate in place: no extra 32-register copy
          if (epi_reads_out(EPI)) {
            // residual chunk: from its TMA smem slot (SWIZZLE_128B rows, as the box landed), or the registers
            int rslot = 0;
            uint32_t rb = 0;
            if (Cfg::RESID_TMA) {
              const int c = tile_it * NUNITS + u;
              rslot = c % (RSLOTS > 0 ? RSLOTS : 1);
              mbar_wait(rfull_bar(rslot), (c / (RSLOTS > 0 ? RSLOTS : 1)) & 1);
              rb = rslot0 + rslot * Cfg::RSLOT_BYTES;
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const float4 b = (n + 4 * j < ep.n_valid) ? __ldg(reinterpret_cast<const float4*>(ep.bias + n) + j)
                                                        : make_float4(0.f, 0.f, 0.f, 0.f);
              float4 xv;
              if (Cfg::RESID_TMA)
                ld_shared_v4(rb + sw128_off(r_in_tile, j), xv.x, xv.y, xv.z, xv.w);
              else
                xv = make_float4(xa[4 * j + 0], xa[4 * j + 1], xa[4 * j + 2], xa[4 * j + 3]);
              if (EPI == WM3_EPI_GELU_GRAD_F32) {  // in-place GELU backward: out held the pre-activation
                v[4 * j + 0] = v[4 * j + 0] * ginv * gelu_grad(xv.x + b.x);
                v[4 * j + 1] = v[4 * j + 1] * ginv * gelu_grad(xv.y + b.y);
                v[4 * j + 2] = v[4 * j + 2] * ginv * gelu_grad(xv.z + b.z);
                v[4 * j + 3] = v[4 * j + 3] * ginv * gelu_grad(xv.w + b.w);
                if (row_ok)
                  gmax = fmaxf(gmax, fmaxf(fmaxf(fabsf(v[4 * j + 0]), fabsf(v[4 * j + 1])),
                                           fmaxf(fabsf(v[4 * j + 2]), fabsf(v[4 * j + 3]))));
              } else {
                v[4 * j + 0] += b.x + xv.x;
                v[4 * j + 1] += b.y + xv.y;
                v[4 * j + 2] += b.z + xv.z;
                v[4 * j + 3] += b.w + xv.w;
              }
            }
            if (Cfg::RESID_TMA) {
              // the slot's next TMA load (async proxy) must not overtake these generic-proxy reads
              fence_proxy_async();
              __syncwarp();
              if (lane == 0) mbar_arrive(rempty_bar(rslot));
            }
            if (ep.ln_prod) {
              // the updated stream as the next GEMM's fp16 operand, and its row statistics
              float s1b = 0.f, s2b = 0.f;  // packed pairs: (even, odd) column partial sums
#pragma unroll
              for (int e = 0; e < 32; e += 2) {
                const float ta = (n + e < ep.n_valid) ? v[e] : 0.f;
                const float tb = (n + e + 1 < ep.n_valid) ? v[e + 1] : 0.f;
                ffma2(ln_s1, s1b, ta, tb, 1.f, 1.f, ln_s1, s1b);
                ffma2(ln_s2, s2b, ta, tb, ta, tb, ln_s2, s2b);
              }
              ln_s1 += s1b;
              ln_s2 += s2b;
              if (row_ok) {
                elem_t* dst = static_cast<elem_t*>(ep.fold.xh_out) + static_cast<size_t>(row) * ep.fold.ld_xh + n;
                if (n + 32 <= ep.n_valid) {
#pragma unroll
                  for (int h = 0; h < 2; ++h) {
                    uint32_t w8[8];
#pragma unroll
                    for (int e = 0; e < 8; ++e) w8[e] = pack_elem(v[16 * h + 2 * e], v[16 * h + 2 * e + 1]);
                    stg256(dst + 16 * h, w8);
                  }
                } else {
#pragma unroll
                  for (int e = 0; e < 32; ++e)
                    if (n + e < ep.n_valid) dst[e] = to_elem(v[e]);
                }
              }
            }
          }
          // staging row: 8 x 16 B chunks of 4 floats
          if (elected) bulk_wait_read<Cfg::STAGING_PER_GROUP - 1>();
          named_bar_sync(bar_id, 128);
          const uint32_t st = staging0 + (g * Cfg::STAGING_PER_GROUP + sbuf) * Cfg::STAGING_BYTES;
#pragma unroll
          for (int j = 0; j < 8; ++j)
            st_shared_v4(st + sw128_off(r_in_tile, j), __float_as_uint(v[4 * j]), __float_as_uint(v[4 * j + 1]),
                         __float_as_uint(v[4 * j + 2]), __float_as_uint(v[4 * j + 3]));
        } else {
          uint32_t r0[32], r1[32];
          tmem_ld32(taddr + u * CW, r0);
          tmem_ld32(taddr + u * CW + 32, r1);
          tmem_ld_wait();
          float v[64];
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            v[e] = __uint_as_float(r0[e]);
            v[32 + e] = __uint_as_float(r1[e]);
          }
          if (cons) {
            // folded LayerNorm: rstd * acc - rstd * mean * c[col] + d[col]   (d = b + beta . W, in ep.bias)
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const bool okc = n + 4 * j < ep.n_valid;
              const float4 b = okc ? __ldg(reinterpret_cast<const float4*>(ep.bias + n) + j) : make_float4(0.f, 0.f, 0.f, 0.f);
              const float4 c = okc ? __ldg(reinterpret_cast<const float4*>(ep.fold.fold_c + n) + j)
                                   : make_float4(0.f, 0.f, 0.f, 0.f);
              float t0, t1, t2, t3;  // packed pairs: two FFMA2 per two columns
              ffma2(t0, t1, -ln_rmu, -ln_rmu, c.x, c.y, b.x, b.y);
              ffma2(t2, t3, -ln_rmu, -ln_rmu, c.z, c.w, b.z, b.w);
              ffma2(v[4 * j + 0], v[4 * j + 1], v[4 * j + 0], v[4 * j + 1], ln_rstd, ln_rstd, t0, t1);
              ffma2(v[4 * j + 2], v[4 * j + 3], v[4 * j + 2], v[4 * j + 3], ln_rstd, ln_rstd, t2, t3);
            }
          } else {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const float4 b = (n + 4 * j < ep.n_valid) ? __ldg(reinterpret_cast<const float4*>(ep.bias + n) + j)
                                                        : make_float4(0.f, 0.f, 0.f, 0.f);
              v[4 * j + 0] += b.x; v[4 * j + 1] += b.y; v[4 * j + 2] += b.z; v[4 * j + 3] += b.w;
            }
          }
#if !defined(WM3_OPERAND_BF16) && WM3_GELU_VARIANT == 2
          constexpr bool gelu_h2 = (EPI == WM3_EPI_BIAS_GELU_BF16);  // f16x2 GELU straight to packed pairs
#else
          constexpr bool gelu_h2 = false;
#endif
          if (EPI == WM3_EPI_BIAS_GELU_BF16 && !gelu_h2) {
#pragma unroll
            for (int e = 0; e < 64; ++e) v[e] = gelu_epi(v[e]);
          }
          if (EPI == WM3_EPI_QKV_ROPE) {
            const int sec = ep.rope.heads * ep.rope.dhp;
            if (n < 2 * sec) rope_chunk(ep.rope, row, M, (n % sec) % ep.rope.dhp, v);
          }
          uint32_t pk[32];
#pragma unroll
          for (int e = 0; e < 32; ++e)
            pk[e] = gelu_h2 ? gelu_tanh_h2(v[2 * e], v[2 * e + 1]) : pack_elem(v[2 * e], v[2 * e + 1]);
          if (EPI == WM3_EPI_QKV_ROPE && ep.has_halo && row_ok && n >= ep.halo.col_lo) {
            // fused halo exchange: this row's 64 columns also go to a neighbour's K/V grid over NVLink
            const int r = prow;
            elem_t* dst = nullptr;
            if (ep.halo.up != nullptr && r < ep.halo.n_up)
              dst = static_cast<elem_t*>(ep.halo.up) +
                    (plane * ep.halo.up_plane_stride + ep.halo.up_row_off + r) * ep.halo.ld + n;
            else if (ep.halo.dn != nullptr && r >= ep.plane_rows - ep.halo.n_dn)
              dst = static_cast<elem_t*>(ep.halo.dn) +
                    (plane * ep.halo.dn_plane_stride + ep.halo.dn_row_off + (r - (ep.plane_rows - ep.halo.n_dn))) *
                        ep.halo.ld + n;
            if (dst != nullptr) {
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                uint32_t w[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) w[e] = pk[8 * q + e];
                stg256(dst + 16 * q, w);
              }
            }
          }
          if (elected) bulk_wait_read<Cfg::STAGING_PER_GROUP - 1>();
          named_bar_sync(bar_id, 128);
          const uint32_t st = staging0 + (g * Cfg::STAGING_PER_GROUP + sbuf) * Cfg::STAGING_BYTES;
#pragma unroll
          for (int j = 0; j < 8; ++j)
            st_shared_v4(st + sw128_off(r_in_tile, j), pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
        }
        fence_proxy_async();
        named_bar_sync(bar_id, 128);
        if (elected) {
          const uint32_t st = staging0 + (g * Cfg::STAGING_PER_GROUP + sbuf) * Cfg::STAGING_BYTES;
          tma_store_3d(&tmOut, st, n, r0, plane);  // rows past the plane end are clipped
          bulk_commit();
        }
        if (Cfg::STAGING_PER_GROUP > 1) sbuf ^= 1;
      }
      if (EPI == WM3_EPI_BIAS_RESID_F32 && ep.ln_prod && row_ok) {
        float* so = ep.fold.stats_out + static_cast<size_t>(row) * (2 * WM3_LN_SLOTS) + 2 * ((tile % nn) * 2 + g);
        *reinterpret_cast<float2*>(so) = make_float2(ln_s1, ln_s2);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (CG == 2)
          mbar_arrive_cluster_relaxed(tempty_leader0 + 8u * acc);  // the leader's MMA thread reuses the accumulator
        else
          mbar_arrive(tempty_bar(acc));
      }
      acc ^= 1;
      if (acc == 0) aphase ^= 1;
    }
    if (elected) bulk_wait<0>();
    if (EPI == WM3_EPI_GELU_GRAD_F32 && ep.amax_out != nullptr) {
#pragma unroll
      for (int o = 16; o; o >>= 1) gmax = fmaxf(gmax, __shfl_xor_sync(0xffffffffu, gmax, o));
      if (lane == 0) atomicMax(ep.amax_out, __float_as_uint(gmax));  // order-independent: deterministic
    }
    if (EPI == WM3_EPI_QKV_ROPE && ep.has_halo) __threadfence_system();  // peer halo rows visible system-wide
  }
  tc_fence_before();
  if (CG == 2)
    cluster_sync();  // the pair's MMAs read this CTA's smem and write its TMEM until the last tile
  else
    __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    if (CG == 2)
      tmem_dealloc_cg2(tmem_base, Cfg::TMEM_COLS);
    else
      tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
  }
}

template <int BN, int EPI, int CG>
static int launch_gemm(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& to, int M, int N, int K,
                       const EpiParams& ep, cudaStream_t stream) {
  using Cfg = GemmCfg<BN, CG, EPI>;
  auto kern = gemm_tc_kernel<BN, EPI, CG>;
  if (ensure_smem_attr(reinterpret_cast<const void*>(kern), Cfg::SMEM, "gemm")) return -1;
  const int ntiles = ep.planes * ep.tiles_per_plane * ((N + BN - 1) / BN);
  if (CG == 1) {
    const int grid = ntiles < sm_count() ? ntiles : sm_count();
    if (launch_pdl(kern, dim3(grid), dim3(GEMM_THREADS), Cfg::SMEM, stream, ta, tb, to, M, N, K, ep)) return -1;
    return check_launch("gemm_tc_kernel");
  }
  const int pairs = (ntiles < sm_count() / 2) ? ntiles : sm_count() / 2;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * pairs);
  cfg.blockDim = dim3(GEMM_THREADS);
  cfg.dynamicSmemBytes = Cfg::SMEM;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, ta, tb, to, M, N, K, ep);
  if (e != cudaSuccess) return set_error("gemm_tc_kernel (pair) launch: %s", cudaGetErrorString(e));
  return check_launch("gemm_tc_kernel");
}

template <int BN, int CG>
static int dispatch_epi(int epi, const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& to, int M, int N,
                        int K, const EpiParams& ep, cudaStream_t s) {
  switch (epi) {
    case WM3_EPI_F32: return launch_gemm<BN, WM3_EPI_F32, CG>(ta, tb, to, M, N, K, ep, s);
    case WM3_EPI_BIAS_BF16: return launch_gemm<BN, WM3_EPI_BIAS_BF16, CG>(ta, tb, to, M, N, K, ep, s);
    case WM3_EPI_BIAS_GELU_BF16: return launch_gemm<BN, WM3_EPI_BIAS_GELU_BF16, CG>(ta, tb, to, M, N, K, ep, s);
    case WM3_EPI_BIAS_RESID_F32: return launch_gemm<BN, WM3_EPI_BIAS_RESID_F32, CG>(ta, tb, to, M, N, K, ep, s);
    case WM3_EPI_GELU_GRAD_F32: return launch_gemm<BN, WM3_EPI_GELU_GRAD_F32, CG>(ta, tb, to, M, N, K, ep, s);
    case WM3_EPI_QKV_ROPE: return launch_gemm<BN, WM3_EPI_QKV_ROPE, CG>(ta, tb, to, M, N, K, ep, s);
    default: return set_error("wm3_linear: unknown epilogue %d", epi);
  }
}

struct OutPlanes {
  int planes, plane_rows;      // GEMM rows = planes x plane_rows (band tokens in order)
  long long plane_stride;      // destination rows between consecutive planes
  int row_off;                 // destination row of GEMM row 0
};

static int linear_impl(const void* a, int lda, const void* b, int ldb, int m, int n, int k, int epi, void* out,
                       int ldo, int n_valid, const float* bias, const wm3_rope_t* rope, const OutPlanes& op,
                       void* stream, const wm3_halo_t* halo = nullptr, const wm3_ln_fold_t* fold = nullptr,
                       bool mn = false, const unsigned* gscale = nullptr, int ksplit = 1,
                       unsigned* amax_out = nullptr) {
  if (m <= 0 || n <= 0 || k <= 0) return set_error("wm3_linear: bad sizes m=%d n=%d k=%d", m, n, k);
  const bool f32_out = (epi == WM3_EPI_F32 || epi_reads_out(epi));
  if ((lda % 8) || (ldb % 8) || (ldo % (f32_out ? 4 : 8)))
    return set_error("wm3_linear: pitches must be multiples of 8 (bf16) / 4 (f32 out)");
  if (n % 32) return set_error("wm3_linear: n=%d must be a multiple of 32", n);
  if (n_valid <= 0 || n_valid > n) return set_error("wm3_linear: n_valid=%d outside (0, %d]", n_valid, n);
  if ((n_valid * (f32_out ? 4 : 2)) % 16)
    return set_error("wm3_linear: n_valid=%d rows must span a multiple of 16 bytes (TMA store)", n_valid);
  if (epi != WM3_EPI_F32 && bias == nullptr) return set_error("wm3_linear: bias required");
  if (op.planes < 1 || static_cast<long long>(op.planes) * op.plane_rows != m || op.plane_stride < op.plane_rows)
    return set_error("wm3_linear: %d planes x %d rows (stride %lld) do not tile m=%d", op.planes, op.plane_rows,
                     op.plane_stride, m);
  if (epi_reads_out(epi) && op.planes != 1) return set_error("wm3_linear: residual output must be 2D");
  if (epi == WM3_EPI_QKV_ROPE && rope != nullptr) {
    if (reinterpret_cast<uintptr_t>(rope->dr) % 32 || rope->col == nullptr)
      return set_error("wm3_linear: rope dr table must be 32-byte aligned and the column table given");
    if (rope->rows < 1 || rope->cols < 1 || rope->split < 0 || rope->split > 64 ||
        (rope->period > 0 && rope->period % (rope->rows * rope->cols)))
      return set_error("wm3_linear: bad rope geometry (rows %d cols %d period %d split %d)", rope->rows, rope->cols,
                       rope->period, rope->split);
  }
  EpiParams ep{};
  ep.resid = reinterpret_cast<const float*>(out);
  ep.ld_resid = ldo;
  ep.resid_v8 = (ldo % 8 == 0) && (reinterpret_cast<uintptr_t>(out) % 32 == 0);
  ep.bias = bias;
  ep.gscale = gscale;
  ep.ksplit = ksplit;
  ep.amax_out = amax_out;
  if (ksplit > 1 && (epi != WM3_EPI_F32 || op.planes != ksplit || op.row_off != 0 || (k + GEMM_BK - 1) / GEMM_BK < ksplit))
    return set_error("wm3_linear: bad split-K (%d splits, %d planes, k=%d)", ksplit, op.planes, k);
  ep.n_valid = n_valid;
  ep.plane_rows = op.plane_rows;
  ep.planes = op.planes;
  const int bn = (n >= 256) ? 256 : 128;
  // CTA pairs for the wide GEMMs (WM3_GEMM_CG=1 forces single-CTA tiles: A/B aid)
  static const int cg_env = [] {
    const char* e = getenv("WM3_GEMM_CG");
    return e ? atoi(e) : 2;
  }();
  // every wide GEMM runs as CTA pairs; the short-K residual GEMM (O-proj, K = 1024) was faster as single-CTA
  // tiles while its residual came through per-thread loads, and is faster as pairs since the residual streams
  // in by TMA (0.195 vs 0.204 ms isolated)
  const int cg = (bn == 256 && cg_env == 2) ? 2 : 1;
  ep.tiles_per_plane = (op.plane_rows + GEMM_BM * cg - 1) / (GEMM_BM * cg);
  // Narrow pair tiles (256 x 128) for outputs whose 256 x 256 tiles leave most of their last wave idle (a
  // latitude band's 1024-wide GEMMs at 8 GPUs: 156 tiles for 74 pairs).  Off by default: measured per tile they
  // are ~30 % less efficient (half the MMA per operand byte), which costs more than the idle tail — O-proj / W2
  // at M = 9900: 29 / 80 us on 256-wide tiles, 33 / 94 us on 128-wide.  Same per-element arithmetic, so
  // results do not depend on the choice.  WM3_GEMM_NARROW=1 heuristic, 2 always (A/B, tests).
  static const int narrow_env = [] {
    const char* e = getenv("WM3_GEMM_NARROW");
    return e ? atoi(e) : 0;
  }();
  bool narrow = false;
  if (cg == 2 && narrow_env != 0 && fold == nullptr && !mn && ksplit == 1) {
    const long long mt = static_cast<long long>(op.planes) * ep.tiles_per_plane;
    const long long pairs = sm_count() / 2;
    const long long r256 = (mt * ((n + 255) / 256) + pairs - 1) / pairs;
    const long long r128 = (mt * ((n + 127) / 128) + pairs - 1) / pairs;
    narrow = narrow_env == 2 || static_cast<double>(r128) * 0.5 * 1.08 < static_cast<double>(r256);
  }
  if (halo != nullptr) {
    if (epi != WM3_EPI_QKV_ROPE) return set_error("wm3_linear: halo stores need the QKV epilogue");
    if ((halo->ld % 16) || (halo->col_lo % 64) || halo->n_up < 0 || halo->n_dn < 0 ||
        halo->n_up > op.plane_rows || halo->n_dn > op.plane_rows ||
        (reinterpret_cast<uintptr_t>(halo->up) % 32) || (reinterpret_cast<uintptr_t>(halo->dn) % 32))
      return set_error("wm3_linear: bad halo descriptor (ld %% 16, col_lo %% 64, row counts, 32 B alignment)");
    ep.halo = *halo;
    ep.has_halo = 1;
  }
  if (fold != nullptr) {
    ep.fold = *fold;
    ep.ln_prod = fold->xh_out != nullptr || fold->stats_out != nullptr;
    ep.ln_cons = fold->row_stats != nullptr;
    const int ntile_n = (n + bn - 1) / bn;
    if (ep.ln_prod && (epi != WM3_EPI_BIAS_RESID_F32 || fold->xh_out == nullptr || fold->stats_out == nullptr ||
                       (fold->ld_xh % 16) || fold->ld_xh < n_valid || (reinterpret_cast<uintptr_t>(fold->xh_out) % 32) ||
                       2 * ntile_n > WM3_LN_SLOTS || (n_valid % 2)))
      return set_error("wm3_linear: bad LayerNorm-fold producer (residual epilogue, xh and stats, ld_xh %% 16, "
                       "<= %d column tiles)", WM3_LN_SLOTS / 2);
    if (ep.ln_cons && (epi == WM3_EPI_BIAS_RESID_F32 || epi == WM3_EPI_F32 || fold->fold_c == nullptr))
      return set_error("wm3_linear: bad LayerNorm-fold consumer (16-bit epilogue and fold_c required)");
  }
  if (epi == WM3_EPI_QKV_ROPE) {
    if (rope == nullptr) return set_error("wm3_linear: rope descriptor required");
    ep.rope = *rope;
    if (ep.rope.dhp != 64 && ep.rope.dhp != 128) return set_error("wm3_linear: dhp must be 64 or 128");
  }
  CUtensorMap ta, tb, to;
  ep.mn = mn ? 1 : 0;
  const int am = ksplit > 1 ? op.plane_rows : m;  // split-K: every output plane reads the same A rows
  if (mn) {  // A [k][m], B [k][n] row-major: 64 x 64 boxes (M / N inner)
    if (make_tmap_2d_bf16(&ta, a, am, k, lda, 64, GEMM_BK)) return -1;
    if (make_tmap_2d_bf16(&tb, b, n, k, ldb, 64, GEMM_BK)) return -1;
  } else {
    if (make_tmap_2d_bf16(&ta, a, k, am, lda, GEMM_BK, GEMM_BM)) return -1;
    if (make_tmap_2d_bf16(&tb, b, k, n, ldb, GEMM_BK, (narrow ? 128 : bn) / cg)) return -1;  // each CTA of a pair loads half
  }
  {
    const int cw = f32_out ? 32 : 64;
    const size_t esz = f32_out ? 4 : 2;
    const char* base = reinterpret_cast<const char*>(out) + static_cast<size_t>(op.row_off) * ldo * esz;
    uint64_t dims[3] = {static_cast<uint64_t>(n_valid), static_cast<uint64_t>(op.plane_rows),
                        static_cast<uint64_t>(op.planes)};
    uint64_t strides[2] = {static_cast<uint64_t>(ldo), static_cast<uint64_t>(op.plane_stride) * ldo};
    uint32_t box[3] = {static_cast<uint32_t>(cw), static_cast<uint32_t>(GEMM_BM), 1};
    if (make_tmap(&to, base, f32_out ? TMAP_F32 : TMAP_BF16, 3, dims, strides, box, nullptr)) return -1;
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (narrow) return dispatch_epi<128, 2>(epi, ta, tb, to, m, n, k, ep, s);
  if (bn == 256)
    return cg == 2 ? dispatch_epi<256, 2>(epi, ta, tb, to, m, n, k, ep, s)
                   : dispatch_epi<256, 1>(epi, ta, tb, to, m, n, k, ep, s);
  return dispatch_epi<128, 1>(epi, ta, tb, to, m, n, k, ep, s);
}

}  // namespace wm3

using namespace wm3;

extern "C" int wm3_linear(const void* a, int lda, const void* b, int ldb, int m, int n, int k, int epi, void* out,
                          int ldo, int n_valid, const float* bias, const wm3_rope_t* rope, void* stream) {
  const OutPlanes op{1, m, m, 0};
  return linear_impl(a, lda, b, ldb, m, n, k, epi, out, ldo, n_valid, bias, rope, op, stream);
}

extern "C" int wm3_linear_gelu_grad(const void* a, int lda, const void* b, int ldb, int m, int n, int k,
                                    float* preact_inout, int ldo, const float* bias, const unsigned* amax_bits,
                                    unsigned* out_amax_bits, void* stream) {
  const OutPlanes op{1, m, m, 0};
  return linear_impl(a, lda, b, ldb, m, n, k, WM3_EPI_GELU_GRAD_F32, preact_inout, ldo, n, bias, nullptr, op, stream,
                     nullptr, nullptr, false, amax_bits, 1, out_amax_bits);
}

extern "C" int wm3_linear_planes(const void* a, int lda, const void* b, int ldb, int m, int n, int k, int epi,
                                 void* out, int ldo, int n_valid, const float* bias, const wm3_rope_t* rope,
                                 int planes, int plane_rows, long long plane_stride, int row_off, void* stream) {
  const OutPlanes op{planes, plane_rows, plane_stride, row_off};
  return linear_impl(a, lda, b, ldb, m, n, k, epi, out, ldo, n_valid, bias, rope, op, stream);
}

extern "C" int wm3_linear_planes_halo(const void* a, int lda, const void* b, int ldb, int m, int n, int k, int epi,
                                      void* out, int ldo, int n_valid, const float* bias, const wm3_rope_t* rope,
                                      int planes, int plane_rows, long long plane_stride, int row_off,
                                      const wm3_halo_t* halo, void* stream) {
  const OutPlanes op{planes, plane_rows, plane_stride, row_off};
  return linear_impl(a, lda, b, ldb, m, n, k, epi, out, ldo, n_valid, bias, rope, op, stream, halo);
}

extern "C" int wm3_linear_fold(const void* a, int lda, const void* b, int ldb, int m, int n, int k, int epi, void* out,
                               int ldo, int n_valid, const float* bias, const wm3_rope_t* rope, int planes,
                               int plane_rows, long long plane_stride, int row_off, const wm3_halo_t* halo,
                               const wm3_ln_fold_t* fold, void* stream) {
  const OutPlanes op{planes, plane_rows, plane_stride, row_off};
  return linear_impl(a, lda, b, ldb, m, n, k, epi, out, ldo, n_valid, bias, rope, op, stream, halo, fold);
}

namespace wm3 {
__global__ void halo_signal_kernel(int* a, int* b, int epoch) {
  __threadfence_system();
  if (a != nullptr) asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(a), "r"(epoch) : "memory");
  if (b != nullptr) asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(b), "r"(epoch) : "memory");
}
__global__ void halo_wait_kernel(const int* flags, int n, int epoch) {
  const long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    int v;
    for (;;) {
      asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(flags + i) : "memory");
      if (v >= epoch) break;
      __nanosleep(200);
      if (clock64() - t0 > 20000000000LL) __trap();  // ~10 s: a neighbour never signalled
    }
  }
  __threadfence_system();
}
}  // namespace wm3

extern "C" int wm3_halo_signal(int* peer_flag_a, int* peer_flag_b, int epoch, void* stream) {
  halo_signal_kernel<<<1, 1, 0, reinterpret_cast<cudaStream_t>(stream)>>>(peer_flag_a, peer_flag_b, epoch);
  return check_launch("halo_signal_kernel");
}

extern "C" int wm3_halo_wait(const int* flags, int n, int epoch, void* stream) {
  if (n <= 0) return 0;
  halo_wait_kernel<<<1, 1, 0, reinterpret_cast<cudaStream_t>(stream)>>>(flags, n, epoch);
  return check_launch("halo_wait_kernel");
}

// C[m][n] (fp32) = sum_t A[t][m] B[t][n]: both operands row-major over the reduction axis (the backward's
// weight gradients over tokens, autodiff.py:350 matmul VJP), read as MN-major tiles: no transposed copies.
namespace wm3 {
// out[r][c] = sum over s = 0 .. splits-1 in order of part[s][r][c] (split-K partials, [splits][m][n] dense)
__global__ void splitk_reduce_kernel(const float* __restrict__ part, int splits, int m, int n, float* __restrict__ out,
                                     int ldo) {
  const size_t plane = static_cast<size_t>(m) * n;
  const int n4 = n / 4;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < static_cast<size_t>(m) * n4;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const size_t r = i / n4, c = 4 * (i - r * n4);
    float4 acc = __ldg(reinterpret_cast<const float4*>(part + r * n + c));
    for (int sp = 1; sp < splits; ++sp) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(part + sp * plane + r * n + c));
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    *reinterpret_cast<float4*>(out + r * ldo + c) = acc;
  }
}
}  // namespace wm3

// Splits of the K range for an MN-major C = A^T B of m x n on CTA-pair tiles of 256 x 256: the count in [1, 16]
// that minimises (waves of tiles x splits over the pairs) / splits — the long-K weight gradients (K = tokens)
// have few output tiles (16 for a 1024 x 1024 weight: 22 % of the pairs) — limited by the scratch and by >= 8
// k-blocks per split.
static int choose_ksplit(int m, int n, int k, size_t scratch_floats) {
  const int pairs = sm_count() / 2;
  const int tiles = ((m + 255) / 256) * ((n + 255) / 256);
  const int nk = (k + GEMM_BK - 1) / GEMM_BK;
  int best = 1;
  double best_t = static_cast<double>((tiles + pairs - 1) / pairs);
  for (int sp = 2; sp <= 16; ++sp) {
    if (nk / sp < 8 || static_cast<size_t>(sp) * m * n > scratch_floats) break;
    const double t = static_cast<double>((tiles * sp + pairs - 1) / pairs) / sp + 0.02;  // + reduce pass
    if (t < best_t) { best_t = t; best = sp; }
  }
  return best;
}

extern "C" int wm3_linear_tn_split_count(int m, int n, int k) {
  return choose_ksplit(m, n, k, static_cast<size_t>(-1));
}

extern "C" int wm3_linear_tn_split(const void* a, int lda, const void* b, int ldb, int m, int n, int k, float* out,
                                   int ldo, float* scratch, size_t scratch_floats, void* stream) {
  if ((m % 64) || (n % 64)) return set_error("wm3_linear_tn_split: m=%d and n=%d must be multiples of 64", m, n);
  const int sp = scratch != nullptr ? choose_ksplit(m, n, k, scratch_floats) : 1;
  if (sp == 1) {
    const OutPlanes op{1, m, m, 0};
    return linear_impl(a, lda, b, ldb, m, n, k, WM3_EPI_F32, out, ldo, n, nullptr, nullptr, op, stream, nullptr,
                       nullptr, true);
  }
  const OutPlanes op{sp, m, m, 0};
  if (linear_impl(a, lda, b, ldb, sp * m, n, k, WM3_EPI_F32, scratch, n, n, nullptr, nullptr, op, stream, nullptr,
                  nullptr, true, nullptr, sp))
    return -1;
  const long long n4 = static_cast<long long>(m) * n / 4;
  const int blocks = static_cast<int>(n4 / 256 + 1 < 148 * 8 ? n4 / 256 + 1 : 148 * 8);
  splitk_reduce_kernel<<<blocks, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(scratch, sp, m, n, out, ldo);
  return check_launch("splitk_reduce_kernel");
}

extern "C" int wm3_linear_tn(const void* a, int lda, const void* b, int ldb, int m, int n, int k, float* out, int ldo,
                             void* stream) {
  if ((m % 64) || (n % 64)) return set_error("wm3_linear_tn: m=%d and n=%d must be multiples of 64", m, n);
  const OutPlanes op{1, m, m, 0};
  return linear_impl(a, lda, b, ldb, m, n, k, WM3_EPI_F32, out, ldo, n, nullptr, nullptr, op, stream, nullptr,
                     nullptr, true);
}
