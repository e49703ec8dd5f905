// K1: fused 3D neighborhood attention forward on tcgen05 (reference attention.py:173-178,
// window arithmetic grid.py:96-130).
//
// Work item = (query tile, head).  A query tile is a TD x TH x TW box of tokens (<= 128 queries, one per
// TMEM lane).  The union of the tile's windows is walked as a list of key chunks, each a run of rows of
// one depth plane x a contiguous (mod W) run of columns, <= 128 keys.
//
// Persistent, warp-specialised CTA (one per SM, 320 threads):
//   warp 9      TMA producer (one thread): the Q tile (4D box TD x TH x TW) and each chunk's K and V head
//               slices (4D box ncp x nrpc) into SWIZZLE_128B tiles: 3 K slots (freed by Q K^T), 2 V slots
//               (freed by P V), K issued one chunk ahead of V; completion via mbarrier transaction counts
//   warp 8      MMA issuer (one thread): S = Q K^T into one of two TMEM S buffers (M128 N128 K=dhp, both
//               operands from smem), O += P V with P read from TMEM (M128 N=dhp K=128, V MN-major from its
//               TMA tile), O accumulated in TMEM across chunks; S_{j+1} is issued before PV_j
//   warps 0-7   softmax (one thread per query row and key-column half, two warps per TMEM lane quarter):
//               window bitmask built from the same integer formula as grid.py (bump on depth/rows, wrap on
//               cols), fp32 running max / sum with lazy O rescaling (only when the max grows by > 2^8),
//               exp2, P (fp16) -> TMEM (double-buffered); finally O / l -> ctx rows.
// The logits never leave the SM.  Output ctx rows are bf16 [T][heads][dhp] = the O-proj GEMM operand.
#include "common.cuh"
#include "launch.h"
#include "window.cuh"
#include "../../include/wm3.h"

namespace wm3 {

struct NaParams {
  elem_t* out;
  int ldo;
  int depth, rows, cols, rows_global, row0, halo_lo, rows_ext;
  int heads, dhp, wd, wh, ww;
  int TD, TH, TW, ntd, nth, ntw, nitems;
  int ncp, nrpc;  // key-chunk box: ncp columns x nrpc rows (fixed for every tile)
  float scale_log2;
  int dbg;  // profiling switch (WM3_NA_DEBUG): 1 = skip the softmax arithmetic, 2 = also skip the MMAs
};

// warps 0-7 softmax (warp w: TMEM lanes 32 (w % 4).., key / O columns half w / 4), 8 MMA, 9 TMA producer
constexpr int NA_SOFTMAX_WARPS = 8;
constexpr int NA_MMA_WARP = 8;
constexpr int NA_TMA_WARP = 9;
constexpr int NA_THREADS = 320;
constexpr uint32_t NA_TILE = 32768;  // 128 rows x 256 B
constexpr int NA_KSLOTS = 3;         // K frees after Q K^T: three slots give the TMA two chunks of lead time
constexpr int NA_VSLOTS = 2;         // V frees after P V
// smem: Q | K0 K1 K2 | V0 V1 | barriers (256 B) | row-max / row-sum exchange (2 KB)
constexpr uint32_t NA_SMEM_BODY = (1 + NA_KSLOTS + NA_VSLOTS) * NA_TILE;
constexpr uint32_t NA_SMEM = NA_SMEM_BODY + 1024 /*align*/ + 256 /*barriers*/ + 2048 /*exchange*/;
// TMEM columns: S0 [0,128) S1 [128,256) O [256,384) P0 [384,448) P1 [448,512) (P: fp16 pairs per column)
constexpr uint32_t NA_TMEM_O = 256, NA_TMEM_P = 384;
constexpr float NA_RESCALE_LOG2 = 8.0f;

struct TileGeo {
  int head, d0, d1, h0, h1, w0, w1;
  int kd_lo, kr_lo, kr_hi, pc0, ncp, nrpc, nrchunks, nparts, nchunks;
};

// Key patch of a tile: depth planes [kd_lo, kd_hi), rows [kr_lo, kr_hi) (global, bumped like grid.py:96-101),
// columns either the whole circle (pc0 = 0, ncp = W) or the arc [pc0, pc0 + ncp) with pc0 = w0 - hw, which
// may cross the longitude seam.  A crossing arc is fetched as two TMA boxes of the same shape: part 0 at
// origin pc0 and part 1 at origin pc0 -/+ W; out-of-range columns of each box are zero-filled by TMA and
// masked, so together the two parts hold every key of the arc exactly once.
DEVI TileGeo tile_geo(const NaParams& p, int item) {
  TileGeo g;
  const int ntiles = p.ntd * p.nth * p.ntw;
  g.head = item / ntiles;
  const int tile = item - g.head * ntiles;
  const int tw_i = tile % p.ntw;
  const int th_i = (tile / p.ntw) % p.nth;
  const int td_i = tile / (p.ntw * p.nth);
  g.d0 = td_i * p.TD; g.d1 = min(g.d0 + p.TD, p.depth);
  g.h0 = th_i * p.TH; g.h1 = min(g.h0 + p.TH, p.rows);
  g.w0 = tw_i * p.TW; g.w1 = min(g.w0 + p.TW, p.cols);
  g.kd_lo = bump_start(g.d0, p.depth, p.wd);
  const int kd_hi = bump_start(g.d1 - 1, p.depth, p.wd) + p.wd;
  g.kr_lo = bump_start(g.h0 + p.row0, p.rows_global, p.wh);
  g.kr_hi = bump_start(g.h1 - 1 + p.row0, p.rows_global, p.wh) + p.wh;
  const int hw = (p.ww - 1) / 2;
  g.ncp = p.ncp;
  const bool circle = (p.ncp == p.cols);
  g.pc0 = circle ? 0 : g.w0 - hw;
  const int arc_end = g.w1 - 1 + (p.ww - 1 - hw);  // last column any query of the tile needs
  g.nparts = (!circle && (g.pc0 < 0 || arc_end >= p.cols)) ? 2 : 1;
  g.nrpc = p.nrpc;
  const int nrows_u = g.kr_hi - g.kr_lo;
  g.nrchunks = (nrows_u + g.nrpc - 1) / g.nrpc;
  g.nchunks = (kd_hi - g.kd_lo) * g.nrchunks * g.nparts;
  return g;
}

// chunk j -> depth plane, first key row, column origin and the patch columns [vlo, vhi) it holds
DEVI void chunk_geo(const TileGeo& g, int cols, int j, int& kd, int& kr0, int& nr, int& origin, int& vlo,
                    int& vhi) {
  const int part = j % g.nparts;
  const int jr = j / g.nparts;
  kd = g.kd_lo + jr / g.nrchunks;
  kr0 = g.kr_lo + (jr % g.nrchunks) * g.nrpc;
  nr = min(g.nrpc, g.kr_hi - kr0);
  // patch column cc is global column pc0 + cc; part 0 holds those inside [0, W), part 1 the wrapped ones
  const int in_lo = max(0, -g.pc0), in_hi = min(g.ncp, cols - g.pc0);
  if (part == 0) {
    origin = g.pc0; vlo = in_lo; vhi = in_hi;
  } else if (g.pc0 < 0) {
    origin = g.pc0 + cols; vlo = 0; vhi = in_lo;
  } else {
    origin = g.pc0 - cols; vlo = in_hi; vhi = g.ncp;
  }
}

// bits [a, b) of a 64-bit word (a, b clamped to [0, 64])
DEVI uint64_t bits64(int a, int b) {
  a = max(a, 0);
  b = min(b, 64);
  if (a >= b) return 0ull;
  const uint64_t hi = (b == 64) ? ~0ull : ((1ull << b) - 1ull);
  return hi & ~((1ull << a) - 1ull);
}

__global__ void __launch_bounds__(NA_THREADS, 1)
    natten_fwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmKV, NaParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sQ = smem_u32(smem);
  auto sK = [&](int s) { return sQ + NA_TILE * (1 + s); };
  auto sV = [&](int s) { return sQ + NA_TILE * (1 + NA_KSLOTS + s); };
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + NA_SMEM_BODY);
  const uint32_t b0 = smem_u32(bars);
  const uint32_t bar_qfull = b0 + 0, bar_qempty = b0 + 8;
  auto bar_kfull = [&](int s) { return b0 + 16 + 8 * s; };   // 3
  auto bar_kempty = [&](int s) { return b0 + 40 + 8 * s; };  // 3
  auto bar_vfull = [&](int s) { return b0 + 64 + 8 * s; };   // 2
  auto bar_vempty = [&](int s) { return b0 + 80 + 8 * s; };  // 2
  auto bar_sfull = [&](int s) { return b0 + 96 + 8 * s; };   // 2
  auto bar_sempty = [&](int s) { return b0 + 112 + 8 * s; }; // 2
  auto bar_pempty = [&](int s) { return b0 + 128 + 8 * s; }; // 2
  const uint32_t bar_pfull = b0 + 144, bar_ofull = b0 + 152, bar_oempty = b0 + 160;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 22);

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;

  if (tid == 0) {
    mbar_init(bar_qfull, 1);
    mbar_init(bar_qempty, 1);
    for (int s = 0; s < NA_KSLOTS; ++s) {
      mbar_init(bar_kfull(s), 1);
      mbar_init(bar_kempty(s), 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(bar_vfull(s), 1);
      mbar_init(bar_vempty(s), 1);
      mbar_init(bar_sfull(s), 1);
      mbar_init(bar_sempty(s), NA_SOFTMAX_WARPS);
      mbar_init(bar_pempty(s), 1);
    }
    mbar_init(bar_pfull, NA_SOFTMAX_WARPS);
    mbar_init(bar_ofull, 1);
    mbar_init(bar_oempty, NA_SOFTMAX_WARPS);
    fence_barrier_init();
  }
  if (warp == NA_MMA_WARP) {
    tmem_alloc(smem_u32(tmem_slot), 512);
    tmem_relinquish();
  }
  // Zero the operand tiles once: rows past a box are never written by TMA and V rows feed P V (0 * NaN).
  for (uint32_t off = tid * 16u; off < NA_SMEM_BODY; off += NA_THREADS * 16u) st_shared_v4(sQ + off, 0, 0, 0, 0);
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int sec = p.heads * p.dhp;  // columns per q/k/v section
  const int brow0 = p.row0 - p.halo_lo;

  if (warp == NA_TMA_WARP) {
    // =============================== TMA producer ===============================
    // K runs one chunk ahead of V (K slots free after Q K^T, V slots only after P V).
    if (lane == 0) {
      tma_prefetch(&tmQ);
      tma_prefetch(&tmKV);
      const int halves = p.dhp / 64;
      const uint32_t qbytes = halves * 128u * p.TW * p.TH * p.TD;
      const uint32_t kbytes = halves * 128u * p.ncp * p.nrpc;
      int chunk_ctr = 0, tile_ctr = 0;
      auto load_kv = [&](const TileGeo& g, int j, int c, bool is_v) {
        const int slot = is_v ? (c % NA_VSLOTS) : (c % NA_KSLOTS);
        const int use = is_v ? (c / NA_VSLOTS) : (c / NA_KSLOTS);
        int kd, kr0, nr, origin, vlo, vhi;
        chunk_geo(g, p.cols, j, kd, kr0, nr, origin, vlo, vhi);
        const uint32_t full = is_v ? bar_vfull(slot) : bar_kfull(slot);
        mbar_wait(is_v ? bar_vempty(slot) : bar_kempty(slot), (use & 1) ^ 1);
        mbar_arrive_expect_tx(full, kbytes);
        const int c1 = origin, c2 = kr0 - brow0;  // may be negative / past the edge: TMA zero-fills
        const uint32_t dst = is_v ? sV(slot) : sK(slot);
        const int col = (is_v ? 2 : 1) * sec + g.head * p.dhp;
        for (int h = 0; h < halves; ++h) tma_load_4d(dst + h * 16384u, &tmKV, full, col + 64 * h, c1, c2, kd);
      };
      for (int item = blockIdx.x; item < p.nitems; item += gridDim.x, ++tile_ctr) {
        const TileGeo g = tile_geo(p, item);
        mbar_wait(bar_qempty, (tile_ctr & 1) ^ 1);
        mbar_arrive_expect_tx(bar_qfull, qbytes);
        for (int h = 0; h < halves; ++h)
          tma_load_4d(sQ + h * 16384u, &tmQ, bar_qfull, g.head * p.dhp + 64 * h, g.w0, g.h0 + p.halo_lo, g.d0);
        for (int j = 0; j < g.nchunks; ++j, ++chunk_ctr) {
          load_kv(g, j, chunk_ctr, false);
          if (j > 0) load_kv(g, j - 1, chunk_ctr - 1, true);
        }
        load_kv(g, g.nchunks - 1, chunk_ctr - 1, true);
      }
    }
  } else if (warp == NA_MMA_WARP) {
    // =============================== MMA issuer ===============================
    if (lane == 0) {
      const uint32_t idesc_s = make_idesc(128, 128, 0, 0);
      const uint32_t idesc_o = make_idesc(128, p.dhp, 0, 1);
      const int kb = p.dhp / 64;
      const uint32_t tO = tmem + NA_TMEM_O;
      int chunk_ctr = 0, tile_ctr = 0;
      auto issue_pv = [&](int c, bool first, bool last) {
        const int vs = c % NA_VSLOTS, pb = c & 1;
        mbar_wait(bar_pfull, c & 1);
        mbar_wait(bar_vfull(vs), (c / NA_VSLOTS) & 1);
        if (first) mbar_wait(bar_oempty, (tile_ctr & 1) ^ 1);
        tc_fence_after();
        // O += P V: A = P from TMEM (fp16 pairs, 8 columns per 16 keys), B = V MN-major from its TMA tile
        for (int s = 0; s < (p.dbg >= 2 ? 0 : 8); ++s) {
          const uint64_t bd = make_sdesc_sw128(sV(vs) + s * 2048u, 16384, 1024);
          umma_f16_ts(tO, tmem + NA_TMEM_P + 64 * pb + 8 * s, bd, idesc_o, (!first || s > 0) ? 1u : 0u);
        }
        umma_commit(bar_vempty(vs));
        umma_commit(bar_pempty(pb));
        if (last) umma_commit(bar_ofull);
      };
      for (int item = blockIdx.x; item < p.nitems; item += gridDim.x, ++tile_ctr) {
        const TileGeo g = tile_geo(p, item);
        mbar_wait(bar_qfull, tile_ctr & 1);
        for (int j = 0; j < g.nchunks; ++j, ++chunk_ctr) {
          const int ks = chunk_ctr % NA_KSLOTS, ss = chunk_ctr & 1;
          mbar_wait(bar_kfull(ks), (chunk_ctr / NA_KSLOTS) & 1);
          mbar_wait(bar_sempty(ss), ((chunk_ctr >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t tS = tmem + 128 * ss;
          for (int s = 0; s < (p.dbg >= 2 ? 0 : kb * 4); ++s) {
            const uint32_t off = (s >> 2) * 16384u + (s & 3) * 32u;
            umma_bf16_ss(tS, make_sdesc_sw128(sQ + off, 16, 1024), make_sdesc_sw128(sK(ks) + off, 16, 1024),
                         idesc_s, s > 0 ? 1u : 0u);
          }
          umma_commit(bar_sfull(ss));
          umma_commit(bar_kempty(ks));
          if (j == g.nchunks - 1) umma_commit(bar_qempty);
          if (j > 0) issue_pv(chunk_ctr - 1, j - 1 == 0, false);
        }
        issue_pv(chunk_ctr - 1, g.nchunks == 1, true);
      }
    }
  } else if (warp < NA_SOFTMAX_WARPS) {
    // =============================== softmax / epilogue ===============================
    // Warp w owns query rows 32 (w % 4) .. +32 (its TMEM lane quarter) and half h = w / 4 of the key
    // columns (P columns) and of the O columns; the two warps of a quarter combine row maxima and sums
    // through shared memory (named barrier 1 + quarter, 64 threads).
    const int quarter = warp & 3, half = warp >> 2;
    const int row = 32 * quarter + lane;  // query row in the tile
    float* red = reinterpret_cast<float*>(smem + NA_SMEM_BODY + 256);  // [parity][half][128]
    const uint32_t lane_off = static_cast<uint32_t>(32 * quarter) << 16;
    const uint32_t tO = tmem + NA_TMEM_O;
    const int ocols = p.dhp / 2;  // O columns handled by this warp
    const int hw = (p.ww - 1) / 2;
    int chunk_ctr = 0, tile_ctr = 0;
    for (int item = blockIdx.x; item < p.nitems; item += gridDim.x, ++tile_ctr) {
      const TileGeo g = tile_geo(p, item);
      const int qd = g.d0 + row / (p.TH * p.TW);
      const int qh = g.h0 + (row / p.TW) % p.TH;
      const int qw = g.w0 + row % p.TW;
      const bool qvalid = row < p.TD * p.TH * p.TW && qd < g.d1 && qh < g.h1 && qw < g.w1;
      const int q_sd = bump_start(qvalid ? qd : g.d0, p.depth, p.wd);
      const int q_sh = bump_start((qvalid ? qh : g.h0) + p.row0, p.rows_global, p.wh);
      // window columns in patch coordinates: [c_lo, c_lo + ww), taken mod W for a full-circle patch
      const bool circle = (g.ncp == p.cols);
      const int c_lo = circle ? wrap_col((qvalid ? qw : g.w0) - hw, p.cols) : (qvalid ? qw : g.w0) - hw - g.pc0;
      float m_run = -INFINITY, l_run = 0.f;
      for (int j = 0; j < g.nchunks; ++j, ++chunk_ctr) {
        const int ss = chunk_ctr & 1, pb = chunk_ctr & 1;
        int kd, kr0, nr, origin, vlo, vhi;
        chunk_geo(g, p.cols, j, kd, kr0, nr, origin, vlo, vhi);
        // ---- validity bits of this warp's 64 key columns [64 half, 64 half + 64) ----
        uint64_t mk = 0;
        if (qvalid && kd >= q_sd && kd < q_sd + p.wd) {
          const int rlo = max(0, q_sh - kr0), rhi = min(nr, q_sh + p.wh - kr0);
          const int s1lo = max(c_lo, vlo), s1hi = min(c_lo + p.ww, vhi);
          const int s2hi = circle ? c_lo + p.ww - g.ncp : 0;
          const int off = 64 * half;
          for (int rr = rlo; rr < rhi; ++rr) {
            const int base = rr * g.ncp - off;
            mk |= bits64(base + s1lo, base + s1hi);
            if (s2hi > 0) mk |= bits64(base, base + s2hi);
          }
        }
        // ---- S half -> registers ----
        mbar_wait(bar_sfull(ss), (chunk_ctr >> 1) & 1);
        tc_fence_after();
        uint32_t s[64];
        tmem_ld32(tmem + 128 * ss + lane_off + 64 * half, *reinterpret_cast<uint32_t(*)[32]>(s));
        tmem_ld32(tmem + 128 * ss + lane_off + 64 * half + 32, *reinterpret_cast<uint32_t(*)[32]>(s + 32));
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_sempty(ss));
        uint32_t pk[32];
        float alpha = 1.f, lsum = 0.f;
        if (p.dbg) {
#pragma unroll
          for (int i = 0; i < 32; ++i) pk[i] = 0u;
        } else {
          // ---- masked row max (raw scores), combined with the partner warp ----
          // 8 independent accumulators: a serial 64-long FMNMX / FADD chain would be latency-bound.
          const uint32_t mlo = static_cast<uint32_t>(mk), mhi = static_cast<uint32_t>(mk >> 32);
          float mxa[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) mxa[i] = -INFINITY;
#pragma unroll
          for (int k = 0; k < 64; ++k) {
            const bool ok = ((k < 32 ? mlo : mhi) >> (k & 31)) & 1u;
            mxa[k & 7] = ok ? fmaxf(mxa[k & 7], __uint_as_float(s[k])) : mxa[k & 7];
          }
          float mx = fmaxf(fmaxf(fmaxf(mxa[0], mxa[1]), fmaxf(mxa[2], mxa[3])),
                           fmaxf(fmaxf(mxa[4], mxa[5]), fmaxf(mxa[6], mxa[7])));
          float* rbuf = red + (chunk_ctr & 1) * 256;  // parity buffers: the partner may still read the last one
          rbuf[half * 128 + row] = mx;
          named_bar_sync(1 + quarter, 64);
          mx = fmaxf(mx, rbuf[(half ^ 1) * 128 + row]);
          mx = mx * p.scale_log2;
          if (mx > m_run + NA_RESCALE_LOG2) {  // lazy rescale (also covers m_run = -inf); same in both warps
            alpha = exp2f(m_run - mx);
            m_run = mx;
          }
          const float m_use = (m_run == -INFINITY) ? 0.f : m_run;
          float lsa[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) lsa[i] = 0.f;
#pragma unroll
          for (int k = 0; k < 64; k += 2) {
            float p0 = fast_exp2(fmaf(__uint_as_float(s[k]), p.scale_log2, -m_use));
            float p1 = fast_exp2(fmaf(__uint_as_float(s[k + 1]), p.scale_log2, -m_use));
            p0 = (((k < 32 ? mlo : mhi) >> (k & 31)) & 1u) ? p0 : 0.f;
            p1 = (((k + 1 < 32 ? mlo : mhi) >> ((k + 1) & 31)) & 1u) ? p1 : 0.f;
            lsa[(k >> 1) & 7] += p0 + p1;
            pk[k >> 1] = pack_elem(p0, p1);
          }
          lsum = ((lsa[0] + lsa[1]) + (lsa[2] + lsa[3])) + ((lsa[4] + lsa[5]) + (lsa[6] + lsa[7]));
        }
        l_run = l_run * alpha + lsum;  // this warp's share of the row sum
        // ---- P buffer pb free once P V of chunk c-2 retired; a rescale also needs P V of chunk c-1 ----
        mbar_wait(bar_pempty(pb), ((chunk_ctr >> 1) & 1) ^ 1);
        if (j > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {
          mbar_wait(bar_pempty(pb ^ 1), ((chunk_ctr - 1) >> 1) & 1);
          tc_fence_after();
#pragma unroll 1
          for (int c = 0; c < ocols / 32; ++c) {
            uint32_t r[32];
            const uint32_t ta = tO + lane_off + half * ocols + 32 * c;
            tmem_ld32(ta, r);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 32; ++e) r[e] = __float_as_uint(__uint_as_float(r[e]) * alpha);
            tmem_st32(ta, r);
          }
        }
        tc_fence_after();
        tmem_st32(tmem + NA_TMEM_P + 64 * pb + 32 * half + lane_off, pk);  // keys [64 half, +64) of my row
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_pfull);
      }
      // ---- epilogue: O / l -> ctx (row sum = both halves) ----
      float* rl = red + ((chunk_ctr) & 1) * 256;  // the parity buffer no warp of this quarter still reads
      rl[half * 128 + row] = l_run;
      named_bar_sync(1 + quarter, 64);
      const float l_tot = l_run + rl[(half ^ 1) * 128 + row];
      mbar_wait(bar_ofull, tile_ctr & 1);
      tc_fence_after();
      const float inv_l = (qvalid && l_tot > 0.f) ? 1.f / l_tot : 0.f;
      elem_t* orow = p.out + (qvalid ? (static_cast<size_t>((qd * p.rows + qh) * p.cols + qw) * p.ldo +
                                        g.head * p.dhp + half * ocols)
                                     : 0);
#pragma unroll 1
      for (int c = 0; c < ocols / 32; ++c) {
        uint32_t r[32];
        tmem_ld32(tO + lane_off + half * ocols + 32 * c, r);
        tmem_ld_wait();
        if (qvalid) {
          uint4* d4 = reinterpret_cast<uint4*>(orow + 32 * c);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint4 u;
            u.x = pack_elem(__uint_as_float(r[8 * q + 0]) * inv_l, __uint_as_float(r[8 * q + 1]) * inv_l);
            u.y = pack_elem(__uint_as_float(r[8 * q + 2]) * inv_l, __uint_as_float(r[8 * q + 3]) * inv_l);
            u.z = pack_elem(__uint_as_float(r[8 * q + 4]) * inv_l, __uint_as_float(r[8 * q + 5]) * inv_l);
            u.w = pack_elem(__uint_as_float(r[8 * q + 6]) * inv_l, __uint_as_float(r[8 * q + 7]) * inv_l);
            d4[q] = u;
          }
        }
      }
      tc_fence_before();
      named_bar_sync(1 + quarter, 64);  // partner has read rl[] before the next tile writes this parity again
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_oempty);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == NA_MMA_WARP) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

__global__ void natten_windows_kernel(int depth, int rows, int cols, int rows_global, int row0, int wd, int wh,
                                      int ww, int32_t* out) {
  const int T = depth * rows * cols;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < T; t += gridDim.x * blockDim.x) {
    const int c = t % cols, r = (t / cols) % rows, d = t / (cols * rows);
    out[3 * t + 0] = bump_start(d, depth, wd);
    out[3 * t + 1] = bump_start(r + row0, rows_global, wh);
    out[3 * t + 2] = wrap_col(c - (ww - 1) / 2, cols);
  }
}

// Host-side query-tile choice: minimise (#tiles x (#chunks + 1)) over TD x TH x TW <= 128; also returns
// the fixed key-chunk box (ncp columns x nrpc rows, <= 128 keys).
static void choose_tile(int depth, int rows, int cols, int rows_global, int wd, int wh, int ww, int* TD, int* TH,
                        int* TW, int* NCP, int* NRPC) {
  long best = -1;
  for (int td = 1; td <= depth && td <= 128; ++td)
    for (int th = 1; th <= rows && td * th <= 128; ++th)
      for (int tw = 1; tw <= cols && td * th * tw <= 128; ++tw) {
        const int ncp = (tw + ww - 1 >= cols) ? cols : tw + ww - 1;
        if (ncp > 128) continue;
        const int nr_u = (th + wh - 1 < rows_global) ? th + wh - 1 : rows_global;
        const int nd_u = (td + wd - 1 < depth) ? td + wd - 1 : depth;
        const int nrpc = (nr_u < 128 / ncp) ? nr_u : 128 / ncp;
        const int nch = nd_u * ((nr_u + nrpc - 1) / nrpc);
        const long tiles = static_cast<long>((depth + td - 1) / td) * ((rows + th - 1) / th) * ((cols + tw - 1) / tw);
        const long cost = tiles * (nch + 1);
        if (best < 0 || cost < best) {
          best = cost; *TD = td; *TH = th; *TW = tw; *NCP = ncp; *NRPC = nrpc;
        }
      }
}

}  // namespace wm3

using namespace wm3;

extern "C" int wm3_natten_fwd(const void* qkv, int ldqkv, void* out, int ldo, int depth, int rows, int cols,
                              int rows_global, int row0, int halo_lo, int halo_hi, int heads, int dhp, int wd, int wh,
                              int ww, float scale, void* stream) {
  if (dhp != 64 && dhp != 128) return set_error("wm3_natten_fwd: dhp must be 64 or 128 (got %d)", dhp);
  if (wd > depth || wh > rows_global || ww > cols) return set_error("wm3_natten_fwd: window exceeds extents");
  if (ww > 64) return set_error("wm3_natten_fwd: col window %d > 64 unsupported", ww);
  if (row0 < 0 || row0 + rows > rows_global || halo_lo > row0 || row0 + rows + halo_hi > rows_global)
    return set_error("wm3_natten_fwd: bad band rows");
  // the halo must cover every window that reaches outside the band
  if (rows < rows_global) {
    const int need_lo = row0 - bump_start(row0, rows_global, wh);
    const int need_hi = bump_start(row0 + rows - 1, rows_global, wh) + wh - (row0 + rows);
    if (halo_lo < need_lo || halo_hi < need_hi)
      return set_error("wm3_natten_fwd: halos (%d,%d) smaller than window reach (%d,%d)", halo_lo, halo_hi, need_lo,
                       need_hi);
  }
  if ((ldqkv % 8) || (ldo % 8)) return set_error("wm3_natten_fwd: pitches must be multiples of 8");
  if (ldqkv < 3 * heads * dhp) return set_error("wm3_natten_fwd: ldqkv < 3 * heads * dhp");
  NaParams p{};
  p.out = reinterpret_cast<elem_t*>(out);
  p.ldo = ldo;
  p.depth = depth; p.rows = rows; p.cols = cols; p.rows_global = rows_global; p.row0 = row0;
  p.halo_lo = halo_lo; p.rows_ext = rows + halo_lo + halo_hi;
  p.heads = heads; p.dhp = dhp; p.wd = wd; p.wh = wh; p.ww = ww;
  choose_tile(depth, rows, cols, rows_global, wd, wh, ww, &p.TD, &p.TH, &p.TW, &p.ncp, &p.nrpc);
  p.ntd = (depth + p.TD - 1) / p.TD;
  p.nth = (rows + p.TH - 1) / p.TH;
  p.ntw = (cols + p.TW - 1) / p.TW;
  p.nitems = p.ntd * p.nth * p.ntw * heads;
  p.scale_log2 = scale * 1.4426950408889634f;
  {
    const char* e = getenv("WM3_NA_DEBUG");
    p.dbg = e ? atoi(e) : 0;
  }
  const uint64_t wp = cols;
  const uint64_t dims[4] = {static_cast<uint64_t>(3 * heads * dhp), wp, static_cast<uint64_t>(p.rows_ext),
                            static_cast<uint64_t>(depth)};
  const uint64_t strides[3] = {static_cast<uint64_t>(ldqkv), wp * ldqkv, wp * p.rows_ext * ldqkv};
  const uint32_t qbox[4] = {64, static_cast<uint32_t>(p.TW), static_cast<uint32_t>(p.TH), static_cast<uint32_t>(p.TD)};
  const uint32_t kvbox[4] = {64, static_cast<uint32_t>(p.ncp), static_cast<uint32_t>(p.nrpc), 1};
  CUtensorMap tq, tkv;
  if (make_tmap(&tq, qkv, TMAP_BF16, 4, dims, strides, qbox, nullptr)) return -1;
  if (make_tmap(&tkv, qkv, TMAP_BF16, 4, dims, strides, kvbox, nullptr)) return -1;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(natten_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, NA_SMEM);
    if (e != cudaSuccess) return set_error("cudaFuncSetAttribute(natten): %s", cudaGetErrorString(e));
    attr = true;
  }
  const int grid = p.nitems < sm_count() ? p.nitems : sm_count();
  natten_fwd_kernel<<<grid, NA_THREADS, NA_SMEM, reinterpret_cast<cudaStream_t>(stream)>>>(tq, tkv, p);
  return check_launch("natten_fwd_kernel");
}

extern "C" int wm3_natten_windows(int depth, int rows, int cols, int rows_global, int row0, int wd, int wh, int ww,
                                  int32_t* out, void* stream) {
  const int T = depth * rows * cols;
  if (T <= 0) return 0;
  int blocks = (T + 255) / 256;
  if (blocks > 4096) blocks = 4096;
  natten_windows_kernel<<<blocks, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(depth, rows, cols, rows_global,
                                                                                    row0, wd, wh, ww, out);
  return check_launch("natten_windows_kernel");
}
