// K1: fused 3D neighborhood attention forward on tcgen05 (reference attention.py:173-178,
// window arithmetic grid.py:96-130).
//
// Work item = (query tile, head).  A query tile is a TD x TH x TW box of tokens (<= 128 queries, one per
// TMEM lane).  The union of the tile's windows is walked as a list of key chunks, each a run of rows of
// one depth plane x a contiguous (mod W) run of columns, <= 128 keys.
//
// Persistent, warp-specialised CTA (one per SM, 256 threads):
//   warps 5-7   producers: cp.async gathers of the Q tile and of each chunk's K and V head slices into
//               SWIZZLE_128B tiles (double-buffered K/V slots), completion signalled on mbarriers
//   warp 4      MMA issuer (one thread): S = Q K^T into one of two TMEM S buffers (M128 N128 K=dhp),
//               O += P V (M128 N=dhp K=128, V read MN-major), O accumulated in TMEM across chunks;
//               S_{j+1} is issued before PV_j so the tensor core works while softmax runs
//   warps 0-3   softmax (one thread per query row): window bitmask built from the same integer formula
//               as grid.py (bump on depth/rows, wrap on cols), fp32 running max / sum with lazy O
//               rescaling (only when the max grows by > 2^8), exp2, P (bf16) -> smem; finally O / l ->
//               bf16 ctx rows.
// The logits never leave the SM.  Output ctx rows are bf16 [T][heads][dhp] = the O-proj GEMM operand.
#include "common.cuh"
#include "launch.h"
#include "window.cuh"
#include "../../include/wm3.h"

namespace wm3 {

struct NaParams {
  const __nv_bfloat16* qkv;
  int ldqkv;
  __nv_bfloat16* out;
  int ldo;
  int depth, rows, cols, rows_global, row0, halo_lo, rows_ext;
  int heads, dhp, wd, wh, ww;
  int TD, TH, TW, ntd, nth, ntw, nitems;
  float scale_log2;
};

constexpr int NA_THREADS = 256;
constexpr int NA_PRODUCER0 = 160;  // warps 5..7
constexpr int NA_NPRODUCERS = 96;
constexpr uint32_t NA_TILE = 32768;  // 128 rows x 256 B
// smem: Q | K0 V0 | K1 V1 | P
constexpr uint32_t NA_SMEM = 6 * NA_TILE + 1024 /*align*/ + 256 /*barriers*/;
constexpr float NA_RESCALE_LOG2 = 8.0f;

struct TileGeo {
  int head, d0, d1, h0, h1, w0, w1;
  int kd_lo, kr_lo, kr_hi, pc0, ncp, nrpc, nrchunks, nchunks;
};

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
  if ((g.w1 - g.w0) + p.ww - 1 >= p.cols) { g.pc0 = 0; g.ncp = p.cols; }
  else { g.pc0 = g.w0 - hw; g.ncp = (g.w1 - g.w0) + p.ww - 1; }
  const int nrows_u = g.kr_hi - g.kr_lo;
  g.nrpc = min(nrows_u, 128 / g.ncp);
  g.nrchunks = (nrows_u + g.nrpc - 1) / g.nrpc;
  g.nchunks = (kd_hi - g.kd_lo) * g.nrchunks;
  return g;
}

DEVI void chunk_geo(const TileGeo& g, int j, int& kd, int& kr0, int& nr) {
  kd = g.kd_lo + j / g.nrchunks;
  kr0 = g.kr_lo + (j % g.nrchunks) * g.nrpc;
  nr = min(g.nrpc, g.kr_hi - kr0);
}

// bits [a, b) of a 64-bit word (a, b clamped to [0, 64])
DEVI uint64_t bits64(int a, int b) {
  a = max(a, 0);
  b = min(b, 64);
  if (a >= b) return 0ull;
  const uint64_t hi = (b == 64) ? ~0ull : ((1ull << b) - 1ull);
  return hi & ~((1ull << a) - 1ull);
}

__global__ void __launch_bounds__(NA_THREADS, 1) natten_fwd_kernel(NaParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sQ = smem_u32(smem);
  auto sK = [&](int s) { return sQ + NA_TILE * (1 + 2 * s); };
  auto sV = [&](int s) { return sQ + NA_TILE * (2 + 2 * s); };
  const uint32_t sP = sQ + 5 * NA_TILE;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 6 * NA_TILE);
  const uint32_t b0 = smem_u32(bars);
  const uint32_t bar_qfull = b0 + 0, bar_qempty = b0 + 8;
  auto bar_kvfull = [&](int s) { return b0 + 16 + 8 * s; };
  auto bar_kvempty = [&](int s) { return b0 + 32 + 8 * s; };
  auto bar_sfull = [&](int s) { return b0 + 48 + 8 * s; };
  auto bar_sempty = [&](int s) { return b0 + 64 + 8 * s; };
  const uint32_t bar_pfull = b0 + 80, bar_pempty = b0 + 88, bar_ofull = b0 + 96, bar_oempty = b0 + 104;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 14);

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;

  if (tid == 0) {
    mbar_init(bar_qfull, NA_NPRODUCERS);
    mbar_init(bar_qempty, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(bar_kvfull(s), NA_NPRODUCERS);
      mbar_init(bar_kvempty(s), 1);
      mbar_init(bar_sfull(s), 1);
      mbar_init(bar_sempty(s), 4);
    }
    mbar_init(bar_pfull, 4);
    mbar_init(bar_pempty, 1);
    mbar_init(bar_ofull, 1);
    mbar_init(bar_oempty, 4);
    fence_barrier_init();
  }
  if (warp == 4) {
    tmem_alloc(smem_u32(tmem_slot), 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int sec = p.heads * p.dhp;  // columns per q/k/v section
  const int brow0 = p.row0 - p.halo_lo;

  if (tid >= NA_PRODUCER0) {
    // =============================== producers ===============================
    const int pt = tid - NA_PRODUCER0;
    const int cpr = p.dhp >> 3;  // 16-byte chunks per row (8 or 16)
    const int c16 = pt % cpr;
    const int rstep = NA_NPRODUCERS / cpr;
    const int r_first = pt / cpr;
    int chunk_ctr = 0, tile_ctr = 0;
    uint32_t pend0 = 0, pend1 = 0;  // barriers whose cp.async group is still in flight (0 = none)
    auto flush = [&]() {
      if (pend0 | pend1) {
        cp_async_wait<0>();
        fence_proxy_async();
        if (pend0) mbar_arrive(pend0);
        if (pend1) mbar_arrive(pend1);
        pend0 = pend1 = 0;
      }
    };
    auto retire_older = [&](uint32_t newest) {  // all but the newest committed group are complete
      cp_async_wait<1>();
      fence_proxy_async();
      if (pend0) mbar_arrive(pend0);
      if (pend1) mbar_arrive(pend1);
      pend0 = newest;
      pend1 = 0;
    };
    for (int item = blockIdx.x; item < p.nitems; item += gridDim.x, ++tile_ctr) {
      const TileGeo g = tile_geo(p, item);
      // ---- Q tile ----
      flush();
      mbar_wait(bar_qempty, (tile_ctr & 1) ^ 1);
      {
        const __nv_bfloat16* qb = p.qkv + g.head * p.dhp + c16 * 8;
        const int tq = p.TD * p.TH * p.TW;
        for (int r = r_first; r < 128; r += rstep) {
          const int rd = g.d0 + r / (p.TH * p.TW), rh = g.h0 + (r / p.TW) % p.TH, rw = g.w0 + r % p.TW;
          const bool ok = r < tq && rd < g.d1 && rh < g.h1 && rw < g.w1;
          const size_t tok = ok ? static_cast<size_t>((rd * p.rows_ext + rh + p.halo_lo) * p.cols + rw) : 0;
          cp_async_16(sQ + (c16 >> 3) * 16384u + sw128_off(r, c16 & 7), qb + tok * p.ldqkv, ok ? 16u : 0u);
        }
      }
      cp_async_commit();
      pend1 = pend0;
      pend0 = bar_qfull;  // newest
      // ---- K/V chunks ----
      for (int j = 0; j < g.nchunks; ++j, ++chunk_ctr) {
        const int slot = chunk_ctr & 1;
        int kd, kr0, nr;
        chunk_geo(g, j, kd, kr0, nr);
        const int nkeys = nr * g.ncp;
        // The slot frees when PV of chunk c-2 retires, which the MMA thread issues only after S of chunk
        // c-1, which needs chunk c-1's arrival: publish pending groups before blocking.
        if (!mbar_try_wait(bar_kvempty(slot), ((chunk_ctr >> 1) & 1) ^ 1)) {
          flush();
          mbar_wait(bar_kvempty(slot), ((chunk_ctr >> 1) & 1) ^ 1);
        }
        const __nv_bfloat16* kb = p.qkv + sec + g.head * p.dhp + c16 * 8;
        const __nv_bfloat16* vb = kb + sec;
        const uint32_t dk = sK(slot) + (c16 >> 3) * 16384u;
        const uint32_t dv = sV(slot) + (c16 >> 3) * 16384u;
        int rr = r_first / g.ncp, cc = r_first - (r_first / g.ncp) * g.ncp;
        const int step_r = rstep / g.ncp, step_c = rstep - step_r * g.ncp;
        const size_t plane_base = static_cast<size_t>(kd) * p.rows_ext;
        for (int r = r_first; r < 128; r += rstep) {
          const bool ok = r < nkeys;
          const size_t tok =
              ok ? (plane_base + (kr0 + rr - brow0)) * p.cols + wrap_col(g.pc0 + cc, p.cols) : 0;
          const uint32_t so = sw128_off(r, c16 & 7);
          cp_async_16(dk + so, kb + tok * p.ldqkv, ok ? 16u : 0u);
          cp_async_16(dv + so, vb + tok * p.ldqkv, ok ? 16u : 0u);
          rr += step_r;
          cc += step_c;
          if (cc >= g.ncp) { cc -= g.ncp; ++rr; }
        }
        cp_async_commit();
        retire_older(bar_kvfull(slot));
      }
    }
    flush();
  } else if (warp == 4) {
    // =============================== MMA issuer ===============================
    if (lane == 0) {
      const uint32_t idesc_s = make_idesc_bf16(128, 128, 0, 0);
      const uint32_t idesc_o = make_idesc_bf16(128, p.dhp, 0, 1);
      const int kb = p.dhp / 64;
      const uint32_t tO = tmem + 256;
      int chunk_ctr = 0, tile_ctr = 0;
      auto issue_pv = [&](int c, bool first, bool last) {
        const int slot = c & 1;
        mbar_wait(bar_pfull, c & 1);
        if (first) mbar_wait(bar_oempty, (tile_ctr & 1) ^ 1);
        tc_fence_after();
        for (int s = 0; s < 8; ++s) {
          const uint64_t ad = make_sdesc_sw128(sP + (s >> 2) * 16384u + (s & 3) * 32u, 16, 1024);
          const uint64_t bd = make_sdesc_sw128(sV(slot) + s * 2048u, 16384, 1024);
          umma_bf16_ss(tO, ad, bd, idesc_o, (!first || s > 0) ? 1u : 0u);
        }
        umma_commit(bar_kvempty(slot));
        umma_commit(bar_pempty);
        if (last) umma_commit(bar_ofull);
      };
      for (int item = blockIdx.x; item < p.nitems; item += gridDim.x, ++tile_ctr) {
        const TileGeo g = tile_geo(p, item);
        mbar_wait(bar_qfull, tile_ctr & 1);
        const int c0 = chunk_ctr;
        for (int j = 0; j < g.nchunks; ++j, ++chunk_ctr) {
          const int slot = chunk_ctr & 1;
          mbar_wait(bar_kvfull(slot), (chunk_ctr >> 1) & 1);
          mbar_wait(bar_sempty(slot), ((chunk_ctr >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t tS = tmem + 128 * slot;
          for (int s = 0; s < kb * 4; ++s) {
            const uint32_t off = (s >> 2) * 16384u + (s & 3) * 32u;
            umma_bf16_ss(tS, make_sdesc_sw128(sQ + off, 16, 1024), make_sdesc_sw128(sK(slot) + off, 16, 1024),
                         idesc_s, s > 0 ? 1u : 0u);
          }
          umma_commit(bar_sfull(slot));
          if (j == g.nchunks - 1) umma_commit(bar_qempty);
          if (j > 0) issue_pv(chunk_ctr - 1, j - 1 == 0, false);
        }
        issue_pv(chunk_ctr - 1, g.nchunks == 1, true);
        (void)c0;
      }
    }
  } else if (warp < 4) {
    // =============================== softmax / epilogue ===============================
    const uint32_t lane_off = static_cast<uint32_t>(32 * warp) << 16;
    const uint32_t tO = tmem + 256;
    const int hw = (p.ww - 1) / 2;
    int chunk_ctr = 0, tile_ctr = 0;
    for (int item = blockIdx.x; item < p.nitems; item += gridDim.x, ++tile_ctr) {
      const TileGeo g = tile_geo(p, item);
      const int qd = g.d0 + tid / (p.TH * p.TW);
      const int qh = g.h0 + (tid / p.TW) % p.TH;
      const int qw = g.w0 + tid % p.TW;
      const bool qvalid = tid < p.TD * p.TH * p.TW && qd < g.d1 && qh < g.h1 && qw < g.w1;
      const int q_sd = bump_start(qvalid ? qd : g.d0, p.depth, p.wd);
      const int q_sh = bump_start((qvalid ? qh : g.h0) + p.row0, p.rows_global, p.wh);
      // window columns inside the patch: [c_lo, c_lo + ww) mod ncp-circle
      const int c_lo = wrap_col((qvalid ? qw : g.w0) - hw - g.pc0, p.cols);
      float m_run = -INFINITY, l_run = 0.f;
      for (int j = 0; j < g.nchunks; ++j, ++chunk_ctr) {
        const int slot = chunk_ctr & 1;
        int kd, kr0, nr;
        chunk_geo(g, j, kd, kr0, nr);
        // ---- validity bitmask over the 128 key columns of this chunk ----
        uint64_t mk0 = 0, mk1 = 0;
        if (qvalid && kd >= q_sd && kd < q_sd + p.wd) {
          const int rlo = max(0, q_sh - kr0), rhi = min(nr, q_sh + p.wh - kr0);
          const int s1hi = min(c_lo + p.ww, g.ncp);
          const int s2hi = c_lo + p.ww - g.ncp;  // wrapped part (full-circle patch only)
          for (int rr = rlo; rr < rhi; ++rr) {
            const int base = rr * g.ncp;
            mk0 |= bits64(base + c_lo, base + s1hi);
            mk1 |= bits64(base + c_lo - 64, base + s1hi - 64);
            if (s2hi > 0) {
              mk0 |= bits64(base, base + s2hi);
              mk1 |= bits64(base - 64, base + s2hi - 64);
            }
          }
        }
        // ---- S -> registers ----
        mbar_wait(bar_sfull(slot), (chunk_ctr >> 1) & 1);
        tc_fence_after();
        uint32_t s[128];
        {
          uint32_t* s0 = s;
          tmem_ld32(tmem + 128 * slot + lane_off + 0, *reinterpret_cast<uint32_t(*)[32]>(s0));
          tmem_ld32(tmem + 128 * slot + lane_off + 32, *reinterpret_cast<uint32_t(*)[32]>(s0 + 32));
          tmem_ld32(tmem + 128 * slot + lane_off + 64, *reinterpret_cast<uint32_t(*)[32]>(s0 + 64));
          tmem_ld32(tmem + 128 * slot + lane_off + 96, *reinterpret_cast<uint32_t(*)[32]>(s0 + 96));
        }
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_sempty(slot));
        // ---- masked row max (log2 domain) ----
        float mx = -INFINITY;
#pragma unroll
        for (int k = 0; k < 128; ++k) {
          const uint64_t w = k < 64 ? mk0 : mk1;
          const bool ok = (w >> (k & 63)) & 1ull;
          mx = ok ? fmaxf(mx, __uint_as_float(s[k])) : mx;
        }
        mx = mx * p.scale_log2;
        float alpha = 1.f;
        if (mx > m_run + NA_RESCALE_LOG2) {  // lazy rescale (also covers m_run = -inf)
          alpha = exp2f(m_run - mx);
          m_run = mx;
        }
        const float m_use = (m_run == -INFINITY) ? 0.f : m_run;
        float lsum = 0.f;
        uint32_t pk[64];
#pragma unroll
        for (int k = 0; k < 128; k += 2) {
          const uint64_t w = k < 64 ? mk0 : mk1;
          const bool ok0 = (w >> (k & 63)) & 1ull;
          const bool ok1 = (w >> ((k + 1) & 63)) & 1ull;
          const float p0 = ok0 ? exp2f(fmaf(__uint_as_float(s[k]), p.scale_log2, -m_use)) : 0.f;
          const float p1 = ok1 ? exp2f(fmaf(__uint_as_float(s[k + 1]), p.scale_log2, -m_use)) : 0.f;
          lsum += p0 + p1;
          pk[k >> 1] = pack_bf16(p0, p1);
        }
        l_run = l_run * alpha + lsum;
        // ---- P buffer free (previous PV retired) -> rescale O if needed, write P ----
        mbar_wait(bar_pempty, (chunk_ctr & 1) ^ 1);
        tc_fence_after();
        if (j > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll 1
          for (int c = 0; c < p.dhp / 32; ++c) {
            uint32_t r[32];
            tmem_ld32(tO + lane_off + 32 * c, r);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 32; ++e) r[e] = __float_as_uint(__uint_as_float(r[e]) * alpha);
            tmem_st32(tO + lane_off + 32 * c, r);
          }
          tmem_st_wait();
        }
#pragma unroll
        for (int q = 0; q < 16; ++q) {  // keys [8q, 8q+8) -> region q/8, 16B chunk q%8
          st_shared_v4(sP + (q >> 3) * 16384u + sw128_off(tid, q & 7), pk[4 * q], pk[4 * q + 1], pk[4 * q + 2],
                       pk[4 * q + 3]);
        }
        fence_proxy_async();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_pfull);
      }
      // ---- epilogue: O / l -> bf16 ctx ----
      mbar_wait(bar_ofull, tile_ctr & 1);
      tc_fence_after();
      const float inv_l = (qvalid && l_run > 0.f) ? 1.f / l_run : 0.f;
      __nv_bfloat16* orow =
          p.out + (qvalid ? (static_cast<size_t>((qd * p.rows + qh) * p.cols + qw) * p.ldo + g.head * p.dhp) : 0);
#pragma unroll 1
      for (int c = 0; c < p.dhp / 32; ++c) {
        uint32_t r[32];
        tmem_ld32(tO + lane_off + 32 * c, r);
        tmem_ld_wait();
        if (qvalid) {
          uint4* d4 = reinterpret_cast<uint4*>(orow + 32 * c);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint4 u;
            u.x = pack_bf16(__uint_as_float(r[8 * q + 0]) * inv_l, __uint_as_float(r[8 * q + 1]) * inv_l);
            u.y = pack_bf16(__uint_as_float(r[8 * q + 2]) * inv_l, __uint_as_float(r[8 * q + 3]) * inv_l);
            u.z = pack_bf16(__uint_as_float(r[8 * q + 4]) * inv_l, __uint_as_float(r[8 * q + 5]) * inv_l);
            u.w = pack_bf16(__uint_as_float(r[8 * q + 6]) * inv_l, __uint_as_float(r[8 * q + 7]) * inv_l);
            d4[q] = u;
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_oempty);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 4) {
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

// Host-side query-tile choice: minimise (#tiles x (#chunks + 1)) over TD x TH x TW <= 128.
static void choose_tile(int depth, int rows, int cols, int wd, int wh, int ww, int* TD, int* TH, int* TW) {
  long best = -1;
  for (int td = 1; td <= depth && td <= 128; ++td)
    for (int th = 1; th <= rows && td * th <= 128; ++th)
      for (int tw = 1; tw <= cols && td * th * tw <= 128; ++tw) {
        const int ncp = (tw + ww - 1 >= cols) ? cols : tw + ww - 1;
        if (ncp > 128) continue;
        const int nr_u = (th + wh - 1 < rows) ? th + wh - 1 : rows;
        const int nd_u = (td + wd - 1 < depth) ? td + wd - 1 : depth;
        const int nrpc = (nr_u < 128 / ncp) ? nr_u : 128 / ncp;
        const int nch = nd_u * ((nr_u + nrpc - 1) / nrpc);
        const long tiles = static_cast<long>((depth + td - 1) / td) * ((rows + th - 1) / th) * ((cols + tw - 1) / tw);
        const long cost = tiles * (nch + 1);
        if (best < 0 || cost < best) { best = cost; *TD = td; *TH = th; *TW = tw; }
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
  NaParams p{};
  p.qkv = reinterpret_cast<const __nv_bfloat16*>(qkv);
  p.ldqkv = ldqkv;
  p.out = reinterpret_cast<__nv_bfloat16*>(out);
  p.ldo = ldo;
  p.depth = depth; p.rows = rows; p.cols = cols; p.rows_global = rows_global; p.row0 = row0;
  p.halo_lo = halo_lo; p.rows_ext = rows + halo_lo + halo_hi;
  p.heads = heads; p.dhp = dhp; p.wd = wd; p.wh = wh; p.ww = ww;
  choose_tile(depth, rows, cols, wd, wh, ww, &p.TD, &p.TH, &p.TW);
  p.ntd = (depth + p.TD - 1) / p.TD;
  p.nth = (rows + p.TH - 1) / p.TH;
  p.ntw = (cols + p.TW - 1) / p.TW;
  p.nitems = p.ntd * p.nth * p.ntw * heads;
  p.scale_log2 = scale * 1.4426950408889634f;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(natten_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, NA_SMEM);
    if (e != cudaSuccess) return set_error("cudaFuncSetAttribute(natten): %s", cudaGetErrorString(e));
    attr = true;
  }
  const int grid = p.nitems < sm_count() ? p.nitems : sm_count();
  natten_fwd_kernel<<<grid, NA_THREADS, NA_SMEM, reinterpret_cast<cudaStream_t>(stream)>>>(p);
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
