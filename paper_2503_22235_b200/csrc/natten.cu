// K1: fused 3D neighborhood attention forward on tcgen05 (reference attention.py:173-178,
// window arithmetic grid.py:96-130).
//
// Work item = (query tile, head, member).  A query tile is a TD x TH x TW box of tokens (<= 128 queries, one
// per TMEM lane).  The union of the tile's windows is walked as a list of key chunks, each a run of rows of
// one depth plane x a contiguous (mod W) run of columns, <= 128 keys.
//
// Two persistent CTAs per SM (192 threads, 256 TMEM columns and ~100 KB smem each).  Inside a CTA the
// chunk loop is a strict chain S(c) -> softmax(c) -> P V(c) -> S(c + 1); the second CTA on the SM fills
// the tensor core while the first one is in softmax (and vice versa), which hides the handshake latencies
// that a single deeper-pipelined CTA exposes.
//   warp 5      TMA producer (one thread): the Q tile (4D box TD x TH x TW) and each chunk's K and V head
//               slices (4D box ncp x nrpc) into SWIZZLE_128B tiles; K(c + 1) streams in while softmax(c)
//               runs, V(c + 1) while S(c + 1) and softmax(c + 1) run
//   warp 4      MMA issuer (one thread): S = Q K^T into TMEM columns [0, 128) (M128 N128 K=dhp, both operands
//               from smem), then O += P V with P (fp16 pairs) read from TMEM columns [0, 64) where softmax
//               wrote it over S (M128 N=dhp K=128, V MN-major from its TMA tile), O in columns [128, 256)
//   warps 0-3   softmax (one thread per query row, all 128 key columns of the chunk): window bitmask built
//               from the same integer formula as grid.py (bump on depth/rows, wrap on cols), fp32 running
//               max / sum with lazy O rescaling (only when the max grows by > 2^8), exp2, P -> TMEM; at the
//               end of a tile O / l -> ctx rows.
// The logits never leave the SM.  Output ctx rows are bf16 [T][heads][dhp] = the O-proj GEMM operand.
#include <cstdio>
#include <map>
#include <mutex>
#include <tuple>

#include "common.cuh"
#include "launch.h"
#include "window.cuh"
#include "../../include/wm3.h"

namespace wm3 {

// Event trace of one CTA (WM3_NA_TRACE builds only): (event, counter, clock) triples for a timeline of the
// hand-off chain.  Events: 0/1 softmax sfull wait begin/end, 2 softmax P arrive, 3/4 MMA pfull wait
// begin/end, 5/6 MMA vfull wait, 7/8 MMA kfull wait, 9 MMA issue done, 10/11 TMA empty wait, 12/13 ofull wait.
#ifdef WM3_NA_TRACE
constexpr int NA_TRACE_MAX = 1 << 16;
__device__ long long g_na_trace[NA_TRACE_MAX][3];
__device__ int g_na_trace_n;
DEVI void na_ev(int e, int c) {
  if (blockIdx.x != 0 || (threadIdx.x & 31) != 0) return;
  const int i = atomicAdd(&g_na_trace_n, 1);
  if (i < NA_TRACE_MAX) {
    g_na_trace[i][0] = e;
    g_na_trace[i][1] = c;
    g_na_trace[i][2] = clock64();
  }
}
#define NA_EV(e, c) na_ev(e, c)
#else
#define NA_EV(e, c)
#endif

struct NaParams {
  elem_t* out;
  int ldo;
  int batch;  // ensemble members: the K/V grid holds batch * depth planes, member b at planes [b * depth, ...)
  int depth, rows, cols, rows_global, row0, halo_lo, rows_ext;
  int heads, dhp, wd, wh, ww;
  int TD, TH, TW, ntd, nth, ntw, nitems;
  int th_first;   // first global row tile the launch touches (tiles are aligned to global rows, see tile_geo)
  int q_lo, q_hi;  // global query rows this launch computes and stores: [q_lo, q_hi) within the band
  int ncp, nrpc;  // key-chunk box: ncp columns x nrpc rows (fixed for every tile)
  float scale_log2;
  float* lse;  // optional [token][head]: log2-domain log-sum-exp of the row (m + log2 l), for the backward
  const uint8_t* bias_table;  // BIAS: [tile][maxch] B_x images (4 KB each), built once per geometry
  int maxch;
  int heavy_lo, heavy_hi;  // first / last column tile crosses the longitude seam (2 chunk parts: twice the work)
};

#ifndef WM3_NA_SPLIT
#define WM3_NA_SPLIT 1
#endif
// Softmax threads per query row: each handles 64 / NA_SPLIT of the 64 columns of an S half (the partner
// threads of a row sit in warps w and w + 4, which see the same TMEM lanes) and they exchange the row max
// through shared memory, which halves the per-half softmax chain.
constexpr int NA_SPLIT = WM3_NA_SPLIT;
constexpr int NA_SOFTMAX_WARPS = 4 * NA_SPLIT;
constexpr int NA_MMA_WARP = NA_SOFTMAX_WARPS;
constexpr int NA_TMA_WARP = NA_SOFTMAX_WARPS + 1;
constexpr int NA_THREADS = 32 * (NA_SOFTMAX_WARPS + 2);
constexpr int NA_CTAS_PER_SM = 2;
constexpr uint32_t NA_TILE = 32768;  // 128 rows x 256 B
// smem: Q | K | V | barriers (256 B) | row-max / row-sum exchange (2 halves + 1) x NA_SPLIT x 128 floats
// Window mask as one extra K = 16 step of Q K^T (kernel template BIAS): A_x = one-hot query classes (tile
// depth / row / column position, 128 x 16, built once per CTA), B_x = the chunk's key bias (0, or NA_MASKED
// where a class's window misses the key), fp16 in the no-swizzle K-major core-matrix layout (4 KB each).  The
// B_x images of every (tile, chunk) are precomputed once per geometry (natten_bias_table_kernel) and loaded
// with the chunk's K by one bulk copy.  The softmax then needs no per-element mask: a masked logit is ~-3e4
// and never wins the row max; a query whose first key half is entirely masked accumulates garbage that the
// lazy rescale multiplies by exp2(-huge) = 0 as soon as its first real key arrives.
constexpr uint32_t NA_XTRA = 8192;  // A_x and the B_x slot (loaded with K, same lifetime)
constexpr float NA_MASKED = -30000.f;
constexpr uint32_t NA_SMEM_BODY = 3 * NA_TILE + NA_XTRA;
constexpr uint32_t NA_RED_BYTES = NA_SPLIT > 1 ? 3 * NA_SPLIT * 128 * 4 : 0;  // (2 CTAs per SM must fit)
constexpr uint32_t NA_SMEM = NA_SMEM_BODY + 1024 /*align*/ + 256 /*barriers*/ + NA_RED_BYTES;
// TMEM columns (256 per CTA): S / P [0, 128), O [128, 256).  S(c + 1) may overwrite P(c) without a wait
// because tcgen05.mma ops of one thread execute in issue order and S(c + 1) is issued after P V(c).
constexpr uint32_t NA_TMEM_COLS = 256, NA_TMEM_O = 128;
constexpr float NA_RESCALE_LOG2 = 8.0f;
#ifndef WM3_NA_DBG
#define WM3_NA_DBG 0
#endif
// Profiling build switch (tools/build_variant.sh -DWM3_NA_DBG=...), bit flags: 1 skip softmax arithmetic,
// 2 skip Q K^T, 4 skip P V, 8 skip K/V loads.  Compile-time so the product build carries no checks.
constexpr int NA_DBG = WM3_NA_DBG;
#ifndef WM3_NA_EMU
#define WM3_NA_EMU 0
#endif
// Of every 8 key pairs of a half, NA_EMU have their exp2 evaluated on the FMA pipe (exp2_fma2) instead of the
// MUFU, which otherwise is the softmax's binding pipe (64 MUFU.EX2 per thread per 64-key half).
constexpr int NA_EMU = WM3_NA_EMU;

// 2^x for a pair on the FMA / ALU pipes: x = n + f (n = rint(x) by the 1.5 * 2^23 shift, f in [-0.5, 0.5]),
// 2^f by a degree-3 polynomial (relative error 7.5e-5, below the fp16 rounding of P), n added to the exponent
// field.  x is clamped at -125 (masked keys: the result is ~2^-125, i.e. 0 once rounded to fp16).
DEVI void exp2_fma2(float& p0, float& p1, float x0, float x1) {
  x0 = fmaxf(x0, -125.f);
  x1 = fmaxf(x1, -125.f);
  float t0, t1, n0, n1, f0, f1, q0, q1;
  fadd2(t0, t1, x0, x1, 12582912.f, 12582912.f);
  fadd2(n0, n1, t0, t1, -12582912.f, -12582912.f);
  fadd2(f0, f1, x0, x1, -n0, -n1);
  ffma2(q0, q1, f0, f1, 0.05517132207751274f, 0.05517132207751274f, 0.24261054396629333f, 0.24261054396629333f);
  ffma2(q0, q1, q0, q1, f0, f1, 0.6932609677314758f, 0.6932609677314758f);
  ffma2(q0, q1, q0, q1, f0, f1, 0.9999281167984009f, 0.9999281167984009f);
  p0 = __int_as_float(__float_as_int(q0) + (__float_as_int(t0) << 23));
  p1 = __int_as_float(__float_as_int(q1) + (__float_as_int(t1) << 23));
}

struct TileGeo {
  int tile, hb;  // raw tile index (d-, h-, w-major) and head x member index of the work item
  int head, b, d0, d1, h0, h1, w0, w1;
  int kd_lo, kr_lo, kr_hi, pc0, ncp, nrpc, nrchunks, nparts, nchunks;
};

// Key patch of a tile: depth planes [kd_lo, kd_hi), rows [kr_lo, kr_hi) (global, bumped like grid.py:96-101),
// columns either the whole circle (pc0 = 0, ncp = W) or the arc [pc0, pc0 + ncp) with pc0 = w0 - hw, which
// may cross the longitude seam.  A crossing arc is fetched as two TMA boxes of the same shape: part 0 at
// origin pc0 and part 1 at origin pc0 -/+ W; out-of-range columns of each box are zero-filled by TMA and
// masked, so together the two parts hold every key of the arc exactly once.
// Work item -> (head x member, tile).  The seam-crossing column tiles (heavy_lo / heavy_hi: two chunk parts, twice
// the work) come first, for every head and member, then the rest head-major: with the persistent CTAs taking items
// round-robin every CTA gets at most one heavy item, instead of some CTAs collecting them (measured: 8 % of the
// launch lost to the most loaded CTA with a plain head-major order at full scale).
DEVI void item_tile(const NaParams& p, int item, int& hb, int& tile) {
  const int ntiles = p.ntd * p.nth * p.ntw;
  const int nhv = p.heavy_lo + p.heavy_hi;
  const int nh = nhv * p.ntd * p.nth;  // heavy tiles per head x member
  const int nhb = p.nitems / ntiles;
  if (nh == 0) {
    hb = item / ntiles;
    tile = item - hb * ntiles;
    return;
  }
  if (item < nh * nhb) {
    hb = item / nh;
    const int k = item - hb * nh;
    const int dh = k / nhv, v = k - dh * nhv;
    tile = dh * p.ntw + ((p.heavy_lo && v == 0) ? 0 : p.ntw - 1);
  } else {
    const int j = item - nh * nhb, nl = ntiles - nh, nlw = p.ntw - nhv;
    hb = j / nl;
    const int k = j - hb * nl;
    const int dh = k / nlw;
    tile = dh * p.ntw + p.heavy_lo + (k - dh * nlw);
  }
}

DEVI TileGeo tile_geo_raw(const NaParams& p, int hb, int tile) {
  TileGeo g;
  g.tile = tile;
  g.hb = hb;
  g.head = hb / p.batch;
  g.b = hb - g.head * p.batch;
  const int tw_i = tile % p.ntw;
  const int th_i = (tile / p.ntw) % p.nth;
  const int td_i = tile / (p.ntw * p.nth);
  g.d0 = td_i * p.TD; g.d1 = min(g.d0 + p.TD, p.depth);
  // Rows are GLOBAL and the row tiles are aligned to multiples of TH of the global grid, whatever the band:
  // a query then sees the same key chunks, in the same order and slot positions, whether its band is the
  // whole latent or one of N latitude bands, so N-band results are bitwise the single-GPU ones.  Tile rows
  // outside the band are not stored; key rows outside the band's grid are zero-filled by TMA and masked.
  g.h0 = (p.th_first + th_i) * p.TH; g.h1 = min(g.h0 + p.TH, p.rows_global);
  g.w0 = tw_i * p.TW; g.w1 = min(g.w0 + p.TW, p.cols);
  g.kd_lo = bump_start(g.d0, p.depth, p.wd);
  const int kd_hi = bump_start(g.d1 - 1, p.depth, p.wd) + p.wd;
  g.kr_lo = bump_start(g.h0, p.rows_global, p.wh);
  g.kr_hi = bump_start(g.h1 - 1, p.rows_global, p.wh) + p.wh;
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

DEVI TileGeo tile_geo(const NaParams& p, int item) {
  int hb, tile;
  item_tile(p, item, hb, tile);
  return tile_geo_raw(p, hb, tile);
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

// m |= bits [a, b) of a 128-bit mask held as 4 words (a, b may lie outside [0, 128)); branch-free
DEVI void set_bits128(uint32_t (&m)[4], int a, int b) {
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    const int lo = min(max(a - 32 * w, 0), 32), hi = min(max(b - 32 * w, 0), 32);
    m[w] |= __funnelshift_lc(0u, 0xffffffffu, lo) & ~__funnelshift_lc(0u, 0xffffffffu, hi);
  }
}

// Window bits of one query over a chunk box of nr x ncp keys (key k = rr * ncp + cc): rows [rlo, rhi),
// columns [s1lo, s1hi) plus the wrapped run [0, s2hi) of a full-circle patch.  nr is warp-uniform.
DEVI void window_mask(uint32_t (&m)[4], int nr, int ncp, int rlo, int rhi, int s1lo, int s1hi, int s2hi) {
  m[0] = m[1] = m[2] = m[3] = 0u;
  for (int rr = 0; rr < nr; ++rr) {
    const bool on = rr >= rlo && rr < rhi;
    const int base = rr * ncp;
    set_bits128(m, on ? base + s1lo : 0, on ? base + s1hi : 0);
    set_bits128(m, base, on ? base + s2hi : base);
  }
}

// smem descriptor of a K-major operand in the no-swizzle core-matrix layout: core matrix (8 rows x 16 B) at
// (row / 8) * 256 + (k / 8) * 128 (LBO = 128 B between K-adjacent cores, SBO = 256 B between row groups)
DEVI uint64_t make_sdesc_interleave(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((128u >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((256u >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  return d;  // layout type 0: SWIZZLE_NONE
}
DEVI uint32_t xtra_off(int r, int kc) { return (r >> 3) * 256u + kc * 128u + (r & 7) * 16u; }

// Row `k` of the B_x image of chunk j of tile g: per query class (tile depth td, row th, column tw) 0 if the
// class's window (grid.py bump / wrap, the same formulas as window_mask) holds key k, else NA_MASKED; padding
// keys are masked through their row classes.
DEVI void bx_row(const NaParams& p, const TileGeo& g, int j, int k, uint32_t (&u)[8]) {
  int kd, kr0, nr, origin, vlo, vhi;
  chunk_geo(g, p.cols, j, kd, kr0, nr, origin, vlo, vhi);
  const int rr = k / g.ncp, cc = k - rr * g.ncp;
  const bool key_ok = rr < nr;
  const int kr = kr0 + rr;
  const int hw = (p.ww - 1) / 2;
  const bool circle = (g.ncp == p.cols);
  const uint32_t masked = pack_elem(NA_MASKED, 0.f) & 0xffffu;  // operand encoding (kElemFmt) of the bias
#pragma unroll
  for (int i = 0; i < 8; ++i) u[i] = 0u;  // fp16 0 = open
#pragma unroll
  for (int cl = 0; cl < 16; ++cl) {
    bool ok = true;
    if (cl < p.TD) {
      const int sd = bump_start(min(g.d0 + cl, p.depth - 1), p.depth, p.wd);
      ok = kd >= sd && kd < sd + p.wd;
    } else if (cl < p.TD + p.TH) {
      const int sh = bump_start(min(g.h0 + cl - p.TD, p.rows_global - 1), p.rows_global, p.wh);
      ok = key_ok && kr >= sh && kr < sh + p.wh;
    } else if (cl < p.TD + p.TH + p.TW) {
      const int qw = min(g.w0 + cl - p.TD - p.TH, p.cols - 1);
      const int c_lo = circle ? wrap_col(qw - hw, p.cols) : qw - hw - g.pc0;
      const int s2hi = circle ? c_lo + p.ww - g.ncp : 0;
      ok = (cc >= max(c_lo, vlo) && cc < min(c_lo + p.ww, vhi)) || cc < s2hi;
    }
    if (!ok) u[cl >> 1] |= masked << (16 * (cl & 1));
  }
}

// One block per (tile, chunk slot), one thread per key: the B_x images of every chunk of every tile, in the
// no-swizzle core-matrix layout the MMA descriptor reads (copied into shared memory with one bulk copy).
__global__ void natten_bias_table_kernel(NaParams p, uint8_t* table) {
  const int tile = blockIdx.x / p.maxch, j = blockIdx.x % p.maxch;
  const TileGeo g = tile_geo_raw(p, 0, tile);  // the geometry is head-independent
  if (j >= g.nchunks) return;
  uint32_t u[8];
  bx_row(p, g, j, threadIdx.x, u);
  uint8_t* img = table + static_cast<size_t>(blockIdx.x) * 4096;
  *reinterpret_cast<uint4*>(img + xtra_off(threadIdx.x, 0)) = make_uint4(u[0], u[1], u[2], u[3]);
  *reinterpret_cast<uint4*>(img + xtra_off(threadIdx.x, 1)) = make_uint4(u[4], u[5], u[6], u[7]);
}

template <bool BIAS, int DHP>
__global__ void __launch_bounds__(NA_THREADS, NA_CTAS_PER_SM)
    natten_fwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmKV, NaParams p) {
  griddep_launch_dependents();  // PDL: the next kernel may start its prologue
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sQ = smem_u32(smem), sK = sQ + NA_TILE, sV = sQ + 2 * NA_TILE;
  const uint32_t sXA = sQ + 3 * NA_TILE, sXB = sXA + 4096;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + NA_SMEM_BODY);
  const uint32_t b0 = smem_u32(bars);
  // Every barrier completes once per chunk (or tile) and its waiter always observes a phase before the
  // next one can complete (each completion needs the waiter's own next step), so parity waits never alias.
  const uint32_t bar_qfull = b0 + 0, bar_qempty = b0 + 8, bar_kfull = b0 + 16, bar_kempty = b0 + 24;
  const uint32_t bar_vfull = b0 + 32, bar_vempty = b0 + 40, bar_ofull = b0 + 48, bar_oempty = b0 + 56;
  auto bar_sfull = [&](int h) { return b0 + 64 + 8 * h; };   // S half h of the chunk is in TMEM
  auto bar_pfull = [&](int h) { return b0 + 80 + 8 * h; };   // P half h written by the 4 softmax warps
  auto bar_pvdone = [&](int h) { return b0 + 96 + 8 * h; };  // P V over key half h retired
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 14);
  float* red = reinterpret_cast<float*>(smem + NA_SMEM_BODY + 256);  // [3][NA_SPLIT][128]

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;

  if (tid == 0) {
    mbar_init(bar_qfull, 1);
    mbar_init(bar_qempty, 1);
    mbar_init(bar_kfull, 1);
    mbar_init(bar_kempty, 1);
    mbar_init(bar_vfull, 1);
    mbar_init(bar_vempty, 1);
    mbar_init(bar_ofull, 1);
    mbar_init(bar_oempty, NA_SOFTMAX_WARPS);
    for (int h = 0; h < 2; ++h) {
      mbar_init(bar_sfull(h), 1);
      mbar_init(bar_pfull(h), NA_SOFTMAX_WARPS);
      mbar_init(bar_pvdone(h), 1);
    }
    fence_barrier_init();
  }
  if (warp == NA_MMA_WARP) {
    tmem_alloc(smem_u32(tmem_slot), NA_TMEM_COLS);
    tmem_relinquish();
  }
  // Zero the operand tiles once: rows past a box are never written by TMA and V rows feed P V (0 * NaN).
  for (uint32_t off = tid * 16u; off < NA_SMEM_BODY; off += NA_THREADS * 16u) st_shared_v4(sQ + off, 0, 0, 0, 0);
  if (BIAS && tid < 128) {
    __syncwarp();
    // A_x row `tid`: ones at the query's tile depth / row / column class (td-major lanes)
    uint32_t u[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
    if (tid < p.TD * p.TH * p.TW) {
      const uint32_t one = pack_elem(1.f, 0.f) & 0xffffu;
      const int c3[3] = {tid / (p.TH * p.TW), p.TD + (tid / p.TW) % p.TH, p.TD + p.TH + tid % p.TW};
      for (int i = 0; i < 3; ++i) u[c3[i] >> 1] |= one << (16 * (c3[i] & 1));
    }
    st_shared_v4(sXA + xtra_off(tid, 0), u[0], u[1], u[2], u[3]);
    st_shared_v4(sXA + xtra_off(tid, 1), u[4], u[5], u[6], u[7]);

  }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  griddep_wait();  // PDL: q/k/v are complete from here on
  const int sec = p.heads * p.dhp;  // columns per q/k/v section
  const int brow0 = p.row0 - p.halo_lo;

  if (warp == NA_TMA_WARP) {
    // =============================== TMA producer ===============================
    if (lane == 0) {
      tma_prefetch(&tmQ);
      tma_prefetch(&tmKV);
      constexpr int halves = DHP / 64;
      const uint32_t qbytes = halves * 128u * p.TW * p.TH * p.TD;
      const uint32_t kbytes = halves * 128u * p.ncp * p.nrpc;
      int chunk_ctr = 0, tile_ctr = 0;
      auto load_kv = [&](const TileGeo& g, int item, int j, int c, bool is_v) {
        int kd, kr0, nr, origin, vlo, vhi;
        chunk_geo(g, p.cols, j, kd, kr0, nr, origin, vlo, vhi);
        const uint32_t full = is_v ? bar_vfull : bar_kfull;
        NA_EV(10, c);
        mbar_wait(is_v ? bar_vempty : bar_kempty, (c & 1) ^ 1);
        NA_EV(11, c);
        if (NA_DBG & 8) {
          mbar_arrive(full);
          return;
        }
        const bool with_bx = BIAS && !is_v;  // the chunk's key-bias image rides with K (same slot lifetime)
        mbar_arrive_expect_tx(full, kbytes + (with_bx ? 4096u : 0u));
        const int c1 = origin, c2 = kr0 - brow0;  // may be negative / past the edge: TMA zero-fills
        const uint32_t dst = is_v ? sV : sK;
        const int col = (is_v ? 2 : 1) * sec + g.head * p.dhp;
        for (int h = 0; h < halves; ++h)
          tma_load_4d(dst + h * 16384u, &tmKV, full, col + 64 * h, c1, c2, g.b * p.depth + kd);
        if (with_bx) {
          bulk_load(sXB, p.bias_table + (static_cast<size_t>(g.tile) * p.maxch + j) * 4096, 4096u, full);
        }
      };
      for (int item = blockIdx.x; item < p.nitems; item += gridDim.x, ++tile_ctr) {
        const TileGeo g = tile_geo(p, item);
        mbar_wait(bar_qempty, (tile_ctr & 1) ^ 1);
        mbar_arrive_expect_tx(bar_qfull, qbytes);
        for (int h = 0; h < halves; ++h)
          tma_load_4d(sQ + h * 16384u, &tmQ, bar_qfull, g.head * p.dhp + 64 * h, g.w0, g.h0 - brow0,
                      g.b * p.depth + g.d0);
        for (int j = 0; j < g.nchunks; ++j, ++chunk_ctr) {
          load_kv(g, item, j, chunk_ctr, false);  // K frees after S(c - 1): streams in during softmax(c - 1)
          load_kv(g, item, j, chunk_ctr, true);   // V frees after P V(c - 1)
        }
      }
    }
  } else if (warp == NA_MMA_WARP) {
    // =============================== MMA issuer ===============================
    // Half-chunk software pipeline (key halves h = 0, 1 of 64 keys each):
    //   S0(c) S1(c) | PV0(c) S0(c+1) | PV1(c) S1(c+1) | PV0(c+1) S0(c+2) | ...
    // S_h(c + 1) overwrites the TMEM columns [64 h, 64 h + 64) whose P_h(c) the preceding PV_h(c) reads (in
    // order), so the softmax of half 0 of the next chunk overlaps P V of half 1 of this one.
    // The whole warp walks the schedule (warp-wide waits) so the descriptors are warp-uniform and live in
    // uniform registers; one elected lane issues the MMAs and commits.  (A lane-0-only loop made every MMA a
    // ~27-instruction R2UR.BROADCAST sequence and kept this warp ~80 % busy on the critical path.)
    constexpr int KSTEPS = DHP / 16;
    const uint32_t idesc_s = make_idesc(128, 64, 0, 0);
    const uint32_t idesc_o = make_idesc(128, DHP, 0, 1);
    const uint32_t tO = tmem + NA_TMEM_O;
    const uint64_t dQ = make_sdesc_sw128(sQ, 16, 1024), dK = make_sdesc_sw128(sK, 16, 1024);
    const uint64_t dV = make_sdesc_sw128(sV, 16384, 1024);
    const uint64_t dXA = make_sdesc_interleave(sXA), dXB = make_sdesc_interleave(sXB);
    auto issue_s = [&](int h) {
      // S_h = Q K_h^T: keys [64 h, 64 h + 64) are rows [64 h, +64) of the K tile (SW128 K-major); descriptor
      // start addresses advance in 16-byte units
      if (elect_one()) {
        if (!(NA_DBG & 2)) {
#pragma unroll
          for (int s = 0; s < KSTEPS; ++s) {
            const uint32_t off = ((s >> 2) * 16384u + (s & 3) * 32u) >> 4;
            umma_bf16_ss(tmem + 64 * h, dQ + off, dK + off + h * 512u, idesc_s, s > 0 ? 1u : 0u);
          }
        }
        if (BIAS)  // + window mask: one-hot query classes x key bias (keys 64 h ..)
          umma_bf16_ss(tmem + 64 * h, dXA, dXB + h * 128u, idesc_s, (NA_DBG & 2) ? 0u : 1u);
        umma_commit(bar_sfull(h));
      }
      __syncwarp();
    };
    auto issue_pv = [&](int h, bool first, uint32_t extra_bar) {
      // O += P_h V_h: A = P_h from TMEM columns [64 h, 64 h + 32) (fp16 pairs), B = V rows 64 h.. (MN-major)
      if (elect_one()) {
        if (!(NA_DBG & 4)) {
#pragma unroll
          for (int s = 0; s < 4; ++s)
            umma_f16_ts(tO, tmem + 64 * h + 8 * s, dV + (4 * h + s) * 128u, idesc_o, (!first || s > 0) ? 1u : 0u);
        }
        umma_commit(bar_pvdone(h));
        if (extra_bar) umma_commit(extra_bar);
      }
      __syncwarp();
    };
    auto commit = [&](uint32_t bar) {
      if (elect_one()) umma_commit(bar);
      __syncwarp();
    };
    int chunk_ctr = 0, tile_ctr = 0;
    for (int item = blockIdx.x; item < p.nitems; item += gridDim.x, ++tile_ctr) {
      const TileGeo g = tile_geo(p, item);
      mbar_wait(bar_qfull, tile_ctr & 1);
      // prologue: both S halves of the tile's first chunk
      mbar_wait(bar_kfull, chunk_ctr & 1);
      tc_fence_after();
      issue_s(0);
      issue_s(1);
      commit(bar_kempty);
      if (g.nchunks == 1) commit(bar_qempty);
      for (int j = 0; j < g.nchunks; ++j, ++chunk_ctr) {
        const uint32_t ph = chunk_ctr & 1;
        const bool more = j + 1 < g.nchunks;
        NA_EV(3, 2 * chunk_ctr);
        mbar_wait(bar_pfull(0), ph);
        NA_EV(4, 2 * chunk_ctr);
        mbar_wait(bar_vfull, ph);
        NA_EV(6, chunk_ctr);
        if (j == 0) mbar_wait(bar_oempty, (tile_ctr & 1) ^ 1);
        tc_fence_after();
        issue_pv(0, j == 0, 0u);
        if (more) {
          NA_EV(7, chunk_ctr);
          mbar_wait(bar_kfull, ph ^ 1);
          NA_EV(8, chunk_ctr);
          tc_fence_after();
          issue_s(0);
        }
        NA_EV(3, 2 * chunk_ctr + 1);
        mbar_wait(bar_pfull(1), ph);
        NA_EV(4, 2 * chunk_ctr + 1);
        tc_fence_after();
        issue_pv(1, false, bar_vempty);
        if (!more) commit(bar_ofull);
        if (more) {
          issue_s(1);
          commit(bar_kempty);
          if (j + 1 == g.nchunks - 1) commit(bar_qempty);
        }
      }
    }
  } else {
    // =============================== softmax / epilogue ===============================
    // Thread = (query row = TMEM lane, column sub-range) of the tile.  Online softmax over key halves of 64:
    // masked max (combined across the row's NA_SPLIT threads), lazy max update (O rescaled only when the max
    // grows by > 2^8), exp2, partial row sum, P_h -> TMEM columns [64 h, +32).
    constexpr int CW = 64 / NA_SPLIT;  // S columns per thread per half
    const int g4 = warp & 3, sub = warp >> 2;
    const int row = 32 * g4 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(32 * g4) << 16;
    const uint32_t tS = tmem + lane_off, tO = tmem + NA_TMEM_O + lane_off;
    const int hw = (p.ww - 1) / 2;
    const size_t member_tokens = static_cast<size_t>(p.depth) * p.rows * p.cols;
    constexpr int ocols = DHP / NA_SPLIT;
    const int oc0 = sub * ocols;  // O columns this thread rescales / stores
    int chunk_ctr = 0, tile_ctr = 0;
    for (int item = blockIdx.x; item < p.nitems; item += gridDim.x, ++tile_ctr) {
      const TileGeo g = tile_geo(p, item);
      const int qd = g.d0 + row / (p.TH * p.TW);
      const int qh = g.h0 + (row / p.TW) % p.TH;  // global row
      const int qw = g.w0 + row % p.TW;
      const bool qvalid = row < p.TD * p.TH * p.TW && qd < g.d1 && qh < g.h1 && qh >= p.q_lo &&
                          qh < p.q_hi && qw < g.w1;
      const int q_sd = bump_start(qvalid ? qd : g.d0, p.depth, p.wd);
      const int q_sh = bump_start(qvalid ? qh : g.h0, p.rows_global, p.wh);
      // window columns in patch coordinates: [c_lo, c_lo + ww), taken mod W for a full-circle patch
      const bool circle = (g.ncp == p.cols);
      const int c_lo = circle ? wrap_col((qvalid ? qw : g.w0) - hw, p.cols) : (qvalid ? qw : g.w0) - hw - g.pc0;
      const int s2hi = circle ? c_lo + p.ww - g.ncp : 0;
      float m_run = -INFINITY, l_run = 0.f;
      // window masks depend on (row chunk, part) only, not on the depth plane: cache one per part, keeping
      // only the MWN words of this thread's columns (word h * CW / 32 + i = columns CW * sub + 32 i of half h)
      constexpr int MWN = 4 / NA_SPLIT;
      int key0 = -1, key1 = -1;
      uint32_t mc0[MWN], mc1[MWN];
      auto own_words = [&](const uint32_t (&m)[4], uint32_t (&o)[MWN]) {
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int i = 0; i < CW / 32; ++i) o[h * (CW / 32) + i] = sub ? m[2 * h + i + CW / 32] : m[2 * h + i];
      };
      for (int j = 0; j < g.nchunks; ++j, ++chunk_ctr) {
        int kd, kr0, nr, origin, vlo, vhi;
        chunk_geo(g, p.cols, j, kd, kr0, nr, origin, vlo, vhi);
        const int part = j % g.nparts, key = (j / g.nparts) % g.nrchunks;
        if (!BIAS && ((part == 0 && key != key0) || (part == 1 && key != key1))) {
          uint32_t m4[4];
          window_mask(m4, nr, g.ncp, max(0, q_sh - kr0), min(nr, q_sh + p.wh - kr0), max(c_lo, vlo),
                      min(c_lo + p.ww, vhi), s2hi);
          if (part == 0) {
            own_words(m4, mc0);
            key0 = key;
          } else {
            own_words(m4, mc1);
            key1 = key;
          }
        }
        const bool dok = qvalid && kd >= q_sd && kd < q_sd + p.wd;
        uint32_t mw[MWN];
#pragma unroll
        for (int w = 0; w < MWN; ++w) mw[w] = BIAS ? 0xffffffffu : (dok ? (part == 0 ? mc0[w] : mc1[w]) : 0u);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (threadIdx.x == 0) NA_EV(0, 2 * chunk_ctr + h);
          mbar_wait(bar_sfull(h), chunk_ctr & 1);
          if (threadIdx.x == 0) NA_EV(1, 2 * chunk_ctr + h);
          tc_fence_after();
          uint32_t pk[CW / 2];
          if (NA_DBG & 1) {
#pragma unroll
            for (int i = 0; i < CW / 2; ++i) pk[i] = 0u;
          } else {
            uint32_t x[CW];
            const uint32_t scol = tS + 64 * h + CW * sub;
#pragma unroll
            for (int i = 0; i < CW / 32; ++i)
              tmem_ld32(scol + 32 * i, *reinterpret_cast<uint32_t(*)[32]>(x + 32 * i));
            tmem_ld_wait();
            float mxa[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) mxa[i] = -INFINITY;
#pragma unroll
            for (int k = 0; k < CW; k += 2) {
              const uint32_t wbits = mw[h * (CW / 32) + (k >> 5)];
              const float a0 = ((wbits >> (k & 31)) & 1u) ? __uint_as_float(x[k]) : -INFINITY;
              const float a1 = ((wbits >> ((k + 1) & 31)) & 1u) ? __uint_as_float(x[k + 1]) : -INFINITY;
              x[k] = __float_as_uint(a0);
              x[k + 1] = __float_as_uint(a1);
              mxa[(k >> 1) & 7] = fmaxf(mxa[(k >> 1) & 7], fmaxf(a0, a1));
            }
            float mxl = fmaxf(fmaxf(fmaxf(mxa[0], mxa[1]), fmaxf(mxa[2], mxa[3])),
                              fmaxf(fmaxf(mxa[4], mxa[5]), fmaxf(mxa[6], mxa[7])));
            if (NA_SPLIT > 1) {
              // the barrier also orders the partners' S loads before either overwrites S with P
              red[(h * NA_SPLIT + sub) * 128 + row] = mxl;
              named_bar_sync(1 + g4, 32 * NA_SPLIT);
#pragma unroll
              for (int o = 1; o < NA_SPLIT; ++o) mxl = fmaxf(mxl, red[(h * NA_SPLIT + (sub ^ o)) * 128 + row]);
            }
            const float mx = mxl * p.scale_log2;
            const bool had = m_run != -INFINITY;  // O already holds weight of this row
            float alpha = 1.f;
            if (mx > m_run + NA_RESCALE_LOG2) {  // lazy max update (also covers m_run = -inf)
              alpha = exp2f(m_run - mx);
              m_run = mx;
            }
            // rescaling O needs the one P V that may still be in flight (issued right after the S half just
            // waited on): PV1(c - 1) for half 0, PV0(c) for half 1.  The row's threads agree on `resc`.
            const bool resc = alpha != 1.f && had;
            l_run *= alpha;
            if (__any_sync(0xffffffffu, resc)) {
              if (h == 0) mbar_wait(bar_pvdone(1), (chunk_ctr - 1) & 1);
              else mbar_wait(bar_pvdone(0), chunk_ctr & 1);
              tc_fence_after();
              const float f = resc ? alpha : 1.f;
#pragma unroll 1
              for (int c = oc0; c < oc0 + ocols; c += 32) {
                uint32_t r[32];
                tmem_ld32(tO + c, r);
                tmem_ld_wait();
#pragma unroll
                for (int e = 0; e < 32; ++e) r[e] = __float_as_uint(__uint_as_float(r[e]) * f);
                tmem_st32(tO + c, r);
              }
            }
            const float m_use = (m_run == -INFINITY) ? 0.f : m_run;
            // packed fp32 pairs (FFMA2 / FADD2): scale-and-shift and row sums issue one instruction per two keys
            float lsa[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) lsa[i] = 0.f;
#pragma unroll
            for (int k = 0; k < CW; k += 2) {
              float e0, e1;  // exp2(-inf) = 0
              ffma2(e0, e1, __uint_as_float(x[k]), __uint_as_float(x[k + 1]), p.scale_log2, p.scale_log2, -m_use,
                    -m_use);
              float p0, p1;
              if (NA_EMU > 0 && ((k >> 1) & 7) < NA_EMU) exp2_fma2(p0, p1, e0, e1);  // FMA pipe
              else { p0 = fast_exp2(e0); p1 = fast_exp2(e1); }                      // MUFU

              const int a = (k >> 1) & 3;
              fadd2(lsa[2 * a], lsa[2 * a + 1], lsa[2 * a], lsa[2 * a + 1], p0, p1);
              pk[k >> 1] = pack_elem(p0, p1);
            }
            l_run += ((lsa[0] + lsa[1]) + (lsa[2] + lsa[3])) + ((lsa[4] + lsa[5]) + (lsa[6] + lsa[7]));
          }
          // P_h (fp16 pairs) over S_h columns [64 h, 64 h + 32): this thread's keys -> CW / 2 columns
          if constexpr (CW == 64) tmem_st32(tS + 64 * h, *reinterpret_cast<uint32_t(*)[32]>(pk));
          else tmem_st16(tS + 64 * h + (CW / 2) * sub, *reinterpret_cast<uint32_t(*)[16]>(pk));
          tmem_st_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(bar_pfull(h));
          if (threadIdx.x == 0) NA_EV(2, 2 * chunk_ctr + h);
        }
      }
      // ---- epilogue: O / l -> ctx ----
      if (NA_SPLIT > 1) {
        red[(2 * NA_SPLIT + sub) * 128 + row] = l_run;
        named_bar_sync(1 + g4, 32 * NA_SPLIT);
        float lt = l_run;
#pragma unroll
        for (int o = 1; o < NA_SPLIT; ++o) lt += red[(2 * NA_SPLIT + (sub ^ o)) * 128 + row];
        l_run = lt;
      }
      const float inv_l = (qvalid && l_run > 0.f) ? 1.f / l_run : 0.f;
      if (threadIdx.x == 0) NA_EV(12, tile_ctr);
      mbar_wait(bar_ofull, tile_ctr & 1);
      if (threadIdx.x == 0) NA_EV(13, tile_ctr);
      tc_fence_after();
      const size_t tok = g.b * member_tokens + static_cast<size_t>((qd * p.rows + (qh - p.row0)) * p.cols + qw);
      elem_t* orow = p.out + (qvalid ? tok * p.ldo + g.head * p.dhp : 0);
      if (p.lse != nullptr && qvalid) p.lse[tok * p.heads + g.head] = m_run + __log2f(l_run);
      // this thread's O columns in batches of 32 TMEM columns, then 256-bit stores (whole 32-byte sectors)
#pragma unroll 1
      for (int c0 = oc0; c0 < oc0 + ocols; c0 += 32) {
        uint32_t r[32];
        tmem_ld32(tO + c0, r);
        tmem_ld_wait();
        if (qvalid) {
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            uint32_t u[8];
#pragma unroll
            for (int e = 0; e < 8; ++e)
              u[e] = pack_elem(__uint_as_float(r[16 * q + 2 * e]) * inv_l, __uint_as_float(r[16 * q + 2 * e + 1]) * inv_l);
            stg256(orow + c0 + 16 * q, u);
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
  if (warp == NA_MMA_WARP) {
    tc_fence_after();
    tmem_dealloc(tmem, NA_TMEM_COLS);
  }
}

// ------------------------------------------------------------------------------------------------------------
// Attention backward on tcgen05 (the block VJP's attention step; reference autodiff rules of
// matmul / softmax / take in attention.py:173-178).  Work item = (query tile, head) as in the forward, one CTA
// per SM (320 threads, all 512 TMEM columns, ~205 KB smem).  Per key half h of every chunk:
//   S_h = Q K_h^T (+ window bias), dP_h = dO V_h^T          (M128 N64, TMEM S [0,128), dP [128,256))
//   softmax warps (thread = query row): P = exp2(S * scale_log2 - lse), dS = P (dP - Delta)   (Delta = dO . O)
//     dS_h (fp16) over the S_h columns (A operand of dQ), P_h and dS_h rows into shared memory (SW128)
//   dQ += dS_h K_h                                            (M128 N=dh K=64, TMEM [256,384))
//   dV_h^T = dO^T P_h, dK_h^T = Q^T dS_h                      (M = dh 128, N64, K = 128 queries; TMEM [384,512))
//   drain warps (thread = dh row) store dK_h^T / dV_h^T as per-(item, chunk, half) partials [slot][dh] (fp32)
// dQ leaves once per tile; natten_bwd_reduce_kernel then sums every key's partials over the (tile, chunk, slot)
// entries that hold it, in a fixed order (CSR built from natten_slot_table_kernel), so dK / dV are deterministic
// without atomics.  Operands: dO enters as fp16 scaled by a power of two sigma chosen so |dP|, |Delta| <= 2^13
// (|dP| <= max|dO| * max_k ||v_k||_1), which keeps dS = P (dP - Delta) inside fp16.
struct NaBwd {
  const elem_t* dout;  // dO * sigma (fp16), [token][heads * dhp] (ldd)
  int ldd;
  const elem_t* o;     // O = ctx (fp16), [token][heads * dhp] (ldo)
  int ldo;
  const float* lse;    // [token][heads], log2 domain (forward with lse)
  float* gqkv;         // fp32 [token][3][heads][dhp] (ldg): dQ into the q section (this kernel)
  int ldg;
  float* partial;      // [item][maxch][2 halves][2 (dK, dV)][64 slots][dhp]
  const float* factors;  // device: [0] dQ / dK factor (scale / (sigma s)), [1] dV factor (1 / (sigma s))
};

// transpose of the rotary rotation (attention.py:87-92 backward) on two interleaved pairs (g0, g1), (g2, g3) with pair tables c, s
DEVI float4 rope_t2(float4 g, float2 c, float2 s) {
  return make_float4(g.x * c.x + g.y * s.x, -g.x * s.x + g.y * c.x, g.z * c.y + g.w * s.y, -g.z * s.y + g.w * c.y);
}

constexpr int NB_THREADS = 320;
constexpr int NB_MMA_WARP = 4, NB_TMA_WARP = 5;  // warps 0-3 softmax, 6-9 partial drain
constexpr uint32_t NB_Q = 0, NB_DO = 32768, NB_K = 65536, NB_V = 131072, NB_P = 163840, NB_DS = 180224,
                   NB_XB = 196608, NB_XA = 204800, NB_BODY = 208896;
constexpr uint32_t NB_SMEM = NB_BODY + 1024 + 256;

template <bool BIAS>
__global__ void __launch_bounds__(NB_THREADS, 1)
    natten_bwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmKV,
                      const __grid_constant__ CUtensorMap tmDO, NaParams p, NaBwd bw) {
  constexpr int DHP = 128;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sb = smem_u32(smem);
  const uint32_t sQ = sb + NB_Q, sDO = sb + NB_DO, sV = sb + NB_V, sP = sb + NB_P, sDS = sb + NB_DS, sXA = sb + NB_XA;
  auto sK = [&](int i) { return sb + NB_K + NA_TILE * i; };
  auto sXB = [&](int i) { return sb + NB_XB + 4096u * i; };
  const uint32_t b0 = sb + NB_BODY;
  const uint32_t bar_qfull = b0, bar_qempty = b0 + 8, bar_vfull = b0 + 16, bar_vempty = b0 + 24;
  auto bar_kfull = [&](int i) { return b0 + 32 + 8 * i; };
  auto bar_kempty = [&](int i) { return b0 + 48 + 8 * i; };
  auto bar_sfull = [&](int h) { return b0 + 64 + 8 * h; };  // S_h and dP_h in TMEM
  auto bar_pfull = [&](int h) { return b0 + 80 + 8 * h; };  // dS_h in TMEM, P_h / dS_h in smem
  const uint32_t bar_psfree = b0 + 96;    // the partial MMAs read P / dS smem (once per half)
  const uint32_t bar_partfull = b0 + 104;  // dK^T / dV^T of a half in TMEM
  const uint32_t bar_partempty = b0 + 112; // drained (4 warps)
  const uint32_t bar_dqfull = b0 + 120, bar_dqempty = b0 + 128;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + NB_BODY + 200);

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;
  if (tid == 0) {
    mbar_init(bar_qfull, 1);
    mbar_init(bar_qempty, 1);
    mbar_init(bar_vfull, 1);
    mbar_init(bar_vempty, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(bar_kfull(i), 1);
      mbar_init(bar_kempty(i), 1);
      mbar_init(bar_sfull(i), 1);
      mbar_init(bar_pfull(i), 4);
    }
    mbar_init(bar_psfree, 1);
    mbar_init(bar_partfull, 1);
    mbar_init(bar_partempty, 4);
    mbar_init(bar_dqfull, 1);
    mbar_init(bar_dqempty, 4);
    fence_barrier_init();
  }
  if (warp == NB_MMA_WARP) {
    tmem_alloc(smem_u32(tmem_slot), 512);
    tmem_relinquish();
  }
  for (uint32_t off = tid * 16u; off < NB_BODY; off += NB_THREADS * 16u) st_shared_v4(sb + off, 0, 0, 0, 0);
  if (BIAS && tid < 128) {
    __syncwarp();
    uint32_t u[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
    if (tid < p.TD * p.TH * p.TW) {
      const uint32_t one = pack_elem(1.f, 0.f) & 0xffffu;
      const int c3[3] = {tid / (p.TH * p.TW), p.TD + (tid / p.TW) % p.TH, p.TD + p.TH + tid % p.TW};
      for (int i = 0; i < 3; ++i) u[c3[i] >> 1] |= one << (16 * (c3[i] & 1));
    }
    st_shared_v4(sXA + xtra_off(tid, 0), u[0], u[1], u[2], u[3]);
    st_shared_v4(sXA + xtra_off(tid, 1), u[4], u[5], u[6], u[7]);
  }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int sec = p.heads * DHP;
  const int brow0 = p.row0 - p.halo_lo;
  const int ntiles = p.ntd * p.nth * p.ntw;

  if (warp == NB_TMA_WARP) {
    // ---------------- producer: Q + dO per tile, K (2 slots) and V (1 slot) per chunk ----------------
    if (lane == 0) {
      tma_prefetch(&tmQ);
      tma_prefetch(&tmKV);
      tma_prefetch(&tmDO);
      const uint32_t qbytes = 2 * 128u * p.TW * p.TH * p.TD;
      const uint32_t kbytes = 2 * 128u * p.ncp * p.nrpc;
      int c = 0, t = 0;
      for (int item = blockIdx.x; item < p.nitems; item += gridDim.x, ++t) {
        const TileGeo g = tile_geo(p, item);
        mbar_wait(bar_qempty, (t & 1) ^ 1);
        mbar_arrive_expect_tx(bar_qfull, 2 * qbytes);
        for (int h = 0; h < 2; ++h) {
          tma_load_4d(sQ + h * 16384u, &tmQ, bar_qfull, g.head * DHP + 64 * h, g.w0, g.h0 - brow0,
                      g.b * p.depth + g.d0);
          tma_load_4d(sDO + h * 16384u, &tmDO, bar_qfull, g.head * DHP + 64 * h, g.w0, g.h0 - brow0,
                      g.b * p.depth + g.d0);
        }
        for (int j = 0; j < g.nchunks; ++j, ++c) {
          int kd, kr0, nr, origin, vlo, vhi;
          chunk_geo(g, p.cols, j, kd, kr0, nr, origin, vlo, vhi);
          const int s = c & 1;
          mbar_wait(bar_kempty(s), ((c >> 1) & 1) ^ 1);
          mbar_arrive_expect_tx(bar_kfull(s), kbytes + (BIAS ? 4096u : 0u));
          for (int h = 0; h < 2; ++h)
            tma_load_4d(sK(s) + h * 16384u, &tmKV, bar_kfull(s), sec + g.head * DHP + 64 * h, origin, kr0 - brow0,
                        g.b * p.depth + kd);
          if (BIAS)
            bulk_load(sXB(s), p.bias_table + (static_cast<size_t>(g.tile) * p.maxch + j) * 4096, 4096u,
                      bar_kfull(s));
          mbar_wait(bar_vempty, (c & 1) ^ 1);
          mbar_arrive_expect_tx(bar_vfull, kbytes);
          for (int h = 0; h < 2; ++h)
            tma_load_4d(sV + h * 16384u, &tmKV, bar_vfull, 2 * sec + g.head * DHP + 64 * h, origin, kr0 - brow0,
                        g.b * p.depth + kd);
        }
      }
    }
  } else if (warp == NB_MMA_WARP) {
    // ---------------- MMA issuer ----------------
    const uint32_t idesc_s = make_idesc(128, 64, 0, 0);      // S, dP: K-major Q / dO and K / V rows
    const uint32_t idesc_q = make_idesc(128, DHP, 0, 1);     // dQ: A = dS (TMEM), B = K MN-major
    const uint32_t idesc_p = make_idesc(128, 64, 1, 1);      // dK^T / dV^T: A = Q / dO MN-major, B = dS / P
    const uint64_t dQd = make_sdesc_sw128(sQ, 16, 1024), dDOd = make_sdesc_sw128(sDO, 16, 1024);
    const uint64_t dK0 = make_sdesc_sw128(sK(0), 16, 1024), dV0 = make_sdesc_sw128(sV, 16, 1024);
    const uint64_t dKmn = make_sdesc_sw128(sK(0), 16384, 1024);   // K as an MN-major B (N = dh)
    const uint64_t dQmn = make_sdesc_sw128(sQ, 16384, 1024), dDOmn = make_sdesc_sw128(sDO, 16384, 1024);
    const uint64_t dPs = make_sdesc_sw128(sP, 16384, 1024), dDSs = make_sdesc_sw128(sDS, 16384, 1024);
    const uint64_t dXA = make_sdesc_interleave(sXA), dXB0 = make_sdesc_interleave(sXB(0));
    constexpr uint32_t T16 = NA_TILE >> 4;
    const uint32_t tS = tmem, tDP = tmem + 128, tDQ = tmem + 256, tPK = tmem + 384, tPV = tmem + 448;
    auto issue_s = [&](int h, int ks) {  // S_h and dP_h of the chunk in K slot ks
      if (elect_one()) {
#pragma unroll
        for (int s = 0; s < DHP / 16; ++s) {
          const uint32_t off = ((s >> 2) * 16384u + (s & 3) * 32u) >> 4;
          umma_bf16_ss(tS + 64 * h, dQd + off, dK0 + ks * T16 + off + h * 512u, idesc_s, s > 0 ? 1u : 0u);
        }
        if (BIAS) umma_bf16_ss(tS + 64 * h, dXA, dXB0 + ks * 256u + h * 128u, idesc_s, 1u);
#pragma unroll
        for (int s = 0; s < DHP / 16; ++s) {
          const uint32_t off = ((s >> 2) * 16384u + (s & 3) * 32u) >> 4;
          umma_bf16_ss(tDP + 64 * h, dDOd + off, dV0 + off + h * 512u, idesc_s, s > 0 ? 1u : 0u);
        }
        umma_commit(bar_sfull(h));
      }
      __syncwarp();
    };
    auto commit = [&](uint32_t bar) {
      if (elect_one()) umma_commit(bar);
      __syncwarp();
    };
    int c = 0, t = 0, hc = 0;
    for (int item = blockIdx.x; item < p.nitems; item += gridDim.x, ++t) {
      const TileGeo g = tile_geo(p, item);
      mbar_wait(bar_qfull, t & 1);
      mbar_wait(bar_kfull(c & 1), (c >> 1) & 1);
      mbar_wait(bar_vfull, c & 1);
      tc_fence_after();
      issue_s(0, c & 1);
      issue_s(1, c & 1);
      commit(bar_vempty);
      for (int j = 0; j < g.nchunks; ++j, ++c) {
        const int ks = c & 1;
        const bool more = j + 1 < g.nchunks;
        for (int h = 0; h < 2; ++h, ++hc) {
          mbar_wait(bar_pfull(h), c & 1);
          if (j == 0 && h == 0) mbar_wait(bar_dqempty, (t & 1) ^ 1);
          tc_fence_after();
          if (elect_one()) {
            // dQ += dS_h K_h: A = dS_h from TMEM (fp16 pairs over S_h), B = K rows 64 h.. (MN-major, N = dh)
#pragma unroll
            for (int s = 0; s < 4; ++s)
              umma_f16_ts(tDQ, tS + 64 * h + 8 * s, dKmn + ks * T16 + (4 * h + s) * 128u, idesc_q,
                          (j > 0 || h > 0 || s > 0) ? 1u : 0u);
          }
          __syncwarp();
          mbar_wait(bar_partempty, (hc & 1) ^ 1);
          tc_fence_after();
          if (elect_one()) {
            // dV_h^T = dO^T P_h, dK_h^T = Q^T dS_h over the 128 query rows (K = queries, 16 per MMA)
#pragma unroll
            for (int s = 0; s < 8; ++s) {
              umma_bf16_ss(tPV, dDOmn + s * 128u, dPs + s * 128u, idesc_p, s > 0 ? 1u : 0u);
              umma_bf16_ss(tPK, dQmn + s * 128u, dDSs + s * 128u, idesc_p, s > 0 ? 1u : 0u);
            }
            umma_commit(bar_partfull);
            umma_commit(bar_psfree);
            if (h == 1) umma_commit(bar_kempty(ks));
            if (h == 1 && !more) {
              umma_commit(bar_dqfull);
              umma_commit(bar_qempty);
            }
          }
          __syncwarp();
          if (more) {
            if (h == 0) {
              mbar_wait(bar_kfull((c + 1) & 1), ((c + 1) >> 1) & 1);
              mbar_wait(bar_vfull, (c + 1) & 1);
              tc_fence_after();
            }
            issue_s(h, (c + 1) & 1);
            if (h == 1) commit(bar_vempty);
          }
        }
      }
    }
  } else if (warp < 4) {
    // ---------------- softmax: P, dS per query row; dQ epilogue ----------------
    const int row = 32 * warp + lane;
    const uint32_t lane_off = static_cast<uint32_t>(32 * warp) << 16;
    const uint32_t tS = tmem + lane_off, tDP = tmem + 128 + lane_off, tDQ = tmem + 256 + lane_off;
    const size_t member_tokens = static_cast<size_t>(p.depth) * p.rows * p.cols;
    int c = 0, t = 0, hc = 0;
    for (int item = blockIdx.x; item < p.nitems; item += gridDim.x, ++t) {
      const TileGeo g = tile_geo(p, item);
      const int qd = g.d0 + row / (p.TH * p.TW);
      const int qh = g.h0 + (row / p.TW) % p.TH;
      const int qw = g.w0 + row % p.TW;
      const bool qvalid = row < p.TD * p.TH * p.TW && qd < g.d1 && qh < g.h1 && qh >= p.q_lo && qh < p.q_hi &&
                          qw < g.w1;
      const size_t tok = g.b * member_tokens + static_cast<size_t>((qd * p.rows + (qh - p.row0)) * p.cols + qw);
      const float lse = qvalid ? __ldg(bw.lse + tok * p.heads + g.head) : 0.f;
      // Delta = dO . O of this row (dO from the staged tile, O from global)
      mbar_wait(bar_qfull, t & 1);
      float delta = 0.f;
      if (qvalid) {
        const uint4* orow = reinterpret_cast<const uint4*>(bw.o + tok * bw.ldo + g.head * DHP);
#pragma unroll
        for (int ch = 0; ch < 16; ++ch) {
          uint32_t a0, a1, a2, a3;
          ld_shared_v4u(sDO + (ch >> 3) * 16384u + sw128_off(row, ch & 7), a0, a1, a2, a3);
          const uint4 o4 = __ldg(orow + ch);
          const uint32_t da[4] = {a0, a1, a2, a3}, oa[4] = {o4.x, o4.y, o4.z, o4.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 x = unpack_elem2(da[e]), y = unpack_elem2(oa[e]);
            delta = fmaf(x.x, y.x, fmaf(x.y, y.y, delta));
          }
        }
      }
      for (int j = 0; j < g.nchunks; ++j, ++c) {
        for (int h = 0; h < 2; ++h, ++hc) {
          mbar_wait(bar_sfull(h), c & 1);
          tc_fence_after();
          // the previous half's partial MMAs must be done reading the P / dS staging rows
          mbar_wait(bar_psfree, (hc & 1) ^ 1);
#pragma unroll
          for (int sub = 0; sub < 2; ++sub) {
            uint32_t xs[32], xp[32];
            tmem_ld32(tS + 64 * h + 32 * sub, xs);
            tmem_ld32(tDP + 64 * h + 32 * sub, xp);
            tmem_ld_wait();
            uint32_t pp[16], pd[16];
#pragma unroll
            for (int k = 0; k < 32; k += 2) {
              float e0, e1;
              ffma2(e0, e1, __uint_as_float(xs[k]), __uint_as_float(xs[k + 1]), p.scale_log2, p.scale_log2, -lse,
                    -lse);
              float p0 = qvalid ? fast_exp2(e0) : 0.f, p1 = qvalid ? fast_exp2(e1) : 0.f;
              const float d0 = p0 * (__uint_as_float(xp[k]) - delta), d1 = p1 * (__uint_as_float(xp[k + 1]) - delta);
              pp[k >> 1] = pack_elem(p0, p1);
              pd[k >> 1] = pack_elem(d0, d1);
            }
            // dS (fp16 pairs) over the consumed S columns: A operand of dQ
            tmem_st16(tS + 64 * h + 16 * sub, pd);
            // P / dS rows into the SW128 staging tiles (keys 32 sub .. 32 sub + 31 = 16-byte chunks 4 sub ..)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              st_shared_v4(sP + sw128_off(row, 4 * sub + q), pp[4 * q], pp[4 * q + 1], pp[4 * q + 2], pp[4 * q + 3]);
              st_shared_v4(sDS + sw128_off(row, 4 * sub + q), pd[4 * q], pd[4 * q + 1], pd[4 * q + 2], pd[4 * q + 3]);
            }
          }
          tmem_st_wait();
          fence_proxy_async();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(bar_pfull(h));
        }
      }
      // ---- dQ epilogue ----
      mbar_wait(bar_dqfull, t & 1);
      tc_fence_after();
      const float f = __ldg(bw.factors);
      float* gq = bw.gqkv + tok * bw.ldg + g.head * DHP;
#pragma unroll 1
      for (int c0 = 0; c0 < DHP; c0 += 32) {
        uint32_t r[32];
        tmem_ld32(tDQ + c0, r);
        tmem_ld_wait();
        if (qvalid) {
#pragma unroll
          for (int e = 0; e < 32; e += 4) {
            *reinterpret_cast<float4*>(gq + c0 + e) =
                make_float4(__uint_as_float(r[e]) * f, __uint_as_float(r[e + 1]) * f, __uint_as_float(r[e + 2]) * f,
                            __uint_as_float(r[e + 3]) * f);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_dqempty);
    }
  } else if (warp >= 6) {
    // ---------------- partial drain: thread = dh row ----------------
    const int q4 = warp & 3;
    const int d = 32 * q4 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(32 * q4) << 16;
    int hc = 0;
    for (int item = blockIdx.x; item < p.nitems; item += gridDim.x) {
      const TileGeo g = tile_geo(p, item);
      for (int j = 0; j < g.nchunks; ++j) {
        for (int h = 0; h < 2; ++h, ++hc) {
          mbar_wait(bar_partfull, hc & 1);
          tc_fence_after();
          const size_t raw = static_cast<size_t>(g.hb) * (p.ntd * p.nth * p.ntw) + g.tile;  // reduce-kernel index
          float* base = bw.partial + (((raw * p.maxch + j) * 2 + h) * 2) * 64 * DHP + d;
#pragma unroll
          for (int kv = 0; kv < 2; ++kv) {
#pragma unroll
            for (int c0 = 0; c0 < 64; c0 += 32) {
              uint32_t r[32];
              tmem_ld32(tmem + lane_off + 384 + 64 * kv + c0, r);
              tmem_ld_wait();
#pragma unroll
              for (int e = 0; e < 32; ++e) base[(static_cast<size_t>(kv) * 64 + c0 + e) * DHP] = __uint_as_float(r[e]);
            }
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(bar_partempty);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == NB_MMA_WARP) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// Key token held by every slot of every (tile, chunk): -1 for padding / zero-filled / out-of-grid slots.
__global__ void natten_slot_table_kernel(NaParams p, int32_t* table) {
  const int tile = blockIdx.x / p.maxch, j = blockIdx.x % p.maxch;
  const TileGeo g = tile_geo_raw(p, 0, tile);
  const int k = threadIdx.x;
  int32_t tok = -1;
  if (j < g.nchunks) {
    int kd, kr0, nr, origin, vlo, vhi;
    chunk_geo(g, p.cols, j, kd, kr0, nr, origin, vlo, vhi);
    const int rr = k / g.ncp, cc = k - rr * g.ncp;
    if (rr < nr && cc >= vlo && cc < vhi) {
      const int kr = kr0 + rr;
      const int col = wrap_col(g.pc0 + cc, p.cols);
      if (kr >= 0 && kr < p.rows_global) tok = (kd * p.rows + (kr - p.row0)) * p.cols + col;
    }
  }
  table[static_cast<size_t>(blockIdx.x) * 128 + k] = tok;
}

// dK / dV of every (key token, head): the sum of the partials of the (tile, chunk, slot) entries holding the key,
// in CSR order (fixed), times the factors; one warp per (token, head), 4 channels per lane.
__global__ void natten_bwd_reduce_kernel(const float* __restrict__ partial, const int32_t* __restrict__ off,
                                         const int32_t* __restrict__ ent, int T, int heads, int ntiles, int maxch,
                                         const float* __restrict__ factors, float* __restrict__ gqkv, int ldg,
                                         const float* __restrict__ rope_cos, const float* __restrict__ rope_sin,
                                         unsigned* amax) {
  constexpr int DHP = 128;
  __shared__ float redm[32];
  const int lane = threadIdx.x & 31;
  const int sec = heads * DHP;
  const float fk = __ldg(factors), fv = __ldg(factors + 1);
  float m = 0.f;  // max |dK|, |dV| of this thread's elements (the QKV weight gradient's operand scale)
  // warps stride over the (key token, head) pairs; one atomic per block at the end (thousands of warps
  // hitting one address measured slower than the whole reduction)
  for (int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; wid < T * heads;
       wid += (gridDim.x * blockDim.x) >> 5) {
    const int tk = wid / heads, h = wid - tk * heads;
    float4 ak = make_float4(0.f, 0.f, 0.f, 0.f), av = ak;
    for (int e = off[tk]; e < off[tk + 1]; ++e) {
      const int32_t code = ent[e];  // (tile * maxch + chunk) * 128 + slot
      const int slot = code & 127, tc = code >> 7;
      const int tile = tc / maxch, j = tc - tile * maxch;
      const size_t item = static_cast<size_t>(h) * ntiles + tile;
      const float* base = partial + (((item * maxch + j) * 2 + (slot >> 6)) * 2) * 64 * DHP +
                          static_cast<size_t>(slot & 63) * DHP + 4 * lane;
      const float4 k4 = __ldg(reinterpret_cast<const float4*>(base));
      const float4 v4 = __ldg(reinterpret_cast<const float4*>(base + 64 * DHP));
      ak.x += k4.x; ak.y += k4.y; ak.z += k4.z; ak.w += k4.w;
      av.x += v4.x; av.y += v4.y; av.z += v4.z; av.w += v4.w;
    }
    float* g = gqkv + static_cast<size_t>(tk) * ldg + h * DHP + 4 * lane;
    float4 k4 = make_float4(ak.x * fk, ak.y * fk, ak.z * fk, ak.w * fk);
    if (rope_cos != nullptr) {
      const size_t pi = static_cast<size_t>(tk) * (DHP / 2) + 2 * lane;
      k4 = rope_t2(k4, __ldg(reinterpret_cast<const float2*>(rope_cos + pi)),
                   __ldg(reinterpret_cast<const float2*>(rope_sin + pi)));
    }
    *reinterpret_cast<float4*>(g + sec) = k4;
    const float4 v4 = make_float4(av.x * fv, av.y * fv, av.z * fv, av.w * fv);
    *reinterpret_cast<float4*>(g + 2 * sec) = v4;
    m = fmaxf(m, fmaxf(fmaxf(fmaxf(fabsf(k4.x), fabsf(k4.y)), fmaxf(fabsf(k4.z), fabsf(k4.w))),
                       fmaxf(fmaxf(fabsf(v4.x), fabsf(v4.y)), fmaxf(fabsf(v4.z), fabsf(v4.w)))));
  }
  if (amax != nullptr) {
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) redm[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
      float t = redm[0];
      for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) t = fmaxf(t, redm[w]);
      atomicMax(amax, __float_as_uint(t));
    }
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
static void choose_tile(int depth, int cols, int rows_global, int wd, int wh, int ww, int* TD, int* TH, int* TW,
                        int* NCP, int* NRPC) {
  const int rows = rows_global;  // the tile shape depends on the global grid only (band-invariant results)
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

// Geometry, tensor maps and (once per geometry) the window-bias images of an NA launch.
static int natten_setup(const void* qkv, int ldqkv, void* out, int ldo, int batch, int depth, int rows, int cols,
                        int rows_global, int row0, int halo_lo, int halo_hi, int heads, int dhp, int wd, int wh,
                        int ww, float scale, int q_lo, int q_rows, void* stream, NaParams& p, CUtensorMap& tq,
                        CUtensorMap& tkv, bool& bias) {
  if (dhp != 64 && dhp != 128) return set_error("wm3_natten_fwd: dhp must be 64 or 128 (got %d)", dhp);
  if (batch < 1) return set_error("wm3_natten_fwd: batch must be >= 1 (got %d)", batch);
  if (wd > depth || wh > rows_global || ww > cols) return set_error("wm3_natten_fwd: window exceeds extents");
  if (ww > 64) return set_error("wm3_natten_fwd: col window %d > 64 unsupported", ww);
  if (row0 < 0 || row0 + rows > rows_global || halo_lo > row0 || row0 + rows + halo_hi > rows_global)
    return set_error("wm3_natten_fwd: bad band rows");
  if (q_rows < 1 || q_lo < row0 || q_lo + q_rows > row0 + rows)
    return set_error("wm3_natten_fwd: query rows [%d, %d) outside the band [%d, %d)", q_lo, q_lo + q_rows, row0,
                     row0 + rows);
  // the halo must cover every window that reaches outside the band
  if (rows < rows_global) {
    const int need_lo = row0 - bump_start(row0, rows_global, wh);
    const int need_hi = bump_start(row0 + rows - 1, rows_global, wh) + wh - (row0 + rows);
    if (halo_lo < need_lo || halo_hi < need_hi)
      return set_error("wm3_natten_fwd: halos (%d,%d) smaller than window reach (%d,%d)", halo_lo, halo_hi, need_lo,
                       need_hi);
  }
  if ((ldqkv % 8) || (ldo % 16)) return set_error("wm3_natten_fwd: ldqkv must be a multiple of 8, ldo of 16");
  if (reinterpret_cast<uintptr_t>(out) % 32) return set_error("wm3_natten_fwd: out must be 32-byte aligned");
  if (ldqkv < 3 * heads * dhp) return set_error("wm3_natten_fwd: ldqkv < 3 * heads * dhp");
  p = NaParams{};
  p.out = reinterpret_cast<elem_t*>(out);
  p.ldo = ldo;
  p.batch = batch;
  p.depth = depth; p.rows = rows; p.cols = cols; p.rows_global = rows_global; p.row0 = row0;
  p.halo_lo = halo_lo; p.rows_ext = rows + halo_lo + halo_hi;
  p.heads = heads; p.dhp = dhp; p.wd = wd; p.wh = wh; p.ww = ww;
  choose_tile(depth, cols, rows_global, wd, wh, ww, &p.TD, &p.TH, &p.TW, &p.ncp, &p.nrpc);
  if (const char* e = getenv("WM3_NA_TILE")) {  // A/B aid: "TD,TH,TW" (key box derived as in choose_tile)
    int td, th, tw;
    if (sscanf(e, "%d,%d,%d", &td, &th, &tw) == 3 && td >= 1 && th >= 1 && tw >= 1 && td <= depth && th <= rows_global &&
        tw <= cols && td * th * tw <= 128) {
      const int ncp = (tw + ww - 1 >= cols) ? cols : tw + ww - 1;
      const int nr_u = (th + wh - 1 < rows_global) ? th + wh - 1 : rows_global;
      if (ncp <= 128) {
        p.TD = td; p.TH = th; p.TW = tw; p.ncp = ncp;
        p.nrpc = (nr_u < 128 / ncp) ? nr_u : 128 / ncp;
      }
    }
  }
  p.ntd = (depth + p.TD - 1) / p.TD;
  p.q_lo = q_lo;
  p.q_hi = q_lo + q_rows;
  p.th_first = q_lo / p.TH;
  p.nth = (p.q_hi - 1) / p.TH - p.th_first + 1;
  p.ntw = (cols + p.TW - 1) / p.TW;
  p.nitems = p.ntd * p.nth * p.ntw * heads * batch;
  {  // seam-crossing first / last column tiles (item_tile schedules them first)
    const int hw = (ww - 1) / 2;
    const bool circle = p.ncp == cols;
    const int w0 = (p.ntw - 1) * p.TW, w1 = (w0 + p.TW < cols) ? w0 + p.TW : cols;
    p.heavy_lo = (!circle && hw > 0) ? 1 : 0;
    p.heavy_hi = (!circle && p.ntw > 1 && (w0 - hw < 0 || w1 - 1 + (ww - 1 - hw) >= cols)) ? 1 : 0;
  }
  p.scale_log2 = scale * 1.4426950408889634f;

  const uint64_t wp = cols;
  const uint64_t dims[4] = {static_cast<uint64_t>(3 * heads * dhp), wp, static_cast<uint64_t>(p.rows_ext),
                            static_cast<uint64_t>(batch) * depth};
  const uint64_t strides[3] = {static_cast<uint64_t>(ldqkv), wp * ldqkv, wp * p.rows_ext * ldqkv};
  const uint32_t qbox[4] = {64, static_cast<uint32_t>(p.TW), static_cast<uint32_t>(p.TH), static_cast<uint32_t>(p.TD)};
  const uint32_t kvbox[4] = {64, static_cast<uint32_t>(p.ncp), static_cast<uint32_t>(p.nrpc), 1};
  if (make_tmap(&tq, qkv, TMAP_BF16, 4, dims, strides, qbox, nullptr)) return -1;
  if (make_tmap(&tkv, qkv, TMAP_BF16, 4, dims, strides, kvbox, nullptr)) return -1;
  for (auto kern : {natten_fwd_kernel<true, 64>, natten_fwd_kernel<false, 64>, natten_fwd_kernel<true, 128>,
                    natten_fwd_kernel<false, 128>})
    if (ensure_smem_attr(reinterpret_cast<const void*>(kern), NA_SMEM, "natten")) return -1;
  // window mask in the MMA when the tile's query classes fit the extra K = 16 step (WM3_NA_BIAS=0: softmax mask)
  static const bool bias_env = [] {
    const char* e = getenv("WM3_NA_BIAS");
    return !(e && e[0] == '0');
  }();
  bias = bias_env && p.TD + p.TH + p.TW <= 16;
  {
    // depth planes of a tile's key patch x row chunks x parts: the chunk-slot stride of every per-chunk table
    p.maxch = p.wd + p.TD - 1;
    p.maxch = (p.maxch < depth ? p.maxch : depth) * ((p.wh + p.TH - 1 + p.nrpc - 1) / p.nrpc) * 2;
  }
  if (bias) {
    // B_x images of every (tile, chunk): built once per geometry on this stream, kept for the process (a few
    // tens of MB at full scale, shared by every head, member, block and step)
    const int ntiles = p.ntd * p.nth * p.ntw;
    struct Key {
      // the images depend on the launch's global tile rows only (not on the band or its halos)
      int dev, depth, cols, rows_global, th_first, nth, wd, wh, ww, TD, TH, TW, ncp, nrpc;
      bool operator<(const Key& o) const {
        return std::tie(dev, depth, cols, rows_global, th_first, nth, wd, wh, ww, TD, TH, TW, ncp, nrpc) <
               std::tie(o.dev, o.depth, o.cols, o.rows_global, o.th_first, o.nth, o.wd, o.wh, o.ww, o.TD, o.TH,
                        o.TW, o.ncp, o.nrpc);
      }
    };
    static std::map<Key, uint8_t*> tables;
    static std::mutex mu;
    int dev = 0;
    cudaGetDevice(&dev);
    const Key key{dev, depth, cols, rows_global, p.th_first, p.nth, wd, wh, ww, p.TD, p.TH, p.TW, p.ncp, p.nrpc};
    std::lock_guard<std::mutex> lock(mu);
    auto it = tables.find(key);
    if (it == tables.end()) {
      cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
      cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
      const cudaError_t ce = cudaStreamIsCapturing(s, &cap);
      if (ce != cudaSuccess) {  // e.g. the legacy stream during another thread's global-mode capture
        cudaGetLastError();
        return set_error("wm3_natten_fwd: cannot build the window-mask images now (%s); run this geometry once "
                         "eagerly first", cudaGetErrorString(ce));
      }
      if (cap != cudaStreamCaptureStatusNone)
        return set_error("wm3_natten_fwd: first call for this geometry inside a CUDA graph capture; run it once "
                         "eagerly first (the window-mask images are built then)");
      uint8_t* t = nullptr;
      const size_t bytes = static_cast<size_t>(ntiles) * p.maxch * 4096;
      if (cudaMalloc(&t, bytes) != cudaSuccess) return set_error("wm3_natten_fwd: bias table allocation failed");
      cudaMemsetAsync(t, 0, bytes, s);
      natten_bias_table_kernel<<<ntiles * p.maxch, 128, 0, s>>>(p, t);
      if (check_launch("natten_bias_table_kernel")) {
        cudaFree(t);
        return -1;
      }
      // one-time: the images must be complete before any stream (not only this one) uses them
      if (cudaStreamSynchronize(s) != cudaSuccess) {
        cudaFree(t);
        return set_error("wm3_natten_fwd: bias table build failed");
      }
      it = tables.emplace(key, t).first;
    }
    p.bias_table = it->second;
  }
  return 0;
}

static int natten_launch(const void* qkv, int ldqkv, void* out, int ldo, int batch, int depth, int rows, int cols,
                         int rows_global, int row0, int halo_lo, int halo_hi, int heads, int dhp, int wd, int wh,
                         int ww, float scale, int q_lo, int q_rows, void* stream, float* lse = nullptr) {
  NaParams p;
  CUtensorMap tq, tkv;
  bool bias = false;
  if (natten_setup(qkv, ldqkv, out, ldo, batch, depth, rows, cols, rows_global, row0, halo_lo, halo_hi, heads, dhp,
                   wd, wh, ww, scale, q_lo, q_rows, stream, p, tq, tkv, bias))
    return -1;
  p.lse = lse;
  const int slots = NA_CTAS_PER_SM * sm_count();
  const int grid = p.nitems < slots ? p.nitems : slots;
  auto kern = dhp == 64 ? (bias ? natten_fwd_kernel<true, 64> : natten_fwd_kernel<false, 64>)
                        : (bias ? natten_fwd_kernel<true, 128> : natten_fwd_kernel<false, 128>);
  if (launch_pdl(kern, dim3(grid), dim3(NA_THREADS), NA_SMEM,
                 reinterpret_cast<cudaStream_t>(stream), tq,
                 tkv, p))
    return -1;
  return check_launch("natten_fwd_kernel");
}

extern "C" int wm3_natten_fwd(const void* qkv, int ldqkv, void* out, int ldo, int batch, int depth, int rows, int cols,
                              int rows_global, int row0, int halo_lo, int halo_hi, int heads, int dhp, int wd, int wh,
                              int ww, float scale, void* stream) {
  return natten_launch(qkv, ldqkv, out, ldo, batch, depth, rows, cols, rows_global, row0, halo_lo, halo_hi, heads,
                       dhp, wd, wh, ww, scale, row0, rows, stream);
}

extern "C" int wm3_natten_fwd_rows(const void* qkv, int ldqkv, void* out, int ldo, int batch, int depth, int rows,
                                   int cols, int rows_global, int row0, int halo_lo, int halo_hi, int heads, int dhp,
                                   int wd, int wh, int ww, float scale, int q_lo, int q_rows, void* stream) {
  return natten_launch(qkv, ldqkv, out, ldo, batch, depth, rows, cols, rows_global, row0, halo_lo, halo_hi, heads,
                       dhp, wd, wh, ww, scale, q_lo, q_rows, stream);
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

#ifdef WM3_NA_TRACE
extern "C" int wm3_na_trace(long long* out, int max_events) {
  int n = 0;
  cudaMemcpyFromSymbol(&n, wm3::g_na_trace_n, sizeof(int));
  n = n < max_events ? n : max_events;
  n = n < wm3::NA_TRACE_MAX ? n : wm3::NA_TRACE_MAX;
  cudaMemcpyFromSymbol(out, wm3::g_na_trace, static_cast<size_t>(n) * 3 * sizeof(long long));
  const int zero = 0;
  cudaMemcpyToSymbol(wm3::g_na_trace_n, &zero, sizeof(int));
  return n;
}
#endif

// ---------------------------------------------------------------------------------------------------------------
// Attention backward (natten_bwd_kernel + natten_bwd_reduce_kernel), full domain (no band / halo), batch 1.
// ---------------------------------------------------------------------------------------------------------------
extern "C" int wm3_natten_fwd_lse(const void* qkv, int ldqkv, void* out, int ldo, int depth, int rows, int cols,
                                  int heads, int dhp, int wd, int wh, int ww, float scale, float* lse, void* stream) {
  return natten_launch(qkv, ldqkv, out, ldo, 1, depth, rows, cols, rows, 0, 0, 0, heads, dhp, wd, wh, ww, scale, 0,
                       rows, stream, lse);
}

static int natten_bwd_geom(int depth, int rows, int cols, int heads, int dhp, int wd, int wh, int ww, void* stream,
                           NaParams& p, CUtensorMap& tq, CUtensorMap& tkv, bool& bias) {
  // geometry only: the tensor maps are rebuilt by the launch with the real operands
  void* dummy = reinterpret_cast<void*>(static_cast<uintptr_t>(1) << 20);
  return natten_setup(dummy, 3 * heads * dhp, dummy, heads * dhp, 1, depth, rows, cols, rows, 0, 0, 0, heads, dhp, wd,
                      wh, ww, 1.f, 0, rows, stream, p, tq, tkv, bias);
}

// Tiles and chunk-slot stride of the backward's geometry; supported = 1 when the tcgen05 backward applies
// (head dim padded to 128 and the window mask in the MMA), else the caller uses wm3_bw_natten.
extern "C" int wm3_natten_bwd_info(int depth, int rows, int cols, int heads, int dhp, int wd, int wh, int ww,
                                   int* ntiles, int* maxch, int* supported, void* stream) {
  NaParams p;
  CUtensorMap tq, tkv;
  bool bias = false;
  if (natten_bwd_geom(depth, rows, cols, heads, dhp, wd, wh, ww, stream, p, tq, tkv, bias)) return -1;
  *ntiles = p.ntd * p.nth * p.ntw;
  *maxch = p.maxch;
  *supported = (dhp == 128 && bias) ? 1 : 0;
  return 0;
}

// [tile][maxch][128] key token of every chunk slot (-1: none), for the host-built CSR of the dK / dV reduction.
extern "C" int wm3_natten_slot_table(int depth, int rows, int cols, int heads, int dhp, int wd, int wh, int ww,
                                     int32_t* table, void* stream) {
  NaParams p;
  CUtensorMap tq, tkv;
  bool bias = false;
  if (natten_bwd_geom(depth, rows, cols, heads, dhp, wd, wh, ww, stream, p, tq, tkv, bias)) return -1;
  const int ntiles = p.ntd * p.nth * p.ntw;
  natten_slot_table_kernel<<<ntiles * p.maxch, 128, 0, reinterpret_cast<cudaStream_t>(stream)>>>(p, table);
  return check_launch("natten_slot_table_kernel");
}

extern "C" int wm3_natten_bwd(const void* qkv, int ldqkv, const void* dout, int ldd, const void* o, int ldo,
                              const float* lse, float* gqkv, int ldg, float* partial, const int32_t* csr_off,
                              const int32_t* csr_ent, const float* factors, const float* rope_cos,
                              const float* rope_sin, unsigned* kv_amax, int depth, int rows, int cols, int heads,
                              int dhp, int wd, int wh, int ww, float scale, void* stream) {
  if (dhp != 128) return set_error("wm3_natten_bwd: head dim must be padded to 128 (got %d)", dhp);
  if ((ldd % 8) || (ldo % 8) || (ldg % 4)) return set_error("wm3_natten_bwd: bad leading dimensions");
  NaParams p;
  CUtensorMap tq, tkv;
  bool bias = false;
  if (natten_setup(qkv, ldqkv, const_cast<void*>(o), ldo, 1, depth, rows, cols, rows, 0, 0, 0, heads, dhp, wd, wh, ww,
                   scale, 0, rows, stream, p, tq, tkv, bias))
    return -1;
  if (!bias) return set_error("wm3_natten_bwd: the window mask must fit the MMA bias step (TD + TH + TW <= 16)");
  const uint64_t dims[4] = {static_cast<uint64_t>(heads * dhp), static_cast<uint64_t>(cols),
                            static_cast<uint64_t>(rows), static_cast<uint64_t>(depth)};
  const uint64_t strides[3] = {static_cast<uint64_t>(ldd), static_cast<uint64_t>(cols) * ldd,
                               static_cast<uint64_t>(cols) * rows * ldd};
  const uint32_t box[4] = {64, static_cast<uint32_t>(p.TW), static_cast<uint32_t>(p.TH), static_cast<uint32_t>(p.TD)};
  CUtensorMap tdo;
  if (make_tmap(&tdo, dout, TMAP_BF16, 4, dims, strides, box, nullptr)) return -1;
  NaBwd b{};
  b.dout = reinterpret_cast<const elem_t*>(dout);
  b.ldd = ldd;
  b.o = reinterpret_cast<const elem_t*>(o);
  b.ldo = ldo;
  b.lse = lse;
  b.gqkv = gqkv;
  b.ldg = ldg;
  b.partial = partial;
  b.factors = factors;
  if ((rope_cos == nullptr) != (rope_sin == nullptr)) return set_error("wm3_natten_bwd: give both rotary tables or none");
  if (ensure_smem_attr(reinterpret_cast<const void*>(natten_bwd_kernel<true>), NB_SMEM, "natten_bwd")) return -1;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int grid = p.nitems < sm_count() ? p.nitems : sm_count();
  natten_bwd_kernel<true><<<grid, NB_THREADS, NB_SMEM, s>>>(tq, tkv, tdo, p, b);
  if (check_launch("natten_bwd_kernel")) return -1;
  const int T = depth * rows * cols;
  const int blocks = std::min((T * heads * 32 + 255) / 256, sm_count() * 32);
  natten_bwd_reduce_kernel<<<blocks, 256, 0, s>>>(partial, csr_off, csr_ent, T, heads, p.ntd * p.nth * p.ntw,
                                                  p.maxch, factors, gqkv, ldg, rope_cos, rope_sin, kv_amax);
  return check_launch("natten_bwd_reduce_kernel");
}
