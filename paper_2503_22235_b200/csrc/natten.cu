// K1: fused 3D neighborhood attention forward on tcgen05 (reference attention.py:173-178,
// window arithmetic grid.py:96-130).
//
// One CTA = one (query tile, head).  A query tile is a TD x TH x TW box of tokens (<= 128 queries,
// one per TMEM lane / thread).  The union of the tile's windows is walked as a list of key chunks,
// each a run of rows of one depth plane x a contiguous (mod W) run of columns, <= 128 keys.  Per chunk:
//   cp.async gather of K, V rows (bf16, head slice) into SWIZZLE_128B tiles,
//   S = Q K^T          tcgen05.mma M128 N128, K = dhp, accumulator in TMEM columns [0,128)
//   online softmax     one thread per query row: window mask from the same integer formula as
//                      grid.py (bump on depth/rows, wrap on cols), running max / sum in fp32, exp2
//   P (bf16) -> smem   written over the dead K tile
//   O += P V           tcgen05.mma M128 N=dhp, K = 128 keys, V read MN-major, O in TMEM [128,128+dhp)
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
  int TD, TH, TW, ntd, nth, ntw;
  float scale_log2;
};

constexpr int NA_THREADS = 128;
constexpr uint32_t NA_TILE_BYTES = 32768;  // 128 rows x 256 B (dhp <= 128), or 128 x 128 keys of P
constexpr uint32_t NA_SMEM = 3 * NA_TILE_BYTES + 1024 /*align*/ + 512 /*key info + barriers*/;

// Copy `nrows` rows (head slice, dhp bf16 each) into a SW128 K-major tile; rows >= valid are zero.
// tok_of(row) returns the buffer token index or -1 for padding.
template <class TokFn>
DEVI void gather_rows(uint32_t dst, const __nv_bfloat16* base, int ld, int dhp, TokFn tok_of) {
  const int cpr = dhp / 8;  // 16-byte chunks per row
  const int rows_per_iter = NA_THREADS / cpr;
  const int c = threadIdx.x % cpr;
  for (int r = threadIdx.x / cpr; r < 128; r += rows_per_iter) {
    const int tok = tok_of(r);
    const __nv_bfloat16* src = base + (tok >= 0 ? static_cast<size_t>(tok) * ld + c * 8 : 0);
    const uint32_t d = dst + (c >> 3) * 16384u + sw128_off(r, c & 7);
    cp_async_16(d, src, tok >= 0 ? 16u : 0u);
  }
}

__global__ void __launch_bounds__(NA_THREADS, 2) natten_fwd_kernel(NaParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sQ = smem_u32(smem);
  const uint32_t sK = sQ + NA_TILE_BYTES;  // K tile, then P tile (aliased)
  const uint32_t sV = sK + NA_TILE_BYTES;
  int16_t* key_rr = reinterpret_cast<int16_t*>(smem + 3 * NA_TILE_BYTES);
  int16_t* key_cc = key_rr + 128;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 3 * NA_TILE_BYTES + 512);
  const uint32_t bar_s = smem_u32(bars);
  const uint32_t bar_o = smem_u32(bars + 1);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2);

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int head = blockIdx.y;
  const int tile = blockIdx.x;
  const int tw_i = tile % p.ntw;
  const int th_i = (tile / p.ntw) % p.nth;
  const int td_i = tile / (p.ntw * p.nth);
  const int d0 = td_i * p.TD, d1 = min(d0 + p.TD, p.depth);
  const int h0 = th_i * p.TH, h1 = min(h0 + p.TH, p.rows);  // local rows
  const int w0 = tw_i * p.TW, w1 = min(w0 + p.TW, p.cols);

  // this thread's query
  const int qd = d0 + tid / (p.TH * p.TW);
  const int qh = h0 + (tid / p.TW) % p.TH;
  const int qw = w0 + tid % p.TW;
  const bool qvalid = tid < p.TD * p.TH * p.TW && qd < d1 && qh < h1 && qw < w1;
  const int hw = (p.ww - 1) / 2;
  const int q_sd = bump_start(qvalid ? qd : d0, p.depth, p.wd);
  const int q_sh = bump_start((qvalid ? qh : h0) + p.row0, p.rows_global, p.wh);  // global row start

  // key union of the tile (grid.py:121-123 applied to the tile's extreme queries; bump is monotone)
  const int kd_lo = bump_start(d0, p.depth, p.wd);
  const int kd_hi = bump_start(d1 - 1, p.depth, p.wd) + p.wd;
  const int kr_lo = bump_start(h0 + p.row0, p.rows_global, p.wh);
  const int kr_hi = bump_start(h1 - 1 + p.row0, p.rows_global, p.wh) + p.wh;
  const int nrows_u = kr_hi - kr_lo;
  int pc0, ncp;
  if ((w1 - w0) + p.ww - 1 >= p.cols) { pc0 = 0; ncp = p.cols; }
  else { pc0 = w0 - hw; ncp = (w1 - w0) + p.ww - 1; }
  const int nrpc = min(nrows_u, 128 / ncp);
  const int nrchunks = (nrows_u + nrpc - 1) / nrpc;
  const int nchunks = (kd_hi - kd_lo) * nrchunks;
  const int brow0 = p.row0 - p.halo_lo;  // global row of buffer row 0
  // column offset of this query's window inside the patch: valid cc iff (cc - q_cc0) mod W < ww
  const int q_cc0 = wrap_col((qvalid ? qw : w0) - hw - pc0, p.cols);

  if (tid == 0) {
    mbar_init(bar_s, 1);
    mbar_init(bar_o, 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    tmem_alloc(smem_u32(tmem_slot), 256);
    tmem_relinquish();
  }

  const int sec = p.heads * p.dhp;  // columns per q/k/v section
  const __nv_bfloat16* qbase = p.qkv + head * p.dhp;
  const __nv_bfloat16* kbase = p.qkv + sec + head * p.dhp;
  const __nv_bfloat16* vbase = p.qkv + 2 * sec + head * p.dhp;

  // Q tile
  gather_rows(sQ, qbase, p.ldqkv, p.dhp, [&](int r) -> int {
    const int rd = d0 + r / (p.TH * p.TW), rh = h0 + (r / p.TW) % p.TH, rw = w0 + r % p.TW;
    if (r >= p.TD * p.TH * p.TW || rd >= d1 || rh >= h1 || rw >= w1) return -1;
    return (rd * p.rows_ext + rh + p.halo_lo) * p.cols + rw;
  });
  cp_async_commit();

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS = tmem;         // columns [0,128)
  const uint32_t tO = tmem + 128;   // columns [128, 128+dhp)
  const uint32_t lane_off = static_cast<uint32_t>(32 * warp) << 16;

  float m_run = -INFINITY, l_run = 0.f;
  uint32_t ph_s = 0, ph_o = 0;
  const uint32_t idesc_s = make_idesc_bf16(128, 128, 0, 0);
  const uint32_t idesc_o = make_idesc_bf16(128, p.dhp, 0, 1);
  const int kblocks = p.dhp / 64;

  for (int j = 0; j < nchunks; ++j) {
    const int kd = kd_lo + j / nrchunks;
    const int kr0 = kr_lo + (j % nrchunks) * nrpc;
    const int nr = min(nrpc, kr_hi - kr0);
    const int nkeys = nr * ncp;
    // K/V gather for this chunk (K buffer is free: the previous PV has retired)
    auto tok_of = [&](int r) -> int {
      if (r >= nkeys) return -1;
      const int rr = r / ncp, cc = r - (r / ncp) * ncp;
      return (kd * p.rows_ext + (kr0 + rr - brow0)) * p.cols + wrap_col(pc0 + cc, p.cols);
    };
    gather_rows(sK, kbase, p.ldqkv, p.dhp, tok_of);
    gather_rows(sV, vbase, p.ldqkv, p.dhp, tok_of);
    cp_async_commit();
    {
      const int r = tid;
      key_rr[r] = r < nkeys ? static_cast<int16_t>(kr0 + r / ncp) : static_cast<int16_t>(-30000);
      key_cc[r] = r < nkeys ? static_cast<int16_t>(r % ncp) : static_cast<int16_t>(0);
    }
    cp_async_wait<0>();
    fence_proxy_async();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
#pragma unroll 1
      for (int s = 0; s < kblocks * 4; ++s) {
        const uint32_t off = (s >> 2) * 16384u + (s & 3) * 32u;
        umma_bf16_ss(tS, make_sdesc_sw128(sQ + off, 16, 1024), make_sdesc_sw128(sK + off, 16, 1024), idesc_s,
                     s > 0 ? 1u : 0u);
      }
      umma_commit(bar_s);
    }
    mbar_wait(bar_s, ph_s);
    ph_s ^= 1;
    tc_fence_after();

    // ---- softmax over this chunk (row = query) ----
    const bool depth_ok = qvalid && (kd - q_sd) >= 0 && (kd - q_sd) < p.wd;
    float mx = -INFINITY;
#pragma unroll 1
    for (int sl = 0; sl < 4; ++sl) {
      uint32_t r[32];
      tmem_ld32(tS + lane_off + 32 * sl, r);
      tmem_ld_wait();
#pragma unroll
      for (int e = 0; e < 32; ++e) {
        const int k = 32 * sl + e;
        const int dr = key_rr[k] - q_sh;
        int dc = key_cc[k] - q_cc0;
        dc += dc < 0 ? p.cols : 0;
        const bool ok = depth_ok && dr >= 0 && dr < p.wh && dc < p.ww;
        const float v = ok ? __uint_as_float(r[e]) * p.scale_log2 : -INFINITY;
        mx = fmaxf(mx, v);
      }
    }
    const float m_new = fmaxf(m_run, mx);
    const float m_use = (m_new == -INFINITY) ? 0.f : m_new;
    const float alpha = exp2f(m_run - m_use);  // m_run = -inf -> 0
    float lsum = 0.f;
    // P goes over the dead K tile
#pragma unroll 1
    for (int sl = 0; sl < 4; ++sl) {
      uint32_t r[32];
      tmem_ld32(tS + lane_off + 32 * sl, r);
      tmem_ld_wait();
      uint32_t pk[16];
#pragma unroll
      for (int e = 0; e < 32; e += 2) {
        float pv[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int k = 32 * sl + e + u;
          const int dr = key_rr[k] - q_sh;
          int dc = key_cc[k] - q_cc0;
          dc += dc < 0 ? p.cols : 0;
          const bool ok = depth_ok && dr >= 0 && dr < p.wh && dc < p.ww;
          pv[u] = ok ? exp2f(__uint_as_float(r[e + u]) * p.scale_log2 - m_use) : 0.f;
          lsum += pv[u];
        }
        pk[e / 2] = pack_bf16(pv[0], pv[1]);
      }
      // keys [32sl, 32sl+32) -> region (sl/2), 16B chunks ((sl%2)*4 .. +4)
      const uint32_t region = sK + (sl >> 1) * 16384u;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t addr = region + sw128_off(tid, (sl & 1) * 4 + q);
        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(pk[4 * q]), "r"(pk[4 * q + 1]),
                     "r"(pk[4 * q + 2]), "r"(pk[4 * q + 3])
                     : "memory");
      }
    }
    l_run = l_run * alpha + lsum;
    m_run = m_new;
    // rescale the running O (previous PV retired: we waited on bar_o at the end of the last chunk)
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
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
#pragma unroll 1
      for (int s = 0; s < 8; ++s) {  // 128 keys, 16 per MMA
        const uint64_t ad = make_sdesc_sw128(sK + (s >> 2) * 16384u + (s & 3) * 32u, 16, 1024);
        const uint64_t bd = make_sdesc_sw128(sV + s * 2048u, 16384, 1024);
        umma_bf16_ss(tO, ad, bd, idesc_o, (j > 0 || s > 0) ? 1u : 0u);
      }
      umma_commit(bar_o);
    }
    mbar_wait(bar_o, ph_o);
    ph_o ^= 1;
    tc_fence_after();
  }

  // ---- epilogue: O / l -> bf16 ctx ----
  const float inv_l = (qvalid && l_run > 0.f) ? 1.f / l_run : 0.f;
  __nv_bfloat16* orow =
      p.out + (qvalid ? (static_cast<size_t>((qd * p.rows + qh) * p.cols + qw) * p.ldo + head * p.dhp) : 0);
#pragma unroll 1
  for (int c = 0; c < p.dhp / 32; ++c) {
    uint32_t r[32];
    tmem_ld32(tO + lane_off + 32 * c, r);
    tmem_ld_wait();
    if (qvalid) {
      float v[32];
#pragma unroll
      for (int e = 0; e < 32; ++e) v[e] = __uint_as_float(r[e]) * inv_l;
      uint4* d4 = reinterpret_cast<uint4*>(orow + 32 * c);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint4 u;
        u.x = pack_bf16(v[8 * q + 0], v[8 * q + 1]);
        u.y = pack_bf16(v[8 * q + 2], v[8 * q + 3]);
        u.z = pack_bf16(v[8 * q + 4], v[8 * q + 5]);
        u.w = pack_bf16(v[8 * q + 6], v[8 * q + 7]);
        d4[q] = u;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 256);
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
  p.scale_log2 = scale * 1.4426950408889634f;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(natten_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, NA_SMEM);
    if (e != cudaSuccess) return set_error("cudaFuncSetAttribute(natten): %s", cudaGetErrorString(e));
    attr = true;
  }
  dim3 grid(p.ntd * p.nth * p.ntw, heads);
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
