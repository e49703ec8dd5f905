// Persistent warp-specialised tcgen05 GEMM with fused epilogues (K2-K5 of DESIGN.md).
//
//   C[M, N] = A[M, K] * B[N, K]^T     A: activations bf16 (K-major), B: weights bf16 pre-transposed
//                                     to (out, in) so both operands are K-major SWIZZLE_128B tiles.
// Roles (one CTA per SM, 256 threads):
//   warp 0      TMA producer: A/B k-blocks into a STAGES-deep smem ring (mbarrier full/empty)
//   warp 1      MMA issuer: one thread issues tcgen05.mma 128xBNx16, accumulator in TMEM,
//               double-buffered (2 x BN columns) so the epilogue of tile i overlaps MMAs of tile i+1
//   warp 2      TMEM allocator
//   warps 4..7  epilogue: tcgen05.ld 32 columns at a time, bias / GELU / residual / rotary, store
// Reference semantics: attention.py:142-143 (_linear), :167-171 (q,k,v + rotary), :179 and :183
// (residual adds), :182 (exact-erf GELU, autodiff.py:372-382).
#include "common.cuh"
#include "launch.h"
#include "../../include/wm3.h"

namespace wm3 {

struct EpiParams {
  void* out;
  int ldo;
  int n_valid;
  const float* bias;
  wm3_rope_t rope;
};

constexpr int GEMM_BM = 128;
constexpr int GEMM_BK = 64;
constexpr int GEMM_THREADS = 256;

template <int BN>
struct GemmCfg {
  static constexpr int STAGES = (BN == 256) ? 4 : 6;
  static constexpr uint32_t A_BYTES = GEMM_BM * GEMM_BK * 2;
  static constexpr uint32_t B_BYTES = BN * GEMM_BK * 2;
  static constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr uint32_t SMEM = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
  static constexpr uint32_t TMEM_COLS = 2 * BN;
};

DEVI void store_bf16x32(__nv_bfloat16* dst, const float* v, int nvalid) {
  if (nvalid >= 32) {
    uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint4 u;
      u.x = pack_bf16(v[8 * q + 0], v[8 * q + 1]);
      u.y = pack_bf16(v[8 * q + 2], v[8 * q + 3]);
      u.z = pack_bf16(v[8 * q + 4], v[8 * q + 5]);
      u.w = pack_bf16(v[8 * q + 6], v[8 * q + 7]);
      d4[q] = u;
    }
  } else {
    for (int e = 0; e < nvalid; ++e) dst[e] = __float2bfloat16_rn(v[e]);
  }
}

template <int EPI>
DEVI void epi_simple_chunk(const EpiParams& ep, uint32_t (&r)[32], int row, int n) {
  float v[32];
#pragma unroll
  for (int e = 0; e < 32; ++e) v[e] = __uint_as_float(r[e]);
  const int nvalid = min(32, ep.n_valid - n);
  if (nvalid <= 0) return;
  if (EPI != WM3_EPI_F32 && ep.bias != nullptr) {
    if (nvalid >= 32) {
      const float4* b4 = reinterpret_cast<const float4*>(ep.bias + n);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        float4 b = __ldg(b4 + q);
        v[4 * q + 0] += b.x; v[4 * q + 1] += b.y; v[4 * q + 2] += b.z; v[4 * q + 3] += b.w;
      }
    } else {
      for (int e = 0; e < nvalid; ++e) v[e] += __ldg(ep.bias + n + e);
    }
  }
  if (EPI == WM3_EPI_BIAS_GELU_BF16) {
#pragma unroll
    for (int e = 0; e < 32; ++e) v[e] = gelu_erf(v[e]);
  }
  if (EPI == WM3_EPI_F32 || EPI == WM3_EPI_BIAS_RESID_F32) {
    float* dst = reinterpret_cast<float*>(ep.out) + static_cast<size_t>(row) * ep.ldo + n;
    if (nvalid >= 32) {
      float4* d4 = reinterpret_cast<float4*>(dst);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        float4 o = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        if (EPI == WM3_EPI_BIAS_RESID_F32) {
          float4 x = d4[q];
          o.x += x.x; o.y += x.y; o.z += x.z; o.w += x.w;
        }
        d4[q] = o;
      }
    } else {
      for (int e = 0; e < nvalid; ++e) dst[e] = (EPI == WM3_EPI_BIAS_RESID_F32 ? dst[e] : 0.f) + v[e];
    }
  } else {
    __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(ep.out) + static_cast<size_t>(row) * ep.ldo + n;
    store_bf16x32(dst, v, nvalid);
  }
}

// q/k/v + bias, rotary (NeoX half split, attention.py:87-92) on the q and k sections.
template <int BN>
DEVI void epi_qkv_rope(const EpiParams& ep, uint32_t taddr, int row, int n0, int M) {
  const wm3_rope_t& rp = ep.rope;
  const int dhp = rp.dhp;
  const int half = dhp >> 1;
  const int heads_per_tile = BN / dhp;
  const int qk_cols = 2 * rp.heads * dhp;
  // token coordinates (global row for the rotary phase; attention.py:242 uses global (d,h,w))
  int t = row < M ? row : 0;
  const int c = t % rp.cols;
  const int rr = (t / rp.cols) % rp.rows + rp.row0;
  const int d = t / (rp.cols * rp.rows);
  const float* cd = rp.rope_cos + (0 * rp.emax + d) * 64;
  const float* ch = rp.rope_cos + (1 * rp.emax + rr) * 64;
  const float* cw = rp.rope_cos + (2 * rp.emax + c) * 64;
  const float* sd = rp.rope_sin + (0 * rp.emax + d) * 64;
  const float* sh = rp.rope_sin + (1 * rp.emax + rr) * 64;
  const float* sw = rp.rope_sin + (2 * rp.emax + c) * 64;
  const int pd = rp.pd, pdr = rp.pd + rp.pr;
  for (int hh = 0; hh < heads_per_tile; ++hh) {
    for (int cc = 0; cc < dhp / 64; ++cc) {
      const int j0 = 32 * cc;
      const int col1 = hh * dhp + j0;
      const int col2 = col1 + half;
      uint32_t r1[32], r2[32];
      tmem_ld32(taddr + col1, r1);
      tmem_ld32(taddr + col2, r2);
      tmem_ld_wait();
      const int n1 = n0 + col1, n2 = n0 + col2;
      if (row >= M || n1 >= ep.n_valid) continue;
      float a[32], b[32];
#pragma unroll
      for (int e = 0; e < 32; ++e) {
        a[e] = __uint_as_float(r1[e]) + __ldg(ep.bias + n1 + e);
        b[e] = __uint_as_float(r2[e]) + __ldg(ep.bias + n2 + e);
      }
      if (n1 < qk_cols) {
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          const int j = j0 + e;
          const float* cp = j < pd ? cd : (j < pdr ? ch : cw);
          const float* sp = j < pd ? sd : (j < pdr ? sh : sw);
          const float cs = __ldg(cp + j), sn = __ldg(sp + j);
          const float x1 = a[e], x2 = b[e];
          a[e] = x1 * cs - x2 * sn;
          b[e] = x1 * sn + x2 * cs;
        }
      }
      __nv_bfloat16* base = reinterpret_cast<__nv_bfloat16*>(ep.out) + static_cast<size_t>(row) * ep.ldo;
      store_bf16x32(base + n1, a, min(32, ep.n_valid - n1));
      store_bf16x32(base + n2, b, min(32, ep.n_valid - n2));
    }
  }
}

template <int BN, int EPI>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M, int N,
                   int K, EpiParams ep) {
  using Cfg = GemmCfg<BN>;
  constexpr int STAGES = Cfg::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = smem_u32(smem);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::STAGE_BYTES);
  const uint32_t bar0 = smem_u32(bars);
  auto full_bar = [&](int s) { return bar0 + 8u * s; };
  auto empty_bar = [&](int s) { return bar0 + 8u * (STAGES + s); };
  auto tfull_bar = [&](int a) { return bar0 + 8u * (2 * STAGES + a); };
  auto tempty_bar = [&](int a) { return bar0 + 8u * (2 * STAGES + 2 + a); };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 4);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int nm = (M + GEMM_BM - 1) / GEMM_BM;
  const int nn = (N + BN - 1) / BN;
  const int ntiles = nm * nn;
  const int nk = (K + GEMM_BK - 1) / GEMM_BK;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(empty_bar(s), 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull_bar(a), 1);
      mbar_init(tempty_bar(a), 4);
    }
    fence_barrier_init();
  }
  if (warp == 2) {
    tmem_alloc(smem_u32(tmem_slot), Cfg::TMEM_COLS);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int m0 = (tile / nn) * GEMM_BM;
        const int n0 = (tile % nn) * BN;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(empty_bar(stage), phase ^ 1);
          const uint32_t sa = sbase + stage * Cfg::STAGE_BYTES;
          const uint32_t sb = sa + Cfg::A_BYTES;
          mbar_arrive_expect_tx(full_bar(stage), Cfg::STAGE_BYTES);
          tma_load_2d(sa, &tmA, full_bar(stage), kb * GEMM_BK, m0);
          tma_load_2d(sb, &tmB, full_bar(stage), kb * GEMM_BK, n0);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = make_idesc_bf16(GEMM_BM, BN, 0, 0);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t aphase = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        mbar_wait(tempty_bar(acc), aphase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(full_bar(stage), phase);
          tc_fence_after();
          const uint32_t sa = sbase + stage * Cfg::STAGE_BYTES;
          const uint32_t sb = sa + Cfg::A_BYTES;
#pragma unroll
          for (int k = 0; k < GEMM_BK / 16; ++k) {
            const uint64_t ad = make_sdesc_sw128(sa + k * 32, 16, 1024);
            const uint64_t bd = make_sdesc_sw128(sb + k * 32, 16, 1024);
            umma_bf16_ss(d_tmem, ad, bd, idesc, (kb | k) != 0 ? 1u : 0u);
          }
          umma_commit(empty_bar(stage));
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        umma_commit(tfull_bar(acc));
        acc ^= 1;
        if (acc == 0) aphase ^= 1;
      }
    }
  } else if (warp >= 4) {
    const int q = warp & 3;
    int acc = 0;
    uint32_t aphase = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      const int m0 = (tile / nn) * GEMM_BM;
      const int n0 = (tile % nn) * BN;
      mbar_wait(tfull_bar(acc), aphase);
      tc_fence_after();
      const int row = m0 + 32 * q + lane;
      const uint32_t taddr = tmem_base + acc * BN + (static_cast<uint32_t>(32 * q) << 16);
      if (EPI == WM3_EPI_QKV_ROPE) {
        epi_qkv_rope<BN>(ep, taddr, row, n0, M);
      } else {
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
          uint32_t r[32];
          tmem_ld32(taddr + 32 * c, r);
          tmem_ld_wait();
          if (row < M) epi_simple_chunk<EPI>(ep, r, row, n0 + 32 * c);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty_bar(acc));
      acc ^= 1;
      if (acc == 0) aphase ^= 1;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
  }
}

template <int BN, int EPI>
static int launch_gemm(const CUtensorMap& ta, const CUtensorMap& tb, int M, int N, int K, const EpiParams& ep,
                       cudaStream_t stream) {
  using Cfg = GemmCfg<BN>;
  auto kern = gemm_tc_kernel<BN, EPI>;
  static bool attr_done = false;
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    if (e != cudaSuccess) return set_error("cudaFuncSetAttribute(gemm): %s", cudaGetErrorString(e));
    attr_done = true;
  }
  const int ntiles = ((M + GEMM_BM - 1) / GEMM_BM) * ((N + BN - 1) / BN);
  const int grid = ntiles < sm_count() ? ntiles : sm_count();
  kern<<<grid, GEMM_THREADS, Cfg::SMEM, stream>>>(ta, tb, M, N, K, ep);
  return check_launch("gemm_tc_kernel");
}

template <int BN>
static int dispatch_epi(int epi, const CUtensorMap& ta, const CUtensorMap& tb, int M, int N, int K,
                        const EpiParams& ep, cudaStream_t s) {
  switch (epi) {
    case WM3_EPI_F32: return launch_gemm<BN, WM3_EPI_F32>(ta, tb, M, N, K, ep, s);
    case WM3_EPI_BIAS_BF16: return launch_gemm<BN, WM3_EPI_BIAS_BF16>(ta, tb, M, N, K, ep, s);
    case WM3_EPI_BIAS_GELU_BF16: return launch_gemm<BN, WM3_EPI_BIAS_GELU_BF16>(ta, tb, M, N, K, ep, s);
    case WM3_EPI_BIAS_RESID_F32: return launch_gemm<BN, WM3_EPI_BIAS_RESID_F32>(ta, tb, M, N, K, ep, s);
    case WM3_EPI_QKV_ROPE: return launch_gemm<BN, WM3_EPI_QKV_ROPE>(ta, tb, M, N, K, ep, s);
    default: return set_error("wm3_linear: unknown epilogue %d", epi);
  }
}

}  // namespace wm3

using namespace wm3;

extern "C" int wm3_linear(const void* a, int lda, const void* b, int ldb, int m, int n, int k, int epi, void* out,
                          int ldo, int n_valid, const float* bias, const wm3_rope_t* rope, void* stream) {
  if (m <= 0 || n <= 0 || k <= 0) return set_error("wm3_linear: bad sizes m=%d n=%d k=%d", m, n, k);
  const bool f32_out = (epi == WM3_EPI_F32 || epi == WM3_EPI_BIAS_RESID_F32);
  if ((lda % 8) || (ldb % 8) || (ldo % (f32_out ? 4 : 8)))
    return set_error("wm3_linear: pitches must be multiples of 8 (bf16) / 4 (f32 out)");
  if (n % 32) return set_error("wm3_linear: n=%d must be a multiple of 32", n);
  if (epi != WM3_EPI_F32 && bias == nullptr) return set_error("wm3_linear: bias required");
  EpiParams ep{};
  ep.out = out;
  ep.ldo = ldo;
  ep.n_valid = n_valid;
  ep.bias = bias;
  if (epi == WM3_EPI_QKV_ROPE) {
    if (rope == nullptr) return set_error("wm3_linear: rope descriptor required");
    ep.rope = *rope;
    if (ep.rope.dhp != 64 && ep.rope.dhp != 128) return set_error("wm3_linear: dhp must be 64 or 128");
  }
  const int bn = (n >= 256) ? 256 : 128;
  if (epi == WM3_EPI_QKV_ROPE && (bn % ep.rope.dhp)) return set_error("wm3_linear: tile/head mismatch");
  CUtensorMap ta, tb;
  if (make_tmap_2d_bf16(&ta, a, k, m, lda, GEMM_BK, GEMM_BM)) return -1;
  if (make_tmap_2d_bf16(&tb, b, k, n, ldb, GEMM_BK, bn)) return -1;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  return bn == 256 ? dispatch_epi<256>(epi, ta, tb, m, n, k, ep, s) : dispatch_epi<128>(epi, ta, tb, m, n, k, ep, s);
}
