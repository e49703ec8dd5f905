// Reverse-mode pieces of one processor block (reference autodiff.py backward rules of layernorm :400-424, gelu
// :372-382, matmul :350-369, the attention gather / softmax / matmuls attention.py:166-178 and the rotary
// rotation :87-92).  The block VJP (paper_2503_22235_b200/backward.py) chains them with the forward GEMM kernel:
// every weight / input gradient GEMM runs on the tcgen05 GEMM (gemm.cu) with 16-bit operands, so gradients are
// cast with a per-tensor power-of-two scale (wm3_bw_amax) that puts their largest magnitude near 2^14 — fp16
// holds them without underflow — and the consumers of the fp32 GEMM results divide the scale back out.
//
// Everything here is deterministic: maxima use order-independent atomicMax, sums run in a fixed order (column
// sums as fixed row chunks + an ordered second pass; the attention key gradients walk an inverse neighbor list
// sorted by query), so a recomputed segment's gradients are bitwise those of the first computation (the
// reference's checkpoint / offload parity contract, autodiff.py:893-924, offload.py:287-412).
#include <cmath>

#include "common.cuh"
#include "launch.h"
#include "../../include/wm3.h"

namespace wm3 {

DEVI float to_f(__half v) { return __half2float(v); }
DEVI float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }

// Row strips: block b takes rows b, b + grid, ...; its threads sweep the columns (4 at a time when the rows are
// 16-byte aligned), so there is no per-element 64-bit index division; one atomic per block.
__global__ void bw_amax_kernel(const float* __restrict__ x, int rows, int cols, int ld, unsigned* amax_bits) {
  __shared__ float red[32];
  float m = 0.f;
  const bool v4 = (cols % 4 == 0) && (ld % 4 == 0) && (reinterpret_cast<uintptr_t>(x) % 16 == 0);
  for (int r = blockIdx.x; r < rows; r += gridDim.x) {
    const float* xr = x + static_cast<size_t>(r) * ld;
    if (v4) {
      for (int c = 4 * threadIdx.x; c < cols; c += 4 * blockDim.x) {
        const float4 q = __ldg(reinterpret_cast<const float4*>(xr + c));
        m = fmaxf(m, fmaxf(fmaxf(fabsf(q.x), fabsf(q.y)), fmaxf(fabsf(q.z), fabsf(q.w))));
      }
    } else {
      for (int c = threadIdx.x; c < cols; c += blockDim.x) m = fmaxf(m, fabsf(xr[c]));
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (threadIdx.x == 0) atomicMax(amax_bits, __float_as_uint(m));
  }
}

// dst = operand(src * scale), row-major [rows][ld_dst] (columns >= cols zero) or transposed [cols][ld_dst]
// (columns >= rows zero); src fp32 (f32 = 1) or 16-bit operand.  32 x 32 tiles through shared memory.
__global__ void bw_cast_kernel(const void* __restrict__ src, int f32, int rows, int cols, int lds,
                               elem_t* __restrict__ dst, int ldd, int transpose, const unsigned* amax_bits) {
  __shared__ float tile[32][33];
  const float s = grad_scale(amax_bits);
  const int tr = blockIdx.y * 32, tc = blockIdx.x * 32;  // tile origin in dst coordinates
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8 threads
  if (!transpose) {  // (row-major casts take bw_cast_rows_kernel; kept for completeness)
    for (int i = ty; i < 32; i += 8) {
      const int r = tr + i, c = tc + tx;
      if (r >= rows || c >= ldd) continue;
      float v = 0.f;
      if (c < cols) {
        const size_t o = static_cast<size_t>(r) * lds + c;
        v = f32 ? static_cast<const float*>(src)[o] : unpack_elem2(static_cast<const uint16_t*>(src)[o]).x;
      }
      dst[static_cast<size_t>(r) * ldd + c] = to_elem(v * s);
    }
    return;
  }
  // dst [cols][ldd] = src^T: dst row = src column
  for (int i = ty; i < 32; i += 8) {
    const int sr = tc + i, sc = tr + tx;  // read src (row sr = dst column, col sc = dst row), coalesced over sc
    float v = 0.f;
    if (sr < rows && sc < cols) {
      const size_t o = static_cast<size_t>(sr) * lds + sc;
      v = f32 ? static_cast<const float*>(src)[o] : unpack_elem2(static_cast<const uint16_t*>(src)[o]).x;
    }
    tile[i][tx] = v;
  }
  __syncthreads();
  for (int i = ty; i < 32; i += 8) {
    const int dr = tr + i, dc = tc + tx;
    if (dr < cols && dc < ldd) dst[static_cast<size_t>(dr) * ldd + dc] = to_elem(tile[tx][i] * s);
  }
}

// Row-major fp32 -> 16-bit operand copy (times the scale), 8 elements per thread-step: two 16-byte loads, one
// 16-byte store; columns in [cols, ldd) are zero.  Needs cols, lds, ldd multiples of 8 and aligned bases.
__global__ void bw_cast_rows_kernel(const float* __restrict__ src, int rows, int cols, int lds, elem_t* __restrict__ dst,
                                    int ldd, const unsigned* amax_bits) {
  const float s = grad_scale(amax_bits);
  for (int r = blockIdx.x; r < rows; r += gridDim.x) {
    const float* sr = src + static_cast<size_t>(r) * lds;
    elem_t* dr = dst + static_cast<size_t>(r) * ldd;
    for (int c = 8 * threadIdx.x; c < ldd; c += 8 * blockDim.x) {
      uint4 o = make_uint4(0u, 0u, 0u, 0u);
      if (c < cols) {
        const float4 a = __ldg(reinterpret_cast<const float4*>(sr + c));
        const float4 b = __ldg(reinterpret_cast<const float4*>(sr + c + 4));
        o = make_uint4(pack_elem(a.x * s, a.y * s), pack_elem(a.z * s, a.w * s), pack_elem(b.x * s, b.y * s),
                       pack_elem(b.z * s, b.w * s));
      }
      *reinterpret_cast<uint4*>(dr + c) = o;
    }
  }
}

// partial[chunk][c] = sum over rows [chunk * 256, +256) of src[r][c] (optionally times src2[r][c]), row order
constexpr int BW_CHUNK = 256;
__global__ void bw_colsum_partial_kernel(const float* __restrict__ src, const float* __restrict__ src2, int rows,
                                         int cols, int ld, float* __restrict__ partial) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cols) return;
  const int r0 = blockIdx.y * BW_CHUNK, r1 = min(rows, r0 + BW_CHUNK);
  float acc = 0.f;
  for (int r = r0; r < r1; ++r) {
    const float v = src[static_cast<size_t>(r) * ld + c];
    acc += src2 != nullptr ? v * src2[static_cast<size_t>(r) * ld + c] : v;
  }
  partial[static_cast<size_t>(blockIdx.y) * cols + c] = acc;
}

// Vectorised column sums over one BW_CHUNK-row chunk (cols, leading dims multiple of 4, 16-byte aligned bases):
// block = 256 columns x 4 row groups, thread (quad q, group k) adds rows r0 + k, r0 + k + 4, ... of columns
// 4q .. 4q + 3 with 16-byte loads, and the 4 group sums are added in group order through shared memory into
// partial[chunk][c] — a fixed order, and 4x the bytes in flight of one float per thread.  MODE 0: v = g;
// MODE 1: v = g * a (product sums); MODE 2: v = (g / scale) * gelu'(a + bias), stored to out; MODE 3: v = g, and
// the 16-bit operand copy v * scale(in_scale_bits) stored to out ([rows][ldo], columns [cols, ldo) zero — the
// cast and the bias gradient in one pass once the producer has left max |g| in in_scale_bits).  With amax_bits,
// also atomicMax of max |v| (one per block).
template <int MODE>
__global__ void __launch_bounds__(256) bw_colsum4_kernel(const float* __restrict__ g, int ldg,
                                                         const float* __restrict__ a, int lda,
                                                         const float* __restrict__ bias,
                                                         const unsigned* in_scale_bits, int rows, int cols,
                                                         float* __restrict__ out, int ldo,
                                                         float* __restrict__ partial, unsigned* amax_bits) {
  __shared__ float red[4][257];
  __shared__ float redm[8];
  const int q = threadIdx.x & 63, k = threadIdx.x >> 6;
  const int c = blockIdx.x * 256 + 4 * q;
  const bool ok = c < cols;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  float m = 0.f;
  if (ok) {
    const int r0 = blockIdx.y * BW_CHUNK, r1 = min(rows, r0 + BW_CHUNK);
    float inv = 1.f;
    float4 b = make_float4(0.f, 0.f, 0.f, 0.f);
    if (MODE == 2) {
      inv = 1.f / grad_scale(in_scale_bits);
      b = __ldg(reinterpret_cast<const float4*>(bias + c));
    }
    const float sc = MODE == 3 ? grad_scale(in_scale_bits) : 1.f;
#pragma unroll 4
    for (int r = r0 + k; r < r1; r += 4) {
      float4 v = __ldg(reinterpret_cast<const float4*>(g + static_cast<size_t>(r) * ldg + c));
      if (MODE == 1) {
        const float4 w = __ldg(reinterpret_cast<const float4*>(a + static_cast<size_t>(r) * lda + c));
        v.x *= w.x; v.y *= w.y; v.z *= w.z; v.w *= w.w;
      } else if (MODE == 3) {  // operand copy times the scale (the cast), column sums of the unscaled values
        *reinterpret_cast<uint2*>(reinterpret_cast<elem_t*>(out) + static_cast<size_t>(r) * ldo + c) =
            make_uint2(pack_elem(v.x * sc, v.y * sc), pack_elem(v.z * sc, v.w * sc));
      } else if (MODE == 2) {
        const float4 z = __ldg(reinterpret_cast<const float4*>(a + static_cast<size_t>(r) * lda + c));
        v.x = v.x * inv * gelu_grad(z.x + b.x);
        v.y = v.y * inv * gelu_grad(z.y + b.y);
        v.z = v.z * inv * gelu_grad(z.z + b.z);
        v.w = v.w * inv * gelu_grad(z.w + b.w);
        *reinterpret_cast<float4*>(out + static_cast<size_t>(r) * ldo + c) = v;
      }
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
      m = fmaxf(m, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
    }
  }
  if (MODE == 3 && !ok && c < ldo) {  // operand padding columns [cols, ldo) are zero
    const int r0 = blockIdx.y * BW_CHUNK, r1 = min(rows, r0 + BW_CHUNK);
    for (int r = r0 + k; r < r1; r += 4)
      *reinterpret_cast<uint2*>(reinterpret_cast<elem_t*>(out) + static_cast<size_t>(r) * ldo + c) = make_uint2(0u, 0u);
  }
  red[k][4 * q + 0] = acc.x;
  red[k][4 * q + 1] = acc.y;
  red[k][4 * q + 2] = acc.z;
  red[k][4 * q + 3] = acc.w;
  if (amax_bits != nullptr) {
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) redm[threadIdx.x >> 5] = m;
  }
  __syncthreads();
  const int cc = blockIdx.x * 256 + threadIdx.x;
  if (cc < cols)
    partial[static_cast<size_t>(blockIdx.y) * cols + cc] =
        ((red[0][threadIdx.x] + red[1][threadIdx.x]) + red[2][threadIdx.x]) + red[3][threadIdx.x];
  if (amax_bits != nullptr && threadIdx.x == 0) {
    float t = redm[0];
#pragma unroll
    for (int w = 1; w < 8; ++w) t = fmaxf(t, redm[w]);
    atomicMax(amax_bits, __float_as_uint(t));
  }
}

static inline bool aligned16(const void* p) { return p == nullptr || reinterpret_cast<uintptr_t>(p) % 16 == 0; }

// One pass for a gradient that needs both its column sums (a bias gradient) and its max |x| (the operand
// scale of the next cast): bw_colsum_partial_kernel's fixed row chunks plus one atomicMax per block.  With `a`
// set it first applies the GELU derivative, out = (g / scale) * gelu'(a + bias) (bw_gelu_kernel), and stores
// it — the GELU backward, the bias gradient and the scale of the W1 operands read the tensor once.
__global__ void bw_colsum_amax_kernel(const float* __restrict__ g, int ldg, const float* __restrict__ a, int lda,
                                      const float* __restrict__ bias, const unsigned* in_scale_bits, int rows,
                                      int cols, float* __restrict__ out, int ldo, float* __restrict__ partial,
                                      unsigned* amax_bits) {
  __shared__ float red[32];
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  float acc = 0.f, m = 0.f;
  if (c < cols) {
    const int r0 = blockIdx.y * BW_CHUNK, r1 = min(rows, r0 + BW_CHUNK);
    if (a != nullptr) {
      const float inv = 1.f / grad_scale(in_scale_bits), b = __ldg(bias + c);
#pragma unroll 4
      for (int r = r0; r < r1; ++r) {
        const float z = a[static_cast<size_t>(r) * lda + c] + b;
        const float d =
            0.5f * (1.f + erff(z * 0.70710678118654752f)) + z * 0.39894228040143268f * __expf(-0.5f * z * z);
        const float v = g[static_cast<size_t>(r) * ldg + c] * inv * d;
        out[static_cast<size_t>(r) * ldo + c] = v;
        acc += v;
        m = fmaxf(m, fabsf(v));
      }
    } else {
#pragma unroll 4
      for (int r = r0; r < r1; ++r) {
        const float v = g[static_cast<size_t>(r) * ldg + c];
        acc += v;
        m = fmaxf(m, fabsf(v));
      }
    }
    partial[static_cast<size_t>(blockIdx.y) * cols + c] = acc;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (threadIdx.x == 0) atomicMax(amax_bits, __float_as_uint(m));
  }
}

// out[c] = (sum over k of partial[k][c]) / scale.  Block: 32 columns x 8 lanes groups; group q adds partials
// q, q + 8, q + 16, ... in order, then the 8 group sums are added in group order (a fixed order for any launch).
__global__ void __launch_bounds__(256) bw_colsum_final_kernel(const float* __restrict__ partial, int chunks, int cols,
                                                              const unsigned* amax_bits, float* __restrict__ out) {
  __shared__ float red[8][33];
  const int cl = threadIdx.x & 31, q = threadIdx.x >> 5, c = blockIdx.x * 32 + cl;
  float acc = 0.f;
  if (c < cols) {
#pragma unroll 4
    for (int k = q; k < chunks; k += 8) acc += __ldg(partial + static_cast<size_t>(k) * cols + c);
  }
  red[q][cl] = acc;
  __syncthreads();
  if (q == 0 && c < cols) {
    float t = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) t += red[k][cl];
    out[c] = t / grad_scale(amax_bits);
  }
}

// The forward's GELU activation rebuilt from the stored pre-activation: out = operand(GELU(a + bias)) with the
// W1 GEMM epilogue's exact arithmetic (gemm.cu WM3_EPI_BIAS_GELU_BF16: fp32 a + bias, then the same GELU and
// packing), so it is bitwise the forward's activation without re-running the W1 GEMM.  8 elements per
// thread-step; cols, lda, ldo multiples of 8.
__global__ void bw_gelu_fwd_kernel(const float* __restrict__ a, int lda, const float* __restrict__ bias, int rows,
                                   int cols, elem_t* __restrict__ out, int ldo) {
  for (int r = blockIdx.x; r < rows; r += gridDim.x) {
    const float* ar = a + static_cast<size_t>(r) * lda;
    elem_t* orow = out + static_cast<size_t>(r) * ldo;
    for (int c = 8 * threadIdx.x; c < cols; c += 8 * blockDim.x) {
      float v[8];
      const float4 x0 = __ldg(reinterpret_cast<const float4*>(ar + c));
      const float4 x1 = __ldg(reinterpret_cast<const float4*>(ar + c + 4));
      const float4 b0 = __ldg(reinterpret_cast<const float4*>(bias + c));
      const float4 b1 = __ldg(reinterpret_cast<const float4*>(bias + c + 4));
      v[0] = x0.x + b0.x; v[1] = x0.y + b0.y; v[2] = x0.z + b0.z; v[3] = x0.w + b0.w;
      v[4] = x1.x + b1.x; v[5] = x1.y + b1.y; v[6] = x1.z + b1.z; v[7] = x1.w + b1.w;
      uint32_t pk[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
#if !defined(WM3_OPERAND_BF16) && WM3_GELU_VARIANT == 2
        pk[e] = gelu_tanh_h2(v[2 * e], v[2 * e + 1]);
#else
        pk[e] = pack_elem(gelu_epi(v[2 * e]), gelu_epi(v[2 * e + 1]));
#endif
      }
      *reinterpret_cast<uint4*>(orow + c) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
    }
  }
}

// out = (g / scale) * gelu'(a + bias), exact-erf GELU derivative Phi(z) + z phi(z) (autodiff.py:372-382)
__global__ void bw_gelu_kernel(const float* __restrict__ g, int ldg, const float* __restrict__ a, int lda,
                               const float* __restrict__ bias, int rows, int cols, const unsigned* amax_bits,
                               float* __restrict__ out, int ldo) {
  const float inv = 1.f / grad_scale(amax_bits);
  for (int r = blockIdx.x; r < rows; r += gridDim.x) {  // row strips (see bw_amax_kernel)
    const float* gr = g + static_cast<size_t>(r) * ldg;
    const float* ar = a + static_cast<size_t>(r) * lda;
    float* orow = out + static_cast<size_t>(r) * ldo;
    for (int c = threadIdx.x; c < cols; c += blockDim.x) {
      const float z = ar[c] + __ldg(bias + c);
      const float d = 0.5f * (1.f + erff(z * 0.70710678118654752f)) + z * 0.39894228040143268f * __expf(-0.5f * z * z);
      orow[c] = gr[c] * inv * d;
    }
  }
}

// LayerNorm backward per row (one warp), forward statistics recomputed as layernorm_kernel does (mean, biased
// variance, eps): ghat = (g / scale) * gamma, gx = rstd * (ghat - mean(ghat) - xhat * mean(ghat * xhat)) (+ add);
// gxh[r][c] = (g / scale) * xhat (gain gradient = its column sum), gsc[r][c] = g / scale (bias gradient).
__global__ void bw_layernorm_kernel(const float* __restrict__ x, int ldx, int rows, int n, float eps,
                                    const float* __restrict__ gamma, const float* __restrict__ g, int ldg,
                                    const unsigned* amax_bits, const float* __restrict__ add, float* __restrict__ gx,
                                    float* __restrict__ gxh, float* __restrict__ gsc, unsigned* gx_amax) {
  __shared__ float redm[8];
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  float gm = 0.f;  // max |gx| of this warp's row (gx_amax: the next operand scale without another pass)
  if (warp < rows) {
    const float inv = 1.f / grad_scale(amax_bits);
    const float* xr = x + static_cast<size_t>(warp) * ldx;
    const float* gr = g + static_cast<size_t>(warp) * ldg;
    float s = 0.f;
    for (int c = lane; c < n; c += 32) s += xr[c];
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const float mu = s / n;
    float q = 0.f;
    for (int c = lane; c < n; c += 32) {
      const float d = xr[c] - mu;
      q += d * d;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
    const float rstd = rsqrtf(q / n + eps);
    float a1 = 0.f, a2 = 0.f;
    for (int c = lane; c < n; c += 32) {
      const float xh = (xr[c] - mu) * rstd;
      const float gh = gr[c] * inv * gamma[c];
      a1 += gh;
      a2 += gh * xh;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      a1 += __shfl_xor_sync(0xffffffffu, a1, o);
      a2 += __shfl_xor_sync(0xffffffffu, a2, o);
    }
    a1 /= n;
    a2 /= n;
    for (int c = lane; c < n; c += 32) {
      const size_t o = static_cast<size_t>(warp) * n + c;
      const float xh = (xr[c] - mu) * rstd;
      const float gu = gr[c] * inv;
      const float gh = gu * gamma[c];
      const float gv = rstd * (gh - a1 - xh * a2) + (add != nullptr ? add[o] : 0.f);
      gx[o] = gv;
      gm = fmaxf(gm, fabsf(gv));
      gxh[o] = gu * xh;
      if (gsc != nullptr) gsc[o] = gu;
    }
  }
  if (gx_amax != nullptr) {  // block-level max, one atomic per block (order-independent)
#pragma unroll
    for (int o = 16; o; o >>= 1) gm = fmaxf(gm, __shfl_xor_sync(0xffffffffu, gm, o));
    if (lane == 0) redm[threadIdx.x >> 5] = gm;
    __syncthreads();
    if (threadIdx.x == 0) {
      float t = redm[0];
      for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) t = fmaxf(t, redm[w]);
      atomicMax(gx_amax, __float_as_uint(t));
    }
  }
}

// Attention backward, query side (one warp per (token, head)): logits over the token's K window keys
// (neighbor table, grid.py K order) recomputed from the rotated q, k exactly as scored (scale after rotary),
// softmax in fp32, dP_k = g_ctx . v_k, D = sum_k p_k dP_k, dS_k = p_k (dP_k - D), g_q = scale * sum_k dS_k k_k.
// Stores P and dS [T][heads][K] for the key side.  qkv: [T][3][heads][dhp] (16-bit), g_ctx [T][heads * dhp]
// fp32 with scale `amax_bits`; g_out [T][3][heads][dhp] fp32 (q section written here).
__global__ void bw_na_query_kernel(const elem_t* __restrict__ qkv, int ldq, const int64_t* __restrict__ nbr, int T,
                                   int K, int heads, int dhp, float scale, const float* __restrict__ gctx, int ldc,
                                   const unsigned* amax_bits, float* __restrict__ P, float* __restrict__ dS,
                                   float* __restrict__ gout, int ldg, float* __restrict__ work) {
  const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (wid >= T * heads) return;
  const int t = wid / heads, h = wid - t * heads;
  const int sec = heads * dhp;
  const float inv = 1.f / grad_scale(amax_bits);
  const int per = dhp / 32;  // 2 or 4 channels per lane
  float qv[4], gc[4], acc[4];
  for (int e = 0; e < per; ++e) {
    const int c = lane * per + e;
    qv[e] = to_f(qkv[static_cast<size_t>(t) * ldq + h * dhp + c]);
    gc[e] = gctx[static_cast<size_t>(t) * ldc + h * dhp + c] * inv;
    acc[e] = 0.f;
  }
  float* s = work + static_cast<size_t>(wid) * 2 * K;  // logits, then dP
  float mx = -INFINITY;
  for (int k = 0; k < K; ++k) {
    const int64_t j = nbr[static_cast<size_t>(t) * K + k];
    const elem_t* kr = qkv + static_cast<size_t>(j) * ldq + sec + h * dhp;
    const elem_t* vr = kr + sec;
    float d = 0.f, dp = 0.f;
    for (int e = 0; e < per; ++e) {
      const int c = lane * per + e;
      d += qv[e] * to_f(kr[c]);
      dp += gc[e] * to_f(vr[c]);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      d += __shfl_xor_sync(0xffffffffu, d, o);
      dp += __shfl_xor_sync(0xffffffffu, dp, o);
    }
    d *= scale;
    mx = fmaxf(mx, d);
    if (lane == 0) {
      s[k] = d;
      s[K + k] = dp;
    }
  }
  __syncwarp();
  float l = 0.f;
  for (int k = lane; k < K; k += 32) l += expf(s[k] - mx);
#pragma unroll
  for (int o = 16; o; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
  float dsum = 0.f;
  for (int k = lane; k < K; k += 32) dsum += expf(s[k] - mx) / l * s[K + k];
#pragma unroll
  for (int o = 16; o; o >>= 1) dsum += __shfl_xor_sync(0xffffffffu, dsum, o);
  const size_t pbase = (static_cast<size_t>(t) * heads + h) * K;
  for (int k = lane; k < K; k += 32) {
    const float p = expf(s[k] - mx) / l;
    P[pbase + k] = p;
    dS[pbase + k] = p * (s[K + k] - dsum);
  }
  __syncwarp();
  for (int k = 0; k < K; ++k) {
    const float ds = dS[pbase + k];
    const int64_t j = nbr[static_cast<size_t>(t) * K + k];
    const elem_t* kr = qkv + static_cast<size_t>(j) * ldq + sec + h * dhp;
    for (int e = 0; e < per; ++e)
      acc[e] += ds * to_f(kr[lane * per + e]);
  }
  for (int e = 0; e < per; ++e) gout[static_cast<size_t>(t) * ldg + h * dhp + lane * per + e] = acc[e] * scale;
}

// Attention backward, key side (one warp per (key token, head)): the inverse neighbor list of key j (entries
// (t, k) with nbr[t][k] = j, sorted by t) gives g_k = scale * sum dS[t][h][k] q_t and g_v = sum P[t][h][k] g_ctx_t,
// in a fixed order.
__global__ void bw_na_key_kernel(const elem_t* __restrict__ qkv, int ldq, const int* __restrict__ inv_off,
                                 const int* __restrict__ inv_ent, int T, int K, int heads, int dhp, float scale,
                                 const float* __restrict__ gctx, int ldc, const unsigned* amax_bits,
                                 const float* __restrict__ P, const float* __restrict__ dS, float* __restrict__ gout,
                                 int ldg) {
  const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (wid >= T * heads) return;
  const int j = wid / heads, h = wid - j * heads;
  const int sec = heads * dhp;
  const float inv = 1.f / grad_scale(amax_bits);
  const int per = dhp / 32;
  float gk[4] = {0.f, 0.f, 0.f, 0.f}, gv[4] = {0.f, 0.f, 0.f, 0.f};
  for (int e = inv_off[j]; e < inv_off[j + 1]; ++e) {
    const int t = inv_ent[2 * e], k = inv_ent[2 * e + 1];
    const size_t pi = (static_cast<size_t>(t) * heads + h) * K + k;
    const float ds = dS[pi], p = P[pi];
    for (int c = 0; c < per; ++c) {
      const int ch = lane * per + c;
      gk[c] += ds * to_f(qkv[static_cast<size_t>(t) * ldq + h * dhp + ch]);
      gv[c] += p * gctx[static_cast<size_t>(t) * ldc + h * dhp + ch] * inv;
    }
  }
  for (int c = 0; c < per; ++c) {
    const int ch = lane * per + c;
    gout[static_cast<size_t>(j) * ldg + sec + h * dhp + ch] = gk[c] * scale;
    gout[static_cast<size_t>(j) * ldg + 2 * sec + h * dhp + ch] = gv[c];
  }
}

// In place on the q and k sections of g [T][3][heads][dhp]: the transpose of the rotary rotation of the
// interleaved pairs (2i, 2i + 1) (forward: v0' = v0 c - v1 s, v1' = v0 s + v1 c), cos / sin [T][dhp / 2].
__global__ void bw_rope_kernel(float* __restrict__ g, int ldg, int T, int heads, int dhp,
                               const float* __restrict__ cs, const float* __restrict__ sn, int sections = 2,
                               unsigned* amax = nullptr) {
  const int half = dhp / 2;
  if (ldg % 4 == 0 && dhp % 4 == 0) {  // row strips, two pairs per thread-step (16-byte I/O)
    __shared__ float redm[32];
    const int w = sections * heads * dhp;
    float m = 0.f;  // max |rotated value| (amax: the operand scale of the q section)
    for (int t = blockIdx.x; t < T; t += gridDim.x) {
      float* gr = g + static_cast<size_t>(t) * ldg;
      const float* ct = cs + static_cast<size_t>(t) * half;
      const float* st = sn + static_cast<size_t>(t) * half;
      for (int c = 4 * threadIdx.x; c < w; c += 4 * blockDim.x) {
        const int pr = (c % dhp) >> 1;
        const float4 v = *reinterpret_cast<const float4*>(gr + c);
        const float2 cc = __ldg(reinterpret_cast<const float2*>(ct + pr));
        const float2 ss = __ldg(reinterpret_cast<const float2*>(st + pr));
        const float4 r = make_float4(v.x * cc.x + v.y * ss.x, -v.x * ss.x + v.y * cc.x, v.z * cc.y + v.w * ss.y,
                                     -v.z * ss.y + v.w * cc.y);
        *reinterpret_cast<float4*>(gr + c) = r;
        m = fmaxf(m, fmaxf(fmaxf(fabsf(r.x), fabsf(r.y)), fmaxf(fabsf(r.z), fabsf(r.w))));
      }
    }
    if (amax != nullptr) {
#pragma unroll
      for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
      if ((threadIdx.x & 31) == 0) redm[threadIdx.x >> 5] = m;
      __syncthreads();
      if (threadIdx.x == 0) {
        float t = redm[0];
        for (int k = 1; k < static_cast<int>(blockDim.x >> 5); ++k) t = fmaxf(t, redm[k]);
        atomicMax(amax, __float_as_uint(t));
      }
    }
    return;
  }
  const long long n = static_cast<long long>(T) * sections * heads * half;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int pr = static_cast<int>(i % half);
    long long rest = i / half;
    const int hs = static_cast<int>(rest % (sections * heads));  // section (q / k) x head
    const int t = static_cast<int>(rest / (sections * heads));
    float* p = g + static_cast<size_t>(t) * ldg + static_cast<size_t>(hs) * dhp + 2 * pr;
    const float c = cs[static_cast<size_t>(t) * half + pr], s = sn[static_cast<size_t>(t) * half + pr];
    const float g0 = p[0], g1 = p[1];
    p[0] = g0 * c + g1 * s;
    p[1] = -g0 * s + g1 * c;
  }
}

static int grid_for(long long n, int threads) {
  long long b = (n + threads - 1) / threads;
  if (b > 148LL * 32) b = 148LL * 32;
  return static_cast<int>(b < 1 ? 1 : b);
}

}  // namespace wm3

using namespace wm3;

extern "C" int wm3_bw_amax(const float* x, int rows, int cols, int ld, unsigned* amax_bits, void* stream) {
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (cudaMemsetAsync(amax_bits, 0, sizeof(unsigned), s) != cudaSuccess) return set_error("wm3_bw_amax: memset");
  bw_amax_kernel<<<rows < 148 * 8 ? rows : 148 * 8, 256, 0, s>>>(x, rows, cols, ld, amax_bits);
  return check_launch("bw_amax_kernel");
}

extern "C" int wm3_bw_cast(const void* src, int src_f32, int rows, int cols, int lds, void* dst, int ldd,
                           int transpose, const unsigned* amax_bits, void* stream) {
  if (rows < 1 || cols < 1) return set_error("wm3_bw_cast: empty");
  if (!transpose && src_f32 && cols % 8 == 0 && lds % 8 == 0 && ldd % 8 == 0 &&
      reinterpret_cast<uintptr_t>(src) % 16 == 0 && reinterpret_cast<uintptr_t>(dst) % 16 == 0) {
    bw_cast_rows_kernel<<<rows < 148 * 8 ? rows : 148 * 8, 128, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
        static_cast<const float*>(src), rows, cols, lds, reinterpret_cast<elem_t*>(dst), ldd, amax_bits);
    return check_launch("bw_cast_rows_kernel");
  }
  const int drows = transpose ? cols : rows;
  dim3 grid((ldd + 31) / 32, (drows + 31) / 32);
  bw_cast_kernel<<<grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      src, src_f32, rows, cols, lds, reinterpret_cast<elem_t*>(dst), ldd, transpose, amax_bits);
  return check_launch("bw_cast_kernel");
}

extern "C" int wm3_bw_colsum(const float* src, const float* src2, int rows, int cols, int ld, const unsigned* amax_bits,
                             float* partial, float* out, void* stream) {
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int chunks = (rows + BW_CHUNK - 1) / BW_CHUNK;
  if (cols % 4 == 0 && ld % 4 == 0 && aligned16(src) && aligned16(src2)) {
    if (src2 != nullptr)
      bw_colsum4_kernel<1><<<dim3((cols + 255) / 256, chunks), 256, 0, s>>>(src, ld, src2, ld, nullptr, nullptr, rows,
                                                                            cols, nullptr, 0, partial, nullptr);
    else
      bw_colsum4_kernel<0><<<dim3((cols + 255) / 256, chunks), 256, 0, s>>>(src, ld, nullptr, 0, nullptr, nullptr,
                                                                            rows, cols, nullptr, 0, partial, nullptr);
    if (check_launch("bw_colsum4_kernel")) return -1;
  } else {
    bw_colsum_partial_kernel<<<dim3((cols + 127) / 128, chunks), 128, 0, s>>>(src, src2, rows, cols, ld, partial);
    if (check_launch("bw_colsum_partial_kernel")) return -1;
  }
  bw_colsum_final_kernel<<<(cols + 31) / 32, 256, 0, s>>>(partial, chunks, cols, amax_bits, out);
  return check_launch("bw_colsum_final_kernel");
}

extern "C" int wm3_bw_cast_colsum(const float* src, int rows, int cols, int lds, void* dst, int ldd,
                                  const unsigned* amax_bits, float* partial, float* colsum, void* stream) {
  if (rows < 1 || cols < 1 || ldd < cols) return set_error("wm3_bw_cast_colsum: bad shape");
  if ((cols % 4) || (lds % 4) || (ldd % 4) || !aligned16(src) || reinterpret_cast<uintptr_t>(dst) % 8)
    return set_error("wm3_bw_cast_colsum: cols / pitches multiples of 4, aligned bases required");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int chunks = (rows + BW_CHUNK - 1) / BW_CHUNK;
  bw_colsum4_kernel<3><<<dim3((ldd + 255) / 256, chunks), 256, 0, s>>>(
      src, lds, nullptr, 0, nullptr, amax_bits, rows, cols, reinterpret_cast<float*>(dst), ldd, partial, nullptr);
  if (check_launch("bw_colsum4_kernel")) return -1;
  bw_colsum_final_kernel<<<(cols + 31) / 32, 256, 0, s>>>(partial, chunks, cols, nullptr, colsum);
  return check_launch("bw_colsum_final_kernel");
}

extern "C" int wm3_bw_colsum_amax(const float* g, int ldg, const float* a, int lda, const float* bias,
                                  const unsigned* in_scale_bits, int rows, int cols, float* out, int ldo,
                                  float* partial, float* colsum, unsigned* amax_bits, void* stream) {
  if (rows < 1 || cols < 1) return set_error("wm3_bw_colsum_amax: empty");
  if (a != nullptr && (out == nullptr || bias == nullptr)) return set_error("wm3_bw_colsum_amax: GELU needs out, bias");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (cudaMemsetAsync(amax_bits, 0, sizeof(unsigned), s) != cudaSuccess) return set_error("wm3_bw_colsum_amax: memset");
  const int chunks = (rows + BW_CHUNK - 1) / BW_CHUNK;
  const bool v4 = cols % 4 == 0 && ldg % 4 == 0 && aligned16(g) &&
                  (a == nullptr || (lda % 4 == 0 && ldo % 4 == 0 && aligned16(a) && aligned16(out) && aligned16(bias)));
  if (v4) {
    if (a != nullptr)
      bw_colsum4_kernel<2><<<dim3((cols + 255) / 256, chunks), 256, 0, s>>>(g, ldg, a, lda, bias, in_scale_bits, rows,
                                                                            cols, out, ldo, partial, amax_bits);
    else
      bw_colsum4_kernel<0><<<dim3((cols + 255) / 256, chunks), 256, 0, s>>>(g, ldg, nullptr, 0, nullptr, nullptr, rows,
                                                                            cols, nullptr, 0, partial, amax_bits);
    if (check_launch("bw_colsum4_kernel")) return -1;
  } else {
    bw_colsum_amax_kernel<<<dim3((cols + 255) / 256, chunks), 256, 0, s>>>(g, ldg, a, lda, bias, in_scale_bits, rows,
                                                                           cols, out, ldo, partial, amax_bits);
    if (check_launch("bw_colsum_amax_kernel")) return -1;
  }
  bw_colsum_final_kernel<<<(cols + 31) / 32, 256, 0, s>>>(partial, chunks, cols, nullptr, colsum);
  return check_launch("bw_colsum_final_kernel");
}

extern "C" int wm3_bw_gelu_fwd(const float* a, int lda, const float* bias, int rows, int cols, void* out, int ldo,
                               void* stream) {
  if (rows < 1 || cols < 1 || cols % 8 || lda % 8 || ldo % 8) return set_error("wm3_bw_gelu_fwd: shape");
  bw_gelu_fwd_kernel<<<rows < 148 * 8 ? rows : 148 * 8, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      a, lda, bias, rows, cols, static_cast<elem_t*>(out), ldo);
  return check_launch("bw_gelu_fwd_kernel");
}

extern "C" int wm3_bw_gelu(const float* g, int ldg, const float* a, int lda, const float* bias, int rows, int cols,
                           const unsigned* amax_bits, float* out, int ldo, void* stream) {
  bw_gelu_kernel<<<rows < 148 * 8 ? rows : 148 * 8, 256, 0,
                   reinterpret_cast<cudaStream_t>(stream)>>>(g, ldg, a, lda, bias, rows, cols, amax_bits, out, ldo);
  return check_launch("bw_gelu_kernel");
}

extern "C" int wm3_bw_layernorm(const float* x, int ldx, int rows, int n, float eps, const float* gamma, const float* g,
                                int ldg, const unsigned* amax_bits, const float* add, float* gx, float* gxh, float* gsc,
                                unsigned* gx_amax, void* stream) {
  const int threads = 256, blocks = (rows * 32 + threads - 1) / threads;
  bw_layernorm_kernel<<<blocks, threads, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      x, ldx, rows, n, eps, gamma, g, ldg, amax_bits, add, gx, gxh, gsc, gx_amax);
  return check_launch("bw_layernorm_kernel");
}

extern "C" int wm3_bw_natten(const void* qkv, int ldq, const int64_t* nbr, const int* inv_off, const int* inv_ent, int T,
                             int K, int heads, int dhp, float scale, const float* gctx, int ldc,
                             const unsigned* amax_bits, float* P, float* dS, float* work, float* gout, int ldg,
                             void* stream) {
  if (dhp != 64 && dhp != 128) return set_error("wm3_bw_natten: dhp must be 64 or 128");
  if (ldg < 3 * heads * dhp) return set_error("wm3_bw_natten: ldg < 3 * heads * dhp");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int threads = 256, blocks = (T * heads * 32 + threads - 1) / threads;
  bw_na_query_kernel<<<blocks, threads, 0, s>>>(reinterpret_cast<const elem_t*>(qkv), ldq, nbr, T, K, heads, dhp,
                                                scale, gctx, ldc, amax_bits, P, dS, gout, ldg, work);
  if (check_launch("bw_na_query_kernel")) return -1;
  bw_na_key_kernel<<<blocks, threads, 0, s>>>(reinterpret_cast<const elem_t*>(qkv), ldq, inv_off, inv_ent, T, K, heads,
                                              dhp, scale, gctx, ldc, amax_bits, P, dS, gout, ldg);
  return check_launch("bw_na_key_kernel");
}

extern "C" int wm3_bw_rope_q(float* g, int ldg, int T, int heads, int dhp, const float* cos_t, const float* sin_t,
                             unsigned* amax, void* stream) {
  if ((ldg % 4) || (dhp % 4)) return set_error("wm3_bw_rope_q: ldg and dhp must be multiples of 4");
  bw_rope_kernel<<<T < 148 * 8 ? T : 148 * 8, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(g, ldg, T, heads, dhp,
                                                                                               cos_t, sin_t, 1, amax);
  return check_launch("bw_rope_kernel");
}

extern "C" int wm3_bw_rope(float* g, int ldg, int T, int heads, int dhp, const float* cos_t, const float* sin_t,
                           void* stream) {
  bw_rope_kernel<<<grid_for(static_cast<long long>(T) * heads * dhp, 256), 256, 0,
                   reinterpret_cast<cudaStream_t>(stream)>>>(g, ldg, T, heads, dhp, cos_t, sin_t);
  return check_launch("bw_rope_kernel");
}

// ---------------------------------------------------------------------------------------------------------------
// Operands of the tcgen05 attention backward (natten.cu wm3_natten_bwd): dO as fp16 scaled by a power of two
// sigma with sigma * max|g_ctx| * max_k ||v_k||_1 <= 2^13 (so |dP| and |Delta| <= 2^13 and dS = P (dP - Delta) fits
// fp16), and the unscale factors of dQ / dK (scale / (sigma s)) and dV (1 / (sigma s)), s = the g_ctx grad scale.
// ---------------------------------------------------------------------------------------------------------------
__global__ void bw_na_prep_reduce_kernel(const elem_t* __restrict__ qkv, int ldq, int T, int heads, int dhp,
                                         const float* __restrict__ gctx, int ldc, unsigned* __restrict__ maxima) {
  // maxima[0] = max |g_ctx| over the (T, heads * dhp) block, maxima[1] = max over (token, head) of sum |v|;
  // one warp per (token, head) at a time, lanes over the channels (coalesced), one atomic pair per warp
  const int sec = heads * dhp;
  const int lane = threadIdx.x & 31;
  const long long nw = static_cast<long long>(gridDim.x) * (blockDim.x >> 5);
  float mg = 0.f, mv = 0.f;
  for (long long w = blockIdx.x * static_cast<long long>(blockDim.x >> 5) + (threadIdx.x >> 5);
       w < static_cast<long long>(T) * heads; w += nw) {
    const int t = static_cast<int>(w / heads), h = static_cast<int>(w - static_cast<long long>(t) * heads);
    const elem_t* v = qkv + static_cast<size_t>(t) * ldq + 2 * sec + h * dhp;
    const float* g = gctx + static_cast<size_t>(t) * ldc + h * dhp;
    float l1 = 0.f;
    for (int c = lane; c < dhp; c += 32) {
      l1 += fabsf(to_f(v[c]));
      mg = fmaxf(mg, fabsf(g[c]));
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) l1 += __shfl_xor_sync(0xffffffffu, l1, o);
    mv = fmaxf(mv, l1);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) mg = fmaxf(mg, __shfl_xor_sync(0xffffffffu, mg, o));
  if (lane == 0) {
    atomicMax(maxima, __float_as_uint(mg));
    atomicMax(maxima + 1, __float_as_uint(mv));
  }
}

__global__ void bw_na_prep_scale_kernel(const float* __restrict__ gctx, int ldc, int T, int cols,
                                        const unsigned* __restrict__ maxima, const unsigned* gscale_bits, float scale,
                                        elem_t* __restrict__ dout, int ldd, float* __restrict__ factors) {
  const float bound = __uint_as_float(maxima[0]) * __uint_as_float(maxima[1]);
  const float sigma = (bound > 0.f && isfinite(bound)) ? exp2f(floorf(log2f(8192.f / bound))) : 1.f;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const float s = grad_scale(gscale_bits);
    factors[0] = scale / (sigma * s);
    factors[1] = 1.f / (sigma * s);
  }
  if (cols % 8 == 0 && ldc % 4 == 0 && ldd % 8 == 0) {  // row strips, 8 elements per thread-step (16-byte I/O)
    for (int t = blockIdx.x; t < T; t += gridDim.x) {
      const float* gr = gctx + static_cast<size_t>(t) * ldc;
      elem_t* dr = dout + static_cast<size_t>(t) * ldd;
      for (int c = 8 * threadIdx.x; c < cols; c += 8 * blockDim.x) {
        const float4 a = __ldg(reinterpret_cast<const float4*>(gr + c));
        const float4 b = __ldg(reinterpret_cast<const float4*>(gr + c + 4));
        *reinterpret_cast<uint4*>(dr + c) =
            make_uint4(pack_elem(a.x * sigma, a.y * sigma), pack_elem(a.z * sigma, a.w * sigma),
                       pack_elem(b.x * sigma, b.y * sigma), pack_elem(b.z * sigma, b.w * sigma));
      }
    }
    return;
  }
  const long long n = static_cast<long long>(T) * cols;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int t = static_cast<int>(i / cols), c = static_cast<int>(i - static_cast<long long>(t) * cols);
    dout[static_cast<size_t>(t) * ldd + c] = to_elem(gctx[static_cast<size_t>(t) * ldc + c] * sigma);
  }
}

extern "C" int wm3_bw_na_prep(const void* qkv, int ldq, int T, int heads, int dhp, const float* gctx, int ldc,
                              const unsigned* gscale_bits, float scale, void* dout, int ldd, unsigned* maxima,
                              float* factors, void* stream) {
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  cudaMemsetAsync(maxima, 0, 2 * sizeof(unsigned), s);
  bw_na_prep_reduce_kernel<<<148 * 8, 256, 0, s>>>(
      reinterpret_cast<const elem_t*>(qkv), ldq, T, heads, dhp, gctx, ldc, maxima);
  if (check_launch("bw_na_prep_reduce_kernel")) return -1;
  bw_na_prep_scale_kernel<<<T < 148 * 8 ? T : 148 * 8, 128, 0, s>>>(
      gctx, ldc, T, heads * dhp, maxima, gscale_bits, scale, reinterpret_cast<elem_t*>(dout), ldd, factors);
  return check_launch("bw_na_prep_scale_kernel");
}
