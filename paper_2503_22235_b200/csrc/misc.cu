// Small bandwidth-bound kernels: neighbor-table export (bit-exact window arithmetic) and LayerNorm.
#include "common.cuh"
#include "launch.h"
#include "window.cuh"
#include "../../include/wm3.h"

namespace wm3 {

// grid.py:96-130.  One thread per (token, key) entry; token index is global over (depth, rows, cols),
// the table covers global rows [row0, row0 + nrows).
__global__ void neighbor_table_kernel(int depth, int rows, int cols, int wd, int wh, int ww, int row0, int nrows,
                                      int64_t* __restrict__ out) {
  const int K = wd * wh * ww;
  const long long total = static_cast<long long>(depth) * nrows * cols * K;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int kk = static_cast<int>(i % K);
    const long long t = i / K;
    const int c = static_cast<int>(t % cols);
    const int r = static_cast<int>((t / cols) % nrows) + row0;
    const int d = static_cast<int>(t / (static_cast<long long>(cols) * nrows));
    const int kw = kk % ww;
    const int kh = (kk / ww) % wh;
    const int kd = kk / (ww * wh);
    const int dd = bump_start(d, depth, wd) + kd;
    const int hh = bump_start(r, rows, wh) + kh;
    const int cc = wrap_col(c + kw - (ww - 1) / 2, cols);
    out[i] = (static_cast<int64_t>(dd) * rows + hh) * cols + cc;
  }
}

// autodiff.py:400-424: mean, biased variance, eps, gain/bias; one warp per row, fp32 statistics.
template <int NV>
__global__ void layernorm_kernel(const float* __restrict__ x, int ldx, int m, int n, const float* __restrict__ gain,
                                 const float* __restrict__ bias, float eps, elem_t* __restrict__ out, int ldo) {
  griddep_launch_dependents();  // PDL: the next kernel may start its prologue
  griddep_wait();
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= m) return;
  const float* xr = x + static_cast<size_t>(warp) * ldx;
  elem_t* orow = out + static_cast<size_t>(warp) * ldo;
  const bool vec = (n % 4 == 0) && (ldx % 4 == 0) && (n <= NV * 128);
  if (vec) {
    float4 v[NV];
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c = (i * 32 + lane) * 4;
      v[i] = c < n ? *reinterpret_cast<const float4*>(xr + c) : make_float4(0.f, 0.f, 0.f, 0.f);
      s += v[i].x + v[i].y + v[i].z + v[i].w;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const float mu = s / n;
    float q = 0.f;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c = (i * 32 + lane) * 4;
      if (c < n) {
        const float a = v[i].x - mu, b = v[i].y - mu, cc = v[i].z - mu, d = v[i].w - mu;
        q += a * a + b * b + cc * cc + d * d;
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
    const float inv = rsqrtf(q / n + eps);
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c = (i * 32 + lane) * 4;
      if (c < n) {
        const float4 g = __ldg(reinterpret_cast<const float4*>(gain + c));
        const float4 b = __ldg(reinterpret_cast<const float4*>(bias + c));
        uint2 pk;
        pk.x = pack_elem((v[i].x - mu) * inv * g.x + b.x, (v[i].y - mu) * inv * g.y + b.y);
        pk.y = pack_elem((v[i].z - mu) * inv * g.z + b.z, (v[i].w - mu) * inv * g.w + b.w);
        *reinterpret_cast<uint2*>(orow + c) = pk;
      }
    }
  } else {
    float s = 0.f;
    for (int c = lane; c < n; c += 32) s += xr[c];
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const float mu = s / n;
    float q = 0.f;
    for (int c = lane; c < n; c += 32) { const float a = xr[c] - mu; q += a * a; }
    for (int o = 16; o; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
    const float inv = rsqrtf(q / n + eps);
    for (int c = lane; c < n; c += 32) orow[c] = to_elem((xr[c] - mu) * inv * gain[c] + bias[c]);
  }
  for (int c = n + lane; c < ldo; c += 32) orow[c] = to_elem(0.f);
}

DEVI float2 ln_row_stats(float s1, float s2, int n, float eps) {
  const float inv_n = 1.f / static_cast<float>(n);
  const float mu = s1 * inv_n;
  const float rstd = rsqrtf(fmaxf(fmaf(-mu, mu, s2 * inv_n), 0.f) + eps);
  return make_float2(rstd, rstd * mu);
}

// Producer partials -> (rstd, rstd * mean) per row (include/wm3.h wm3_ln_fold_finalize); one thread per row.
__global__ void ln_fold_finalize_kernel(const float* __restrict__ stats, int parts, int n, float eps, int m,
                                        float2* __restrict__ row_stats) {
  griddep_launch_dependents();
  griddep_wait();
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= m) return;
  const float4* sp = reinterpret_cast<const float4*>(stats + static_cast<size_t>(r) * (2 * WM3_LN_SLOTS));
  float s1 = 0.f, s2 = 0.f;
  for (int i = 0; i < (parts + 1) / 2; ++i) {
    const float4 v = __ldg(sp + i);
    s1 += v.x;
    s2 += v.y;
    if (2 * i + 1 < parts) {
      s1 += v.z;
      s2 += v.w;
    }
  }
  row_stats[r] = ln_row_stats(s1, s2, n, eps);
}

// Start of a LayerNorm-folded chain (include/wm3.h wm3_ln_fold_prep): one warp per row writes the fp16 copy of
// the row (pad columns zero) and the row's (rstd, rstd * mean).
template <int NV>
__global__ void ln_fold_prep_kernel(const float* __restrict__ x, int ldx, int m, int n, elem_t* __restrict__ xh,
                                    int ld_xh, float eps, float2* __restrict__ row_stats) {
  griddep_launch_dependents();
  griddep_wait();
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= m) return;
  const float* xr = x + static_cast<size_t>(warp) * ldx;
  elem_t* orow = xh + static_cast<size_t>(warp) * ld_xh;
  float s1 = 0.f, s2 = 0.f;
  if ((n % 4 == 0) && (ldx % 4 == 0) && (n <= NV * 128)) {
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c = (i * 32 + lane) * 4;
      if (c < n) {
        const float4 v = *reinterpret_cast<const float4*>(xr + c);
        s1 += (v.x + v.y) + (v.z + v.w);
        s2 = fmaf(v.x, v.x, fmaf(v.y, v.y, fmaf(v.z, v.z, fmaf(v.w, v.w, s2))));
        uint2 pk;
        pk.x = pack_elem(v.x, v.y);
        pk.y = pack_elem(v.z, v.w);
        *reinterpret_cast<uint2*>(orow + c) = pk;
      }
    }
  } else {
    for (int c = lane; c < n; c += 32) {
      const float v = xr[c];
      s1 += v;
      s2 = fmaf(v, v, s2);
      orow[c] = to_elem(v);
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    s2 += __shfl_xor_sync(0xffffffffu, s2, o);
  }
  for (int c = n + lane; c < ld_xh; c += 32) orow[c] = to_elem(0.f);
  if (lane == 0) row_stats[warp] = ln_row_stats(s1, s2, n, eps);
}

}  // namespace wm3

using namespace wm3;

extern "C" int wm3_ln_fold_finalize(const float* stats, int parts, int n, float eps, int m, float* row_stats,
                                    void* stream) {
  if (m <= 0) return 0;
  if (n <= 0 || parts < 1 || parts > WM3_LN_SLOTS) return set_error("wm3_ln_fold_finalize: bad sizes");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (launch_pdl(ln_fold_finalize_kernel, dim3((m + 255) / 256), dim3(256), 0, s, stats, parts, n, eps, m,
                 reinterpret_cast<float2*>(row_stats)))
    return -1;
  return check_launch("ln_fold_finalize_kernel");
}

extern "C" int wm3_ln_fold_prep(const float* x, int ldx, int m, int n, void* xh, int ld_xh, float eps,
                                float* row_stats, void* stream) {
  if (m <= 0) return 0;
  if (n <= 0 || ld_xh < n || ldx < n) return set_error("wm3_ln_fold_prep: bad sizes (n %d ld_xh %d)", n, ld_xh);
  const int threads = 256;
  const int blocks = (m * 32 + threads - 1) / threads;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  auto* o = reinterpret_cast<elem_t*>(xh);
  auto kern = (n <= 256) ? ln_fold_prep_kernel<2> : (n <= 1024) ? ln_fold_prep_kernel<8> : ln_fold_prep_kernel<16>;
  if (launch_pdl(kern, dim3(blocks), dim3(threads), 0, s, x, ldx, m, n, o, ld_xh, eps,
                 reinterpret_cast<float2*>(row_stats)))
    return -1;
  return check_launch("ln_fold_prep_kernel");
}

extern "C" int wm3_neighbor_table(int depth, int rows, int cols, int wd, int wh, int ww, int row0, int nrows,
                                  int64_t* out, void* stream) {
  if (wd > depth || wh > rows || ww > cols || wd < 1 || wh < 1 || ww < 1)
    return set_error("wm3_neighbor_table: window (%d,%d,%d) exceeds extents (%d,%d,%d)", wd, wh, ww, depth, rows, cols);
  if (row0 < 0 || nrows < 0 || row0 + nrows > rows) return set_error("wm3_neighbor_table: bad row band");
  const long long total = static_cast<long long>(depth) * nrows * cols * wd * wh * ww;
  if (total == 0) return 0;
  long long blocks = (total + 255) / 256;
  if (blocks > 148LL * 32) blocks = 148LL * 32;
  neighbor_table_kernel<<<static_cast<int>(blocks), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      depth, rows, cols, wd, wh, ww, row0, nrows, out);
  return check_launch("neighbor_table_kernel");
}

extern "C" int wm3_layernorm_bf16(const float* x, int ldx, int m, int n, const float* gain, const float* bias,
                                  float eps, void* out_bf16, int ldo, void* stream) {
  if (m <= 0) return 0;
  if (n <= 0 || ldo < n) return set_error("wm3_layernorm_bf16: bad sizes");
  const int threads = 256;
  const int blocks = (m * 32 + threads - 1) / threads;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  auto* o = reinterpret_cast<elem_t*>(out_bf16);
  auto kern = (n <= 256) ? layernorm_kernel<2> : (n <= 1024) ? layernorm_kernel<8> : layernorm_kernel<16>;
  if (launch_pdl(kern, dim3(blocks), dim3(threads), 0, s, x, ldx, m, n, gain, bias, eps, o, ldo)) return -1;
  return check_launch("layernorm_kernel");
}

extern "C" int wm3_operand_dtype(void) { return wm3::kElemFmt == 0 ? WM3_DTYPE_F16 : WM3_DTYPE_BF16; }
