// Forecast verification metrics on the device (reference evaluation.py:37-190), so decoded fields and
// ensemble members never leave HBM: cos-latitude weighted squared error per (time, row) and the per-row
// zonal power spectrum, each optionally of the mean of the leading k ensemble members (computed on the fly).
// Accumulation is float64 with a fixed reduction order (one CTA per (time, row)), so results are
// deterministic run to run.
#include "common.cuh"
#include "launch.h"
#include "../../include/wm3.h"

namespace wm3 {

constexpr int MT_THREADS = 256;

template <typename T>
DEVI double member_mean(const T* f, long long mstride, int k, size_t idx) {
  double s = 0.0;
  for (int j = 0; j < k; ++j) s += static_cast<double>(f[static_cast<long long>(j) * mstride + idx]);
  return k == 1 ? s : s / k;
}

DEVI double block_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) s += red[w];  // fixed order
  return s;
}

// partial[t * rows + r] = w[r] * sum_c (mean_k(a)[t, r, c] - b[t, r, c])^2   (evaluation.py:45-52)
template <typename T>
__global__ void __launch_bounds__(MT_THREADS) sq_err_rows_kernel(const T* __restrict__ a, long long mstride, int k,
                                                                   const T* __restrict__ b,
                                                                   const double* __restrict__ w, int rows, int cols,
                                                                   double* __restrict__ partial) {
  __shared__ double red[MT_THREADS / 32];
  const int r = blockIdx.x % rows;
  const size_t base = static_cast<size_t>(blockIdx.x) * cols;
  double s = 0.0;
  for (int c = threadIdx.x; c < cols; c += blockDim.x) {
    const double d = member_mean(a, mstride, k, base + c) - static_cast<double>(b[base + c]);
    s = fma(d, d, s);
  }
  s = block_sum(s, red);
  if (threadIdx.x == 0) partial[blockIdx.x] = w[r] * s;
}

// out[img, r, m] = mean-square zonal power of wavenumber m along row r (evaluation.py:59-75): a direct DFT
// with an exact periodic twiddle table (angle index m * c mod W), bins 1..W/2-1 (or W/2 for odd W) doubled.
template <typename T>
__global__ void __launch_bounds__(MT_THREADS) zonal_power_kernel(const T* __restrict__ f, long long mstride, int k,
                                                                   int cols, double* __restrict__ out) {
  extern __shared__ double sh[];
  double* row = sh;
  double* cs = sh + cols;
  double* sn = sh + 2 * cols;
  const size_t base = static_cast<size_t>(blockIdx.x) * cols;
  for (int c = threadIdx.x; c < cols; c += blockDim.x) {
    row[c] = member_mean(f, mstride, k, base + c);
    double s_, c_;
    sincospi(2.0 * c / cols, &s_, &c_);
    cs[c] = c_;
    sn[c] = s_;
  }
  __syncthreads();
  const int nb = cols / 2 + 1;
  const double inv = 1.0 / (static_cast<double>(cols) * cols);
  for (int m = threadIdx.x; m < nb; m += blockDim.x) {
    double re = 0.0, im = 0.0;
    int kk = 0;
    for (int c = 0; c < cols; ++c) {
      re = fma(row[c], cs[kk], re);
      im = fma(row[c], sn[kk], im);
      kk += m;
      if (kk >= cols) kk -= cols;
    }
    double p = (re * re + im * im) * inv;
    const bool interior = (m > 0) && !((cols % 2 == 0) && m == cols / 2);
    if (interior) p *= 2.0;
    out[static_cast<size_t>(blockIdx.x) * nb + m] = p;
  }
}

}  // namespace wm3

using namespace wm3;

extern "C" int wm3_sq_err_rows(int dtype, const void* a, long long member_stride, int k, const void* b,
                               const double* w_rows, int times, int rows, int cols, double* partial, void* stream) {
  if (times <= 0 || rows <= 0 || cols <= 0 || k < 1) return set_error("wm3_sq_err_rows: bad sizes");
  const dim3 grid(static_cast<unsigned>(times) * rows);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (dtype == 0)
    sq_err_rows_kernel<float><<<grid, MT_THREADS, 0, s>>>(static_cast<const float*>(a), member_stride, k,
                                                          static_cast<const float*>(b), w_rows, rows, cols, partial);
  else if (dtype == 1)
    sq_err_rows_kernel<double><<<grid, MT_THREADS, 0, s>>>(static_cast<const double*>(a), member_stride, k,
                                                           static_cast<const double*>(b), w_rows, rows, cols,
                                                           partial);
  else
    return set_error("wm3_sq_err_rows: dtype must be 0 (f32) or 1 (f64)");
  return check_launch("sq_err_rows_kernel");
}

extern "C" int wm3_zonal_power(int dtype, const void* field, long long member_stride, int k, int imgs, int rows,
                               int cols, double* out, void* stream) {
  if (imgs <= 0 || rows <= 0 || cols <= 0 || k < 1) return set_error("wm3_zonal_power: bad sizes");
  const size_t smem = 3 * sizeof(double) * cols;
  if (smem > 200 * 1024) return set_error("wm3_zonal_power: %d columns exceed the shared-memory row stage", cols);
  const dim3 grid(static_cast<unsigned>(imgs) * rows);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e = cudaSuccess;
  if (dtype == 0) {
    e = cudaFuncSetAttribute(zonal_power_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem));
    if (e == cudaSuccess)
      zonal_power_kernel<float><<<grid, MT_THREADS, smem, s>>>(static_cast<const float*>(field), member_stride, k,
                                                               cols, out);
  } else if (dtype == 1) {
    e = cudaFuncSetAttribute(zonal_power_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem));
    if (e == cudaSuccess)
      zonal_power_kernel<double><<<grid, MT_THREADS, smem, s>>>(static_cast<const double*>(field), member_stride,
                                                                k, cols, out);
  } else {
    return set_error("wm3_zonal_power: dtype must be 0 (f32) or 1 (f64)");
  }
  if (e != cudaSuccess) return set_error("cudaFuncSetAttribute(zonal_power): %s", cudaGetErrorString(e));
  return check_launch("zonal_power_kernel");
}
