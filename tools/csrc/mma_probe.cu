// Micro-benchmark of tcgen05.mma issue/execution rates for the shapes the kernels use (profiling aid; not on
// the forecast path).  One CTA per SM; one thread issues `reps` groups of 8 K=16 MMAs and waits for each group.
#include "../../paper_2503_22235_b200/csrc/common.cuh"
#include "../../paper_2503_22235_b200/csrc/launch.h"

namespace wm3 {

__global__ void __launch_bounds__(128, 1) mma_probe_kernel(int mode, int n, int reps, long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sA = smem_u32(smem), sB = sA + 32768;
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (uint32_t off = threadIdx.x * 16u; off < 98304u; off += 128 * 16u) st_shared_v4(sA + off, 0, 0, 0, 0);
  fence_proxy_async();
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar), 1);
    fence_barrier_init();
  }
  if (threadIdx.x < 32) {
    tmem_alloc(smem_u32(&slot), 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const bool pipelined = mode >= 16;
  mode &= 15;
  if (threadIdx.x == 0) {
    const uint32_t idesc = make_idesc(128, n, 0, mode == 2 ? 1 : 0);
    uint32_t ph = 0;
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      for (int s = 0; s < 8; ++s) {
        if (mode == 0) {  // SS, both K-major (S = Q K^T)
          const uint32_t off = (s >> 2) * 16384u + (s & 3) * 32u;
          umma_bf16_ss(tmem, make_sdesc_sw128(sA + off, 16, 1024), make_sdesc_sw128(sB + off, 16, 1024), idesc,
                       s > 0 ? 1u : 0u);
        } else if (mode == 1) {  // TS: A from TMEM, B K-major
          const uint32_t off = (s >> 2) * 16384u + (s & 3) * 32u;
          umma_f16_ts(tmem, tmem + 384 + 8 * s, make_sdesc_sw128(sB + off, 16, 1024), idesc, s > 0 ? 1u : 0u);
        } else {  // TS with B MN-major (P V)
          umma_f16_ts(tmem, tmem + 384 + 8 * s, make_sdesc_sw128(sB + s * 2048u, 16384, 1024), idesc,
                      s > 0 ? 1u : 0u);
        }
      }
      if (!pipelined || r == reps - 1) {
        umma_commit(smem_u32(&bar));
        mbar_wait(smem_u32(&bar), ph);
        ph ^= 1;
      }
    }
    out[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

}  // namespace wm3

using namespace wm3;

extern "C" int mma_probe(int mode, int n, int reps, int ctas, long long* out_cycles, void* stream) {
  const int smem = 98304 + 1024;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(mma_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  mma_probe_kernel<<<ctas, 128, smem, reinterpret_cast<cudaStream_t>(stream)>>>(mode, n, reps, out_cycles);
  return check_launch("mma_probe_kernel");
}
