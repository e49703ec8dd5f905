// Host-side helpers shared by the kernel translation units (definitions in host.cu).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace wm3 {

// Record a printf-style message as the thread's last error; returns -1.
int set_error(const char* fmt, ...);
// cudaGetLastError after a launch; returns 0 or -1 (with message).
int check_launch(const char* what);
int sm_count();
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (device, kernel, size); thread-safe.
int ensure_smem_attr(const void* func, int bytes, const char* what);

// 2D bf16 tensor map (inner = contiguous extent, outer = rows, pitch in elements), SWIZZLE_128B,
// OOB elements zero-filled.  Box = (box_inner, box_outer); box_inner * 2 must be 128.
int make_tmap_2d_bf16(CUtensorMap* map, const void* ptr, uint64_t inner, uint64_t outer, uint64_t pitch_elems,
                      uint32_t box_inner, uint32_t box_outer);
enum { TMAP_BF16 = 0, TMAP_F32 = 1 };
// General tensor map (SWIZZLE_128B, zero OOB fill), rank <= 5; strides in elements for dims 1..rank-1.
int make_tmap(CUtensorMap* map, const void* ptr, int dtype, int rank, const uint64_t* dims,
              const uint64_t* strides_elems, const uint32_t* box, const uint32_t* elem_strides);
// make_tmap with the shared-memory swizzle chosen (32 / 64 / 128 bytes; make_tmap uses 128)
int make_tmap_swz(CUtensorMap* map, const void* ptr, int dtype, int rank, const uint64_t* dims,
                  const uint64_t* strides_elems, const uint32_t* box, const uint32_t* elem_strides, int swizzle_bytes);
// General bf16 tensor map, rank <= 5; strides in elements for dims 1..rank-1.
int make_tmap_bf16(CUtensorMap* map, const void* ptr, int rank, const uint64_t* dims, const uint64_t* strides_elems,
                   const uint32_t* box, const uint32_t* elem_strides);

// Launch with programmatic dependent launch (PDL): the kernel may be scheduled while the previous kernel on
// the stream drains; it must execute griddep_wait() (common.cuh) before touching memory the previous kernels
// produce or consume.  Every wm3 kernel does, right after its prologue (barriers, TMEM, tensor-map prefetch),
// so the prologue and launch latency overlap the predecessor's tail.  Opt-in (WM3_PDL=1): see host.cu.
bool pdl_enabled();
template <typename... KArgs, typename... Args>
int launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
  if (e != cudaSuccess) return set_error("launch: %s", cudaGetErrorString(e));
  return 0;
}

}  // namespace wm3
