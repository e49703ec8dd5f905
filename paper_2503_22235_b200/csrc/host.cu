// C-ABI plumbing: error reporting, device properties, TMA descriptor encoding.
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <mutex>
#include <set>
#include <utility>

#include "launch.h"
#include "../../include/wm3.h"

namespace wm3 {

static thread_local char g_err[1024] = "";

int set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return -1;
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error("%s launch failed: %s", what, cudaGetErrorString(e));
  return 0;
}

bool pdl_enabled() {
  // Off by default: measured on B200 the CUDA-graph rollout ran 4.5 % slower with PDL (2.80 vs 2.68 ms per
  // block, alternating A/B, tools/rollout_time.py) and the eager block step was unchanged.  WM3_PDL=1 enables.
  static const bool on = [] {
    const char* e = getenv("WM3_PDL");
    return e && atoi(e) != 0;
  }();
  return on;
}

int sm_count() {
  // per device (a process may drive several GPUs); cached per (thread, device)
  static thread_local int cached_dev = -1, n = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev != cached_dev) {
    n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
    cached_dev = dev;
  }
  return n;
}

int ensure_smem_attr(const void* func, int bytes, const char* what) {
  // cudaFuncSetAttribute applies to the current device only: remember (device, kernel, size) triples, under a
  // lock so concurrent host threads (one per GPU) stay correct
  static std::mutex mu;
  static std::set<std::pair<std::pair<int, const void*>, int>> done;
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_pair(std::make_pair(dev, func), bytes);
  std::lock_guard<std::mutex> lock(mu);
  if (done.count(key)) return 0;
  const cudaError_t e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) return set_error("cudaFuncSetAttribute(%s): %s", what, cudaGetErrorString(e));
  done.insert(key);
  return 0;
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

int make_tmap(CUtensorMap* map, const void* ptr, int dtype, int rank, const uint64_t* dims,
              const uint64_t* strides_elems, const uint32_t* box, const uint32_t* elem_strides) {
  return make_tmap_swz(map, ptr, dtype, rank, dims, strides_elems, box, elem_strides, 128);
}

int make_tmap_swz(CUtensorMap* map, const void* ptr, int dtype, int rank, const uint64_t* dims,
                  const uint64_t* strides_elems, const uint32_t* box, const uint32_t* elem_strides, int swizzle_bytes) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return set_error("cuTensorMapEncodeTiled unavailable");
  const uint64_t esz = dtype == TMAP_F32 ? 4 : 2;
  cuuint64_t d[5], st[4];
  cuuint32_t b[5], es[5];
  for (int i = 0; i < rank; ++i) {
    d[i] = dims[i];
    b[i] = box[i];
    es[i] = elem_strides ? elem_strides[i] : 1;
  }
  for (int i = 0; i + 1 < rank; ++i) st[i] = strides_elems[i] * esz;
  CUresult r = fn(map, dtype == TMAP_F32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank,
                  const_cast<void*>(ptr), d, st, b, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                      : (swizzle_bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_128B),
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return set_error("cuTensorMapEncodeTiled failed (%d): rank %d dims %llu %llu %llu box %u %u", int(r), rank,
                     (unsigned long long)dims[0], (unsigned long long)(rank > 1 ? dims[1] : 0),
                     (unsigned long long)(rank > 2 ? dims[2] : 0), box[0], rank > 1 ? box[1] : 0);
  return 0;
}

int make_tmap_bf16(CUtensorMap* map, const void* ptr, int rank, const uint64_t* dims, const uint64_t* strides_elems,
                   const uint32_t* box, const uint32_t* elem_strides) {
  return make_tmap(map, ptr, TMAP_BF16, rank, dims, strides_elems, box, elem_strides);
}

int make_tmap_2d_bf16(CUtensorMap* map, const void* ptr, uint64_t inner, uint64_t outer, uint64_t pitch_elems,
                      uint32_t box_inner, uint32_t box_outer) {
  uint64_t dims[2] = {inner, outer};
  uint64_t strides[1] = {pitch_elems};
  uint32_t box[2] = {box_inner, box_outer};
  return make_tmap(map, ptr, TMAP_BF16, 2, dims, strides, box, nullptr);
}

}  // namespace wm3

extern "C" const char* wm3_last_error(void) { return wm3::g_err; }
extern "C" int wm3_version(void) { return 2; }
extern "C" int wm3_sm_count(void) { return wm3::sm_count(); }
