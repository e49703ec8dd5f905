// Neighborhood window arithmetic shared by every kernel that needs it (bit-exact with grid.py).
#pragma once

namespace wm3 {

// grid.py:96-101: start = clip(i - (w-1)//2, 0, E - w).  (w-1)//2 is non-negative, so C division
// agrees with Python's floor division here.
__host__ __device__ __forceinline__ int bump_start(int i, int extent, int window) {
  int s = i - (window - 1) / 2;
  const int hi = extent - window;
  s = s < 0 ? 0 : s;
  return s > hi ? hi : s;
}

// grid.py:123: (c) mod W with Python semantics (result in [0, W)) for possibly negative c.
__host__ __device__ __forceinline__ int wrap_col(int c, int cols) {
  int r = c % cols;
  return r < 0 ? r + cols : r;
}

}  // namespace wm3
