// common.cuh — shared device/host helpers for the sm_100a kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/harpia_b200.h"

namespace hb {

constexpr int kNumSMs = 148;  // B200; grids are sized from the device query anyway

// A (Z, Y, X) block of the current stage input: local z in [0, nz), clamp-to-edge
// at every face (the reference pads each chunk with mode="edge"/"nearest").
template <typename T>
struct Block3 {
  const T* __restrict__ p;
  int64_t nz, ny, nx;
};

__host__ __device__ __forceinline__ int64_t clamp64(int64_t v, int64_t lo, int64_t hi) {
  return v < lo ? lo : (v > hi ? hi : v);
}
__host__ __device__ __forceinline__ int clampi(int v, int lo, int hi) {
  return v < lo ? lo : (v > hi ? hi : v);
}

template <typename T> __device__ __forceinline__ float to_f32(T v) { return (float)v; }

// Order-preserving u32 key for float32 (total order; -0 < +0; NaNs last).
__device__ __forceinline__ uint32_t f32_key(float f) {
  uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float key_f32(uint32_t k) {
  uint32_t u = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
  return __uint_as_float(u);
}

inline int dtype_size(int dt) { return dt == HB_U8 ? 1 : (dt == HB_U16 ? 2 : 4); }

// Per-launch bookkeeping the executor reports (hb_report.kernel_launches).
struct LaunchCounter {
  int64_t n = 0;
};

}  // namespace hb
