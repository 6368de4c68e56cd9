// reduce.cu — pass 1 of the two-pass global operators (chunking.py:282-306),
// for Otsu (threshold.py:30-107): float32 min/max and NumPy-exact histograms.
//
// The histogram reproduces np.histogram(data, bins, range=(lo, hi)) bit for
// bit (numpy/lib/_histograms_impl.py, uniform-bin path, NumPy 2 / NEP 50
// promotion): values outside [lo, hi] are dropped; for float32 data the
// offset is the float32 difference v - float32(lo), divided in float64 by
// (hi - lo) and scaled by bins, truncated, then corrected by one against the
// float32 bin edges; integer data runs the same in float64.  Counts are exact
// (per-block shared-memory u32 counters, u64 global atomics).
#include <cuda_runtime.h>

#include "ops.cuh"

namespace hb {
namespace {

constexpr int kRT = 256;

__device__ __forceinline__ unsigned ord_key(float f) {  // total order, -0 < +0
  const unsigned u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__global__ void __launch_bounds__(kRT) k_minmax_f32(const float* __restrict__ p, int64_t n,
                                                     unsigned* __restrict__ acc) {
  unsigned lo = 0xffffffffu, hi = 0u, nan = 0u;
  for (int64_t i = blockIdx.x * (int64_t)kRT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kRT) {
    const float v = __ldg(p + i);
    if (v != v) {
      nan = 1u;
      continue;
    }
    const unsigned k = ord_key(v);
    lo = min(lo, k);
    hi = max(hi, k);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    nan |= __shfl_xor_sync(0xffffffffu, nan, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(acc, lo);
    atomicMax(acc + 1, hi);
    if (nan) atomicOr(acc + 2, 1u);
  }
}

template <typename T, bool F32>
__global__ void __launch_bounds__(kRT)
k_histogram(const T* __restrict__ p, int64_t n, int bins, double lo, double hi, double denom,
            const double* __restrict__ edges, unsigned long long* __restrict__ counts) {
  extern __shared__ unsigned sh[];
  const bool use_sh = bins <= 8192;
  if (use_sh)
    for (int b = threadIdx.x; b < bins; b += kRT) sh[b] = 0u;
  __syncthreads();
  const float lof = (float)lo, hif = (float)hi;
  for (int64_t i = blockIdx.x * (int64_t)kRT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kRT) {
    const T raw = __ldg(p + i);
    int64_t idx;
    if constexpr (F32) {
      const float v = (float)raw;
      if (!(v >= lof && v <= hif)) continue;
      const float d = __fsub_rn(v, lof);
      idx = (int64_t)__dmul_rn(__ddiv_rn((double)d, denom), (double)bins);
      if (idx == bins) idx = bins - 1;
      if (v < (float)edges[idx]) --idx;
      if (idx != bins - 1 && v >= (float)edges[idx + 1]) ++idx;
    } else {
      const double v = (double)raw;
      if (!(v >= lo && v <= hi)) continue;
      idx = (int64_t)__dmul_rn(__ddiv_rn(__dsub_rn(v, lo), denom), (double)bins);
      if (idx == bins) idx = bins - 1;
      if (v < edges[idx]) --idx;
      if (idx != bins - 1 && v >= edges[idx + 1]) ++idx;
    }
    if (use_sh) atomicAdd(&sh[idx], 1u);
    else atomicAdd(&counts[idx], 1ull);
  }
  __syncthreads();
  if (use_sh)
    for (int b = threadIdx.x; b < bins; b += kRT)
      if (sh[b]) atomicAdd(&counts[b], (unsigned long long)sh[b]);
}

inline int rgrid(int64_t n) {
  const int64_t b = (n + kRT - 1) / kRT, cap = (int64_t)kNumSMs * 8;
  return (int)(b < 1 ? 1 : (b < cap ? b : cap));
}

}  // namespace

cudaError_t minmax_f32(const float* p, int64_t n, unsigned* acc, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  k_minmax_f32<<<rgrid(n), kRT, 0, s>>>(p, n, acc);
  return cudaGetLastError();
}

cudaError_t histogram(const void* p, int dt, int64_t n, int bins, double lo, double hi,
                      const double* edges, bool edges_f32, unsigned long long* counts,
                      cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const double denom = hi - lo;  // np.subtract(hi, lo, dtype=float64)
  const size_t smem = bins <= 8192 ? (size_t)bins * 4 : 0;
  const int g = rgrid(n);
  if (dt == HB_F32 && edges_f32) {
    k_histogram<float, true><<<g, kRT, smem, s>>>((const float*)p, n, bins, lo, hi, denom, edges, counts);
  } else {
    switch (dt) {
      case HB_U8: k_histogram<uint8_t, false><<<g, kRT, smem, s>>>((const uint8_t*)p, n, bins, lo, hi, denom, edges, counts); break;
      case HB_U16: k_histogram<uint16_t, false><<<g, kRT, smem, s>>>((const uint16_t*)p, n, bins, lo, hi, denom, edges, counts); break;
      case HB_U32: k_histogram<uint32_t, false><<<g, kRT, smem, s>>>((const uint32_t*)p, n, bins, lo, hi, denom, edges, counts); break;
      case HB_F32: k_histogram<float, false><<<g, kRT, smem, s>>>((const float*)p, n, bins, lo, hi, denom, edges, counts); break;
      default: return cudaErrorInvalidValue;
    }
  }
  return cudaGetLastError();
}

}  // namespace hb
