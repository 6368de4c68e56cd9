// median.cu — (2r+1)^3 median filter, rank = size//2, clamp-to-edge
// (filters.py:78-82 -> scipy median_filter -> rank_filter).  Output dtype is
// the input dtype; the order statistic is exact, so results are bit-exact.
//
// r = 1, 2: forgetful selection in registers (working set N/2+2, each round
// discards the min and max of the set and admits one new sample).
// r >= 3:   per-voxel radix (bit-by-bit) selection over order-preserving keys.
#include "ops.cuh"

namespace hb {
namespace {

constexpr int kThreads = 256;

template <typename K> struct MinMax;
template <> struct MinMax<float> {
  static __device__ __forceinline__ float mn(float a, float b) { return fminf(a, b); }
  static __device__ __forceinline__ float mx(float a, float b) { return fmaxf(a, b); }
};
template <> struct MinMax<uint32_t> {
  static __device__ __forceinline__ uint32_t mn(uint32_t a, uint32_t b) { return min(a, b); }
  static __device__ __forceinline__ uint32_t mx(uint32_t a, uint32_t b) { return max(a, b); }
};

template <typename K>
__device__ __forceinline__ void cs(K& a, K& b) {
  K t = MinMax<K>::mn(a, b);
  b = MinMax<K>::mx(a, b);
  a = t;
}

// Move the minimum of a[0..m) to a[0] and the maximum to a[m-1], keeping the set.
template <int m, typename K>
__device__ __forceinline__ void minmax_to_ends(K* a) {
#pragma unroll
  for (int i = 0; i < m / 2; ++i) cs(a[i], a[m - 1 - i]);
#pragma unroll
  for (int i = 1; i <= (m - 1) / 2; ++i) cs(a[0], a[i]);
#pragma unroll
  for (int i = m / 2; i < m - 1; ++i) cs(a[i], a[m - 1]);
}

template <typename T, typename K> struct Key;
template <> struct Key<float, float> {
  static __device__ __forceinline__ float to(float v) { return v; }
  static __device__ __forceinline__ float from(float k) { return k; }
};
template <typename T> struct Key<T, uint32_t> {
  static __device__ __forceinline__ uint32_t to(T v) { return (uint32_t)v; }
  static __device__ __forceinline__ T from(uint32_t k) { return (T)k; }
};

template <int W, typename T>
struct Window {
  const T* __restrict__ p;
  int64_t row[W][W];  // (zc*ny + yc)*nx for each (dz, dy)
  int64_t xc[W];
  __device__ __forceinline__ T get(int e) const {
    const int a = e / (W * W), b = (e / W) % W, c = e % W;
    return __ldg(p + row[a][b] + xc[c]);
  }
};

template <int m, int next, int N, int W, typename T, typename K>
__device__ __forceinline__ K forgetful_step(K* a, const Window<W, T>& win) {
  minmax_to_ends<m>(a);
  if constexpr (next < N) {
    a[0] = Key<T, K>::to(win.get(next));
    return forgetful_step<m - 1, next + 1, N, W, T, K>(a, win);
  } else {
    static_assert(m == 3, "forgetful selection must end with three candidates");
    return a[1];
  }
}

template <int R, typename T, typename K>
__global__ void __launch_bounds__(kThreads)
k_median_forgetful(const T* __restrict__ in, int64_t nz, int64_t ny, int64_t nx, int64_t zo,
                   int64_t nzo, T* __restrict__ out) {
  constexpr int W = 2 * R + 1;
  constexpr int N = W * W * W;
  constexpr int M0 = N / 2 + 2;
  const int64_t plane = ny * nx;
  const int64_t total = nzo * plane;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t zl = i / plane;
    int64_t rr = i - zl * plane;
    int64_t y = rr / nx;
    int64_t x = rr - y * nx;
    int64_t z = zl + zo;
    Window<W, T> win;
    win.p = in;
#pragma unroll
    for (int a = 0; a < W; ++a) {
      int64_t zc = clamp64(z + a - R, 0, nz - 1);
#pragma unroll
      for (int b = 0; b < W; ++b) win.row[a][b] = (zc * ny + clamp64(y + b - R, 0, ny - 1)) * nx;
      win.xc[a] = clamp64(x + a - R, 0, nx - 1);
    }
    K a[M0];
#pragma unroll
    for (int e = 0; e < M0; ++e) a[e] = Key<T, K>::to(win.get(e));
    K med = forgetful_step<M0, M0, N, W, T, K>(a, win);
    out[i] = Key<T, K>::from(med);
  }
}

template <typename T> __device__ __forceinline__ uint32_t okey(T v) { return (uint32_t)v; }
template <> __device__ __forceinline__ uint32_t okey<float>(float v) { return f32_key(v); }
template <typename T> __device__ __forceinline__ T unkey(uint32_t k) { return (T)k; }
template <> __device__ __forceinline__ float unkey<float>(uint32_t k) { return key_f32(k); }

// Radix selection of the k-th smallest key, one bit per pass, any radius.
template <typename T, int BITS>
__global__ void __launch_bounds__(kThreads)
k_median_radix(const T* __restrict__ in, int64_t nz, int64_t ny, int64_t nx, int64_t zo,
               int64_t nzo, T* __restrict__ out, int R) {
  const int W = 2 * R + 1;
  const int N = W * W * W;
  const int64_t plane = ny * nx;
  const int64_t total = nzo * plane;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t zl = i / plane;
    int64_t rr = i - zl * plane;
    int64_t y = rr / nx;
    int64_t x = rr - y * nx;
    int64_t z = zl + zo;
    uint32_t prefix = 0;
    int k = N / 2;
    for (int bit = BITS - 1; bit >= 0; --bit) {
      const uint32_t hi_mask = (bit == 31) ? 0u : (0xffffffffu << (bit + 1));
      int cnt0 = 0;
      for (int dz = -R; dz <= R; ++dz) {
        int64_t zc = clamp64(z + dz, 0, nz - 1);
        for (int dy = -R; dy <= R; ++dy) {
          const T* row = in + (zc * ny + clamp64(y + dy, 0, ny - 1)) * nx;
          for (int dx = -R; dx <= R; ++dx) {
            uint32_t key = okey<T>(__ldg(row + clamp64(x + dx, 0, nx - 1)));
            cnt0 += (((key ^ prefix) & hi_mask) == 0u) & (((key >> bit) & 1u) == 0u);
          }
        }
      }
      if (k >= cnt0) {
        k -= cnt0;
        prefix |= (1u << bit);
      }
    }
    out[i] = unkey<T>(prefix);
  }
}

inline int grid_for(int64_t n) {
  int64_t b = (n + kThreads - 1) / kThreads;
  int64_t cap = (int64_t)kNumSMs * 16;
  return (int)(b < cap ? (b < 1 ? 1 : b) : cap);
}

template <typename T, typename K, int BITS>
cudaError_t run_median(const DevIn& in, int64_t zo, int64_t nzo, void* out, int r,
                       cudaStream_t s, int64_t* launches) {
  int64_t n = nzo * in.ny * in.nx;
  int g = grid_for(n);
  const T* src = (const T*)in.p;
  T* dst = (T*)out;
  if (r == 1) {
    k_median_forgetful<1, T, K><<<g, kThreads, 0, s>>>(src, in.nz, in.ny, in.nx, zo, nzo, dst);
  } else if (r == 2) {
    k_median_forgetful<2, T, K><<<g, kThreads, 0, s>>>(src, in.nz, in.ny, in.nx, zo, nzo, dst);
  } else {
    k_median_radix<T, BITS><<<g, kThreads, 0, s>>>(src, in.nz, in.ny, in.nx, zo, nzo, dst, r);
  }
  if (launches) *launches += 1;
  return cudaGetLastError();
}

}  // namespace

cudaError_t median(const DevIn& in, int64_t zo, int64_t nzo, void* out, int r,
                   cudaStream_t s, int64_t* launches) {
  if (nzo <= 0) return cudaSuccess;
  switch (in.dt) {
    case HB_U8: return run_median<uint8_t, uint32_t, 8>(in, zo, nzo, out, r, s, launches);
    case HB_U16: return run_median<uint16_t, uint32_t, 16>(in, zo, nzo, out, r, s, launches);
    case HB_U32: return run_median<uint32_t, uint32_t, 32>(in, zo, nzo, out, r, s, launches);
    case HB_F32: return run_median<float, float, 32>(in, zo, nzo, out, r, s, launches);
  }
  return cudaErrorInvalidValue;
}

}  // namespace hb
