// extra.cu — the next local map operators on the same chunk machinery
// (SURVEY.md §8(f) row 2): single Hessian components, Sobel / Prewitt gradient
// magnitude and apply_threshold.  All three are bit-exact restatements:
//   hessian_ab = cd_b(cd_a(g)), cd(f)[i] = 0.5 * (f[clamp(i+1)] - f[clamp(i-1)])
//       in float32 on the exact Gaussian g (filters.py:246-253);
//   sobel / prewitt: per derivative axis, three 3-tap correlate1d passes
//       (z, y, x; f64 accumulation in NI_Correlate1D's symmetric /
//       antisymmetric fold, f32 rounding per pass), total += comp*comp in f32,
//       sqrt (filters.py:187-207);
//   apply_threshold: data > t as uint32 labels with NumPy 2 comparison
//       semantics (float32 data compares against float32(t), integer data in
//       float64) (threshold.py:110-112).
// These are memory-/latency-light per-voxel kernels (one thread per output,
// x fastest, neighbours through L1): not on the benchmarked path.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "ops.cuh"

namespace hb {
namespace {

constexpr int kT = 256;

inline int grid_for(int64_t n) {
  int64_t b = (n + kT - 1) / kT;
  const int64_t cap = (int64_t)kNumSMs * 32;
  return (int)(b < 1 ? 1 : (b < cap ? b : cap));
}

// axes are template parameters: the (z, y, x) position stays in registers
// (a runtime-indexed int[3] lived on the stack and cost ~3x)
template <int A, int B>
__global__ void __launch_bounds__(kT)
k_hessian_comp(const float* __restrict__ g, int64_t gz0, int nz, int ny, int nx, int64_t zo,
               int64_t nzo, float* __restrict__ out) {
  // one output row (z, y) per block iteration: no per-voxel 64-bit division
  for (int64_t row = blockIdx.x; row < nzo * ny; row += gridDim.x) {
    const int zl = (int)(row / ny);
    const int z = (int)(zo + zl), y = (int)(row - (int64_t)zl * ny);
    for (int x = threadIdx.x; x < nx; x += kT) {
      auto at = [&](int qz, int qy, int qx) {
        return __ldg(g + ((int64_t)(qz - gz0) * ny + qy) * nx + qx);
      };
      auto lim = [&](int ax) { return ax == 0 ? nz : (ax == 1 ? ny : nx); };
      // inner cd along A at q (clamped per step), q = (qz, qy, qx)
      auto cd_a = [&](int qz, int qy, int qx) {
        int h[3] = {qz, qy, qx}, l[3] = {qz, qy, qx};
        h[A] = min(h[A] + 1, lim(A) - 1);
        l[A] = max(l[A] - 1, 0);
        return __fmul_rn(0.5f, __fsub_rn(at(h[0], h[1], h[2]), at(l[0], l[1], l[2])));
      };
      int p[3] = {z, y, x}, m[3] = {z, y, x};
      p[B] = min(p[B] + 1, lim(B) - 1);
      m[B] = max(m[B] - 1, 0);
      const float dp = cd_a(p[0], p[1], p[2]);
      const float dm = cd_a(m[0], m[1], m[2]);
      out[row * nx + x] = __fmul_rn(0.5f, __fsub_rn(dp, dm));
    }
  }
}

// one 3-tap correlate1d output, NI_Correlate1D fold order, f64, rounded to f32
__device__ __forceinline__ float corr3(float xm, float x0, float xp, double w0, double w1, int sym) {
  const double m = (double)xm, c = (double)x0, p = (double)xp;
  double acc = __dmul_rn(c, w1);
  if (sym > 0) acc = __dadd_rn(acc, __dmul_rn(__dadd_rn(m, p), w0));
  else acc = __dadd_rn(acc, __dmul_rn(__dsub_rn(m, p), w0));
  return (float)acc;
}

template <typename T>
__global__ void __launch_bounds__(kT)
k_gradmag(const T* __restrict__ in, int nz, int ny, int nx, int64_t zo, int64_t nzo,
          float smooth_mid, float* __restrict__ out) {
  for (int64_t row = blockIdx.x; row < nzo * ny; row += gridDim.x)
  for (int x = threadIdx.x; x < nx; x += kT) {
    const int64_t i = row * nx + x;
    const int zl = (int)(row / ny);
    const int z = (int)(zo + zl), y = (int)(row - (int64_t)zl * ny);
    // the clamped 3x3x3 window (each separable pass clamps along its own axis,
    // which is the same as clamping the window once)
    float v[3][3][3];
#pragma unroll
    for (int dz = 0; dz < 3; ++dz) {
      const int zc = min(max(z + dz - 1, 0), nz - 1);
#pragma unroll
      for (int dy = 0; dy < 3; ++dy) {
        const int yc = min(max(y + dy - 1, 0), ny - 1);
        const T* row = in + ((int64_t)zc * ny + yc) * nx;
#pragma unroll
        for (int dx = 0; dx < 3; ++dx) v[dz][dy][dx] = (float)__ldg(row + min(max(x + dx - 1, 0), nx - 1));
      }
    }
    float total_sq = 0.f;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      // weights (w0 = outer, w1 = centre): deriv [-1, 0, 1] is antisymmetric
      // with w0 = -1; smoothing [1, m, 1] is symmetric with w0 = 1
      const double w0z = d == 0 ? -1.0 : 1.0, w1z = d == 0 ? 0.0 : (double)smooth_mid;
      const double w0y = d == 1 ? -1.0 : 1.0, w1y = d == 1 ? 0.0 : (double)smooth_mid;
      const double w0x = d == 2 ? -1.0 : 1.0, w1x = d == 2 ? 0.0 : (double)smooth_mid;
      const int sz = d == 0 ? -1 : 1, sy = d == 1 ? -1 : 1, sx = d == 2 ? -1 : 1;
      float a[3][3];  // z pass at the 3x3 (y, x) positions
#pragma unroll
      for (int dy = 0; dy < 3; ++dy)
#pragma unroll
        for (int dx = 0; dx < 3; ++dx) a[dy][dx] = corr3(v[0][dy][dx], v[1][dy][dx], v[2][dy][dx], w0z, w1z, sz);
      float b[3];  // y pass at the 3 x positions
#pragma unroll
      for (int dx = 0; dx < 3; ++dx) b[dx] = corr3(a[0][dx], a[1][dx], a[2][dx], w0y, w1y, sy);
      const float comp = corr3(b[0], b[1], b[2], w0x, w1x, sx);
      total_sq = __fadd_rn(total_sq, __fmul_rn(comp, comp));
    }
    out[i] = __fsqrt_rn(total_sq);
  }
}

template <typename T>
__global__ void __launch_bounds__(kT)
k_threshold(const T* __restrict__ in, int64_t n, double t, uint32_t* __restrict__ out) {
  const float tf = (float)t;
  for (int64_t i = blockIdx.x * (int64_t)kT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kT) {
    const T v = __ldg(in + i);
    if constexpr (std::is_same<T, float>::value) out[i] = v > tf ? 1u : 0u;
    else out[i] = (double)v > t ? 1u : 0u;
  }
}

// lbp2d: bit (7 - k) set when neighbour k >= centre, neighbours clockwise from
// the top-left, edge-clamped in y/x; comparisons in the input dtype
template <typename T>
__global__ void __launch_bounds__(kT)
k_lbp2d(const T* __restrict__ in, int ny, int nx, int64_t n, uint8_t* __restrict__ out) {
  const int64_t plane = (int64_t)ny * nx;
  for (int64_t row = blockIdx.x; row < n / nx; row += gridDim.x)
  for (int x = threadIdx.x; x < nx; x += kT) {
    const int64_t i = row * nx + x;
    const int64_t zl = row / ny;
    const int y = (int)(row - zl * ny);
    const T* sl = in + zl * plane;
    const int64_t rr = (int64_t)y * nx + x;
    const T c = __ldg(sl + rr);
    const int ym = max(y - 1, 0) * nx, y0 = y * nx, yp = min(y + 1, ny - 1) * nx;
    const int xm = max(x - 1, 0), xp = min(x + 1, nx - 1);
    const int nb[8] = {ym + xm, ym + x, ym + xp, y0 + xp, yp + xp, yp + x, yp + xm, y0 + xm};
    uint32_t b = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) b |= (__ldg(sl + nb[k]) >= c ? 1u : 0u) << (7 - k);
    out[i] = (uint8_t)b;
  }
}

template <typename T>
__global__ void __launch_bounds__(kT) k_to_f32(const T* __restrict__ in, int64_t n, float* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)kT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kT)
    out[i] = (float)__ldg(in + i);
}

// one Perona-Malik step over the 6 axial neighbours (filters.py:166-183), the
// reference's float32 op order: per axis t = g(fwd)*fwd + g(bwd)*bwd, flux += t
// (flux starts at +0), out = c + dt*flux; fwd = 0 past the last slice of the
// block, bwd = -(c - prev) and 0 at the first
__device__ __forceinline__ float diff_g(float v, float kappa, bool rational) {
  const float sc = __fdiv_rn(v, kappa);
  const float s2 = __fmul_rn(sc, sc);
  return rational ? __fdiv_rn(1.0f, __fadd_rn(1.0f, s2)) : expf(-s2);
}

__global__ void __launch_bounds__(kT)
k_diffusion_step(const float* __restrict__ src, float* __restrict__ dst, int nz, int ny, int nx,
                 float kappa, float dt, bool rational) {
  const int64_t plane = (int64_t)ny * nx;
  for (int64_t row = blockIdx.x; row < (int64_t)nz * ny; row += gridDim.x)
  for (int x = threadIdx.x; x < nx; x += kT) {
    const int64_t i = row * nx + x;
    const int z = (int)(row / ny), y = (int)(row - (int64_t)z * ny);
    const float c = src[i];
    const int crd[3] = {z, y, x}, ext[3] = {nz, ny, nx};
    const int64_t str[3] = {plane, nx, 1};
    float flux = 0.0f;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const float fwd = crd[a] < ext[a] - 1 ? __fsub_rn(src[i + str[a]], c) : 0.0f;
      const float bwd = crd[a] > 0 ? -__fsub_rn(c, src[i - str[a]]) : 0.0f;
      const float t = __fadd_rn(__fmul_rn(diff_g(fwd, kappa, rational), fwd),
                                __fmul_rn(diff_g(bwd, kappa, rational), bwd));
      flux = __fadd_rn(flux, t);
    }
    dst[i] = __fadd_rn(c, __fmul_rn(dt, flux));
  }
}

}  // namespace

cudaError_t diffusion(const DevIn& in, int64_t zo, int64_t nzo, float* out, int iterations,
                      float kappa, float dt, bool rational, float* b0, float* b1, cudaStream_t s,
                      int64_t* launches) {
  if (nzo <= 0) return cudaSuccess;
  const int64_t plane = in.ny * in.nx, n = in.nz * plane;
  const int g = grid_for(n);
  switch (in.dt) {
    case HB_U8: k_to_f32<uint8_t><<<g, kT, 0, s>>>((const uint8_t*)in.p, n, b0); break;
    case HB_U16: k_to_f32<uint16_t><<<g, kT, 0, s>>>((const uint16_t*)in.p, n, b0); break;
    case HB_U32: k_to_f32<uint32_t><<<g, kT, 0, s>>>((const uint32_t*)in.p, n, b0); break;
    case HB_F32: k_to_f32<float><<<g, kT, 0, s>>>((const float*)in.p, n, b0); break;
    default: return cudaErrorInvalidValue;
  }
  if (launches) *launches += 1;
  for (int it = 0; it < iterations; ++it) {
    k_diffusion_step<<<g, kT, 0, s>>>(b0, b1, (int)in.nz, (int)in.ny, (int)in.nx, kappa, dt, rational);
    if (launches) *launches += 1;
    float* t = b0;
    b0 = b1;
    b1 = t;
  }
  cudaError_t e = cudaMemcpyAsync(out, b0 + zo * plane, (size_t)(nzo * plane) * 4,
                                  cudaMemcpyDeviceToDevice, s);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t lbp2d(const DevIn& in, int64_t zo, int64_t nzo, uint8_t* out, cudaStream_t s,
                  int64_t* launches) {
  if (nzo <= 0) return cudaSuccess;
  const int64_t plane = in.ny * in.nx, n = nzo * plane;
  const int g = grid_for(n);
  switch (in.dt) {
    case HB_U8: k_lbp2d<uint8_t><<<g, kT, 0, s>>>((const uint8_t*)in.p + zo * plane, (int)in.ny, (int)in.nx, n, out); break;
    case HB_U16: k_lbp2d<uint16_t><<<g, kT, 0, s>>>((const uint16_t*)in.p + zo * plane, (int)in.ny, (int)in.nx, n, out); break;
    case HB_U32: k_lbp2d<uint32_t><<<g, kT, 0, s>>>((const uint32_t*)in.p + zo * plane, (int)in.ny, (int)in.nx, n, out); break;
    case HB_F32: k_lbp2d<float><<<g, kT, 0, s>>>((const float*)in.p + zo * plane, (int)in.ny, (int)in.nx, n, out); break;
    default: return cudaErrorInvalidValue;
  }
  if (launches) *launches += 1;
  return cudaGetLastError();
}

cudaError_t hessian_stage(const float* g, int64_t gz0, int64_t nz, int64_t ny, int64_t nx,
                          int64_t zo, int64_t nzo, int axis_a, int axis_b, float* out,
                          cudaStream_t s, int64_t* launches) {
  if (nzo <= 0) return cudaSuccess;
  const int gr = grid_for(nzo * ny * nx);
  const int key = axis_a * 3 + axis_b;
#define HB_HC(A, B) \
  case A * 3 + B: k_hessian_comp<A, B><<<gr, kT, 0, s>>>(g, gz0, (int)nz, (int)ny, (int)nx, zo, nzo, out); break;
  switch (key) {
    HB_HC(0, 0) HB_HC(0, 1) HB_HC(0, 2) HB_HC(1, 0) HB_HC(1, 1) HB_HC(1, 2) HB_HC(2, 0) HB_HC(2, 1) HB_HC(2, 2)
    default: return cudaErrorInvalidValue;
  }
#undef HB_HC
  if (launches) *launches += 1;
  return cudaGetLastError();
}

namespace {
// Separable tiled form of k_gradmag: a 32 x 8 tile of outputs streams down z;
// per output slice the three z-passes are shared by the whole tile
// (Zs = smooth, Zd = derivative at every (y, x) of the halo'd tile), then three
// y-pass planes (Ys∘Zs, Yd∘Zs, Ys∘Zd), then the three x-passes per output —
// 8 corr3 per voxel (x1.3 halo) instead of 39, identical arithmetic per pass
// (each pass output is the same f32 the per-voxel kernel rounds to).
constexpr int GT_X = 32, GT_Y = 8, GT_H = GT_Y + 2, GT_W = GT_X + 2;
constexpr int GT_NL = (GT_H * GT_W + kT - 1) / kT;

template <typename T>
__global__ void __launch_bounds__(kT)
k_gradmag_tile(const T* __restrict__ in, int nz, int ny, int nx, int zo, int nzo, int zchunk,
               float smooth_mid, float* __restrict__ out) {
  __shared__ float ring[3][GT_H * GT_W];
  __shared__ float zs[GT_H * GT_W], zd[GT_H * GT_W];
  __shared__ float yss[GT_Y * GT_W], yds[GT_Y * GT_W], ysd[GT_Y * GT_W];
  const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
  const int x0 = blockIdx.x * GT_X, y0 = blockIdx.y * GT_Y;
  const int o0 = blockIdx.z * zchunk, o1 = min(o0 + zchunk, nzo);
  const int64_t plane = (int64_t)ny * nx;
  const double mid = (double)smooth_mid;
  int off[GT_NL];
#pragma unroll
  for (int j = 0; j < GT_NL; ++j) {
    const int i = min(tid + j * kT, GT_H * GT_W - 1);
    const int r = i / GT_W, c = i - r * GT_W;
    off[j] = min(max(y0 - 1 + r, 0), ny - 1) * nx + min(max(x0 - 1 + c, 0), nx - 1);
  }
  auto load = [&](int zb, float (&v)[GT_NL]) {
    const T* sl = in + (int64_t)min(max(zb, 0), nz - 1) * plane;
#pragma unroll
    for (int j = 0; j < GT_NL; ++j) v[j] = (float)__ldg(sl + off[j]);
  };
  auto put = [&](float* dst, const float (&v)[GT_NL]) {
#pragma unroll
    for (int j = 0; j < GT_NL; ++j)
      if (j < GT_NL - 1 || tid + j * kT < GT_H * GT_W) dst[tid + j * kT] = v[j];
  };
  float pre[GT_NL];
  load(zo + o0 - 1, pre);
  put(ring[0], pre);
  load(zo + o0, pre);
  put(ring[1], pre);
  load(zo + o0 + 1, pre);
  const int gx = x0 + tx, gy = y0 + ty;
  for (int o = o0; o < o1; ++o) {
    const int k = o - o0;
    put(ring[(k + 2) % 3], pre);
    __syncthreads();
    if (o + 1 < o1) load(zo + o + 2, pre);
    const float* rm = ring[k % 3];
    const float* rc = ring[(k + 1) % 3];
    const float* rp = ring[(k + 2) % 3];
    for (int i = tid; i < GT_H * GT_W; i += kT) {
      const float m = rm[i], c = rc[i], p = rp[i];
      zs[i] = corr3(m, c, p, 1.0, mid, 1);
      zd[i] = corr3(m, c, p, -1.0, 0.0, -1);
    }
    __syncthreads();
    for (int i = tid; i < GT_Y * GT_W; i += kT) {
      const int r = i / GT_W, c = i - r * GT_W;
      const int a = r * GT_W + c;
      const float s0 = zs[a], s1 = zs[a + GT_W], s2 = zs[a + 2 * GT_W];
      yss[i] = corr3(s0, s1, s2, 1.0, mid, 1);
      yds[i] = corr3(s0, s1, s2, -1.0, 0.0, -1);
      ysd[i] = corr3(zd[a], zd[a + GT_W], zd[a + 2 * GT_W], 1.0, mid, 1);
    }
    __syncthreads();
    if (gx < nx && gy < ny) {
      const int a = ty * GT_W + tx;
      const float gzc = corr3(ysd[a], ysd[a + 1], ysd[a + 2], 1.0, mid, 1);
      const float gyc = corr3(yds[a], yds[a + 1], yds[a + 2], 1.0, mid, 1);
      const float gxc = corr3(yss[a], yss[a + 1], yss[a + 2], -1.0, 0.0, -1);
      float t = __fmul_rn(gzc, gzc);  // 0 + gz^2 == gz^2 exactly
      t = __fadd_rn(t, __fmul_rn(gyc, gyc));
      t = __fadd_rn(t, __fmul_rn(gxc, gxc));
      __stcs(out + (int64_t)o * plane + (int64_t)gy * nx + gx, __fsqrt_rn(t));
    }
  }
}
}  // namespace

cudaError_t gradmag(const DevIn& in, int64_t zo, int64_t nzo, float* out, bool sobel,
                    cudaStream_t s, int64_t* launches) {
  if (nzo <= 0) return cudaSuccess;
  const float mid = sobel ? 2.f : 1.f;
  if (!std::getenv("HB_GRADMAG_NAIVE")) {
    const int gx = (int)((in.nx + GT_X - 1) / GT_X), gy = (int)((in.ny + GT_Y - 1) / GT_Y);
    const int64_t tiles = (int64_t)gx * gy, slots = (int64_t)kNumSMs * 4;
    int64_t split = std::max<int64_t>(1, (2 * slots + tiles - 1) / tiles);
    split = std::min<int64_t>(std::min<int64_t>(split, std::max<int64_t>(1, nzo / 8)), 65535);
    const int zc = (int)((nzo + split - 1) / split);
    dim3 grid(gx, gy, (unsigned)((nzo + zc - 1) / zc));
    const int nz = (int)in.nz, ny = (int)in.ny, nx = (int)in.nx;
    switch (in.dt) {
      case HB_U8: k_gradmag_tile<uint8_t><<<grid, kT, 0, s>>>((const uint8_t*)in.p, nz, ny, nx, (int)zo, (int)nzo, zc, mid, out); break;
      case HB_U16: k_gradmag_tile<uint16_t><<<grid, kT, 0, s>>>((const uint16_t*)in.p, nz, ny, nx, (int)zo, (int)nzo, zc, mid, out); break;
      case HB_U32: k_gradmag_tile<uint32_t><<<grid, kT, 0, s>>>((const uint32_t*)in.p, nz, ny, nx, (int)zo, (int)nzo, zc, mid, out); break;
      case HB_F32: k_gradmag_tile<float><<<grid, kT, 0, s>>>((const float*)in.p, nz, ny, nx, (int)zo, (int)nzo, zc, mid, out); break;
      default: return cudaErrorInvalidValue;
    }
    if (launches) *launches += 1;
    return cudaGetLastError();
  }
  const int g = grid_for(nzo * in.ny * in.nx);
  switch (in.dt) {
    case HB_U8: k_gradmag<uint8_t><<<g, kT, 0, s>>>((const uint8_t*)in.p, (int)in.nz, (int)in.ny, (int)in.nx, zo, nzo, mid, out); break;
    case HB_U16: k_gradmag<uint16_t><<<g, kT, 0, s>>>((const uint16_t*)in.p, (int)in.nz, (int)in.ny, (int)in.nx, zo, nzo, mid, out); break;
    case HB_U32: k_gradmag<uint32_t><<<g, kT, 0, s>>>((const uint32_t*)in.p, (int)in.nz, (int)in.ny, (int)in.nx, zo, nzo, mid, out); break;
    case HB_F32: k_gradmag<float><<<g, kT, 0, s>>>((const float*)in.p, (int)in.nz, (int)in.ny, (int)in.nx, zo, nzo, mid, out); break;
    default: return cudaErrorInvalidValue;
  }
  if (launches) *launches += 1;
  return cudaGetLastError();
}

cudaError_t threshold(const DevIn& in, int64_t zo, int64_t nzo, uint32_t* out, double t,
                      cudaStream_t s, int64_t* launches) {
  if (nzo <= 0) return cudaSuccess;
  const int64_t plane = in.ny * in.nx, n = nzo * plane;
  const int g = grid_for(n);
  switch (in.dt) {
    case HB_U8: k_threshold<uint8_t><<<g, kT, 0, s>>>((const uint8_t*)in.p + zo * plane, n, t, out); break;
    case HB_U16: k_threshold<uint16_t><<<g, kT, 0, s>>>((const uint16_t*)in.p + zo * plane, n, t, out); break;
    case HB_U32: k_threshold<uint32_t><<<g, kT, 0, s>>>((const uint32_t*)in.p + zo * plane, n, t, out); break;
    case HB_F32: k_threshold<float><<<g, kT, 0, s>>>((const float*)in.p + zo * plane, n, t, out); break;
    default: return cudaErrorInvalidValue;
  }
  if (launches) *launches += 1;
  return cudaGetLastError();
}

}  // namespace hb

// ---------------------------------------------------------------------------
// geodesic reconstruction (morphology.py:143-165): the fixed point of
// m <- min(dilate(m, cross(1)), mask) (or max(erode(m, cross(1)), mask)).  The
// reconstruction is the unique fixed point of this monotone map, so in-place
// (chaotic) sweeps reach exactly the reference's Jacobi result, in fewer
// passes; sweeps repeat until one changes nothing.
// ---------------------------------------------------------------------------
namespace hb {
namespace {

template <typename T, bool DIL>
__global__ void __launch_bounds__(kT)
k_geo_check(const T* __restrict__ marker, const T* __restrict__ mask, int64_t n, int* __restrict__ bad) {
  for (int64_t i = blockIdx.x * (int64_t)kT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kT) {
    const T a = marker[i], b = mask[i];
    if (DIL ? a > b : a < b) {
      *bad = 1;
      return;
    }
  }
}

template <typename T, bool DIL>
__global__ void __launch_bounds__(kT)
k_geo_sweep(T* cur, const T* __restrict__ mask, int nz, int ny, int nx, int* __restrict__ changed) {
  const int64_t plane = (int64_t)ny * nx;
  bool any = false;
  // one (z, y) row per block iteration (no per-voxel 64-bit division)
  for (int64_t row = blockIdx.x; row < (int64_t)nz * ny; row += gridDim.x)
  for (int x = threadIdx.x; x < nx; x += kT) {
    const int z = (int)(row / ny), y = (int)(row - (int64_t)z * ny);
    const int64_t i = row * nx + x;
    const T v = cur[i];
    T m = v;
    auto take = [&](int64_t j) {
      const T u = *((volatile const T*)(cur + j));
      m = DIL ? (u > m ? u : m) : (u < m ? u : m);
    };
    if (x > 0) take(i - 1);
    if (x < nx - 1) take(i + 1);
    if (y > 0) take(i - nx);
    if (y < ny - 1) take(i + nx);
    if (z > 0) take(i - plane);
    if (z < nz - 1) take(i + plane);
    const T b = mask[i];
    const T nv = DIL ? (m < b ? m : b) : (m > b ? m : b);
    if (nv != v) {
      cur[i] = nv;
      any = true;
    }
  }
  if (any) *changed = 1;
}

template <typename T, bool DIL>
cudaError_t geo_t(const T* marker, const T* mask, int64_t nz, int64_t ny, int64_t nx, T* out,
                  int* flags, cudaStream_t s, int64_t* sweeps) {
  const int64_t n = nz * ny * nx;
  const int g = grid_for(n);
  int h = 0;
  cudaMemsetAsync(flags, 0, 4, s);
  k_geo_check<T, DIL><<<g, kT, 0, s>>>(marker, mask, n, flags);
  cudaMemcpyAsync(&h, flags, 4, cudaMemcpyDeviceToHost, s);
  cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return e;
  if (h) return cudaErrorInvalidValue;  // marker violates the ordering
  if ((const void*)out != (const void*)marker)
    cudaMemcpyAsync(out, marker, (size_t)n * sizeof(T), cudaMemcpyDeviceToDevice, s);
  int64_t k = 0;
  const int gr = (int)std::min<int64_t>(nz * ny, (int64_t)kNumSMs * 64);
  do {
    cudaMemsetAsync(flags, 0, 4, s);
    k_geo_sweep<T, DIL><<<gr, kT, 0, s>>>(out, mask, (int)nz, (int)ny, (int)nx, flags);
    cudaMemcpyAsync(&h, flags, 4, cudaMemcpyDeviceToHost, s);
    e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return e;
    ++k;
  } while (h);
  if (sweeps) *sweeps = k;
  return cudaGetLastError();
}

}  // namespace

cudaError_t geodesic(const void* marker, const void* mask, int dt, int64_t nz, int64_t ny, int64_t nx,
                     bool dilation, void* out, int* flags, cudaStream_t s, int64_t* sweeps) {
  if (nz * ny * nx <= 0) return cudaSuccess;
#define HB_GEO(T)                                                                                     \
  return dilation ? geo_t<T, true>((const T*)marker, (const T*)mask, nz, ny, nx, (T*)out, flags, s, sweeps) \
                  : geo_t<T, false>((const T*)marker, (const T*)mask, nz, ny, nx, (T*)out, flags, s, sweeps);
  switch (dt) {
    case HB_U8: HB_GEO(uint8_t)
    case HB_U16: HB_GEO(uint16_t)
    case HB_U32: HB_GEO(uint32_t)
    case HB_F32: HB_GEO(float)
  }
#undef HB_GEO
  return cudaErrorInvalidValue;
}

}  // namespace hb
