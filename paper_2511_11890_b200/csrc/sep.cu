// sep.cu — generic separable stencils: one kernel per axis (Z, then Y, then X).
//
// This is the always-available path (any radius, any shape, any dtype) and the
// bit-exact path: in `exact` mode every pass reproduces scipy's NI_Correlate1D
// arithmetic at filters.py:40 — f64 line values, symmetric fold
//     acc = x0*w0;  for d = R..1: acc += (x[-d] + x[+d]) * w[d]
// with separately rounded f64 multiply and add (no FMA contraction), then a
// float32 round per pass.  The fused fast kernel (gauss_fused.cu) is the
// throughput path; this file is its fallback and the LoG smoothing stage.
#include <algorithm>

#include <cstdlib>

#include "ops.cuh"

namespace hb {
namespace {

constexpr int kThreads = 256;

inline int grid_for(int64_t n) {
  int64_t b = (n + kThreads - 1) / kThreads;
  int64_t cap = (int64_t)kNumSMs * 16;
  return (int)(b < cap ? (b < 1 ? 1 : b) : cap);
}

template <typename T>
__device__ __forceinline__ float ldf(const T* p, int64_t i) {
  return (float)__ldg(p + i);
}

template <typename T>
__device__ __forceinline__ float load_base(const void* p, int64_t i) {
  return (float)__ldg(reinterpret_cast<const T*>(p) + i);
}

__device__ __forceinline__ float load_any(const void* p, int dt, int64_t i) {
  switch (dt) {
    case HB_U8: return load_base<uint8_t>(p, i);
    case HB_U16: return load_base<uint16_t>(p, i);
    case HB_U32: return load_base<uint32_t>(p, i);
    default: return load_base<float>(p, i);
  }
}

// MODE: 0 fast gaussian (fp32 fma), 1 exact gaussian (fp64 fold), 2 box sum.
template <typename Tin, int AXIS, int MODE>
__global__ void __launch_bounds__(kThreads)
k_axis_pass(const Tin* __restrict__ in, int64_t nzi, int64_t ny, int64_t nx,
            int64_t zo, int64_t nzo, float* __restrict__ out, Taps taps, EpiArgs epi,
            bool last) {
  const int R = taps.R;
  const int64_t plane = ny * nx;
  const int64_t total = nzo * plane;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t z = i / plane;
    int64_t r = i - z * plane;
    int64_t y = r / nx;
    int64_t x = r - y * nx;
    int64_t len, pos, stride, base;
    if (AXIS == 0) {
      len = nzi; pos = z + zo; stride = plane; base = r;
    } else if (AXIS == 1) {
      len = ny; pos = y; stride = nx; base = z * plane + x;
    } else {
      len = nx; pos = x; stride = 1; base = z * plane + y * nx;
    }
    float result;
    if (MODE == 1) {
      double acc = __dmul_rn((double)ldf(in, base + pos * stride), (double)taps.w[R]);
      for (int d = R; d >= 1; --d) {
        double a = (double)ldf(in, base + clamp64(pos - d, 0, len - 1) * stride);
        double b = (double)ldf(in, base + clamp64(pos + d, 0, len - 1) * stride);
        acc = __dadd_rn(acc, __dmul_rn(__dadd_rn(a, b), (double)taps.w[R - d]));
      }
      result = (float)acc;
    } else if (MODE == 0) {
      float acc = ldf(in, base + pos * stride) * taps.w[R];
      for (int d = R; d >= 1; --d) {
        float a = ldf(in, base + clamp64(pos - d, 0, len - 1) * stride);
        float b = ldf(in, base + clamp64(pos + d, 0, len - 1) * stride);
        acc = fmaf(a + b, taps.w[R - d], acc);
      }
      result = acc;
    } else {
      float acc = ldf(in, base + pos * stride);
      for (int d = 1; d <= R; ++d) {
        acc += ldf(in, base + clamp64(pos - d, 0, len - 1) * stride);
        acc += ldf(in, base + clamp64(pos + d, 0, len - 1) * stride);
      }
      result = acc;
    }
    if (last) {
      if (epi.kind == EPI_UNSHARP) {
        // filters.py:139 — numpy order: (base - g), * amount, base + ...; no FMA
        float b = load_any(epi.orig, epi.orig_dt, (z + epi.orig_zo) * plane + r);
        result = __fadd_rn(b, __fmul_rn(epi.amount, __fsub_rn(b, result)));
      } else if (epi.kind == EPI_BOX_MEAN) {
        result = __fdiv_rn(result, epi.count);
      }
    }
    out[i] = result;
  }
}

template <typename Tin, int MODE>
cudaError_t run3(const DevIn& in, int64_t zo, int64_t nzo, float* out, const Taps& taps,
                 const EpiArgs& epi, float* tmp, cudaStream_t s, int64_t* launches) {
  int64_t n = nzo * in.ny * in.nx;
  int g = grid_for(n);
  EpiArgs none;
  // Z: in -> out, Y: out -> tmp, X: tmp -> out (+ epilogue)
  k_axis_pass<Tin, 0, MODE><<<g, kThreads, 0, s>>>(
      (const Tin*)in.p, in.nz, in.ny, in.nx, zo, nzo, out, taps, none, false);
  k_axis_pass<float, 1, MODE><<<g, kThreads, 0, s>>>(
      out, nzo, in.ny, in.nx, 0, nzo, tmp, taps, none, false);
  k_axis_pass<float, 2, MODE><<<g, kThreads, 0, s>>>(
      tmp, nzo, in.ny, in.nx, 0, nzo, out, taps, epi, true);
  if (launches) *launches += 3;
  return cudaGetLastError();
}

template <int MODE>
cudaError_t dispatch_dt(const DevIn& in, int64_t zo, int64_t nzo, float* out,
                        const Taps& taps, const EpiArgs& epi, float* tmp, cudaStream_t s,
                        int64_t* launches) {
  switch (in.dt) {
    case HB_U8: return run3<uint8_t, MODE>(in, zo, nzo, out, taps, epi, tmp, s, launches);
    case HB_U16: return run3<uint16_t, MODE>(in, zo, nzo, out, taps, epi, tmp, s, launches);
    case HB_U32: return run3<uint32_t, MODE>(in, zo, nzo, out, taps, epi, tmp, s, launches);
    case HB_F32: return run3<float, MODE>(in, zo, nzo, out, taps, epi, tmp, s, launches);
  }
  return cudaErrorInvalidValue;
}

// ---- LoG second stage ------------------------------------------------------
// cd(f)[i] = 0.5f * (f[clamp(i+1)] - f[clamp(i-1)])   (filters.py:234-243)
// second(i) = 0.5f * (cd[clamp(i+1)] - cd[clamp(i-1)])

// One CTA = 32 x 8 (x, y) tile marching down a z-chunk.  Each slice's tile
// plus a 2-voxel x/y halo is staged in smem (cooperative, prefetched one slice
// ahead in registers), so xx and yy come from smem; zz comes from a 5-slice
// register window per thread.  32-bit in-plane math.
constexpr int LD_TX = 32, LD_TY = 8, LD_W = LD_TX + 4, LD_H = LD_TY + 4;
constexpr int LD_PER = (LD_W * LD_H + 255) / 256;

__global__ void __launch_bounds__(256)
k_log_diff(const float* __restrict__ g, int64_t gz0, int nz, int ny, int nx, int64_t zo,
           int nzo, int zchunk, float* __restrict__ out) {
  __shared__ float tile[2][LD_H][LD_W];
  const int tid = threadIdx.x;
  const int x0 = blockIdx.x * LD_TX, y0 = blockIdx.y * LD_TY;
  const int x = x0 + (tid & 31), y = y0 + (tid >> 5);
  const int zs = blockIdx.z * zchunk, ze = min(zs + zchunk, nzo);
  const int64_t plane = (int64_t)ny * nx;
  // loader: element e -> clamped (gy, gx) offset in a slice
  int off[LD_PER];
  bool val[LD_PER];
#pragma unroll
  for (int k = 0; k < LD_PER; ++k) {
    const int e = tid + 256 * k;
    val[k] = e < LD_W * LD_H;
    const int ly = val[k] ? e / LD_W : 0, lx = val[k] ? e % LD_W : 0;
    off[k] = min(max(y0 - 2 + ly, 0), ny - 1) * nx + min(max(x0 - 2 + lx, 0), nx - 1);
  }
  auto fetch = [&](int64_t zb, float (&v)[LD_PER]) {
    const float* src = g + (zb - gz0) * plane;
#pragma unroll
    for (int k = 0; k < LD_PER; ++k) v[k] = val[k] ? __ldg(src + off[k]) : 0.f;
  };
  const bool inside = x < nx && y < ny;
  const float* col = g + (int64_t)min(y, ny - 1) * nx + min(x, nx - 1);
  auto at = [&](int64_t zz) { return __ldg(col + (zz - gz0) * plane); };
  // clamped-index second difference over a window held by accessor f
  auto second = [&](int c, int len, auto f) {
    const int jp = min(c + 1, len - 1), jm = max(c - 1, 0);
    const float dp = __fmul_rn(0.5f, __fsub_rn(f(min(jp + 1, len - 1)), f(max(jp - 1, 0))));
    const float dm = __fmul_rn(0.5f, __fsub_rn(f(min(jm + 1, len - 1)), f(max(jm - 1, 0))));
    return __fmul_rn(0.5f, __fsub_rn(dp, dm));
  };
  float w[5];
  const int64_t zb0 = zo + zs;
#pragma unroll
  for (int k = 0; k < 4; ++k) w[k] = at(min(max(zb0 - 2 + k, (int64_t)0), (int64_t)nz - 1));
  float v[LD_PER];
  fetch(zb0, v);
  int buf = 0;
  for (int zl = zs; zl < ze; ++zl) {
    const int64_t z = zo + zl;
#pragma unroll
    for (int k = 0; k < LD_PER; ++k)
      if (val[k]) (&tile[buf][0][0])[tid + 256 * k] = v[k];
    if (zl + 1 < ze) fetch(z + 1, v);
    w[4] = at(min(z + 2, (int64_t)nz - 1));
    __syncthreads();
    if (inside) {
      const int zi = (int)z;
      const int tx = (tid & 31) + 2, ty = (tid >> 5) + 2;
      float xx, yy, zz;
      if (x >= 2 && x < nx - 2 && y >= 2 && y < ny - 2 && zi >= 2 && zi < nz - 2) {
        // interior: no clamp can trigger -> straight-line, same rounding order
        const float c = tile[buf][ty][tx];
        auto sec = [](float lo2, float ctr, float hi2) {
          const float dp = __fmul_rn(0.5f, __fsub_rn(hi2, ctr));
          const float dm = __fmul_rn(0.5f, __fsub_rn(ctr, lo2));
          return __fmul_rn(0.5f, __fsub_rn(dp, dm));
        };
        xx = sec(tile[buf][ty][tx - 2], c, tile[buf][ty][tx + 2]);
        yy = sec(tile[buf][ty - 2][tx], c, tile[buf][ty + 2][tx]);
        zz = sec(w[0], w[2], w[4]);
      } else {
        auto wz = [&](int i) { return w[i - zi + 2]; };
        zz = second(zi, nz, wz);
        xx = second(x, nx, [&](int i) { return tile[buf][ty][tx + (i - x)]; });
        yy = second(y, ny, [&](int i) { return tile[buf][ty + (i - y)][tx]; });
      }
      out[(int64_t)zl * plane + (int64_t)y * nx + x] = __fadd_rn(__fadd_rn(xx, yy), zz);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) w[k] = w[k + 1];
    buf ^= 1;
  }
}

template <typename Tin, typename Tout>
__global__ void __launch_bounds__(kThreads)
k_copy(const Tin* __restrict__ in, int64_t off, int64_t n, Tout* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (Tout)in[off + i];
}

}  // namespace

cudaError_t gaussian_generic(const DevIn& in, int64_t zo, int64_t nzo, float* out,
                             const Taps& taps, bool exact, const EpiArgs& epi, float* tmp,
                             cudaStream_t s, int64_t* launches) {
  if (nzo <= 0) return cudaSuccess;
  return exact ? dispatch_dt<1>(in, zo, nzo, out, taps, epi, tmp, s, launches)
               : dispatch_dt<0>(in, zo, nzo, out, taps, epi, tmp, s, launches);
}

cudaError_t mean_generic(const DevIn& in, int64_t zo, int64_t nzo, float* out, int r,
                         float* tmp, cudaStream_t s, int64_t* launches) {
  if (nzo <= 0) return cudaSuccess;
  Taps taps;
  taps.R = r;
  EpiArgs epi;
  epi.kind = EPI_BOX_MEAN;
  float size = (float)(2 * r + 1);
  epi.count = size * size * size;
  return dispatch_dt<2>(in, zo, nzo, out, taps, epi, tmp, s, launches);
}

cudaError_t log_diff(const float* g, int64_t gz0, int64_t ngz, int64_t nz, int64_t ny,
                     int64_t nx, int64_t zo, int64_t nzo, float* out, cudaStream_t s,
                     int64_t* launches) {
  (void)ngz;
  if (nzo <= 0) return cudaSuccess;
  if (!std::getenv("HB_LOG_TILE")) {
    const cudaError_t e = log_diff_stream(g, gz0, nz, ny, nx, zo, nzo, out, s, launches);
    if (e != cudaErrorNotSupported) return e;
    cudaGetLastError();
  }
  const int64_t tiles = ((nx + LD_TX - 1) / LD_TX) * ((ny + LD_TY - 1) / LD_TY);
  // short z-chunks: each step's loads are latency-bound, so parallelism (many
  // resident CTAs) hides them; 32 slices keep the window priming cost at ~12%
  const int64_t want = std::max<int64_t>((nzo + 31) / 32, (64 * kNumSMs + tiles - 1) / tiles);
  const int zchunk = (int)std::max<int64_t>(8, (nzo + want - 1) / want);
  dim3 grid((unsigned)((nx + LD_TX - 1) / LD_TX), (unsigned)((ny + LD_TY - 1) / LD_TY),
            (unsigned)((nzo + zchunk - 1) / zchunk));
  k_log_diff<<<grid, 256, 0, s>>>(g, gz0, (int)nz, (int)ny, (int)nx, zo, (int)nzo, zchunk, out);
  if (launches) *launches += 1;
  return cudaGetLastError();
}

cudaError_t copy_slices(const DevIn& in, int64_t zo, int64_t nzo, void* out,
                        cudaStream_t s, int64_t* launches) {
  if (nzo <= 0) return cudaSuccess;
  size_t es = dtype_size(in.dt);
  size_t bytes = (size_t)nzo * in.ny * in.nx * es;
  const char* src = (const char*)in.p + (size_t)zo * in.ny * in.nx * es;
  if (launches) *launches += 1;
  return cudaMemcpyAsync(out, src, bytes, cudaMemcpyDeviceToDevice, s);
}

}  // namespace hb
