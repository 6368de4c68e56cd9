// sep.cu — generic separable stencils: one kernel per axis (Z, then Y, then X).
//
// This is the always-available path (any radius, any shape, any dtype) and the
// bit-exact path: in `exact` mode every pass reproduces scipy's NI_Correlate1D
// arithmetic at filters.py:40 — f64 line values, symmetric fold
//     acc = x0*w0;  for d = R..1: acc += (x[-d] + x[+d]) * w[d]
// with separately rounded f64 multiply and add (no FMA contraction), then a
// float32 round per pass.  The fused fast kernel (gauss_fused.cu) is the
// throughput path; this file is its fallback and the LoG smoothing stage.
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
__device__ __forceinline__ float gat(const float* g, int64_t gz0, int64_t plane, int64_t nx,
                                     int64_t z, int64_t y, int64_t x) {
  return __ldg(g + (z - gz0) * plane + y * nx + x);
}

__global__ void __launch_bounds__(kThreads)
k_log_diff(const float* __restrict__ g, int64_t gz0, int64_t nz, int64_t ny, int64_t nx,
           int64_t zo, int64_t nzo, float* __restrict__ out) {
  const int64_t plane = ny * nx;
  const int64_t total = nzo * plane;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t zl = i / plane;
    int64_t r = i - zl * plane;
    int64_t y = r / nx;
    int64_t x = r - y * nx;
    int64_t z = zl + zo;
    float second[3];
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      int64_t len = ax == 0 ? nx : (ax == 1 ? ny : nz);
      int64_t c = ax == 0 ? x : (ax == 1 ? y : z);
      float d[2];
#pragma unroll
      for (int side = 0; side < 2; ++side) {
        int64_t j = clamp64(side ? c + 1 : c - 1, 0, len - 1);
        int64_t hi = clamp64(j + 1, 0, len - 1), lo = clamp64(j - 1, 0, len - 1);
        float fh, fl;
        if (ax == 0) {
          fh = gat(g, gz0, plane, nx, z, y, hi); fl = gat(g, gz0, plane, nx, z, y, lo);
        } else if (ax == 1) {
          fh = gat(g, gz0, plane, nx, z, hi, x); fl = gat(g, gz0, plane, nx, z, lo, x);
        } else {
          fh = gat(g, gz0, plane, nx, hi, y, x); fl = gat(g, gz0, plane, nx, lo, y, x);
        }
        d[side] = __fmul_rn(0.5f, __fsub_rn(fh, fl));
      }
      second[ax] = __fmul_rn(0.5f, __fsub_rn(d[1], d[0]));
    }
    // LoG := (xx + yy) + zz
    out[i] = __fadd_rn(__fadd_rn(second[0], second[1]), second[2]);
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
  int64_t n = nzo * ny * nx;
  k_log_diff<<<grid_for(n), kThreads, 0, s>>>(g, gz0, nz, ny, nx, zo, nzo, out);
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
