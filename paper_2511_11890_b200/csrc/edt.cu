// edt.cu — exact Euclidean distance transform (quantify.py:115-175) on the
// device, bit for bit: dist2 = inf on foreground, 0 on background; for each
// axis z, y, x every line runs Felzenszwalb & Huttenlocher's lower-envelope
// scan (quantify.py:115-158) in float64 with the reference's operation order
// (explicit __dmul_rn/__dadd_rn/__ddiv_rn: no FMA contraction), then
// sqrt(dist2) in float64 cast to float32 (or dist2 itself when squared).
// One thread per line; the scan's site list and boundaries live in a
// line-interleaved workspace (coalesced across threads).
#include <cuda_runtime.h>

#include <math_constants.h>

#include <algorithm>
#include <cstdlib>

#include "ops.cuh"

namespace hb {
namespace {

constexpr int kET = 128;

template <typename T>
__global__ void __launch_bounds__(256) k_edt_init(const T* __restrict__ in, int64_t n, double* __restrict__ d2) {
  for (int64_t i = blockIdx.x * 256ll + threadIdx.x; i < n; i += (int64_t)gridDim.x * 256)
    d2[i] = in[i] != T(0) ? CUDART_INF : 0.0;
}

// one 1D pass along `axis` for every line; lines enumerate the other two axes
__global__ void __launch_bounds__(kET)
k_edt_axis(const double* __restrict__ f, double* __restrict__ out, int nz, int ny, int nx, int axis,
           double step, int64_t nlines, int* __restrict__ vbuf, double* __restrict__ zbuf) {
  const int64_t L = blockIdx.x * (int64_t)kET + threadIdx.x;
  if (L >= nlines) return;
  const int64_t plane = (int64_t)ny * nx;
  int n;
  int64_t base, stride;
  if (axis == 0) {  // lines over (y, x)
    n = nz;
    stride = plane;
    base = L;
  } else if (axis == 1) {  // lines over (z, x)
    n = ny;
    stride = nx;
    base = (L / nx) * plane + (L % nx);
  } else {  // lines over (z, y)
    n = nx;
    stride = 1;
    base = L * nx;
  }
  auto F = [&](int q) { return f[base + (int64_t)q * stride]; };
  auto V = [&](int k) -> int& { return vbuf[(int64_t)k * nlines + L]; };
  auto Z = [&](int k) -> double& { return zbuf[(int64_t)k * nlines + L]; };
  const double w2 = __dmul_rn(step, step);
  int k = 0;
  V(0) = 0;
  Z(0) = -CUDART_INF;
  Z(1) = CUDART_INF;
  for (int q = 1; q < n; ++q) {
    const double fq = F(q);
    if (fq == CUDART_INF) continue;
    while (true) {
      const int p = V(k);
      const double fp = F(p);
      double s;
      if (fp == CUDART_INF) {
        s = -CUDART_INF;
      } else {
        // ((f[q] + w2*q*q) - (f[p] + w2*p*p)) / (2.0*w2*(q - p))
        const double a = __dadd_rn(fq, __dmul_rn(__dmul_rn(w2, (double)q), (double)q));
        const double b = __dadd_rn(fp, __dmul_rn(__dmul_rn(w2, (double)p), (double)p));
        s = __ddiv_rn(__dsub_rn(a, b), __dmul_rn(__dmul_rn(2.0, w2), (double)(q - p)));
      }
      if (s <= Z(k)) {
        k -= 1;
        if (k < 0) {
          k = 0;
          V(0) = q;
          Z(0) = -CUDART_INF;
          Z(1) = CUDART_INF;
          break;
        }
        continue;
      }
      k += 1;
      V(k) = q;
      Z(k) = s;
      Z(k + 1) = CUDART_INF;
      break;
    }
  }
  k = 0;
  for (int q = 0; q < n; ++q) {
    while (Z(k + 1) < (double)q) ++k;
    const int p = V(k);
    const double fp = F(p);
    const int64_t dq = (int64_t)(q - p) * (q - p);
    out[base + (int64_t)q * stride] = fp != CUDART_INF ? __dadd_rn(fp, __dmul_rn(w2, (double)dq)) : CUDART_INF;
  }
}

// (z, a, b) -> (z, b, a) transpose of float64 planes through a 32 x 33 tile;
// with SQRT the float32 sqrt of the distance is written instead (fused final
// step).  The x-axis scan runs on the transposed block, where its lines are
// the middle axis (coalesced across threads, like the y scan).
template <typename To, bool SQRT>
__global__ void __launch_bounds__(256)
k_edt_transpose(const double* __restrict__ in, To* __restrict__ out, int na, int nb) {
  __shared__ double t[32][33];
  const int z = blockIdx.z;
  const int a0 = blockIdx.y * 32, b0 = blockIdx.x * 32;
  const double* src = in + (int64_t)z * na * nb;
  To* dst = out + (int64_t)z * na * nb;
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int a = a0 + r, b = b0 + threadIdx.x;
    if (a < na && b < nb) t[r][threadIdx.x] = src[(int64_t)a * nb + b];
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int b = b0 + r, a = a0 + threadIdx.x;
    if (a < na && b < nb) {
      const double v = t[threadIdx.x][r];
      if constexpr (SQRT) dst[(int64_t)b * na + a] = (To)__dsqrt_rn(v);
      else dst[(int64_t)b * na + a] = (To)v;
    }
  }
}

__global__ void __launch_bounds__(256) k_edt_sqrt(const double* __restrict__ d2, int64_t n, float* __restrict__ out) {
  for (int64_t i = blockIdx.x * 256ll + threadIdx.x; i < n; i += (int64_t)gridDim.x * 256)
    out[i] = (float)__dsqrt_rn(d2[i]);
}

}  // namespace

size_t edt_workspace_bytes(int64_t nz, int64_t ny, int64_t nx) {
  // per axis: lines * n sites (int) + lines * (n + 1) boundaries (double); the
  // largest axis pass bounds it
  const int64_t v = nz * ny * nx;
  const int64_t lines_max = std::max(ny * nx, std::max(nz * nx, nz * ny));
  return (size_t)(v * 4 + (v + lines_max) * 8) + 256;
}

cudaError_t edt(const void* in, int dt, int64_t nz, int64_t ny, int64_t nx, const double* spacing,
                bool squared, void* out, double* d2a, double* d2b, void* work, cudaStream_t s) {
  const int64_t n = nz * ny * nx;
  if (n <= 0) return cudaSuccess;
  const int g = (int)std::min<int64_t>((n + 255) / 256, (int64_t)kNumSMs * 32);
  switch (dt) {
    case HB_U8: k_edt_init<uint8_t><<<g, 256, 0, s>>>((const uint8_t*)in, n, d2a); break;
    case HB_U16: k_edt_init<uint16_t><<<g, 256, 0, s>>>((const uint16_t*)in, n, d2a); break;
    case HB_U32: k_edt_init<uint32_t><<<g, 256, 0, s>>>((const uint32_t*)in, n, d2a); break;
    case HB_F32: k_edt_init<float><<<g, 256, 0, s>>>((const float*)in, n, d2a); break;
    default: return cudaErrorInvalidValue;
  }
  const int64_t lines[3] = {ny * nx, nz * nx, nz * ny};
  double* src = d2a;
  double* dst = d2b;
  int* vbuf = reinterpret_cast<int*>(work);
  double* zbuf = reinterpret_cast<double*>(reinterpret_cast<char*>(work) + ((size_t)n * 4 + 255) / 256 * 256);
  const bool transpose_x = nz <= 65535 && !std::getenv("HB_EDT_DIRECT_X");
  for (int axis = 0; axis < (transpose_x ? 2 : 3); ++axis) {
    const int64_t nl = lines[axis];
    k_edt_axis<<<(unsigned)((nl + kET - 1) / kET), kET, 0, s>>>(src, dst, (int)nz, (int)ny, (int)nx, axis,
                                                                spacing[axis], nl, vbuf, zbuf);
    std::swap(src, dst);
  }
  if (!transpose_x) {
    if (squared) return cudaMemcpyAsync(out, src, (size_t)n * 8, cudaMemcpyDeviceToDevice, s);
    k_edt_sqrt<<<g, 256, 0, s>>>(src, n, (float*)out);
    return cudaGetLastError();
  }
  // x scan on the (z, x, y) transpose: same per-line arithmetic, coalesced
  const dim3 tb(32, 8);
  k_edt_transpose<double, false><<<dim3((unsigned)((nx + 31) / 32), (unsigned)((ny + 31) / 32), (unsigned)nz), tb, 0, s>>>(
      src, dst, (int)ny, (int)nx);
  std::swap(src, dst);
  k_edt_axis<<<(unsigned)((lines[2] + kET - 1) / kET), kET, 0, s>>>(src, dst, (int)nz, (int)nx, (int)ny, 1,
                                                                    spacing[2], lines[2], vbuf, zbuf);
  std::swap(src, dst);
  const dim3 gb((unsigned)((ny + 31) / 32), (unsigned)((nx + 31) / 32), (unsigned)nz);
  if (squared) k_edt_transpose<double, false><<<gb, tb, 0, s>>>(src, (double*)out, (int)nx, (int)ny);
  else k_edt_transpose<float, true><<<gb, tb, 0, s>>>(src, (float*)out, (int)nx, (int)ny);
  return cudaGetLastError();
}

}  // namespace hb
