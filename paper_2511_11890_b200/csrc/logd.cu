// logd.cu — LoG second stage, streaming form: out = (xx + yy) + zz where
// aa = cd_a(cd_a(g)) and cd(f)[i] = 0.5 * (f[clamp(i+1)] - f[clamp(i-1)])
// (filters.py:234-253: _central_diff / hessian_component, axis 2 = x, 1 = y,
// 0 = z; the clamp applies per cd step).  g is the smoothed volume.
//
// Like the box mean (box.cu) this stage is HBM traffic plus ~20 FP32 ops per
// voxel, so it is built for bytes in flight: a warp owns a 128-column x strip
// (4 columns per lane, 128-bit loads) of RY output rows and marches down z.
// The centre rows of the five slices z-2..z+2 sit in a register ring (one new
// slice per step, loaded a step ahead, rotated by moves); the y halo rows (y-2, y-1, y+RY,
// y+RY+1) of slice z and the strip's x-edge columns are loaded a step ahead
// too (L1/L2 hits: they are other warps' centre rows); x neighbours come from
// the adjacent lanes by shuffle.  Away from the volume faces the straight-line
// form is used; at the faces each operand index is clamped exactly as the
// reference does (identical rounding: the same f32 ops in the same order), so
// the output is bit-identical to the tiled k_log_diff and to the reference
// given the same g.
#include <cuda_runtime.h>

#include <cstdlib>

#include "ops.cuh"

namespace hb {
namespace {

constexpr int LX = 128;  // x columns per warp
#ifndef HB_LOG_MINB
#define HB_LOG_MINB 4  // 128 registers: 16 warps/SM instead of 8 at 179 (LoG 1024^3: 111.6 vs 95-106 Gvox/s; 5-6 spill)
#endif

struct LogArgs {
  const float* g;
  int64_t gz0;  // block slice of g's first slice
  int nz, ny, nx;
  int64_t zo;   // block slice of output 0
  int nzo, zchunk;
  float* out;
};

// cd(cd(f))[c] for the window f(clamp(c - 2 + k)), k = 0..4, with the
// per-step index clamps of the reference (faces only: kept out of line so the
// streaming loop stays small — a 6-way unrolled body with inline face code
// overflowed the instruction cache)
__device__ __noinline__ float sec_general(float w0, float w1, float w2, float w3, float w4, int c,
                                          int n) {
  const float w[5] = {w0, w1, w2, w3, w4};
  const int jp = min(c + 1, n - 1), jm = max(c - 1, 0);
  const float fpp = w[min(jp + 1, n - 1) - c + 2], fpm = w[max(jp - 1, 0) - c + 2];
  const float fmp = w[min(jm + 1, n - 1) - c + 2], fmm = w[max(jm - 1, 0) - c + 2];
  const float dp = __fmul_rn(0.5f, __fsub_rn(fpp, fpm));
  const float dm = __fmul_rn(0.5f, __fsub_rn(fmp, fmm));
  return __fmul_rn(0.5f, __fsub_rn(dp, dm));
}
// interior form (no clamp can trigger): same ops, same order
__device__ __forceinline__ float sec_fast(float lo2, float c, float hi2) {
  const float dp = __fmul_rn(0.5f, __fsub_rn(hi2, c));
  const float dm = __fmul_rn(0.5f, __fsub_rn(c, lo2));
  return __fmul_rn(0.5f, __fsub_rn(dp, dm));
}

__device__ __forceinline__ float comp(const float4& v, int c) {
  return c == 0 ? v.x : (c == 1 ? v.y : (c == 2 ? v.z : v.w));
}

template <int RY, int W>
__global__ void __launch_bounds__(32 * W, HB_LOG_MINB) k_log_stream(const LogArgs a) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int x0 = blockIdx.x * LX;
  const int xl = x0 + 4 * lane;
  const int y0 = (blockIdx.y * W + warp) * RY;
  if (y0 >= a.ny) return;
  const int oz0 = blockIdx.z * a.zchunk;
  const int oz1 = min(oz0 + a.zchunk, a.nzo);
  if (oz0 >= oz1) return;
  const int nx = a.nx, ny = a.ny, nz = a.nz;
  const bool act = xl < nx;
  const int xc = act ? xl : nx - 4;
  const bool clamp_right = xl + 4 >= nx;
  const bool edge_lane = lane == 0 || lane == 31;
  const int e0 = lane == 0 ? max(x0 - 2, 0) : min(x0 + LX, nx - 1);
  const int e1 = lane == 0 ? max(x0 - 1, 0) : min(x0 + LX + 1, nx - 1);
  const bool x_face = xl < 2 || xl + 4 > nx - 2;  // some column of this lane is within 2 of an x face
  const bool y_face = y0 < 2 || y0 + RY > ny - 2;
  const int64_t plane = (int64_t)ny * nx;
  int crow[RY], hrow[4];
#pragma unroll
  for (int r = 0; r < RY; ++r) crow[r] = min(y0 + r, ny - 1) * nx;
  hrow[0] = max(y0 - 2, 0) * nx;
  hrow[1] = max(y0 - 1, 0) * nx;
  hrow[2] = min(y0 + RY, ny - 1) * nx;
  hrow[3] = min(y0 + RY + 1, ny - 1) * nx;
  auto slice = [&](int64_t zb) {  // g slice of block slice clamp(zb)
    const int64_t zc = zb < 0 ? 0 : (zb > nz - 1 ? nz - 1 : zb);
    return a.g + (zc - a.gz0) * plane;
  };
  auto load_centre = [&](int64_t zb, float4 (&c)[RY]) {
    const float* p = slice(zb);
#pragma unroll
    for (int r = 0; r < RY; ++r) c[r] = __ldg(reinterpret_cast<const float4*>(p + crow[r] + xc));
  };

  // ring[k] = centre rows of block slice z - 2 + k (k = 0..4); slice z + 3 is
  // loaded a full step ahead into nxt, then the ring rotates by moves.  The y
  // halo rows of slice z (other warps' centre rows: L1/L2 hits) and the strip's
  // edge columns are loaded a step ahead as well.
  float4 ring[5][RY];
  const int64_t zb0 = a.zo + oz0;
#pragma unroll
  for (int k = 0; k < 5; ++k) load_centre(zb0 - 2 + k, ring[k]);
  float* dst = a.out + (int64_t)oz0 * plane + (int64_t)y0 * nx + xl;
  auto load_halo = [&](int64_t zb, float4 (&h)[4], float (&e)[RY][2]) {
    const float* p = slice(zb);
#pragma unroll
    for (int k = 0; k < 4; ++k) h[k] = __ldg(reinterpret_cast<const float4*>(p + hrow[k] + xc));
    if (edge_lane) {
#pragma unroll
      for (int r = 0; r < RY; ++r) {
        e[r][0] = __ldg(p + crow[r] + e0);
        e[r][1] = __ldg(p + crow[r] + e1);
      }
    }
  };
  float4 hal_n[4];
  float el_n[RY][2] = {};
  load_halo(zb0, hal_n, el_n);

#pragma unroll 1
  for (int o = oz0; o < oz1; ++o) {
    const int64_t z = a.zo + o;
    float4 nxt[RY];
    float4 hal[4];
    float el[RY][2];
#pragma unroll
    for (int k = 0; k < 4; ++k) hal[k] = hal_n[k];
#pragma unroll
    for (int r = 0; r < RY; ++r) el[r][0] = el_n[r][0], el[r][1] = el_n[r][1];
    if (o + 1 < oz1) {
      load_centre(z + 3, nxt);
      load_halo(z + 1, hal_n, el_n);  // the next step's halo, a step ahead
    }
    const bool z_face = z < 2 || z > nz - 3;
    float res[RY][4];
    // ---- zz
#pragma unroll
    for (int r = 0; r < RY; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c)
        res[r][c] = sec_fast(comp(ring[0][r], c), comp(ring[2][r], c), comp(ring[4][r], c));
    if (z_face) {
#pragma unroll
      for (int r = 0; r < RY; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c)
          res[r][c] = sec_general(comp(ring[0][r], c), comp(ring[1][r], c), comp(ring[2][r], c),
                                  comp(ring[3][r], c), comp(ring[4][r], c), (int)z, nz);
    }
    // ---- xx (added first: out = (xx + yy) + zz)
    float xxv[RY][4];
#pragma unroll
    for (int r = 0; r < RY; ++r) {
      const float4 v = ring[2][r];
      const float sl2 = __shfl_up_sync(0xffffffffu, v.z, 1);
      const float sl1 = __shfl_up_sync(0xffffffffu, v.w, 1);
      const float sr1 = __shfl_down_sync(0xffffffffu, v.x, 1);
      const float sr2 = __shfl_down_sync(0xffffffffu, v.y, 1);
      const float l2 = lane == 0 ? el[r][0] : sl2;
      const float l1 = lane == 0 ? el[r][1] : sl1;
      const float r1 = lane == 31 ? el[r][0] : (clamp_right ? v.w : sr1);
      const float r2 = lane == 31 ? el[r][1] : (clamp_right ? v.w : sr2);
      xxv[r][0] = sec_fast(l2, v.x, v.z);
      xxv[r][1] = sec_fast(l1, v.y, v.w);
      xxv[r][2] = sec_fast(v.x, v.z, r1);
      xxv[r][3] = sec_fast(v.y, v.w, r2);
      if (x_face && act) {  // inactive lanes (xl >= nx) would index past the window
        const float xw[8] = {l2, l1, v.x, v.y, v.z, v.w, r1, r2};
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int x = xl + c;
          if (x < 2 || x > nx - 3)
            xxv[r][c] = sec_general(xw[c], xw[c + 1], xw[c + 2], xw[c + 3], xw[c + 4], x, nx);
        }
      }
    }
    // ---- yy and the sum
#pragma unroll
    for (int r = 0; r < RY; ++r) {
      const float4 ym2 = r >= 2 ? ring[2][r - 2] : hal[r];
      const float4 yp2 = r + 2 < RY ? ring[2][r + 2] : hal[r + 4 - RY];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const float yy = sec_fast(comp(ym2, c), comp(ring[2][r], c), comp(yp2, c));
        res[r][c] = __fadd_rn(__fadd_rn(xxv[r][c], yy), res[r][c]);
      }
    }
    if (y_face) {
#pragma unroll
      for (int r = 0; r < RY; ++r) {
        const int y = y0 + r;
        if (y < 2 || y > ny - 3) {
          float4 wr[5];
#pragma unroll
          for (int k = 0; k < 5; ++k) {
            const int rr = r - 2 + k;  // row within [-2, RY+1]
            wr[k] = rr < 0 ? hal[rr + 2] : (rr >= RY ? hal[rr - RY + 2] : ring[2][rr]);
          }
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            // recompute the whole sum with the clamped yy (same op order)
            const float yy = sec_general(comp(wr[0], c), comp(wr[1], c), comp(wr[2], c),
                                         comp(wr[3], c), comp(wr[4], c), y, ny);
            float zz = sec_fast(comp(ring[0][r], c), comp(ring[2][r], c), comp(ring[4][r], c));
            if (z_face)
              zz = sec_general(comp(ring[0][r], c), comp(ring[1][r], c), comp(ring[2][r], c),
                               comp(ring[3][r], c), comp(ring[4][r], c), (int)z, nz);
            res[r][c] = __fadd_rn(__fadd_rn(xxv[r][c], yy), zz);
          }
        }
      }
    }
#pragma unroll
    for (int r = 0; r < RY; ++r)
      if (act && y0 + r < ny)
        __stcs(reinterpret_cast<float4*>(dst + r * nx),
               make_float4(res[r][0], res[r][1], res[r][2], res[r][3]));
    dst += plane;
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int r = 0; r < RY; ++r) ring[k][r] = ring[k + 1][r];
#pragma unroll
    for (int r = 0; r < RY; ++r) ring[4][r] = nxt[r];
  }
}

template <int RY, int W>
cudaError_t launch_log(const LogArgs& a0, cudaStream_t s) {
  LogArgs a = a0;
  auto kern = k_log_stream<RY, W>;
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * W, 0) != cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
  int dev = 0, nsm = kNumSMs;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int gx = (a.nx + LX - 1) / LX;
  const int gy = (a.ny + RY * W - 1) / (RY * W);
  const int64_t tiles = (int64_t)gx * gy, slots = (int64_t)nsm * per_sm;
  double best = 1e300;
  int64_t best_zc = a.nzo;
  for (int split = 1; split <= 512; ++split) {
    const int64_t zc = (a.nzo + split - 1) / split;
    if (split > 1 && zc < 16) break;
    const int64_t ctas = tiles * ((a.nzo + zc - 1) / zc);
    const int64_t waves = (ctas + slots - 1) / slots;
    const double cost = (double)waves * (double)(zc + 4);
    if (cost < best * 0.98) {
      best = cost;
      best_zc = zc;
    }
  }
  a.zchunk = (int)best_zc;
  dim3 grid(gx, gy, (unsigned)((a.nzo + best_zc - 1) / best_zc));
  kern<<<grid, 32 * W, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace

cudaError_t log_diff_stream(const float* g, int64_t gz0, int64_t nz, int64_t ny, int64_t nx,
                            int64_t zo, int64_t nzo, float* out, cudaStream_t s,
                            int64_t* launches) {
  if (nzo <= 0) return cudaSuccess;
  if (nx < 4 || nx % 4 != 0 || ny * nx >= (1ll << 31) || nz >= (1ll << 30)) return cudaErrorNotSupported;
  if ((reinterpret_cast<uintptr_t>(g) % 16) != 0 || (reinterpret_cast<uintptr_t>(out) % 16) != 0)
    return cudaErrorNotSupported;
  LogArgs a;
  a.g = g;
  a.gz0 = gz0;
  a.nz = (int)nz;
  a.ny = (int)ny;
  a.nx = (int)nx;
  a.zo = zo;
  a.nzo = (int)nzo;
  a.out = out;
  cudaError_t e = std::getenv("HB_LOG_RY4") ? launch_log<4, 4>(a, s) : launch_log<2, 4>(a, s);
  if (e == cudaSuccess && launches) *launches += 1;
  return e;
}

}  // namespace hb
