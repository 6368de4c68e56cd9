// gauss_small.cu — fast (fp32) Gaussian for small XY planes (BASELINE
// configs[0]: sigma = 2 on 256^3, the reference's CPU-runnable case), float
// input, R in {2, 4, 6, 8} (filters.py:33-41).
//
// The z-streaming kernels (k_gauss_tri, k_gauss_ws) need many XY tiles to
// fill 148 SMs; a 256^2 plane has 48-64, so they split z into short chunks
// that each pay 2R priming slices and still run one partial wave (256^3:
// 146-159 Gvox/s, 18-19% of HBM).  Here the passes are split instead, so
// every kernel has plenty of independent work:
//   k_fast_z2 : Z pass, TMA 64x8 slice tiles in an 8-deep ring, a thread owns
//               two x-adjacent columns (one FFMA2 lane pair) with a (2R+1)-slot
//               register window -> tmp (stays mostly in the 126 MB L2);
//   k_fast_yx : one 48x32 output tile of one slice per CTA: TMA box from tmp,
//               Y pass on column pairs x 8 rows (LDS.64, FFMA2) into a
//               row-pair-interleaved tile, X pass on row pairs x 6 columns
//               (LDS.128, FFMA2), STG.64 — the Y/X roles of k_gauss_tri
//               without the z ring.
// Pass order Z, Y, X (the reference's); fp32 rounding ~2e-7 (tests: 1e-5).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "ops.cuh"
#include "tma.cuh"

namespace hb {
namespace {

typedef unsigned long long f2;
__device__ __forceinline__ f2 pk(float lo, float hi) {
  f2 d;
  asm("mov.b64 %0, {%1, %2};" : "=l"(d) : "f"(lo), "f"(hi));
  return d;
}
__device__ __forceinline__ void upk(f2 v, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ f2 add2(f2 a, f2 b) {
  f2 d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ f2 mul2(f2 a, f2 b) {
  f2 d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) {
  f2 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

struct SmallArgs {
  f2 w2[17];  // (w_k, w_k)
  int nzi, ny, nx, zo, nzo, zchunk;
};

// symmetric fold of a (2R+1)-window held in f2 slots v(k), k = 0..2R
template <int R, typename F>
__device__ __forceinline__ f2 fold2(F v, const f2* w) {
  f2 e = mul2(v(R), w[R]);
  f2 f = mul2(add2(v(R - 1), v(R + 1)), w[R - 1]);
#pragma unroll
  for (int d = 2; d <= R; ++d) {
    const f2 t = add2(v(R - d), v(R + d));
    if (d % 2 == 0) e = fma2(t, w[R - d], e);
    else f = fma2(t, w[R - d], f);
  }
  return add2(e, f);
}

// ---- Z pass ------------------------------------------------------------------
constexpr int SZ_TX = 64, SZ_TY = 8, SZ_NT = 256, SZ_NST = 8;

template <int R>
__global__ void __launch_bounds__(SZ_NT)
k_fast_z2(const __grid_constant__ CUtensorMap tin, float* __restrict__ tmp, const __grid_constant__ SmallArgs a) {
  constexpr int W = 2 * R + 1;
  __shared__ __align__(128) float stg[SZ_NST][SZ_TY][SZ_TX];
  __shared__ __align__(8) uint64_t bar[SZ_NST];
  const int tid = threadIdx.x, lane = tid & 31, ty = tid >> 5;
  const int x0 = blockIdx.x * SZ_TX, y0 = blockIdx.y * SZ_TY;
  const int zs = blockIdx.z * a.zchunk, ze = min(zs + a.zchunk, a.nzo);
  const int nsl = ze - zs + 2 * R;
  auto zin = [&](int i) { return min(max(a.zo + zs - R + i, 0), a.nzi - 1); };
  constexpr uint32_t BYTES = SZ_TX * SZ_TY * 4;
  if (tid == 0) {
    prefetch_tmap(&tin);
#pragma unroll
    for (int i = 0; i < SZ_NST; ++i) mbar_init(&bar[i], 1);
    fence_mbar_init();
    for (int i = 0; i < SZ_NST && i < nsl; ++i) {
      mbar_expect_tx(&bar[i], BYTES);
      tma_load_3d(&stg[i][0][0], &tin, x0, y0, zin(i), &bar[i]);
    }
  }
  __syncthreads();
  const int gx = x0 + 2 * lane, gy = y0 + ty;
  const bool ok = gy < a.ny && gx < a.nx;  // nx even: gx + 1 < nx too
  const int64_t plane = (int64_t)a.ny * a.nx;
  float* optr = tmp + (int64_t)zs * plane + (int64_t)min(gy, a.ny - 1) * a.nx + min(gx, a.nx - 2);
  f2 ring[W];
  for (int i0 = 0; i0 < nsl; i0 += W) {
#pragma unroll
    for (int u = 0; u < W; ++u) {
      const int i = i0 + u;
      if (i < nsl) {
        const int st = i & (SZ_NST - 1);
        mbar_wait(&bar[st], (uint32_t)((i / SZ_NST) & 1));
        const float2 p = *reinterpret_cast<const float2*>(&stg[st][ty][2 * lane]);
        __syncthreads();  // every thread has read stage st
        if (tid == 0 && i + SZ_NST < nsl) {
          fence_proxy_async();
          mbar_expect_tx(&bar[st], BYTES);
          tma_load_3d(&stg[st][0][0], &tin, x0, y0, zin(i + SZ_NST), &bar[st]);
        }
        ring[u] = pk(p.x, p.y);  // slot u holds slice i (i0 is a multiple of W)
        if (i >= 2 * R) {
          // window position k = slice i - 2R + k -> slot (u + 1 + k) % W
          const f2 r = fold2<R>([&](int k) { return ring[(u + 1 + k) % W]; }, a.w2);
          float r0, r1;
          upk(r, r0, r1);
          if (ok) *reinterpret_cast<float2*>(optr + (int64_t)(i - 2 * R) * plane) = make_float2(r0, r1);
        }
      }
    }
  }
  // let the Y/X pass's CTAs be scheduled once every Z CTA got here (they
  // still wait for this grid's completion before reading tmp)
  asm volatile("griddepcontrol.launch_dependents;");
}

// ---- Y + X pass of one slice tile ------------------------------------------------
constexpr int SY_TX = 48, SY_TY = 32, SY_NT = 128, SY_YR = 8, SY_XC = 6;

template <int R>
struct SGeo {
  static constexpr int NYC = SY_TX + 2 * R;   // columns the y pass produces
  static constexpr int NYP = NYC / 2;
  static constexpr int HB = SY_TY + 2 * R;
  static constexpr int XA = (R + 3) / 4 * 4;  // 16-B aligned TMA start
  static constexpr int XOFF = XA - R;
  static constexpr int WBOX = (XOFF + NYC + 3) / 4 * 4;
  static constexpr int SYP = (2 * NYC + 31) / 32 * 32;  // floats per row pair
  static constexpr int OFF_SY = (HB * WBOX * 4 + 127) / 128 * 128;
  static constexpr int OFF_BAR = OFF_SY + (SY_TY / 2) * SYP * 4;
  static constexpr int SMEM = OFF_BAR + 16 + 128;
  static constexpr int NYI = NYP * (SY_TY / SY_YR);
  static_assert(R % 2 == 0, "even R only");
  static_assert(NYI <= SY_NT, "y items exceed the CTA");
  static_assert((SY_TY / 2) * (SY_TX / SY_XC) == SY_NT, "x items fill the CTA");
};

template <int R>
__global__ void __launch_bounds__(SY_NT)
k_fast_yx(const __grid_constant__ CUtensorMap tm, float* __restrict__ out, const __grid_constant__ SmallArgs a) {
  using G = SGeo<R>;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  float* sIn = reinterpret_cast<float*>(smem);
  float* sY = reinterpret_cast<float*>(smem + G::OFF_SY);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + G::OFF_BAR);
  const int tid = threadIdx.x;
  const int x0 = blockIdx.x * SY_TX, y0 = blockIdx.y * SY_TY, z = blockIdx.z;
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
    prefetch_tmap(&tm);
    // programmatic dependent launch: everything above overlaps the Z pass's
    // tail; tmp is read only after the Z grid has completed (no-op when the
    // kernel is launched without the PDL attribute)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    mbar_expect_tx(bar, G::HB * G::WBOX * 4);
    tma_load_3d(sIn, &tm, x0 - G::XA, y0 - R, z, bar);
  }
  __syncthreads();
  mbar_wait(bar, 0);
  if ((x0 - R < 0) || (x0 + G::NYC - R > a.nx) || (y0 - R < 0) || (y0 + SY_TY + R > a.ny)) {
    clamp_tile<float, SY_NT>(sIn + G::XOFF, G::WBOX, G::HB, G::NYC, y0 - R, x0 - R, a.ny, a.nx, tid);
    __syncthreads();
  }
  // Y pass: column pair ycp x 8 rows, stored row-pair interleaved
  if (tid < G::NYI) {
    const int ycp = tid % G::NYP, yg = tid / G::NYP;
    const float* src = sIn + (SY_YR * yg) * G::WBOX + G::XOFF + 2 * ycp;
    f2 acc[SY_YR];
#pragma unroll
    for (int j = 0; j < SY_YR + 2 * R; ++j) {
      const f2 v = *reinterpret_cast<const f2*>(src + j * G::WBOX);
#pragma unroll
      for (int m = 0; m < SY_YR; ++m) {
        const int k = j - m;
        if (k == 0) acc[m] = mul2(v, a.w2[0]);
        else if (k > 0 && k <= 2 * R) acc[m] = fma2(v, a.w2[k], acc[m]);
      }
    }
    float* dst = sY + (SY_YR / 2 * yg) * G::SYP + 4 * ycp;
#pragma unroll
    for (int q = 0; q < SY_YR / 2; ++q) {
      float r0a, r0b, r1a, r1b;
      upk(acc[2 * q], r0a, r0b);
      upk(acc[2 * q + 1], r1a, r1b);
      *reinterpret_cast<float4*>(dst + q * G::SYP) = make_float4(r0a, r1a, r0b, r1b);
    }
  }
  __syncthreads();
  // X pass: row pair rp x 6 columns
  const int rp = tid / (SY_TX / SY_XC), g = tid % (SY_TX / SY_XC);
  const float* srow = sY + rp * G::SYP + 2 * SY_XC * g;
  constexpr int NXP = SY_XC + 2 * R;
  f2 v[NXP];
#pragma unroll
  for (int i = 0; i < NXP / 2; ++i) {
    const float4 q = *reinterpret_cast<const float4*>(srow + 4 * i);
    v[2 * i] = pk(q.x, q.y);
    v[2 * i + 1] = pk(q.z, q.w);
  }
  float r0[SY_XC], r1[SY_XC];
#pragma unroll
  for (int j = 0; j < SY_XC; ++j) {
    const f2 o = fold2<R>([&](int k) { return v[j + k]; }, a.w2);
    upk(o, r0[j], r1[j]);  // rows 2rp, 2rp + 1 of column 6g + j
  }
  const int gy = y0 + 2 * rp, gx = x0 + SY_XC * g;
  const int64_t plane = (int64_t)a.ny * a.nx;
  float* p0 = out + (int64_t)z * plane + (int64_t)gy * a.nx + gx;
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    if (gy + t >= a.ny) break;
    float* p = p0 + (int64_t)t * a.nx;
    const float* r = t ? r1 : r0;
    if (gx + SY_XC <= a.nx) {
#pragma unroll
      for (int j = 0; j < SY_XC; j += 2) *reinterpret_cast<float2*>(p + j) = make_float2(r[j], r[j + 1]);
    } else {
#pragma unroll
      for (int j = 0; j < SY_XC; ++j)
        if (gx + j < a.nx) p[j] = r[j];
    }
  }
}

template <int R>
cudaError_t launch_small(const DevIn& in, int64_t zo, int64_t nzo, float* out, const Taps& taps,
                         float* tmp, cudaStream_t s) {
  using G = SGeo<R>;
  SmallArgs a;
  for (int k = 0; k < 2 * R + 1; ++k) {
    unsigned int bits = 0;
    std::memcpy(&bits, &taps.w[k], 4);
    a.w2[k] = ((unsigned long long)bits << 32) | bits;
  }
  a.nzi = (int)in.nz;
  a.ny = (int)in.ny;
  a.nx = (int)in.nx;
  a.zo = (int)zo;
  a.nzo = (int)nzo;
  CUtensorMap tz, tm;
  if (!make_tmap_3d(&tz, in.p, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, in.nx, in.ny, in.nz, SZ_TX, SZ_TY))
    return cudaErrorNotSupported;
  if (!make_tmap_3d(&tm, tmp, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, in.nx, in.ny, nzo, G::WBOX, G::HB))
    return cudaErrorNotSupported;
  // Z pass: enough column chunks for ~4 waves of 2-3 CTAs per SM (a
  // direct-load variant without the per-slice CTA barrier measured slower:
  // 50 vs 33 us at 256^3 — too few independent columns to hide the loads)
  const int gx = (int)((in.nx + SZ_TX - 1) / SZ_TX), gy = (int)((in.ny + SZ_TY - 1) / SZ_TY);
  const int64_t tiles = (int64_t)gx * gy, slots = 3 * (int64_t)kNumSMs;
  double best = 1e300;
  int64_t best_zc = nzo;
  for (int split = 1; split <= 512; ++split) {
    const int64_t zc = (nzo + split - 1) / split;
    if (split > 1 && zc < 2 * R + 8) break;
    const int64_t ctas = tiles * ((nzo + zc - 1) / zc);
    const double cost = (double)((ctas + slots - 1) / slots) * (double)(zc + 2 * R);
    if (cost < best * 0.98) {
      best = cost;
      best_zc = zc;
    }
  }
  a.zchunk = (int)best_zc;
  const dim3 gz(gx, gy, (unsigned)((nzo + best_zc - 1) / best_zc));
  // (one TMA pipeline per warp — 64-float row boxes, no CTA barrier per
  // slice — measured 80-82 vs 78 us at 256^3: the small boxes cost more than
  // the barrier)
  k_fast_z2<R><<<gz, SZ_NT, 0, s>>>(tz, tmp, a);
  auto k = k_fast_yx<R>;
  if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM) != cudaSuccess)
    return cudaErrorNotSupported;
  for (int64_t zb = 0; zb < nzo; zb += 65535) {
    const int nzb = (int)std::min<int64_t>(65535, nzo - zb);
    dim3 grid((unsigned)((in.nx + SY_TX - 1) / SY_TX), (unsigned)((in.ny + SY_TY - 1) / SY_TY), (unsigned)nzb);
    // (the tensor map addresses tmp's slices from 0; offset the batch by
    // shifting the output pointer and using a map over the batch's slices)
    if (zb == 0) {
      if (!std::getenv("HB_SMALL_NO_PDL")) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = grid;
        cfg.blockDim = dim3(SY_NT);
        cfg.dynamicSmemBytes = G::SMEM;
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        const cudaError_t e = cudaLaunchKernelEx(&cfg, k, tm, out, a);
        if (e != cudaSuccess) return e;
      } else {
        k<<<grid, SY_NT, G::SMEM, s>>>(tm, out, a);
      }
    } else {
      CUtensorMap tb;
      if (!make_tmap_3d(&tb, tmp + zb * in.ny * in.nx, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, in.nx, in.ny,
                        nzo - zb, G::WBOX, G::HB))
        return cudaErrorNotSupported;
      k<<<grid, SY_NT, G::SMEM, s>>>(tb, out + zb * in.ny * in.nx, a);
    }
  }
  return cudaGetLastError();
}

}  // namespace

// Planes too small for the z-streaming kernels (nx or ny < 384), fast mode,
// float input, plain gaussian (no epilogue), even R <= 8, even nx.
// `tmp`: nzo * ny * nx floats.  NotSupported outside that envelope.
cudaError_t gaussian_small(const DevIn& in, int64_t zo, int64_t nzo, float* out, const Taps& taps,
                           const EpiArgs& epi, float* tmp, cudaStream_t s, int64_t* launches) {
  if (std::getenv("HB_GAUSS_NOSMALL") || in.dt != HB_F32 || epi.kind != EPI_NONE || nzo <= 0 ||
      taps.R < 2 || taps.R > 8 || (taps.R & 1) || in.nx % 4 != 0 || in.nx < 16 || in.ny < 16 ||
      (in.nx >= 384 && in.ny >= 384) || in.nz >= (1 << 30) || (int64_t)in.ny * in.nx >= ((int64_t)1 << 31) ||
      tmp == nullptr)
    return cudaErrorNotSupported;
  cudaError_t e = cudaErrorNotSupported;
  switch (taps.R) {
    case 2: e = launch_small<2>(in, zo, nzo, out, taps, tmp, s); break;
    case 4: e = launch_small<4>(in, zo, nzo, out, taps, tmp, s); break;
    case 6: e = launch_small<6>(in, zo, nzo, out, taps, tmp, s); break;
    case 8: e = launch_small<8>(in, zo, nzo, out, taps, tmp, s); break;
  }
  if (e == cudaSuccess && launches) *launches += 2;
  return e;
}

}  // namespace hb
