// gauss_exact.cu — bit-exact 3D Gaussian (precision="exact"), the smoothing
// stage of LoG (filters.py:246-264) and exact unsharp.
//
// Reproduces scipy's NI_Correlate1D at filters.py:40 pass by pass: axis order
// Z, Y, X; every pass evaluates in f64 with the symmetric fold
//     acc = x0*w0;  for d = R..1:  acc = acc + (x[-d] + x[+d]) * w[d]
// using separately rounded __dadd_rn/__dmul_rn (no FMA contraction), and rounds
// to float32 between passes.  Two kernels instead of three passes:
//   k_exact_z  : Z pass; one thread per (y, x) column marching z with a
//                (2R+1)-deep f64 register window (static slots) -> f32 tmp
//   k_exact_yx : Y then X pass of one slice tile (TMA load, f64 math, f32
//                rounding between the passes) -> output (+ unsharp epilogue)
// HBM: 16 B/voxel (f32 in/out twice); FP64 (64 ops/clk/SM) bounds it at
// ~81 DP ops/voxel for R = 8.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <type_traits>

#include "ops.cuh"
#include "tma.cuh"

namespace hb {
namespace {

struct ExactArgs {
  double w[kMaxTaps];  // f32 taps promoted to f64 (np.asarray(weights, float64))
  int R;
};

template <typename T>
__device__ __forceinline__ double ldd(const T* p) {
  return (double)(float)__ldg(p);  // the reference casts to float32 first (filters.py:38)
}

// fold for one output: window v[0..2R], centre v[R]
template <int R>
__device__ __forceinline__ float fold(const double (&v)[2 * R + 1], const double* w) {
  double acc = __dmul_rn(v[R], w[R]);
#pragma unroll
  for (int d = R; d >= 1; --d) acc = __dadd_rn(acc, __dmul_rn(__dadd_rn(v[R - d], v[R + d]), w[R - d]));
  return (float)acc;
}

// ---- Z pass ----------------------------------------------------------------
constexpr int EZ_T = 128;

template <int R, typename T>
__global__ void __launch_bounds__(EZ_T)
k_exact_z(const T* __restrict__ in, int64_t nz, int64_t plane, int64_t zo, int64_t nzo,
          int zchunk, float* __restrict__ out, const ExactArgs a) {
  constexpr int W = 2 * R + 1;
  const int64_t col = (int64_t)blockIdx.x * EZ_T + threadIdx.x;
  if (col >= plane) return;
  const int64_t z0 = (int64_t)blockIdx.y * zchunk;
  const int64_t z1 = min(z0 + (int64_t)zchunk, nzo);
  const T* src = in + col;
  const double* wv = a.w;
  // window of input slices (block z) zo+z-R .. zo+z+R for output z
  double v[W];
#pragma unroll
  for (int k = 0; k < W - 1; ++k) v[k] = ldd(src + clamp64(zo + z0 - R + k, 0, nz - 1) * plane);
  int64_t z = z0;
  while (z < z1) {
#pragma unroll
    for (int u = 0; u < W; ++u) {
      if (z < z1) {
        // slot layout: v[(u + k) % W] holds window position k; the newest
        // sample (position 2R) goes to slot (u + 2R) % W
        v[(u + W - 1) % W] = ldd(src + clamp64(zo + z + R, 0, nz - 1) * plane);
        double win[W];
#pragma unroll
        for (int k = 0; k < W; ++k) win[k] = v[(u + k) % W];
        out[(z - z0 + z0) * plane + col] = fold<R>(win, wv);
        ++z;
      }
    }
  }
}

// ---- Z pass, TMA-staged (the fast path) ---------------------------------------
// A CTA owns a 64 x 8 column tile and marches a z-chunk; TMA streams one slice
// tile per stage through an 8-deep smem ring (loads run 8 slices ahead, so the
// f64 fold never waits on memory: k_exact_z's one-load-per-step dependency
// left it latency-bound at 36% FP64 busy).  A thread owns two x-adjacent
// columns (one LDS.64 per slice) and keeps their (2R+1)-deep f64 windows in
// registers with static slots (loop unrolled by 2R+1).
constexpr int Z2_TX = 64, Z2_TY = 8, Z2_NT = 256, Z2_NST = 8;

template <typename T> struct ExTma;
template <> struct ExTma<float> { static constexpr CUtensorMapDataType v = CU_TENSOR_MAP_DATA_TYPE_FLOAT32; };
template <> struct ExTma<uint16_t> { static constexpr CUtensorMapDataType v = CU_TENSOR_MAP_DATA_TYPE_UINT16; };
template <> struct ExTma<uint8_t> { static constexpr CUtensorMapDataType v = CU_TENSOR_MAP_DATA_TYPE_UINT8; };

struct Z2Args {
  int nz, ny, nx;  // input block
  int zo, nzo, zchunk;
};

template <int R, typename T>
__global__ void __launch_bounds__(Z2_NT, 2)
k_exact_z2(const __grid_constant__ CUtensorMap tin, float* __restrict__ out, const ExactArgs a,
           const Z2Args b) {
  constexpr int W = 2 * R + 1;
  __shared__ __align__(128) T stg[Z2_NST][Z2_TY][Z2_TX];
  __shared__ __align__(8) uint64_t bar[Z2_NST];
  const int tid = threadIdx.x, lane = tid & 31, ty = tid >> 5;
  const int x0 = blockIdx.x * Z2_TX, y0 = blockIdx.y * Z2_TY;
  const int zs = blockIdx.z * b.zchunk, ze = min(zs + b.zchunk, b.nzo);
  const int nsl = ze - zs + 2 * R;
  auto zin = [&](int i) { return min(max(b.zo + zs - R + i, 0), b.nz - 1); };
  constexpr uint32_t BYTES = Z2_TX * Z2_TY * sizeof(T);
  if (tid == 0) {
    prefetch_tmap(&tin);
#pragma unroll
    for (int i = 0; i < Z2_NST; ++i) mbar_init(&bar[i], 1);
    fence_mbar_init();
    for (int i = 0; i < Z2_NST && i < nsl; ++i) {
      mbar_expect_tx(&bar[i], BYTES);
      tma_load_3d(&stg[i][0][0], &tin, x0, y0, zin(i), &bar[i]);
    }
  }
  __syncthreads();
  const int gx = x0 + 2 * lane, gy = y0 + ty;
  const bool ok = gy < b.ny && gx < b.nx;  // nx is even here, so gx + 1 < nx too
  const int64_t oplane = (int64_t)b.ny * b.nx;
  float* optr = out + ((int64_t)zs * b.ny + min(gy, b.ny - 1)) * b.nx + min(gx, b.nx - 2);
  const double* wv = a.w;
  double v0[W], v1[W];
  for (int i0 = 0; i0 < nsl; i0 += W) {
#pragma unroll
    for (int u = 0; u < W; ++u) {
      const int i = i0 + u;
      if (i < nsl) {
        const int st = i & (Z2_NST - 1);
        mbar_wait(&bar[st], (uint32_t)((i / Z2_NST) & 1));
        const T p0 = stg[st][ty][2 * lane], p1 = stg[st][ty][2 * lane + 1];
        __syncthreads();  // every thread has read stage st
        if (tid == 0 && i + Z2_NST < nsl) {
          fence_proxy_async();
          mbar_expect_tx(&bar[st], BYTES);
          tma_load_3d(&stg[st][0][0], &tin, x0, y0, zin(i + Z2_NST), &bar[st]);
        }
        // slot u holds slice i (i0 is a multiple of W); the reference casts to f32 first
        v0[u] = (double)(float)p0;
        v1[u] = (double)(float)p1;
        if (i >= 2 * R) {
          double w0[W], w1[W];
#pragma unroll
          for (int k = 0; k < W; ++k) {  // window position k = slice i - 2R + k
            w0[k] = v0[(u + 1 + k) % W];
            w1[k] = v1[(u + 1 + k) % W];
          }
          const float r0 = fold<R>(w0, wv), r1 = fold<R>(w1, wv);
          if (ok) *reinterpret_cast<float2*>(optr + (int64_t)(i - 2 * R) * oplane) = make_float2(r0, r1);
        }
      }
    }
  }
}

// ---- fused Y + X pass of one slice tile --------------------------------------
// 320 threads: the Y pass has (64 + 2R) x 4 = 320 items for R = 8, one per
// thread (256 threads ran two rounds for 64 of them); the X pass uses 256
constexpr int EY_TX = 64, EY_TY = 32, EY_NT = 320;

template <int R>
struct EGeo {
  static constexpr int XA = (R + 3) / 4 * 4;  // 16-B aligned TMA x start
  static constexpr int WC = EY_TX + 2 * R;
  static constexpr int HB = EY_TY + 2 * R;
  static constexpr int WBOX = (XA + EY_TX + R + 3) / 4 * 4;
  static constexpr int XOFF = XA - R;
  static constexpr int SY = WC + 1;  // sY pitch (floats)
  static constexpr int SMEM = HB * WBOX * 4 + EY_TY * SY * 4 + 16 + 128;
};

struct YXArgs {
  int ny, nx, nz;    // slices of tmp / out
  const void* orig;  // unsharp: original block input (any dtype) or null
  int orig_dt;
  int64_t orig_zo;   // block z of tmp slice 0
  float amount;
  int zbase;         // first slice of this launch (gridDim.z <= 65535)
};

template <int R, bool UNSHARP, typename To>
__global__ void __launch_bounds__(EY_NT)
k_exact_yx(const __grid_constant__ CUtensorMap tm, float* __restrict__ out, const ExactArgs a,
           const YXArgs b) {
  using G = EGeo<R>;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem =
      smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u)  /* stays in .shared */;
  float* sIn = reinterpret_cast<float*>(smem);
  float* sY = sIn + G::HB * G::WBOX;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sY + EY_TY * G::SY + ((EY_TY * G::SY) & 1));
  const int tid = threadIdx.x;
  const int x0 = blockIdx.x * EY_TX, y0 = blockIdx.y * EY_TY, z = blockIdx.z + b.zbase;
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
    mbar_expect_tx(bar, G::HB * G::WBOX * 4);
    tma_load_3d(sIn, &tm, x0 - G::XA, y0 - R, z, bar);
  }
  const double* wv = a.w;
  __syncthreads();
  mbar_wait(bar, 0);
  if ((x0 - R < 0) || (x0 + EY_TX + R > b.nx) || (y0 - R < 0) || (y0 + EY_TY + R > b.ny)) {
    clamp_tile<float, EY_NT>(sIn + G::XOFF, G::WBOX, G::HB, G::WC, y0 - R, x0 - R, b.ny, b.nx, tid);
    __syncthreads();
  }
  // Y pass: column c, 8 rows per item
  for (int item = tid; item < G::WC * (EY_TY / 8); item += EY_NT) {
    const int c = item % G::WC, g = item / G::WC;
    double v[8 + 2 * R];
#pragma unroll
    for (int j = 0; j < 8 + 2 * R; ++j) v[j] = (double)sIn[(8 * g + j) * G::WBOX + G::XOFF + c];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      double win[2 * R + 1];
#pragma unroll
      for (int k = 0; k < 2 * R + 1; ++k) win[k] = v[j + k];
      sY[(8 * g + j) * G::SY + c] = fold<R>(win, wv);
    }
  }
  __syncthreads();
  // X pass: row r, 8 outputs per thread
  if (tid >= 256) return;
  const int r = tid >> 3, xs = (tid & 7) * 8;
  double v[8 + 2 * R];
#pragma unroll
  for (int j = 0; j < 8 + 2 * R; ++j) v[j] = (double)sY[r * G::SY + xs + j];
  const int gy = y0 + r;
  if (gy >= b.ny) return;
  float res[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    double win[2 * R + 1];
#pragma unroll
    for (int k = 0; k < 2 * R + 1; ++k) win[k] = v[j + k];
    res[j] = fold<R>(win, wv);
  }
  const int64_t rowoff = ((int64_t)z * b.ny + gy) * (int64_t)b.nx;
  if (UNSHARP) {
    const To* orow = reinterpret_cast<const To*>(b.orig) + (b.orig_zo + z) * (int64_t)b.ny * b.nx + (int64_t)gy * b.nx;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int gx = min(x0 + xs + j, b.nx - 1);
      const float base = (float)__ldg(orow + gx);
      res[j] = __fadd_rn(base, __fmul_rn(b.amount, __fsub_rn(base, res[j])));
    }
  }
  float* dst = out + rowoff + x0 + xs;
  if (x0 + xs + 8 <= b.nx && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
    reinterpret_cast<float4*>(dst)[0] = make_float4(res[0], res[1], res[2], res[3]);
    reinterpret_cast<float4*>(dst)[1] = make_float4(res[4], res[5], res[6], res[7]);
  } else {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (x0 + xs + j < b.nx) dst[j] = res[j];
  }
}

template <int R, typename T>
cudaError_t run_exact_r(const DevIn& in, int64_t zo, int64_t nzo, float* out, const Taps& taps,
                        const EpiArgs& epi, float* tmp, cudaStream_t s, int64_t* launches) {
  ExactArgs a;
  a.R = R;
  for (int k = 0; k < 2 * R + 1; ++k) a.w[k] = (double)taps.w[k];
  const int64_t plane = in.ny * in.nx;
  // Z pass -> tmp (nzo slices): TMA-staged kernel when the layout allows it
  bool z_done = false;
  if constexpr (sizeof(T) <= 2 || std::is_same<T, float>::value) {
    CUtensorMap tz;
    if (make_tmap_3d(&tz, in.p, ExTma<T>::v, sizeof(T), in.nx, in.ny, in.nz, Z2_TX, Z2_TY)) {
      Z2Args zb;
      zb.nz = (int)in.nz;
      zb.ny = (int)in.ny;
      zb.nx = (int)in.nx;
      zb.zo = (int)zo;
      zb.nzo = (int)nzo;
      const int gx = (int)((in.nx + Z2_TX - 1) / Z2_TX), gy = (int)((in.ny + Z2_TY - 1) / Z2_TY);
      auto kz = k_exact_z2<R, T>;
      int per_sm = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kz, Z2_NT, 0) != cudaSuccess || per_sm < 1)
        per_sm = 1;
      const int64_t tiles = (int64_t)gx * gy, slots = (int64_t)kNumSMs * per_sm;
      double best = 1e300;
      int64_t best_zc = nzo;
      for (int split = 1; split <= 512; ++split) {
        const int64_t zc = (nzo + split - 1) / split;
        if (split > 1 && zc < 8 * R + 8) break;
        const int64_t ctas = tiles * ((nzo + zc - 1) / zc);
        const double cost = (double)((ctas + slots - 1) / slots) * (double)(zc + 2 * R);
        if (cost < best * 0.98) {
          best = cost;
          best_zc = zc;
        }
      }
      zb.zchunk = (int)best_zc;
      dim3 grid(gx, gy, (unsigned)((nzo + best_zc - 1) / best_zc));
      kz<<<grid, Z2_NT, 0, s>>>(tz, tmp, a, zb);
      if (launches) *launches += 1;
      z_done = true;
    }
  }
  if (!z_done) {
    const int64_t cols = (plane + EZ_T - 1) / EZ_T;
    // enough column-chunks in flight to hide the per-step load latency (the
    // window priming costs 2R extra L2 reads per chunk)
    int64_t want = std::max<int64_t>((nzo + 127) / 128, (32 * kNumSMs + cols - 1) / cols);
    int zchunk = (int)std::max<int64_t>(std::min<int64_t>(nzo, 4 * R + 8), (nzo + want - 1) / want);
    dim3 grid((unsigned)cols, (unsigned)((nzo + zchunk - 1) / zchunk));
    k_exact_z<R, T><<<grid, EZ_T, 0, s>>>((const T*)in.p, in.nz, plane, zo, nzo, zchunk, tmp, a);
    if (launches) *launches += 1;
  }
  // Y+X pass tmp -> out
  using G = EGeo<R>;
  CUtensorMap tm;
  if (!make_tmap_3d(&tm, tmp, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, in.nx, in.ny, nzo, G::WBOX, G::HB))
    return cudaErrorNotSupported;
  YXArgs b;
  b.ny = (int)in.ny;
  b.nx = (int)in.nx;
  b.nz = (int)nzo;
  b.orig = epi.orig;
  b.orig_dt = epi.orig_dt;
  b.orig_zo = epi.orig_zo;
  b.amount = epi.amount;
  for (int64_t zb = 0; zb < nzo; zb += 65535) {
    b.zbase = (int)zb;
    dim3 grid((unsigned)((in.nx + EY_TX - 1) / EY_TX), (unsigned)((in.ny + EY_TY - 1) / EY_TY),
              (unsigned)std::min<int64_t>(65535, nzo - zb));
    if (epi.kind == EPI_UNSHARP) {
      auto k = k_exact_yx<R, true, T>;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM);
      k<<<grid, EY_NT, G::SMEM, s>>>(tm, out, a, b);
    } else {
      auto k = k_exact_yx<R, false, T>;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM);
      k<<<grid, EY_NT, G::SMEM, s>>>(tm, out, a, b);
    }
  }
  if (launches) *launches += 1;
  return cudaGetLastError();
}

template <typename T>
cudaError_t dispatch_r(const DevIn& in, int64_t zo, int64_t nzo, float* out, const Taps& taps,
                       const EpiArgs& epi, float* tmp, cudaStream_t s, int64_t* launches) {
  switch (taps.R) {
    case 1: return run_exact_r<1, T>(in, zo, nzo, out, taps, epi, tmp, s, launches);
    case 2: return run_exact_r<2, T>(in, zo, nzo, out, taps, epi, tmp, s, launches);
    case 3: return run_exact_r<3, T>(in, zo, nzo, out, taps, epi, tmp, s, launches);
    case 4: return run_exact_r<4, T>(in, zo, nzo, out, taps, epi, tmp, s, launches);
    case 5: return run_exact_r<5, T>(in, zo, nzo, out, taps, epi, tmp, s, launches);
    case 6: return run_exact_r<6, T>(in, zo, nzo, out, taps, epi, tmp, s, launches);
    case 7: return run_exact_r<7, T>(in, zo, nzo, out, taps, epi, tmp, s, launches);
    case 8: return run_exact_r<8, T>(in, zo, nzo, out, taps, epi, tmp, s, launches);
  }
  return cudaErrorNotSupported;
}

}  // namespace

cudaError_t gaussian_exact_fused(const DevIn& in, int64_t zo, int64_t nzo, float* out,
                                 const Taps& taps, const EpiArgs& epi, float* tmp,
                                 cudaStream_t s, int64_t* launches) {
  if (nzo <= 0) return cudaSuccess;
  if (taps.R > 8 || in.nx < 8 || in.ny < 8 || (in.nx % 4) != 0) return cudaErrorNotSupported;
  if (epi.kind == EPI_UNSHARP && (epi.orig != in.p || epi.orig_dt != in.dt)) return cudaErrorNotSupported;
  switch (in.dt) {
    case HB_U8: return dispatch_r<uint8_t>(in, zo, nzo, out, taps, epi, tmp, s, launches);
    case HB_U16: return dispatch_r<uint16_t>(in, zo, nzo, out, taps, epi, tmp, s, launches);
    case HB_U32: return dispatch_r<uint32_t>(in, zo, nzo, out, taps, epi, tmp, s, launches);
    case HB_F32: return dispatch_r<float>(in, zo, nzo, out, taps, epi, tmp, s, launches);
  }
  return cudaErrorNotSupported;
}

}  // namespace hb
