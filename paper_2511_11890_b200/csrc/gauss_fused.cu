// gauss_fused.cu — single-pass fused 3D separable stencil (fast fp32 mode):
// Gaussian (filters.py:33-41), box mean (filters.py:66-75) and the unsharp
// epilogue (filters.py:136-139), one HBM read + one HBM write per voxel.
//
// CTA = 48 x 32 output tile marching down a z-chunk.  Per input slice:
//   1. TMA (cp.async.bulk.tensor.3d) lands the halo'd (48+2R) x (32+2R) slice in
//      a 3..6-stage smem ring (mbarrier completion); x/y faces outside the volume
//      are zero-filled by TMA and then clamp-fixed in smem (border tiles only).
//   2. Y pass (first): each thread filters one column of 8 rows -> sY.
//   3. X pass: each thread filters a 6-wide row segment -> 6 values that enter
//      a (2R+1)-deep register ring (the z window, static indexing via switch).
//   4. Z pass: once 2R+1 slices are in the ring, the 6 outputs are written to
//      smem and one thread issues a TMA bulk store of the 48 x 32 output tile.
// The pass order (Y, X, Z) differs from the reference's (Z, Y, X); fp32
// rounding differences stay ~1e-7 relative (tests pin <= 1e-5).  The exact
// (bit-identical) mode lives in sep.cu.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "ops.cuh"
#include "tma.cuh"

namespace hb {

// ---------------------------------------------------------------------------
// host: tensor-map encoder through the runtime's driver entry point
// ---------------------------------------------------------------------------
namespace {
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn g_encode = nullptr;
std::once_flag g_encode_once;

EncodeTiledFn encoder() {
  std::call_once(g_encode_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<EncodeTiledFn>(fn);
    cudaGetLastError();
  });
  return g_encode;
}
}  // namespace

bool make_tmap_3d(CUtensorMap* map, const void* base, CUtensorMapDataType dt, int elem_bytes,
                  int64_t nx, int64_t ny, int64_t nz, int box_x, int box_y) {
  EncodeTiledFn enc = encoder();
  if (!enc) return false;
  if ((reinterpret_cast<uintptr_t>(base) & 15) != 0) return false;
  if ((nx * elem_bytes) % 16 != 0) return false;
  if (box_x > 256 || box_y > 256 || (box_x * elem_bytes) % 16 != 0) return false;
  if (nx >= (1ll << 32) || ny >= (1ll << 32) || nz >= (1ll << 32)) return false;
  cuuint64_t dims[3] = {(cuuint64_t)nx, (cuuint64_t)ny, (cuuint64_t)nz};
  cuuint64_t strides[2] = {(cuuint64_t)(nx * elem_bytes), (cuuint64_t)(nx * ny * elem_bytes)};
  cuuint32_t box[3] = {(cuuint32_t)box_x, (cuuint32_t)box_y, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, dt, 3, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

namespace {

constexpr int TY = 32, NT = 256;

enum { MODE_GAUSS = 0, MODE_BOX = 1 };

struct FusedArgs {
  float w[kMaxTaps];
  int nzi;       // slices of the input block
  int zo;        // block z of output slice 0
  int nzo;       // output slices
  int zchunk;    // output slices per CTA
  int nx, ny;
  float count;   // box: (2r+1)^3
  float inv_count;  // RN(1 / count)
  // unsharp epilogue
  const void* orig;
  float amount;
};

template <typename T> struct TmaType;
template <> struct TmaType<float> { static constexpr CUtensorMapDataType v = CU_TENSOR_MAP_DATA_TYPE_FLOAT32; };
template <> struct TmaType<uint16_t> { static constexpr CUtensorMapDataType v = CU_TENSOR_MAP_DATA_TYPE_UINT16; };
template <> struct TmaType<uint8_t> { static constexpr CUtensorMapDataType v = CU_TENSOR_MAP_DATA_TYPE_UINT8; };

template <int R, typename Tin>
struct Geo {
  // Tile width: 48 x 32 with 6 outputs per thread for small radii; 32 x 32 with
  // 4 outputs per thread for R >= 4 so the 17-deep register ring (68 regs)
  // leaves room for two CTAs (16 warps) per SM.
  static constexpr int TX = R >= 4 ? 32 : 48;
  static constexpr int SEG = TX / 8;                                    // outputs per thread (x)
  // sY pitch: conflict-free LDS.64 in the X pass (80 = 16 mod 32 for 6-wide
  // segments; 50 = 2 mod 4 for 4-wide segments)
  static constexpr int SYS = R >= 4 ? 50 : 80;
  static constexpr int WC = TX + 2 * R;                                 // halo'd width
  static constexpr int HB = TY + 2 * R;                                 // halo'd height
  static constexpr int ALIGN = 16 / (int)sizeof(Tin);                   // 16 B in elements
  // The box's first x must be 16-B aligned in global memory (measured on B200:
  // unaligned negative starts raise "illegal instruction"), so the box starts
  // XA >= R columns left of the tile and the halo begins XOFF columns in.
  static constexpr int XA = (R + ALIGN - 1) / ALIGN * ALIGN;
  static constexpr int XOFF = XA - R;
  static constexpr int WBOX = (XA + TX + R + ALIGN - 1) / ALIGN * ALIGN;  // smem row pitch
  static constexpr int STAGE_BYTES = HB * WBOX * (int)sizeof(Tin);
  static constexpr int STAGE_PITCH = (STAGE_BYTES + 127) / 128 * 128;
  static constexpr int NST = R <= 1 ? 4 : (R <= 3 ? 6 : 3);            // TMA ring depth
  static constexpr int MINB = R <= 1 ? 3 : 2;                           // CTAs per SM
  static constexpr int RING = 2 * R + 1;
  static constexpr int SY_BYTES = 2 * TY * SYS * 4;
  // triple-buffered output tile: the store of output o-3 is known complete
  // (thread 0's wait_group.read<1> in iteration o-1 precedes this iteration's
  // barrier), so all threads may overwrite its buffer without racing the TMA
  static constexpr int SOUT_BYTES = 3 * TY * TX * 4;
  static constexpr int OFF_SY = NST * STAGE_PITCH;
  static constexpr int OFF_SOUT = OFF_SY + SY_BYTES;
  static constexpr int OFF_BAR = OFF_SOUT + SOUT_BYTES;
  static constexpr int SMEM = OFF_BAR + NST * 8 + 128;  // +128 for base alignment
  static_assert(WC <= SYS, "halo'd tile wider than the sY pitch");
};

template <typename T>
__device__ __forceinline__ float cvt(T v) { return (float)v; }

template <int R, typename Tin, int MODE, bool UNSHARP>
__global__ void __launch_bounds__(NT, Geo<R, Tin>::MINB)
k_sep3d_fused(const __grid_constant__ CUtensorMap tin, const __grid_constant__ CUtensorMap tout,
              const FusedArgs a) {
  using G = Geo<R, Tin>;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem =
      smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u)  /* stays in .shared */;
  Tin* sIn = reinterpret_cast<Tin*>(smem);
  float* sY = reinterpret_cast<float*>(smem + G::OFF_SY);
  float* sOut = reinterpret_cast<float*>(smem + G::OFF_SOUT);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + G::OFF_BAR);

  const int tid = threadIdx.x;
  const int x0 = blockIdx.x * G::TX, y0 = blockIdx.y * TY;
  const int z0 = blockIdx.z * a.zchunk;
  const int z1 = min(z0 + a.zchunk, a.nzo);
  const int nsl = (z1 - z0) + 2 * R;  // input slices this CTA consumes
  const bool border = (x0 - R < 0) || (x0 + G::TX + R > a.nx) || (y0 - R < 0) || (y0 + TY + R > a.ny);

  const float* w = a.w;  // taps stay in the constant bank (FFMA c[] operand)

  auto zin_of = [&](int s) { return min(max(a.zo + z0 - R + s, 0), a.nzi - 1); };

  if (tid == 0) {
    prefetch_tmap(&tin);
    prefetch_tmap(&tout);
#pragma unroll
    for (int i = 0; i < G::NST; ++i) mbar_init(&bar[i], 1);
    fence_mbar_init();
#pragma unroll
    for (int i = 0; i < G::NST; ++i) {
      if (i < nsl) {
        mbar_expect_tx(&bar[i], G::HB * G::WBOX * sizeof(Tin));
        tma_load_3d(sIn + i * (G::STAGE_PITCH / sizeof(Tin)), &tin, x0 - G::XA, y0 - R, zin_of(i), &bar[i]);
      }
    }
  }
  __syncthreads();

  // Y-pass mapping: column c of the halo'd tile, 8 output rows starting at 8g
  const int yc = tid % G::WC, yg = tid / G::WC;
  const bool y_active = yg < TY / 8;
  // X-pass mapping: warp -> 4 rows, lane -> (row r, 6-wide segment j)
  const int lane = tid & 31, warp = tid >> 5;
  const int xr = 4 * warp + (lane >> 3);  // output row in tile (0..31)
  const int xj = (lane & 7) * G::SEG;        // output col start in tile

  float ring[G::RING][G::SEG];
#pragma unroll
  for (int u = 0; u < G::RING; ++u)
#pragma unroll
    for (int m = 0; m < G::SEG; ++m) ring[u][m] = 0.f;

  for (int s = 0; s < nsl; ++s) {
    const int st = s % G::NST;
    Tin* stage = sIn + st * (G::STAGE_PITCH / sizeof(Tin));
    mbar_wait(&bar[st], (uint32_t)((s / G::NST) & 1));
    if (border) {
      // clamp-to-edge fix-up of the zero-filled out-of-volume parts
      clamp_tile<Tin, NT>(stage + G::XOFF, G::WBOX, G::HB, G::WC, y0 - R, x0 - R, a.ny, a.nx, tid);
      fence_proxy_async();  // generic writes before the stage is re-filled by TMA
      __syncthreads();
    }
    // ---- Y pass: sIn -> sY[s&1] -------------------------------------------
    float* sYb = sY + (s & 1) * TY * G::SYS;
    if (y_active) {
      float v[8 + 2 * R];
#pragma unroll
      for (int j = 0; j < 8 + 2 * R; ++j) v[j] = cvt(stage[(8 * yg + j) * G::WBOX + G::XOFF + yc]);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        float acc;
        if (MODE == MODE_GAUSS) {
          acc = v[j + R] * w[R];
#pragma unroll
          for (int d = R; d >= 1; --d) acc = fmaf(v[j + R - d] + v[j + R + d], w[R - d], acc);
        } else {
          acc = v[j];
#pragma unroll
          for (int k = 1; k < 2 * R + 1; ++k) acc += v[j + k];
        }
        sYb[(8 * yg + j) * G::SYS + yc] = acc;
      }
    }
    __syncthreads();
    if (tid == 0) {
      // refill this stage with slice s + NST (all Y-pass reads of it are done)
      if (s + G::NST < nsl) {
        fence_proxy_async();
        mbar_expect_tx(&bar[st], G::HB * G::WBOX * sizeof(Tin));
        tma_load_3d(stage, &tin, x0 - G::XA, y0 - R, zin_of(s + G::NST), &bar[st]);
      }
      // store the output tile produced in the previous iteration
      const int o_prev = s - 1 - 2 * R;
      if (o_prev >= 0) {
        tma_store_3d(&tout, sOut + (o_prev % 3) * TY * G::TX, x0, y0, z0 + o_prev);
        bulk_commit();
        bulk_wait_read<1>();  // the store before it has finished reading its buffer
      }
    }
    // ---- X pass: sY -> 6 values -------------------------------------------
    float xo[G::SEG];
    {
      float v[G::SEG + 2 * R];
      const float* row = sYb + xr * G::SYS + xj;
#pragma unroll
      for (int i = 0; i < (G::SEG + 2 * R) / 2; ++i) {
        const float2 t = *reinterpret_cast<const float2*>(row + 2 * i);
        v[2 * i] = t.x;
        v[2 * i + 1] = t.y;
      }
#pragma unroll
      for (int m = 0; m < G::SEG; ++m) {
        float acc;
        if (MODE == MODE_GAUSS) {
          acc = v[m + R] * w[R];
#pragma unroll
          for (int d = R; d >= 1; --d) acc = fmaf(v[m + R - d] + v[m + R + d], w[R - d], acc);
        } else {
          acc = v[m];
#pragma unroll
          for (int k = 1; k < 2 * R + 1; ++k) acc += v[m + k];
        }
        xo[m] = acc;
      }
    }
    // ---- ring insert + Z pass ----------------------------------------------
    const int o = s - 2 * R;  // output slice produced now (if >= 0)
    float zo_[G::SEG];
    bool have = false;
    switch (s % G::RING) {
#define HB_RING_CASE(U)                                                           \
  case U:                                                                         \
    if constexpr (U < G::RING) {                                                  \
      _Pragma("unroll") for (int m = 0; m < G::SEG; ++m) ring[U][m] = xo[m];         \
      if (o >= 0) {                                                               \
        have = true;                                                              \
        _Pragma("unroll") for (int m = 0; m < G::SEG; ++m) {                         \
          float acc;                                                              \
          if (MODE == MODE_GAUSS) {                                               \
            acc = ring[(U + 1 + R) % G::RING][m] * w[R];                          \
            _Pragma("unroll") for (int d = R; d >= 1; --d) acc =                  \
                fmaf(ring[(U + 1 + R - d) % G::RING][m] + ring[(U + 1 + R + d) % G::RING][m], \
                     w[R - d], acc);                                              \
          } else {                                                                \
            acc = ring[(U + 1) % G::RING][m];                                     \
            _Pragma("unroll") for (int k = 1; k < G::RING; ++k) acc +=            \
                ring[(U + 1 + k) % G::RING][m]; /* z order: plan invariant */     \
          }                                                                       \
          zo_[m] = acc;                                                           \
        }                                                                         \
      }                                                                           \
    }                                                                             \
    break;
      HB_RING_CASE(0) HB_RING_CASE(1) HB_RING_CASE(2) HB_RING_CASE(3) HB_RING_CASE(4)
      HB_RING_CASE(5) HB_RING_CASE(6) HB_RING_CASE(7) HB_RING_CASE(8) HB_RING_CASE(9)
      HB_RING_CASE(10) HB_RING_CASE(11) HB_RING_CASE(12) HB_RING_CASE(13) HB_RING_CASE(14)
      HB_RING_CASE(15) HB_RING_CASE(16)
#undef HB_RING_CASE
      default: break;
    }
    if (have) {
      if (MODE == MODE_BOX) {
        // correctly rounded sum / count (an FMA-refined reciprocal is bit-identical,
        // tools/microbench/divtest.cu, but measured slower here)
#pragma unroll
        for (int m = 0; m < G::SEG; ++m) zo_[m] = __fdiv_rn(zo_[m], a.count);
      }
      if (UNSHARP) {
        const int gy = y0 + xr;
        const int64_t zb = (int64_t)a.zo + z0 + o;
        const Tin* orow = reinterpret_cast<const Tin*>(a.orig) + (zb * a.ny + min(gy, a.ny - 1)) * (int64_t)a.nx;
#pragma unroll
        for (int m = 0; m < G::SEG; ++m) {
          const int gx = min(x0 + xj + m, a.nx - 1);
          const float b = cvt(__ldg(orow + gx));
          zo_[m] = __fadd_rn(b, __fmul_rn(a.amount, __fsub_rn(b, zo_[m])));
        }
      }
      float* dst = sOut + (o % 3) * TY * G::TX + xr * G::TX + xj;
#pragma unroll
      for (int m = 0; m < G::SEG; m += 2) *reinterpret_cast<float2*>(dst + m) = make_float2(zo_[m], zo_[m + 1]);
      fence_proxy_async();
    }
  }
  __syncthreads();
  if (tid == 0) {
    const int o_last = nsl - 1 - 2 * R;
    if (o_last >= 0) {
      tma_store_3d(&tout, sOut + (o_last % 3) * TY * G::TX, x0, y0, z0 + o_last);
      bulk_commit();
    }
    bulk_wait<0>();
  }
}

template <int R, typename Tin, int MODE, bool UNSHARP>
cudaError_t launch(const DevIn& in, int64_t zo, int64_t nzo, float* out, const Taps& taps,
                   const EpiArgs& epi, cudaStream_t s) {
  using G = Geo<R, Tin>;
  CUtensorMap tin, tout;
  if (!make_tmap_3d(&tin, in.p, TmaType<Tin>::v, sizeof(Tin), in.nx, in.ny, in.nz, G::WBOX, G::HB))
    return cudaErrorNotSupported;
  if (!make_tmap_3d(&tout, out, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, in.nx, in.ny, nzo, G::TX, TY))
    return cudaErrorNotSupported;
  FusedArgs a;
  for (int k = 0; k < 2 * R + 1; ++k) a.w[k] = taps.w[k];
  a.nzi = (int)in.nz;
  a.zo = (int)zo;
  a.nzo = (int)nzo;
  a.nx = (int)in.nx;
  a.ny = (int)in.ny;
  a.count = epi.count;
  a.inv_count = 1.0f / epi.count;
  a.orig = epi.orig;
  a.amount = epi.amount;
  const int gx = (int)((in.nx + G::TX - 1) / G::TX), gy = (int)((in.ny + TY - 1) / TY);
  // z-chunking: balance waves of (148 * MINB) resident CTAs against the 2R-slice
  // priming cost of every chunk
  const int64_t tiles = (int64_t)gx * gy;
  const int64_t slots = (int64_t)kNumSMs * G::MINB;
  double best = 1e300;
  int best_split = 1;
  for (int split = 1; split <= 256; ++split) {
    int64_t zc = (nzo + split - 1) / split;
    if (split > 1 && zc < 4 * R + 8) break;
    int64_t ctas = tiles * ((nzo + zc - 1) / zc);
    int64_t waves = (ctas + slots - 1) / slots;
    double cost = (double)waves * (double)(zc + 2 * R);
    if (cost < best * 0.98) {
      best = cost;
      best_split = split;
    }
  }
  a.zchunk = (int)((nzo + best_split - 1) / best_split);
  dim3 grid(gx, gy, (unsigned)((nzo + a.zchunk - 1) / a.zchunk));
  auto kern = k_sep3d_fused<R, Tin, MODE, UNSHARP>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM);
  kern<<<grid, NT, G::SMEM, s>>>(tin, tout, a);
  return cudaGetLastError();
}

template <int MODE, bool UNSHARP, typename Tin>
cudaError_t dispatch_r(int R, const DevIn& in, int64_t zo, int64_t nzo, float* out,
                       const Taps& taps, const EpiArgs& epi, cudaStream_t s) {
  switch (R) {
    case 1: return launch<1, Tin, MODE, UNSHARP>(in, zo, nzo, out, taps, epi, s);
    case 2: return launch<2, Tin, MODE, UNSHARP>(in, zo, nzo, out, taps, epi, s);
    case 3: return launch<3, Tin, MODE, UNSHARP>(in, zo, nzo, out, taps, epi, s);
    case 4: if (MODE == MODE_GAUSS) return launch<4, Tin, MODE, UNSHARP>(in, zo, nzo, out, taps, epi, s); break;
    case 5: if (MODE == MODE_GAUSS) return launch<5, Tin, MODE, UNSHARP>(in, zo, nzo, out, taps, epi, s); break;
    case 6: if (MODE == MODE_GAUSS) return launch<6, Tin, MODE, UNSHARP>(in, zo, nzo, out, taps, epi, s); break;
    case 7: if (MODE == MODE_GAUSS) return launch<7, Tin, MODE, UNSHARP>(in, zo, nzo, out, taps, epi, s); break;
    case 8: if (MODE == MODE_GAUSS) return launch<8, Tin, MODE, UNSHARP>(in, zo, nzo, out, taps, epi, s); break;
  }
  return cudaErrorNotSupported;
}

template <int MODE, bool UNSHARP>
cudaError_t dispatch_dt(int R, const DevIn& in, int64_t zo, int64_t nzo, float* out,
                        const Taps& taps, const EpiArgs& epi, cudaStream_t s) {
  switch (in.dt) {
    case HB_F32: return dispatch_r<MODE, UNSHARP, float>(R, in, zo, nzo, out, taps, epi, s);
    case HB_U16: return dispatch_r<MODE, UNSHARP, uint16_t>(R, in, zo, nzo, out, taps, epi, s);
    case HB_U8: return dispatch_r<MODE, UNSHARP, uint8_t>(R, in, zo, nzo, out, taps, epi, s);
  }
  return cudaErrorNotSupported;
}


// ===========================================================================
// k_gauss_p2 — packed-FP32 Gaussian / unsharp (fast mode), 2 <= R <= 8.
//
// A 17-tap separable pass costs 17 FP ops per voxel per axis, so the Gaussian
// is bound by the FP32 pipe, not HBM (51 ops/voxel -> ~730 Gvox/s at 128
// FMA lanes/clk/SM).  Every pass here runs on FFMA2/FADD2 pairs, which halves
// the FP issue slots so loads, stores and ring traffic fit beside the math:
//   Y pass (first, over the halo'd width): an item = one x-adjacent column
//     pair x 4 rows (160 items: 5 of 8 warps busy; 8-row items were 5% slower
//     from the imbalance), scatter form (acc[m] += w[j-m] * row j), pairs come
//     straight out of the TMA rows as one LDS.64;
//   X pass: a thread owns a row pair (y, y+1) x two x positions; sY is stored
//     row-pair interleaved, so one LDS.128 yields two x columns of a row pair;
//     computed inside the ring switch so results land in the ring slot (no
//     MOVs), two partial sums per output to shorten the FFMA2 chain;
//   Z pass: a (2R+1)-slot register ring of row pairs, symmetric fold.
// Tile 64 x 16 outputs, 256 threads, 2 CTAs/SM; weights live in uniform
// registers (FFMA2 takes a UR pair operand).  TMA ring / border clamp /
// triple-buffered TMA output tile exactly as k_sep3d_fused.
// Measured (B200, sigma=2, 1024^3): 260 Gvox/s vs 240 for the scalar kernel;
// ncu: FP pipe 47% busy, shared-memory wavefronts 66% of peak (0.72 per
// output: the X pass re-reads 18 row pairs per 2 outputs), issue 51% at 16
// warps/SM (the 17-slot ring pins 118 registers) -> latency/smem bound.
// ===========================================================================
namespace p2 {
typedef unsigned long long f2;
__device__ __forceinline__ f2 pk(float lo, float hi) {
  f2 d;
  asm("mov.b64 %0, {%1, %2};" : "=l"(d) : "f"(lo), "f"(hi));
  return d;
}
__device__ __forceinline__ void upk(f2 v, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ f2 add(f2 a, f2 b) {
  f2 d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ f2 mul(f2 a, f2 b) {
  f2 d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ f2 fma(f2 a, f2 b, f2 c) {
  f2 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
template <typename T> __device__ __forceinline__ f2 load_pair(const T* p) {
  return pk((float)p[0], (float)p[1]);
}
template <> __device__ __forceinline__ f2 load_pair<float>(const float* p) {
  return *reinterpret_cast<const f2*>(p);
}
}  // namespace p2

struct P2Args {
  unsigned long long w2[kMaxTaps > 17 ? 17 : kMaxTaps];  // (w_k, w_k) pairs
  float w1[kMaxTaps > 17 ? 17 : kMaxTaps];               // w_k (FFMA constant operands)
  int nzi, zo, nzo, zchunk, nx, ny;
  const void* orig;
  float amount;
};

constexpr int P2_TX = 64, P2_TY = 16, P2_NT = 256;

template <int R, typename Tin, int P2_YR>
struct GeoP2 {
  static constexpr int WC = P2_TX + 2 * R;                     // halo'd width
  static constexpr int HB = P2_TY + 2 * R;                     // halo'd height
  static constexpr int ALIGN = 16 / (int)sizeof(Tin);
  static constexpr int XA = (R + ALIGN - 1) / ALIGN * ALIGN;   // 16-B aligned box start
  static constexpr int XOFF = XA - R;                          // stage col of halo col 0
  static constexpr int YC0 = XOFF & ~1;                        // even first Y column
  static constexpr int YOFF = XOFF - YC0;                      // Y col of halo col 0
  static constexpr int NYC = (YOFF + WC + 1) / 2 * 2;          // Y columns (even)
  static constexpr int NYP = NYC / 2;                          // Y column pairs
  static constexpr int WBOX0 = (XA + P2_TX + R) > (YC0 + NYC) ? (XA + P2_TX + R) : (YC0 + NYC);
  static constexpr int WBOX = (WBOX0 + ALIGN - 1) / ALIGN * ALIGN;
  static constexpr int STAGE_BYTES = HB * WBOX * (int)sizeof(Tin);
  static constexpr int STAGE_PITCH = (STAGE_BYTES + 127) / 128 * 128;
  static constexpr int NST = 3;
  static constexpr int RING = 2 * R + 1;
  static constexpr int NYI = NYP * (P2_TY / P2_YR);            // Y-pass items
  // X pass: R >= 6 reads 4 x positions of a row from a row-major sY in scalar
  // FP32 (halves the X pass's shared-memory bytes, the bottleneck at large R);
  // smaller R keep the FFMA2 row-pair X pass on a row-pair interleaved sY
  static constexpr bool XQ = R >= 6;
  static constexpr int SYP = NYC + 4;                          // sY pitch (floats / f2)
  static constexpr int SY_BYTES = XQ ? 2 * P2_TY * SYP * 4 : 2 * (P2_TY / 2) * SYP * 8;
  static constexpr int SOUT_BYTES = 3 * P2_TY * P2_TX * 4;     // triple-buffered
  static constexpr int OFF_SY = NST * STAGE_PITCH;
  static constexpr int OFF_SOUT = OFF_SY + SY_BYTES;
  static constexpr int OFF_BAR = OFF_SOUT + SOUT_BYTES;
  static constexpr int SMEM = OFF_BAR + NST * 8 + 128;
  static_assert(NYI <= P2_NT, "Y-pass items exceed the CTA");
  static_assert(P2_TY * (P2_TX / 4) == P2_NT, "one thread per (row, 4 x) / (row pair, 2 x)");
};

template <int R, typename Tin, bool UNSHARP, int P2_YR>
__global__ void __launch_bounds__(P2_NT, 2)
k_gauss_p2(const __grid_constant__ CUtensorMap tin, const __grid_constant__ CUtensorMap tout,
           const __grid_constant__ P2Args a) {
  using G = GeoP2<R, Tin, P2_YR>;
  using namespace p2;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem =
      smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u)  /* stays in .shared */;
  Tin* sIn = reinterpret_cast<Tin*>(smem);
  float* sY = reinterpret_cast<float*>(smem + G::OFF_SY);
  float* sOut = reinterpret_cast<float*>(smem + G::OFF_SOUT);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + G::OFF_BAR);
  const int tid = threadIdx.x;
  const int x0 = blockIdx.x * P2_TX, y0 = blockIdx.y * P2_TY;
  const int z0 = blockIdx.z * a.zchunk;
  const int z1 = min(z0 + a.zchunk, a.nzo);
  const int nsl = (z1 - z0) + 2 * R;
  const bool border =
      (x0 - R < 0) || (x0 + P2_TX + R > a.nx) || (y0 - R < 0) || (y0 + P2_TY + R > a.ny);
  auto zin_of = [&](int s) { return min(max(a.zo + z0 - R + s, 0), a.nzi - 1); };
  const f2* W = a.w2;  // kernel-param bank -> uniform registers

  if (tid == 0) {
    prefetch_tmap(&tin);
    prefetch_tmap(&tout);
#pragma unroll
    for (int i = 0; i < G::NST; ++i) mbar_init(&bar[i], 1);
    fence_mbar_init();
#pragma unroll
    for (int i = 0; i < G::NST; ++i)
      if (i < nsl) {
        mbar_expect_tx(&bar[i], G::HB * G::WBOX * sizeof(Tin));
        tma_load_3d(sIn + i * (G::STAGE_PITCH / sizeof(Tin)), &tin, x0 - G::XA, y0 - R, zin_of(i),
                    &bar[i]);
      }
  }
  __syncthreads();
  // Y item: column pair ycp, rows [P2_YR * yg, P2_YR * yg + P2_YR)
  const int ycp = tid % G::NYP, yg = tid / G::NYP;
  const bool y_active = tid < G::NYI;
  // X/Z ownership: XQ: row yr, x positions 4*xq .. 4*xq+3 (ring of two x pairs);
  // otherwise row pair yp, x positions 2*sg, 2*sg+1 (ring of two row pairs)
  const int yr = tid / (P2_TX / 4), xq = tid % (P2_TX / 4);
  const int yp = tid / (P2_TX / 2), sg = tid % (P2_TX / 2);
  f2 ring[G::RING][2];
#pragma unroll
  for (int u = 0; u < G::RING; ++u) ring[u][0] = ring[u][1] = 0ull;

  for (int s = 0; s < nsl; ++s) {
    const int st = s % G::NST;
    Tin* stage = sIn + st * (G::STAGE_PITCH / sizeof(Tin));
    mbar_wait(&bar[st], (uint32_t)((s / G::NST) & 1));
    if (border) {
      clamp_tile<Tin, P2_NT>(stage + G::XOFF, G::WBOX, G::HB, G::WC, y0 - R, x0 - R, a.ny, a.nx, tid);
      fence_proxy_async();
      __syncthreads();
    }
    // ---- Y pass (column pairs, scatter form) -> sY --------------------------
    float* sYb = sY + (s & 1) * P2_TY * G::SYP;  // same float count in both layouts
    if (y_active) {
      f2 acc[P2_YR];
      const Tin* src = stage + (P2_YR * yg) * G::WBOX + G::YC0 + 2 * ycp;
#pragma unroll
      for (int j = 0; j < P2_YR + 2 * R; ++j) {
        const f2 v = load_pair<Tin>(src + j * G::WBOX);
#pragma unroll
        for (int m = 0; m < P2_YR; ++m) {
          const int k = j - m;
          if (k == 0) acc[m] = mul(v, W[0]);
          else if (k > 0 && k <= 2 * R) acc[m] = fma(v, W[k], acc[m]);
        }
      }
      if constexpr (G::XQ) {
#pragma unroll
        for (int m = 0; m < P2_YR; ++m)  // row m: columns (c, c+1), one STS.64
          *reinterpret_cast<f2*>(sYb + (P2_YR * yg + m) * G::SYP + 2 * ycp) = acc[m];
      } else {
        f2* sYp = reinterpret_cast<f2*>(sYb);
#pragma unroll
        for (int m = 0; m < P2_YR; m += 2) {  // row pair: [(c,r0),(c,r1)],[(c+1,r0),(c+1,r1)]
          float a0, a1, b0, b1;
          upk(acc[m], a0, a1);
          upk(acc[m + 1], b0, b1);
          uint4 q;
          q.x = __float_as_uint(a0);
          q.y = __float_as_uint(b0);
          q.z = __float_as_uint(a1);
          q.w = __float_as_uint(b1);
          *reinterpret_cast<uint4*>(sYp + ((P2_YR * yg + m) / 2) * G::SYP + 2 * ycp) = q;
        }
      }
    }
    __syncthreads();
    if (tid == 0) {
      if (s + G::NST < nsl) {
        fence_proxy_async();
        mbar_expect_tx(&bar[st], G::HB * G::WBOX * sizeof(Tin));
        tma_load_3d(stage, &tin, x0 - G::XA, y0 - R, zin_of(s + G::NST), &bar[st]);
      }
      const int o_prev = s - 1 - 2 * R;
      if (o_prev >= 0) {
        tma_store_3d(&tout, sOut + (o_prev % 3) * P2_TY * P2_TX, x0, y0, z0 + o_prev);
        bulk_commit();
        bulk_wait_read<1>();
      }
    }
    // ---- X pass: 4 x positions of one row in scalar FP32 (the shifted taps of
    // x-adjacent outputs do not form aligned register pairs), 20 floats in
    // five LDS.128 -> half the shared-memory bytes of a row-pair X pass, which
    // kept the LSU pipe 71% busy; results land straight in the ring slot as
    // two x pairs.  Two partial sums per output halve the dependent chain.
    auto xpass_q = [&](f2& out0, f2& out1) {
      float xa[4], xb[4];
      const float* row = sYb + yr * G::SYP + G::YOFF + 4 * xq;
      auto tap = [&](int c, float v) {
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          const int k = c - m;
          const float wk = a.w1[k < 0 ? 0 : (k > 2 * R ? 0 : k)];
          if (k == 0) xa[m] = v * wk;
          else if (k == R + 1) xb[m] = v * wk;
          else if (k > 0 && k <= R) xa[m] = fmaf(v, wk, xa[m]);
          else if (k > R + 1 && k <= 2 * R) xb[m] = fmaf(v, wk, xb[m]);
        }
      };
      if (G::YOFF == 0) {
#pragma unroll
        for (int i = 0; i < (4 + 2 * R + 3) / 4; ++i) {
          const float4 q = *reinterpret_cast<const float4*>(row + 4 * i);
          tap(4 * i, q.x);
          tap(4 * i + 1, q.y);
          tap(4 * i + 2, q.z);
          tap(4 * i + 3, q.w);
        }
      } else {
#pragma unroll
        for (int c = 0; c < 4 + 2 * R; ++c) tap(c, row[c]);
      }
      out0 = pk(xa[0] + xb[0], xa[1] + xb[1]);
      out1 = pk(xa[2] + xb[2], xa[3] + xb[3]);
    };
    auto xpass_rp = [&](f2& out0, f2& out1) {  // row-pair FFMA2 X pass (small R)
      f2 xa[2], xb[2];
      const f2* row = reinterpret_cast<const f2*>(sYb) + yp * G::SYP + G::YOFF + 2 * sg;
      auto tap = [&](int c, f2 v) {
#pragma unroll
        for (int m = 0; m < 2; ++m) {
          const int k = c - m;
          if (k == 0) xa[m] = mul(v, W[0]);
          else if (k == R + 1) xb[m] = mul(v, W[k]);
          else if (k > 0 && k <= R) xa[m] = fma(v, W[k], xa[m]);
          else if (k > R + 1 && k <= 2 * R) xb[m] = fma(v, W[k], xb[m]);
        }
      };
      if (G::YOFF == 0) {
#pragma unroll
        for (int i = 0; i < (2 + 2 * R) / 2; ++i) {
          f2 v0, v1;  // one LDS.128: columns 2i, 2i+1 of the row pair
          asm volatile("ld.shared.v2.b64 {%0, %1}, [%2];"
                       : "=l"(v0), "=l"(v1)
                       : "r"(smem_u32(row + 2 * i)));
          tap(2 * i, v0);
          tap(2 * i + 1, v1);
        }
      } else {
#pragma unroll
        for (int c = 0; c < 2 + 2 * R; ++c) tap(c, row[c]);
      }
      out0 = add(xa[0], xb[0]);
      out1 = add(xa[1], xb[1]);
    };
    auto xpass = [&](f2& out0, f2& out1) {
      if constexpr (G::XQ) xpass_q(out0, out1);
      else xpass_rp(out0, out1);
    };
    // ---- ring + Z pass (symmetric fold) --------------------------------------
    const int o = s - 2 * R;
    f2 zr[2];
    bool have = false;
    switch (s % G::RING) {
#define HB_P2_CASE(U)                                                                        \
  case U:                                                                                    \
    if constexpr (U < G::RING) {                                                             \
      xpass(ring[U][0], ring[U][1]);                                                         \
      if (o >= 0) {                                                                          \
        have = true;                                                                         \
        _Pragma("unroll") for (int m = 0; m < 2; ++m) {                                      \
          f2 acc = mul(ring[(U + 1 + R) % G::RING][m], W[R]);                                \
          _Pragma("unroll") for (int d = R; d >= 1; --d) acc =                               \
              fma(add(ring[(U + 1 + R - d) % G::RING][m], ring[(U + 1 + R + d) % G::RING][m]), \
                  W[R - d], acc);                                                            \
          zr[m] = acc;                                                                       \
        }                                                                                    \
      }                                                                                      \
    }                                                                                        \
    break;
      HB_P2_CASE(0) HB_P2_CASE(1) HB_P2_CASE(2) HB_P2_CASE(3) HB_P2_CASE(4) HB_P2_CASE(5)
      HB_P2_CASE(6) HB_P2_CASE(7) HB_P2_CASE(8) HB_P2_CASE(9) HB_P2_CASE(10) HB_P2_CASE(11)
      HB_P2_CASE(12) HB_P2_CASE(13) HB_P2_CASE(14) HB_P2_CASE(15) HB_P2_CASE(16)
#undef HB_P2_CASE
      default: break;
    }
    if (have) {
      float r[4];  // XQ: row yr at x = 4xq..4xq+3; else rows 2yp (r0, r1), 2yp+1 (r2, r3) at x 2sg, 2sg+1
      if constexpr (G::XQ) {
        upk(zr[0], r[0], r[1]);
        upk(zr[1], r[2], r[3]);
      } else {
        upk(zr[0], r[0], r[2]);
        upk(zr[1], r[1], r[3]);
      }
      if (UNSHARP) {
        const int64_t zb = (int64_t)a.zo + z0 + o;
        const Tin* ob = reinterpret_cast<const Tin*>(a.orig);
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          const int gy = G::XQ ? y0 + yr : y0 + 2 * yp + (m >> 1);
          const int gx = G::XQ ? x0 + 4 * xq + m : x0 + 2 * sg + (m & 1);
          const float b = (float)__ldg(ob + (zb * a.ny + min(gy, a.ny - 1)) * (int64_t)a.nx + min(gx, a.nx - 1));
          r[m] = __fadd_rn(b, __fmul_rn(a.amount, __fsub_rn(b, r[m])));
        }
      }
      float* tile = sOut + (o % 3) * P2_TY * P2_TX;
      if constexpr (G::XQ) {
        *reinterpret_cast<float4*>(tile + yr * P2_TX + 4 * xq) = make_float4(r[0], r[1], r[2], r[3]);
      } else {
        *reinterpret_cast<float2*>(tile + (2 * yp) * P2_TX + 2 * sg) = make_float2(r[0], r[1]);
        *reinterpret_cast<float2*>(tile + (2 * yp + 1) * P2_TX + 2 * sg) = make_float2(r[2], r[3]);
      }
      fence_proxy_async();
    }
  }
  __syncthreads();
  if (tid == 0) {
    const int o_last = nsl - 1 - 2 * R;
    if (o_last >= 0) {
      tma_store_3d(&tout, sOut + (o_last % 3) * P2_TY * P2_TX, x0, y0, z0 + o_last);
      bulk_commit();
    }
    bulk_wait<0>();
  }
}

template <int R, typename Tin, bool UNSHARP, int P2_YR>
cudaError_t launch_p2(const DevIn& in, int64_t zo, int64_t nzo, float* out, const Taps& taps,
                      const EpiArgs& epi, cudaStream_t s) {
  using G = GeoP2<R, Tin, P2_YR>;
  CUtensorMap tin, tout;
  if (!make_tmap_3d(&tin, in.p, TmaType<Tin>::v, sizeof(Tin), in.nx, in.ny, in.nz, G::WBOX, G::HB))
    return cudaErrorNotSupported;
  if (!make_tmap_3d(&tout, out, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, in.nx, in.ny, nzo, P2_TX, P2_TY))
    return cudaErrorNotSupported;
  P2Args a;
  for (int k = 0; k < 2 * R + 1; ++k) {
    unsigned int b = 0;
    std::memcpy(&b, &taps.w[k], 4);
    a.w2[k] = ((unsigned long long)b << 32) | b;
    a.w1[k] = taps.w[k];
  }
  a.nzi = (int)in.nz;
  a.zo = (int)zo;
  a.nzo = (int)nzo;
  a.nx = (int)in.nx;
  a.ny = (int)in.ny;
  a.orig = epi.orig;
  a.amount = epi.amount;
  auto kern = k_gauss_p2<R, Tin, UNSHARP, P2_YR>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM);
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, P2_NT, G::SMEM) != cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
  const int gx = (int)((in.nx + P2_TX - 1) / P2_TX), gy = (int)((in.ny + P2_TY - 1) / P2_TY);
  const int64_t tiles = (int64_t)gx * gy;
  const int64_t slots = (int64_t)kNumSMs * per_sm;
  double best = 1e300;
  int best_split = 1;
  for (int split = 1; split <= 256; ++split) {
    int64_t zc = (nzo + split - 1) / split;
    if (split > 1 && zc < 4 * R + 8) break;
    int64_t ctas = tiles * ((nzo + zc - 1) / zc);
    int64_t waves = (ctas + slots - 1) / slots;
    double cost = (double)waves * (double)(zc + 2 * R);
    if (cost < best * 0.98) {
      best = cost;
      best_split = split;
    }
  }
  a.zchunk = (int)((nzo + best_split - 1) / best_split);
  dim3 grid(gx, gy, (unsigned)((nzo + a.zchunk - 1) / a.zchunk));
  kern<<<grid, P2_NT, G::SMEM, s>>>(tin, tout, a);
  return cudaGetLastError();
}

template <bool UNSHARP, typename Tin>
cudaError_t dispatch_p2(int R, const DevIn& in, int64_t zo, int64_t nzo, float* out,
                        const Taps& taps, const EpiArgs& epi, cudaStream_t s) {
  switch (R) {
    case 2: return launch_p2<2, Tin, UNSHARP, 4>(in, zo, nzo, out, taps, epi, s);
    case 3: return launch_p2<3, Tin, UNSHARP, 4>(in, zo, nzo, out, taps, epi, s);
    case 4: return launch_p2<4, Tin, UNSHARP, 4>(in, zo, nzo, out, taps, epi, s);
    case 5: return launch_p2<5, Tin, UNSHARP, 4>(in, zo, nzo, out, taps, epi, s);
    case 6: return launch_p2<6, Tin, UNSHARP, 4>(in, zo, nzo, out, taps, epi, s);
    case 7: return launch_p2<7, Tin, UNSHARP, 4>(in, zo, nzo, out, taps, epi, s);
    case 8: return launch_p2<8, Tin, UNSHARP, 4>(in, zo, nzo, out, taps, epi, s);
  }
  return cudaErrorNotSupported;
}

template <bool UNSHARP>
cudaError_t dispatch_p2_dt(int R, const DevIn& in, int64_t zo, int64_t nzo, float* out,
                           const Taps& taps, const EpiArgs& epi, cudaStream_t s) {
  switch (in.dt) {
    case HB_F32: return dispatch_p2<UNSHARP, float>(R, in, zo, nzo, out, taps, epi, s);
    case HB_U16: return dispatch_p2<UNSHARP, uint16_t>(R, in, zo, nzo, out, taps, epi, s);
    case HB_U8: return dispatch_p2<UNSHARP, uint8_t>(R, in, zo, nzo, out, taps, epi, s);
  }
  return cudaErrorNotSupported;
}


bool envelope_ok(const DevIn& in, int64_t nzo) {
  if (nzo <= 0) return false;
  if (in.nx < 8 || in.ny < 8) return false;  // tiny shapes: generic path
  if (in.nz >= (1 << 30) || in.nx >= (1 << 30) || in.ny >= (1 << 30)) return false;
  return true;
}

}  // namespace

cudaError_t gaussian_fused(const DevIn& in, int64_t zo, int64_t nzo, float* out, const Taps& taps,
                           const EpiArgs& epi, cudaStream_t s, int64_t* launches) {
  if (!envelope_ok(in, nzo) || taps.R > 8) return cudaErrorNotSupported;
  cudaError_t e = cudaErrorNotSupported;
  if (epi.kind == EPI_UNSHARP && (epi.orig != in.p || epi.orig_dt != in.dt)) return cudaErrorNotSupported;
  // warp-specialised kernel first (HB_GAUSS_P2=1: the single-role packed one)
  if (taps.R >= 2 && !std::getenv("HB_GAUSS_SCALAR")) {
    e = gaussian_tri(in, zo, nzo, out, taps, epi, s, launches);
    if (e != cudaErrorNotSupported) return e;
    cudaGetLastError();
    e = gaussian_ws(in, zo, nzo, out, taps, epi, s, launches);
    if (e != cudaErrorNotSupported) return e;
    cudaGetLastError();
  }
  // packed-FP32 kernel for R >= 2 (HB_GAUSS_SCALAR=1 selects the scalar one)
  if (taps.R >= 2 && !std::getenv("HB_GAUSS_SCALAR")) {
    e = epi.kind == EPI_UNSHARP ? dispatch_p2_dt<true>(taps.R, in, zo, nzo, out, taps, epi, s)
                                : dispatch_p2_dt<false>(taps.R, in, zo, nzo, out, taps, epi, s);
    if (e != cudaErrorNotSupported) {
      if (e == cudaSuccess && launches) *launches += 1;
      return e;
    }
    cudaGetLastError();
  }
  if (epi.kind == EPI_UNSHARP) {
    e = dispatch_dt<MODE_GAUSS, true>(taps.R, in, zo, nzo, out, taps, epi, s);
  } else {
    e = dispatch_dt<MODE_GAUSS, false>(taps.R, in, zo, nzo, out, taps, epi, s);
  }
  if (e == cudaSuccess && launches) *launches += 1;
  return e;
}

cudaError_t mean_fused(const DevIn& in, int64_t zo, int64_t nzo, float* out, int r,
                       cudaStream_t s, int64_t* launches) {
  if (!envelope_ok(in, nzo) || r > 3) return cudaErrorNotSupported;
  Taps taps;
  taps.R = r;
  for (int k = 0; k < 2 * r + 1; ++k) taps.w[k] = 1.f;
  EpiArgs epi;
  epi.kind = EPI_BOX_MEAN;
  float size = (float)(2 * r + 1);
  epi.count = size * size * size;
  cudaError_t e = dispatch_dt<MODE_BOX, false>(r, in, zo, nzo, out, taps, epi, s);
  if (e == cudaSuccess && launches) *launches += 1;
  return e;
}

}  // namespace hb
