// gauss_ws.cu — warp-specialised fused 3D Gaussian / unsharp (fast fp32 mode),
// 2 <= R <= 8 (sigma <= 2): filters.py:33-41 (gaussian), filters.py:136-139
// (unsharp epilogue).  One HBM read + one HBM write per voxel.
//
// CTA = 64 x 16 output tile marching down a z-chunk, two warp roles that
// never meet at a CTA-wide barrier:
//
//   Y warps (NYW = ceil(items / 32)): per input slice, wait for its TMA
//     stage (mbarrier tx), filter the halo'd 80-column tile along y —
//     column pairs x 4 rows per thread, packed FP32 (FFMA2), one LDS.64 per
//     input row pair — into a 4-deep ring of y-filtered slices (sY), then
//     arrive on that slot's FULL barrier.  A named barrier among the Y warps
//     retires the TMA stage and thread 0 refills it (slice s + 4).
//   X/Z warps (8 warps, 256 threads): thread (row, 4 x) waits on FULL,
//     filters its 4 outputs along x (scalar FFMA from five LDS.128 — the
//     shifted taps of x-adjacent outputs do not form register pairs), arrives
//     on the slot's EMPTY barrier, keeps the results in a (2R+1)-slot
//     register ring of x-pairs, and once the ring is primed runs the z pass
//     (symmetric fold, FFMA2) and stores the 4 outputs with one STG.128.
//
// The slice loop is unrolled by the ring period so every ring index is a
// compile-time register (no switch / indirect branch); producer/consumer
// slack of up to 4 slices replaces the lock-step __syncthreads of the
// single-role kernel (k_gauss_p2, whose ncu profile showed barrier and
// fixed-latency stalls as the top two reasons with 5 of 8 warps busy in the
// y pass).  Pass order (Y, X, Z) differs from the reference's (Z, Y, X): fp32
// rounding stays ~2e-7 relative (tests pin <= 1e-5); the exact mode is
// gauss_exact.cu.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <type_traits>

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
template <typename T> __device__ __forceinline__ f2 load_pair(const T* p) {
  return pk((float)p[0], (float)p[1]);
}
template <> __device__ __forceinline__ f2 load_pair<float>(const float* p) {
  return *reinterpret_cast<const f2*>(p);
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// clamp-to-edge fix-up of a TMA-staged halo'd tile (zero-filled outside the
// volume), synchronising only the NT threads of the Y role (named barrier 1)
template <typename T, int NT>
__device__ __forceinline__ void clamp_tile_y(T* st, int pitch, int h, int w, int gy0, int gx0,
                                             int ny, int nx, int tid) {
  const int r_lo = max(0, -gy0), r_hi = min(h, ny - gy0);
  if (r_lo > 0 || r_hi < h) {
    const int nbad = r_lo + (h - r_hi);
    for (int e = tid; e < nbad * w; e += NT) {
      const int i = e / w, c = e - i * w;
      const int r = i < r_lo ? i : r_hi + (i - r_lo);
      const int src = i < r_lo ? r_lo : r_hi - 1;
      st[r * pitch + c] = st[src * pitch + c];
    }
    named_sync(1, NT);
  }
  const int c_lo = max(0, -gx0), c_hi = min(w, nx - gx0);
  if (c_lo > 0 || c_hi < w) {
    const int nbc = c_lo + (w - c_hi);
    for (int e = tid; e < h * nbc; e += NT) {
      const int r = e / nbc, i = e - r * nbc;
      const int c = i < c_lo ? i : c_hi + (i - c_lo);
      const int src = i < c_lo ? c_lo : c_hi - 1;
      st[r * pitch + c] = st[r * pitch + src];
    }
  }
}

template <typename T> struct TmaT;
template <> struct TmaT<float> { static constexpr CUtensorMapDataType v = CU_TENSOR_MAP_DATA_TYPE_FLOAT32; };
template <> struct TmaT<uint16_t> { static constexpr CUtensorMapDataType v = CU_TENSOR_MAP_DATA_TYPE_UINT16; };
template <> struct TmaT<uint8_t> { static constexpr CUtensorMapDataType v = CU_TENSOR_MAP_DATA_TYPE_UINT8; };

constexpr int TY = 16;
constexpr int YR = 4;  // rows per y item

struct WSArgs {
  unsigned long long w2[17];  // (w_k, w_k) pairs for FFMA2 (uniform registers)
  float w1[17];               // w_k for the scalar x pass (constant-bank operands)
  int nzi, zo, nzo, zchunk, nx, ny;
  float amount;
};

// TX = 64: 256 X/Z threads (8 warps) + 160 Y threads (5 warps); TX = 48: 192 +
// 128 (6 + 4 warps) — 48 columns make the y items (32 column pairs x 4 row
// groups) exactly four warps and leave 102 registers per thread at two CTAs
// per SM (the 64-wide tile spills its ring at that occupancy).
template <int R, typename Tin, int TX_>
struct Geo {
  static constexpr int TX = TX_;
  static constexpr int XQ = TX / 4;          // x quads per row
  static constexpr int XZT = XQ * TY;        // X/Z threads (4 outputs each)
  static constexpr int WC = TX + 2 * R;
  static constexpr int HB = TY + 2 * R;
  static constexpr int ALIGN = 16 / (int)sizeof(Tin);
  static constexpr int XA = (R + ALIGN - 1) / ALIGN * ALIGN;  // 16-B aligned box start
  static constexpr int XOFF = XA - R;                         // stage col of halo col 0
  static constexpr int YC0 = XOFF & ~1;                       // even first y column
  static constexpr int YOFF = XOFF - YC0;                     // sY col of halo col 0
  static constexpr int NYC = (YOFF + WC + 1) / 2 * 2;
  static constexpr int NYP = NYC / 2;
  static constexpr int WBOX0 = (XA + TX + R) > (YC0 + NYC) ? (XA + TX + R) : (YC0 + NYC);
  static constexpr int WBOX = (WBOX0 + ALIGN - 1) / ALIGN * ALIGN;
  static constexpr int STAGE_BYTES = HB * WBOX * (int)sizeof(Tin);
  static constexpr int STAGE_PITCH = (STAGE_BYTES + 127) / 128 * 128;
  static constexpr int NST = 4;  // TMA stages
  static constexpr int NSY = 4;  // y-filtered slices in flight
  static constexpr int RING = 2 * R + 1;
  static constexpr int NYI = NYP * (TY / YR);
  static constexpr int NYW = (NYI + 31) / 32;
  static constexpr int NYT = NYW * 32;
  static constexpr int NT = XZT + NYT;
  // sY row pitch: = 16 (mod 32) floats, so the 8-thread phases of the x pass's
  // LDS.128 that straddle two rows hit disjoint banks
  static constexpr int SYP = (NYC + 15) / 32 * 32 + 16;
  static constexpr int SY_SLICE = TY * SYP;
  static constexpr int OFF_SY = NST * STAGE_PITCH;
  static constexpr int OFF_BAR = OFF_SY + NSY * SY_SLICE * 4;
  static constexpr int SMEM = OFF_BAR + (NST + 2 * NSY) * 8 + 128;
  static_assert(XZT % 32 == 0, "X/Z role must be whole warps");
};

#ifndef HB_SLEEP_NS
#define HB_SLEEP_NS 0  // measured: no gain from a suspend hint over plain try_wait
#endif
// mbarrier wait with a suspend-time hint: the warp sleeps until the phase
// completes (or the hint expires) instead of spinning try_wait + branch
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
#if HB_SLEEP_NS == 0
  mbar_wait(bar, parity);
  return;
#endif
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAITS_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
      "@!P1 bra WAITS_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity), "r"(HB_SLEEP_NS)
      : "memory");
}

template <typename Tin> struct Vec4;
template <> struct Vec4<float> {
  static __device__ __forceinline__ void get(const float* p, float* v) {
    const float4 q = __ldg(reinterpret_cast<const float4*>(p));
    v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
  }
};
template <> struct Vec4<uint16_t> {
  static __device__ __forceinline__ void get(const uint16_t* p, float* v) {
    const ushort4 q = __ldg(reinterpret_cast<const ushort4*>(p));
    v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
  }
};
template <> struct Vec4<uint8_t> {
  static __device__ __forceinline__ void get(const uint8_t* p, float* v) {
    const uchar4 q = __ldg(reinterpret_cast<const uchar4*>(p));
    v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
  }
};

template <int R, typename Tin, bool UNSHARP, int TX>
__global__ void __launch_bounds__(Geo<R, Tin, TX>::NT, 2)
k_gauss_ws(const __grid_constant__ CUtensorMap tin, const Tin* __restrict__ orig,
           float* __restrict__ out, const __grid_constant__ WSArgs a) {
  using G = Geo<R, Tin, TX>;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  Tin* sIn = reinterpret_cast<Tin*>(smem);
  float* sY = reinterpret_cast<float*>(smem + G::OFF_SY);
  uint64_t* bar_tma = reinterpret_cast<uint64_t*>(smem + G::OFF_BAR);
  uint64_t* bar_full = bar_tma + G::NST;
  uint64_t* bar_empty = bar_full + G::NSY;

  const int tid = threadIdx.x;
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
  const int z0 = blockIdx.z * a.zchunk;
  const int z1 = min(z0 + a.zchunk, a.nzo);
  const int nsl = (z1 - z0) + 2 * R;  // input slices this CTA consumes
  auto zin_of = [&](int s) { return min(max(a.zo + z0 - R + s, 0), a.nzi - 1); };

  if (tid == 0) {
#pragma unroll
    for (int i = 0; i < G::NST; ++i) mbar_init(&bar_tma[i], 1);
#pragma unroll
    for (int i = 0; i < G::NSY; ++i) {
      mbar_init(&bar_full[i], G::NYT);
      mbar_init(&bar_empty[i], G::XZT);
    }
    fence_mbar_init();
  }
  __syncthreads();  // the only CTA-wide barrier

  if (tid >= G::XZT) {
    // =================== Y role: TMA producer + y pass ======================
    const int yt = tid - G::XZT;
    const bool border =
        (x0 - R < 0) || (x0 + TX + R > a.nx) || (y0 - R < 0) || (y0 + TY + R > a.ny);
    if (yt == 0) {
      prefetch_tmap(&tin);
#pragma unroll
      for (int i = 0; i < G::NST; ++i)
        if (i < nsl) {
          mbar_expect_tx(&bar_tma[i], G::HB * G::WBOX * sizeof(Tin));
          tma_load_3d(sIn + i * (G::STAGE_PITCH / sizeof(Tin)), &tin, x0 - G::XA, y0 - R,
                      zin_of(i), &bar_tma[i]);
        }
    }
    const int ycp = yt % G::NYP, yg = yt / G::NYP;
    const bool active = yt < G::NYI;
    const f2* W = a.w2;
    const int src_off = (YR * yg) * G::WBOX + G::YC0 + 2 * ycp;
    const int dst_off = (YR * yg) * G::SYP + 2 * ycp;
    int st = 0, b = 0;          // TMA stage / sY slot of slice s
    uint32_t ph_t = 0, ph_e = 1;  // their phases (EMPTY starts released)
    for (int s = 0; s < nsl; ++s) {
      Tin* stage = sIn + st * (G::STAGE_PITCH / sizeof(Tin));
      mbar_wait_sleep(&bar_tma[st], ph_t);
      if (border) {
        clamp_tile_y<Tin, G::NYT>(stage + G::XOFF, G::WBOX, G::HB, G::WC, y0 - R, x0 - R, a.ny,
                                  a.nx, yt);
        fence_proxy_async();
        named_sync(1, G::NYT);
      }
      if (s >= G::NSY) mbar_wait_sleep(&bar_empty[b], ph_e);
      if (active) {
        f2 acc[YR];
        const Tin* src = stage + src_off;
#pragma unroll
        for (int j = 0; j < YR + 2 * R; ++j) {
          const f2 v = load_pair<Tin>(src + j * G::WBOX);
#pragma unroll
          for (int m = 0; m < YR; ++m) {
            const int k = j - m;
            if (k == 0) acc[m] = mul2(v, W[0]);
            else if (k > 0 && k <= 2 * R) acc[m] = fma2(v, W[k], acc[m]);
          }
        }
        float* dst = sY + b * G::SY_SLICE + dst_off;
#pragma unroll
        for (int m = 0; m < YR; ++m) *reinterpret_cast<f2*>(dst + m * G::SYP) = acc[m];
      }
      mbar_arrive(&bar_full[b]);
      named_sync(1, G::NYT);  // every Y thread is done reading stage st
      if (yt == 0 && s + G::NST < nsl) {
        fence_proxy_async();
        mbar_expect_tx(&bar_tma[st], G::HB * G::WBOX * sizeof(Tin));
        tma_load_3d(stage, &tin, x0 - G::XA, y0 - R, zin_of(s + G::NST), &bar_tma[st]);
      }
      if (++st == G::NST) { st = 0; ph_t ^= 1u; }
      if (++b == G::NSY) { b = 0; if (s >= G::NSY) ph_e ^= 1u; else ph_e = 0u; }
    }
    return;
  }

  // ===================== X/Z role: x pass, ring, z pass ======================
  const int yr = tid / G::XQ, xq = tid - yr * G::XQ;
  const int gy = y0 + yr, gx = x0 + 4 * xq;
  const bool live = gy < a.ny && gx < a.nx;  // nx % 4 == 0: the 4 outputs are all in or out
  const f2* W = a.w2;
  float* optr = out + ((int64_t)z0 * a.ny + min(gy, a.ny - 1)) * a.nx + min(gx, a.nx - 4);
  const int64_t oplane = (int64_t)a.ny * a.nx;
  const Tin* obase = UNSHARP ? orig + ((int64_t)(a.zo + z0) * a.ny + min(gy, a.ny - 1)) * a.nx +
                                   min(gx, a.nx - 4)
                             : nullptr;
  const float* const row0 = sY + yr * G::SYP + G::YOFF + 4 * xq;
  const float* row = row0;   // this thread's row in sY slot b
  int b = 0;
  uint32_t ph = 0;
  f2 ring[G::RING][2];

  auto xpass = [&](f2& out0, f2& out1) {
    mbar_wait_sleep(&bar_full[b], ph);
    float xa[4], xb[4];
    auto tap = [&](int c, float v) {
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const int k = c - m;
        if (k == 0) xa[m] = v * a.w1[0];
        else if (k == R + 1) xb[m] = v * a.w1[R + 1];
        else if (k > 0 && k <= R) xa[m] = fmaf(v, a.w1[k], xa[m]);
        else if (k > R + 1 && k <= 2 * R) xb[m] = fmaf(v, a.w1[k], xb[m]);
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
    mbar_arrive(&bar_empty[b]);  // the slot's values are in registers
    if (++b == G::NSY) {
      b = 0;
      ph ^= 1u;
      row = row0;
    } else {
      row += G::SY_SLICE;
    }
    out0 = pk(xa[0] + xb[0], xa[1] + xb[1]);
    out1 = pk(xa[2] + xb[2], xa[3] + xb[3]);
  };

  for (int s0 = 0; s0 < nsl; s0 += G::RING) {
#pragma unroll
    for (int u = 0; u < G::RING; ++u) {
      const int s = s0 + u;
      if (s < nsl) {
        xpass(ring[u][0], ring[u][1]);
        const int o = s - 2 * R;  // output slice produced now
        if (o >= 0) {
          f2 zr[2];
#pragma unroll
          for (int m = 0; m < 2; ++m) {
            f2 acc = mul2(ring[(u + 1 + R) % G::RING][m], W[R]);
#pragma unroll
            for (int d = R; d >= 1; --d)
              acc = fma2(add2(ring[(u + 1 + R - d) % G::RING][m], ring[(u + 1 + R + d) % G::RING][m]),
                         W[R - d], acc);
            zr[m] = acc;
          }
          float r[4];
          upk(zr[0], r[0], r[1]);
          upk(zr[1], r[2], r[3]);
          if (UNSHARP) {
            float bse[4];
            Vec4<Tin>::get(obase + (int64_t)o * oplane, bse);
#pragma unroll
            for (int m = 0; m < 4; ++m) r[m] = __fadd_rn(bse[m], __fmul_rn(a.amount, __fsub_rn(bse[m], r[m])));
          }
          if (live) *reinterpret_cast<float4*>(optr + (int64_t)o * oplane) = make_float4(r[0], r[1], r[2], r[3]);
        }
      }
    }
  }
}

template <int R, typename Tin, bool UNSHARP, int TX>
cudaError_t launch_ws(const DevIn& in, int64_t zo, int64_t nzo, float* out, const Taps& taps,
                      const EpiArgs& epi, cudaStream_t s) {
  using G = Geo<R, Tin, TX>;
  if (in.nx % 4 != 0 || (reinterpret_cast<uintptr_t>(out) & 15) != 0) return cudaErrorNotSupported;
  CUtensorMap tin;
  if (!make_tmap_3d(&tin, in.p, TmaT<Tin>::v, sizeof(Tin), in.nx, in.ny, in.nz, G::WBOX, G::HB))
    return cudaErrorNotSupported;
  WSArgs a;
  for (int k = 0; k < 2 * R + 1; ++k) {
    unsigned int bits = 0;
    std::memcpy(&bits, &taps.w[k], 4);
    a.w2[k] = ((unsigned long long)bits << 32) | bits;
    a.w1[k] = taps.w[k];
  }
  a.nzi = (int)in.nz;
  a.zo = (int)zo;
  a.nzo = (int)nzo;
  a.nx = (int)in.nx;
  a.ny = (int)in.ny;
  a.amount = epi.amount;
  auto kern = k_gauss_ws<R, Tin, UNSHARP, TX>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM);
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, G::NT, G::SMEM) != cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
  const int gx = (int)((in.nx + TX - 1) / TX), gy = (int)((in.ny + TY - 1) / TY);
  // z-split: balance waves of resident CTAs against each chunk's 2R priming slices
  const int64_t tiles = (int64_t)gx * gy;
  const int64_t slots = (int64_t)kNumSMs * per_sm;
  double best = 1e300;
  int best_split = 1;
  for (int split = 1; split <= 256; ++split) {
    const int64_t zc = (nzo + split - 1) / split;
    if (split > 1 && zc < 2 * R + 8) break;
    const int64_t ctas = tiles * ((nzo + zc - 1) / zc);
    const int64_t waves = (ctas + slots - 1) / slots;
    const double cost = (double)waves * (double)(zc + 2 * R);
    if (cost < best * 0.98) {
      best = cost;
      best_split = split;
    }
  }
  a.zchunk = (int)((nzo + best_split - 1) / best_split);
  dim3 grid(gx, gy, (unsigned)((nzo + a.zchunk - 1) / a.zchunk));
  kern<<<grid, G::NT, G::SMEM, s>>>(tin, static_cast<const Tin*>(in.p), out, a);
  return cudaGetLastError();
}

// Tile width: 64 by default — at 1024^3, 26 warps/SM with a partly spilled
// ring (72 registers) ran ~8% faster than the unspilled 48-wide tile's 20
// warps; HB_GWS_TX=48 selects the narrower tile (better on some small grids,
// e.g. 512^3: 250 vs 200 Gvox/s, from wave quantisation).
template <int R, typename Tin, bool UNSHARP>
cudaError_t launch_tx(const DevIn& in, int64_t zo, int64_t nzo, float* out, const Taps& taps,
                      const EpiArgs& epi, cudaStream_t s) {
  const char* v = std::getenv("HB_GWS_TX");
  return (v && std::atoi(v) == 48) ? launch_ws<R, Tin, UNSHARP, 48>(in, zo, nzo, out, taps, epi, s)
                                   : launch_ws<R, Tin, UNSHARP, 64>(in, zo, nzo, out, taps, epi, s);
}

template <bool UNSHARP, typename Tin>
cudaError_t dispatch_r(int R, const DevIn& in, int64_t zo, int64_t nzo, float* out,
                       const Taps& taps, const EpiArgs& epi, cudaStream_t s) {
  switch (R) {
    case 2: return launch_tx<2, Tin, UNSHARP>(in, zo, nzo, out, taps, epi, s);
    case 3: return launch_tx<3, Tin, UNSHARP>(in, zo, nzo, out, taps, epi, s);
    case 4: return launch_tx<4, Tin, UNSHARP>(in, zo, nzo, out, taps, epi, s);
    case 5: return launch_tx<5, Tin, UNSHARP>(in, zo, nzo, out, taps, epi, s);
    case 6: return launch_tx<6, Tin, UNSHARP>(in, zo, nzo, out, taps, epi, s);
    case 7: return launch_tx<7, Tin, UNSHARP>(in, zo, nzo, out, taps, epi, s);
    case 8: return launch_tx<8, Tin, UNSHARP>(in, zo, nzo, out, taps, epi, s);
  }
  return cudaErrorNotSupported;
}

}  // namespace

// NotSupported outside the envelope (the caller falls back to k_gauss_p2 /
// the generic kernels): 2 <= R <= 8, nx % 4 == 0, TMA-compatible layout.
cudaError_t gaussian_ws(const DevIn& in, int64_t zo, int64_t nzo, float* out, const Taps& taps,
                        const EpiArgs& epi, cudaStream_t s, int64_t* launches) {
  if (taps.R < 2 || taps.R > 8 || nzo <= 0 || in.nx < 8 || in.ny < 8 || in.nz >= (1 << 30) ||
      in.nx >= (1 << 30) || in.ny >= (1 << 30) || std::getenv("HB_GAUSS_P2"))
    return cudaErrorNotSupported;
  if (epi.kind == EPI_UNSHARP && (epi.orig != in.p || epi.orig_dt != in.dt))
    return cudaErrorNotSupported;
  if (epi.kind != EPI_UNSHARP && epi.kind != EPI_NONE) return cudaErrorNotSupported;
  cudaError_t e = cudaErrorNotSupported;
  const bool un = epi.kind == EPI_UNSHARP;
  switch (in.dt) {
    case HB_F32: e = un ? dispatch_r<true, float>(taps.R, in, zo, nzo, out, taps, epi, s)
                        : dispatch_r<false, float>(taps.R, in, zo, nzo, out, taps, epi, s); break;
    case HB_U16: e = un ? dispatch_r<true, uint16_t>(taps.R, in, zo, nzo, out, taps, epi, s)
                        : dispatch_r<false, uint16_t>(taps.R, in, zo, nzo, out, taps, epi, s); break;
    case HB_U8: e = un ? dispatch_r<true, uint8_t>(taps.R, in, zo, nzo, out, taps, epi, s)
                       : dispatch_r<false, uint8_t>(taps.R, in, zo, nzo, out, taps, epi, s); break;
  }
  if (e == cudaSuccess && launches) *launches += 1;
  return e;
}

}  // namespace hb
