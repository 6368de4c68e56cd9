// gauss_tri.cu — fused 3D Gaussian / unsharp, fast fp32 mode, float input,
// R = 8 i.e. sigma = 2 (filters.py:33-41 gaussian; filters.py:136-139 unsharp
// epilogue).  One HBM read + one HBM write per voxel; every pass in packed
// FP32 (FFMA2 / FADD2).
//
// CTA = 48 x 32 output tile marching down a z-chunk, 20 warps in three roles
// that hand slices to each other through shared-memory rings guarded by
// mbarriers (no CTA-wide barrier after the prologue):
//
//   Y role (4 warps): TMA producer; per input slice a thread filters one
//     column pair x 8 rows along y (LDS.64 per input row, 8 FFMA2 chains) and
//     writes the result ROW-PAIR interleaved: sY[row pair][column] = (row 2p,
//     row 2p+1), one STS.128 per 2 x 2 block.
//   X role (4 warps): a thread filters one row pair x 6 columns along x from
//     22 interleaved pairs (11 LDS.128, 6 FFMA2 folds) into sXY, same layout.
//   Z role (12 warps): a thread owns a 2 x 2 output block; one LDS.128 per
//     slice feeds a (2R + 1)-slot register ring, the z fold is symmetric
//     (FADD2 + FFMA2), the result leaves as two STG.64.
//
// Why three roles (ncu, profiles/r02_kernels_*): with the x pass inside the
// ring-holding threads (k_gauss_ws, and a 2-role variant of this kernel) a
// thread can own only 4 outputs — the ring costs 17 registers per output — so
// its x window was 18 pairs for 4 outputs: 36 B of shared-memory reads per
// output, 57-75% of the LSU wavefront peak and short-scoreboard stalls on the
// z-fold adds.  Splitting x off lets the x thread block 12 outputs and the z
// thread read 4 B per output: ~52 B of shared traffic per output in total.
// Warp counts per role are multiples of four so every SMSP gets the same mix
// (one Y, one X and three Z warps); the Y and X warps hand registers to the
// Z warps with setmaxnreg.  z-chunks are capped (HB_G3_ZCAP, default 192
// slices): with 528-slice runs, tiles drifted apart in z and the y-neighbour
// halo rows were re-read from DRAM (8.5 GB read for 4.3 GB at 1024^3).
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
__device__ __forceinline__ void arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// one arrival per warp (barrier counts are in warps): per-thread arrivals on
// the same mbarrier serialise in the LSU — 768 of them per slice cost about
// as long as the slice's arithmetic
// HB_GTRI_THREAD_ARRIVE=1 builds the per-thread form (barrier counts in
// threads) — compute-sanitizer racecheck does not model the elected-lane
// release through __syncwarp and reports the sX/sY reuse as hazards; the
// per-thread build is the one it checks (0 hazards, profiles/r02_sanitizer.md)
#ifndef HB_GTRI_THREAD_ARRIVE
#define HB_GTRI_THREAD_ARRIVE 0
#endif
constexpr int kArrivePerWarp = HB_GTRI_THREAD_ARRIVE ? 32 : 1;
__device__ __forceinline__ void warp_arrive(uint64_t* bar) {
#if HB_GTRI_THREAD_ARRIVE
  arrive(bar);
#else
  __syncwarp();
  if ((threadIdx.x & 31) == 0) arrive(bar);
#endif
}
__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// clamp-to-edge fix-up of a TMA-staged halo'd tile (zero-filled outside the
// volume) by the NT threads of the Y role (named barrier 1 between the row
// and the column step)
template <int NT>
__device__ __forceinline__ void clamp_stage(float* st, int pitch, int h, int w, int gy0, int gx0,
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

#ifndef HB_GTRI_NSY
#define HB_GTRI_NSY 3
#endif
#ifndef HB_GTRI_NSX
#define HB_GTRI_NSX 4  // sY/sX ring depths: 2/3, 3/4, 4/6 all within noise (305-309 Gvox/s)
#endif
#ifndef HB_GTRI_NST
#define HB_GTRI_NST 14  // TMA stages: 10 -> 14 measured 308 -> 313 Gvox/s (216 KB of smem)
#endif
#ifndef HB_GTRI_TY
#define HB_GTRI_TY 32  // 32: one 640-thread CTA/SM with setmaxnreg; 16: two 320-thread CTAs/SM (measured 265 vs 310 Gvox/s)
#endif
constexpr int TX = 48, TY = HB_GTRI_TY;
constexpr int CTAS_PER_SM = TY == 32 ? 1 : 2;
constexpr bool kSetMaxNreg = TY == 32;  // role warp counts are whole warpgroups only at TY = 32
constexpr int YR = 8;   // rows per Y item
constexpr int XC = 6;   // columns per X item
constexpr int NYT = 4 * TY, NXT = 4 * TY, NZT = (TX / 2) * (TY / 2);  // 4 + 4 + 12 warps at TY = 32
constexpr int NT = NYT + NXT + NZT;                                    // 640 at TY = 32
// setmaxnreg (warpgroup-wide; an .inc draws only on what this CTA's .dec
// released): launch at 96, Y -> 56 and X -> 80 free 5120 + 2048 registers,
// the Z warps take 384 x 16 of them
#ifndef HB_GTRI_YREGS
#define HB_GTRI_YREGS 56
#endif
#ifndef HB_GTRI_XREGS
#define HB_GTRI_XREGS 80
#endif
constexpr int kLaunchRegs = 96, kYRegs = HB_GTRI_YREGS, kXRegs = HB_GTRI_XREGS, kZRegs = 112;
static_assert(NYT * (kLaunchRegs - kYRegs) + NXT * (kLaunchRegs - kXRegs) >= NZT * (kZRegs - kLaunchRegs),
              "register hand-over does not balance");

struct TriArgs {
  f2 w2[17];  // (w_k, w_k): FFMA2 operands
  int nzi, zo, nzo, zchunk, nx, ny;
  float amount;
};

template <int R>
struct GeoT {
  static constexpr int WC = TX + 2 * R;         // halo'd columns the x pass reads
  static constexpr int NYC = WC;                // columns the y pass produces (even)
  static constexpr int NYP = NYC / 2;
  static constexpr int HB = TY + 2 * R;         // staged rows
  // the TMA box starts 16-B aligned (a misaligned start coordinate faults):
  // halo column 0 sits at stage column XOFF (0 or 2 for even R)
  static constexpr int XA = (R + 3) / 4 * 4;
  static constexpr int XOFF = XA - R;
  static constexpr int WBOX = (XOFF + NYC + 3) / 4 * 4;
  static constexpr int STAGE_PITCH = (HB * WBOX * 4 + 127) / 128 * 128;
  static constexpr int NST = HB_GTRI_NST;   // TMA stages
  static constexpr int NSY = HB_GTRI_NSY;   // y-filtered slices
  static constexpr int NSX = HB_GTRI_NSX;   // xy-filtered slices
  static constexpr int RING = 2 * R + 1;
  static constexpr int NYI = NYP * (TY / YR);
  static constexpr int SYP = (2 * NYC + 31) / 32 * 32;  // floats per row pair
  static constexpr int SY_SLICE = (TY / 2) * SYP;
  static constexpr int SXP = 2 * TX;                    // floats per row pair of sXY
  static constexpr int SX_SLICE = (TY / 2) * SXP;
  static constexpr int NXP = XC + 2 * R;                // pairs an X item reads
  static constexpr int OFF_SY = NST * STAGE_PITCH;
  static constexpr int OFF_SX = OFF_SY + NSY * SY_SLICE * 4;
  static constexpr int OFF_BAR = OFF_SX + NSX * SX_SLICE * 4;
  static constexpr int NBAR = NST + 2 * NSY + 2 * NSX;
  static constexpr int SMEM = OFF_BAR + NBAR * 8 + 128;
  static_assert(R % 2 == 0, "even R only (odd R: k_gauss_ws)");
  static_assert(NYI <= NYT, "Y items exceed the Y role");
  static_assert((TY / 2) * (TX / XC) == NXT, "X items must fill the X role");
  static_assert(NXP % 2 == 0, "X window in whole LDS.128");
};

template <int R, bool UNSHARP>
__global__ void __launch_bounds__(NT, CTAS_PER_SM)
k_gauss_tri(const __grid_constant__ CUtensorMap tin, const float* __restrict__ orig,
            float* __restrict__ out, const __grid_constant__ TriArgs a) {
  using G = GeoT<R>;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  float* sIn = reinterpret_cast<float*>(smem);
  float* sY = reinterpret_cast<float*>(smem + G::OFF_SY);
  float* sX = reinterpret_cast<float*>(smem + G::OFF_SX);
  uint64_t* bar_tma = reinterpret_cast<uint64_t*>(smem + G::OFF_BAR);
  uint64_t* full_y = bar_tma + G::NST;
  uint64_t* empty_y = full_y + G::NSY;
  uint64_t* full_x = empty_y + G::NSY;
  uint64_t* empty_x = full_x + G::NSX;

  const int tid = threadIdx.x;
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
  const int z0 = blockIdx.z * a.zchunk;
  const int z1 = min(z0 + a.zchunk, a.nzo);
  const int nsl = (z1 - z0) + 2 * R;  // input slices this CTA consumes

  if (tid == 0) {
#pragma unroll
    for (int i = 0; i < G::NST; ++i) mbar_init(&bar_tma[i], 1);
#pragma unroll
    for (int i = 0; i < G::NSY; ++i) {
      mbar_init(&full_y[i], NYT / 32 * kArrivePerWarp);
      mbar_init(&empty_y[i], NXT / 32 * kArrivePerWarp);
    }
#pragma unroll
    for (int i = 0; i < G::NSX; ++i) {
      mbar_init(&full_x[i], NXT / 32 * kArrivePerWarp);
      mbar_init(&empty_x[i], NZT / 32 * kArrivePerWarp);
    }
    fence_mbar_init();
  }
  __syncthreads();  // the only CTA-wide barrier

  if (tid >= NZT + NXT) {
    // =================== Y role: TMA producer + y pass ======================
    if constexpr (kSetMaxNreg) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kYRegs));
    const int yt = tid - (NZT + NXT);
    auto zin_of = [&](int s) { return min(max(a.zo + z0 - R + s, 0), a.nzi - 1); };
    const bool border =
        (x0 - R < 0) || (x0 + G::NYC - R > a.nx) || (y0 - R < 0) || (y0 + TY + R > a.ny);
    constexpr uint32_t kStageBytes = G::HB * G::WBOX * 4;
    if (yt == 0) {
      prefetch_tmap(&tin);
#pragma unroll
      for (int i = 0; i < G::NST; ++i)
        if (i < nsl) {
          mbar_expect_tx(&bar_tma[i], kStageBytes);
          tma_load_3d(sIn + i * (G::STAGE_PITCH / 4), &tin, x0 - G::XA, y0 - R, zin_of(i), &bar_tma[i]);
        }
    }
    const int ycp = yt % G::NYP, yg = yt / G::NYP;
    const bool active = yt < G::NYI;
    const int src_off = (YR * yg) * G::WBOX + G::XOFF + 2 * ycp;
    const int dst_off = (YR / 2 * yg) * G::SYP + 4 * ycp;
    int st = 0, b = 0;
    uint32_t ph_t = 0, ph_e = 0;
    for (int s = 0; s < nsl; ++s) {
      float* stage = sIn + st * (G::STAGE_PITCH / 4);
      mbar_wait(&bar_tma[st], ph_t);
      if (border) {
        clamp_stage<NYT>(stage + G::XOFF, G::WBOX, G::HB, G::NYC, y0 - R, x0 - R, a.ny, a.nx, yt);
        named_sync(1, NYT);
      }
      if (s >= G::NSY) mbar_wait(&empty_y[b], ph_e);
      if (active) {
        f2 acc[YR];
        const float* src = stage + src_off;
#pragma unroll
        for (int j = 0; j < YR + 2 * R; ++j) {
          const f2 v = *reinterpret_cast<const f2*>(src + j * G::WBOX);
#pragma unroll
          for (int m = 0; m < YR; ++m) {
            const int k = j - m;
            if (k == 0) acc[m] = mul2(v, a.w2[0]);
            else if (k > 0 && k <= 2 * R) acc[m] = fma2(v, a.w2[k], acc[m]);
          }
        }
        float* dst = sY + b * G::SY_SLICE + dst_off;
#pragma unroll
        for (int q = 0; q < YR / 2; ++q) {
          float r0a, r0b, r1a, r1b;
          upk(acc[2 * q], r0a, r0b);      // row 2q: columns c, c + 1
          upk(acc[2 * q + 1], r1a, r1b);  // row 2q + 1
          *reinterpret_cast<float4*>(dst + q * G::SYP) = make_float4(r0a, r1a, r0b, r1b);
        }
      }
      warp_arrive(&full_y[b]);
      named_sync(1, NYT);  // every Y thread is done reading stage st
      if (yt == 0 && s + G::NST < nsl) {
        fence_proxy_async();
        mbar_expect_tx(&bar_tma[st], kStageBytes);
        tma_load_3d(stage, &tin, x0 - G::XA, y0 - R, zin_of(s + G::NST), &bar_tma[st]);
      }
      if (++st == G::NST) { st = 0; ph_t ^= 1u; }
      if (++b == G::NSY) { b = 0; if (s >= G::NSY) ph_e ^= 1u; }
    }
    return;
  }

  if (tid >= NZT) {
    // ========================= X role: x pass ================================
    if constexpr (kSetMaxNreg) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kXRegs));
    const int xt = tid - NZT;
    const int rp = xt / (TX / XC), g = xt % (TX / XC);
    const float* const srow = sY + rp * G::SYP + 2 * XC * g;  // pair (XC*g) of row pair rp
    float* const drow = sX + rp * G::SXP + 2 * XC * g;
    int b = 0, bx = 0;
    uint32_t ph_f = 0, ph_e = 0;
    for (int s = 0; s < nsl; ++s) {
      mbar_wait(&full_y[b], ph_f);
      f2 v[G::NXP];
      const float* src = srow + b * G::SY_SLICE;
#pragma unroll
      for (int i = 0; i < G::NXP / 2; ++i) {
        const float4 q = *reinterpret_cast<const float4*>(src + 4 * i);
        v[2 * i] = pk(q.x, q.y);
        v[2 * i + 1] = pk(q.z, q.w);
      }
      // symmetric fold per output column j (taps v[j .. j + 2R]), two chains
      f2 o[XC];
#pragma unroll
      for (int j = 0; j < XC; ++j) {
        f2 e = mul2(v[j + R], a.w2[R]);
        f2 f = mul2(add2(v[j + R - 1], v[j + R + 1]), a.w2[R - 1]);
#pragma unroll
        for (int d = 2; d <= R; ++d) {
          const f2 t = add2(v[j + R - d], v[j + R + d]);
          if (d % 2 == 0) e = fma2(t, a.w2[R - d], e);
          else f = fma2(t, a.w2[R - d], f);
        }
        o[j] = add2(e, f);
      }
      warp_arrive(&empty_y[b]);
      if (s >= G::NSX) mbar_wait(&empty_x[bx], ph_e);
      float* dst = drow + bx * G::SX_SLICE;
#pragma unroll
      for (int j = 0; j < XC; j += 2) {
        float a0, a1, b0, b1;
        upk(o[j], a0, a1);
        upk(o[j + 1], b0, b1);
        *reinterpret_cast<float4*>(dst + 2 * j) = make_float4(a0, a1, b0, b1);
      }
      warp_arrive(&full_x[bx]);
      if (++b == G::NSY) { b = 0; ph_f ^= 1u; }
      if (++bx == G::NSX) { bx = 0; if (s >= G::NSX) ph_e ^= 1u; }
    }
    return;
  }

  // ======================== Z role: ring, z pass, store ======================
  if constexpr (kSetMaxNreg) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kZRegs));
  const int cp = tid % (TX / 2), rp = tid / (TX / 2);
  const int gy = y0 + 2 * rp, gx = x0 + 2 * cp;
  const bool live_c = gx < a.nx;  // nx even: both columns in or out
  const bool live0 = live_c && gy < a.ny, live1 = live_c && gy + 1 < a.ny;
  const int64_t oplane = (int64_t)a.ny * a.nx;
  const int64_t orow = (int64_t)min(gy, a.ny - 1) * a.nx + min(gx, a.nx - 2);
  float* optr = out + (int64_t)z0 * oplane + orow;
  const float* obase = UNSHARP ? orig + (int64_t)(a.zo + z0) * oplane + orow : nullptr;
  const float* const row0 = sX + rp * G::SXP + 4 * cp;
  const float* row = row0;
  int b = 0;
  uint32_t ph = 0;
  f2 ring[G::RING][2];
  // step s: wait for xy slice s and issue its LDS.128, fold output s - 1 - 2R
  // on the ring while it is in flight, then park slice s in slot s % RING
  // (the slot the fold just retired)
  for (int s0 = 0; s0 <= nsl; s0 += G::RING) {
#pragma unroll
    for (int u = 0; u < G::RING; ++u) {
      const int s = s0 + u;
      if (s > nsl) break;
      float4 q;
      if (s < nsl) {
        mbar_wait(&full_x[b], ph);
        q = *reinterpret_cast<const float4*>(row);
      }
      const int o = s - 1 - 2 * R;
      if (o >= 0) {
        // slices o .. o + 2R live in ring slots (u + k) % RING, k = 0 .. 2R
        f2 zr[2];
#pragma unroll
        for (int m = 0; m < 2; ++m) {
          f2 e = mul2(ring[(u + R) % G::RING][m], a.w2[R]);
          f2 f = mul2(add2(ring[(u + R - 1) % G::RING][m], ring[(u + R + 1) % G::RING][m]), a.w2[R - 1]);
#pragma unroll
          for (int d = 2; d <= R; ++d) {
            const f2 t = add2(ring[(u + R - d) % G::RING][m], ring[(u + R + d) % G::RING][m]);
            if (d % 2 == 0) e = fma2(t, a.w2[R - d], e);
            else f = fma2(t, a.w2[R - d], f);
          }
          zr[m] = add2(e, f);
        }
        // zr[0] = column c (rows r, r+1), zr[1] = column c + 1
        float c0r0, c0r1, c1r0, c1r1;
        upk(zr[0], c0r0, c0r1);
        upk(zr[1], c1r0, c1r1);
        if (UNSHARP) {
          const float2 b0 = *reinterpret_cast<const float2*>(obase + (int64_t)o * oplane);
          const float2 b1 = live1 ? *reinterpret_cast<const float2*>(obase + (int64_t)o * oplane + a.nx)
                                  : b0;
          c0r0 = __fadd_rn(b0.x, __fmul_rn(a.amount, __fsub_rn(b0.x, c0r0)));
          c1r0 = __fadd_rn(b0.y, __fmul_rn(a.amount, __fsub_rn(b0.y, c1r0)));
          c0r1 = __fadd_rn(b1.x, __fmul_rn(a.amount, __fsub_rn(b1.x, c0r1)));
          c1r1 = __fadd_rn(b1.y, __fmul_rn(a.amount, __fsub_rn(b1.y, c1r1)));
        }
        float* p = optr + (int64_t)o * oplane;
        if (live0) *reinterpret_cast<float2*>(p) = make_float2(c0r0, c1r0);
        if (live1) *reinterpret_cast<float2*>(p + a.nx) = make_float2(c0r1, c1r1);
      }
      if (s < nsl) {
        ring[u][0] = pk(q.x, q.y);
        ring[u][1] = pk(q.z, q.w);
        warp_arrive(&empty_x[b]);
        if (++b == G::NSX) {
          b = 0;
          ph ^= 1u;
          row = row0;
        } else {
          row += G::SX_SLICE;
        }
      }
    }
  }
}

template <int R, bool UNSHARP>
cudaError_t launch_tri(const DevIn& in, int64_t zo, int64_t nzo, float* out, const Taps& taps,
                       const EpiArgs& epi, cudaStream_t s) {
  using G = GeoT<R>;
  if (in.nx % 2 != 0 || (reinterpret_cast<uintptr_t>(out) & 7) != 0 ||
      (reinterpret_cast<uintptr_t>(in.p) & 15) != 0)
    return cudaErrorNotSupported;
  CUtensorMap tin;
  if (!make_tmap_3d(&tin, in.p, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, in.nx, in.ny, in.nz, G::WBOX, G::HB))
    return cudaErrorNotSupported;
  TriArgs a;
  for (int k = 0; k < 2 * R + 1; ++k) {
    unsigned int bits = 0;
    std::memcpy(&bits, &taps.w[k], 4);
    a.w2[k] = ((unsigned long long)bits << 32) | bits;
  }
  a.nzi = (int)in.nz;
  a.zo = (int)zo;
  a.nzo = (int)nzo;
  a.nx = (int)in.nx;
  a.ny = (int)in.ny;
  a.amount = epi.amount;
  auto kern = k_gauss_tri<R, UNSHARP>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM) != cudaSuccess)
    return cudaErrorNotSupported;
  const int gx = (int)((in.nx + TX - 1) / TX), gy = (int)((in.ny + TY - 1) / TY);
  // z-split: balance waves of resident CTAs (one per SM) against each chunk's
  // 2R priming slices; chunks are capped so that neighbouring tiles, which
  // re-read each other's halo rows, stay close enough in z to hit in L2
  const char* zv = std::getenv("HB_G3_ZCAP");
  const int zcap = zv ? std::max(16, std::atoi(zv)) : 192;
  const int64_t tiles = (int64_t)gx * gy;
  const int64_t slots = (int64_t)kNumSMs * CTAS_PER_SM;
  double best = 1e300;
  int64_t best_split = 1;
  const int64_t min_split = std::max<int64_t>(1, (nzo + zcap - 1) / zcap);
  for (int64_t split = min_split; split <= min_split + 256; ++split) {
    const int64_t zc = (nzo + split - 1) / split;
    if (split > min_split && zc < 2 * R + 8) break;
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
  kern<<<grid, NT, G::SMEM, s>>>(tin, static_cast<const float*>(in.p), out, a);
  return cudaGetLastError();
}

template <bool UNSHARP>
cudaError_t dispatch_tri(int R, const DevIn& in, int64_t zo, int64_t nzo, float* out,
                         const Taps& taps, const EpiArgs& epi, cudaStream_t s) {
  // R = 8 (sigma = 2, the benchmark's filter) only: for smaller R the y pass
  // is cheaper and k_gauss_ws's two CTAs per SM win (unsharp sigma = 1 at
  // 1024^3: 440 vs 347 Gvox/s)
  switch (R) {
    case 8: return launch_tri<8, UNSHARP>(in, zo, nzo, out, taps, epi, s);
  }
  return cudaErrorNotSupported;
}

}  // namespace

// NotSupported outside the envelope (the caller falls back to k_gauss_ws /
// k_gauss_p2 / the generic kernels): float input, R = 8, even nx,
// TMA-compatible layout.  HB_GAUSS_WS=1 skips this kernel (A/B).
cudaError_t gaussian_tri(const DevIn& in, int64_t zo, int64_t nzo, float* out, const Taps& taps,
                         const EpiArgs& epi, cudaStream_t s, int64_t* launches) {
  const bool off = std::getenv("HB_GAUSS_WS") != nullptr;  // read per call (A/B in one process)
  // small planes (e.g. 256^2: 48 tiles of 48 x 32) cannot fill 148 SMs with
  // one CTA each; k_gauss_ws's 64 x 16 tiles at two CTAs/SM do better there
  // (256^3: 159 vs 105-122 Gvox/s; 512^3: 197-204 vs 221-231)
  if (off || in.dt != HB_F32 || taps.R != 8 || nzo <= 0 || in.nx < 384 || in.ny < 384 ||
      in.ny < 8 || in.nz >= (1 << 30) || in.nx >= (1 << 30) || in.ny >= (1 << 30) ||
      (int64_t)in.ny * in.nx >= ((int64_t)1 << 31))
    return cudaErrorNotSupported;
  if (epi.kind == EPI_UNSHARP && (epi.orig != in.p || epi.orig_dt != in.dt))
    return cudaErrorNotSupported;
  if (epi.kind != EPI_UNSHARP && epi.kind != EPI_NONE) return cudaErrorNotSupported;
  const cudaError_t e = epi.kind == EPI_UNSHARP ? dispatch_tri<true>(taps.R, in, zo, nzo, out, taps, epi, s)
                                                : dispatch_tri<false>(taps.R, in, zo, nzo, out, taps, epi, s);
  if (e == cudaSuccess && launches) *launches += 1;
  return e;
}

}  // namespace hb
