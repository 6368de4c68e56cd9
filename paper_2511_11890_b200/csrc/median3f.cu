// median3f.cu — 3x3x3 median of float32 (filters.py:78-82 -> scipy
// median_filter -> rank_filter, rank 13 of 27, clamp-to-edge).  The order
// statistic is one of the inputs, so the result is bit-exact.
//
// Same plane / merge / select networks as k_median3_plane (median.cu), with
// the overhead that made up ~46 of its 154 instructions per voxel removed
// (ncu source view, profiles/r02_kernels_*):
//   * the input tile arrives by TMA (one 3D box per slice into a 6-deep
//     mbarrier ring) instead of 3 LDG + address arithmetic + STS per thread;
//   * no order-preserving key conversion on the way in or out: minima are
//     FMNMX / FMNMX3 on the floats (IEEE order, -0 < +0), and the partner
//     maximum of a compare-exchange is a + b - min on the raw bit patterns
//     (IMAD, exact mod 2^32: min is one of the two inputs), which moves half
//     of every compare-exchange to the FMA pipe;
//   * 32-bit per-CTA bookkeeping, predicated STG.64 stores;
//   * the 3x3 tableau's exchanges in min/max (ALU-only) form: the kernel is
//     issue-bound with ALU-pipe headroom, and an ALU exchange is 2 issue
//     slots against 3 (1024^3: 231 -> 244 Gvox/s).
// The TMA box starts 16-B aligned at x0 - 4 (a misaligned start coordinate
// faults), so a thread reads its x-1 .. x+2 columns as three LDS.64.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "median_nets.h"
#include "ops.cuh"
#include "tma.cuh"

namespace hb {
namespace {

#ifndef HB_M3_TAB_IMAD
#define HB_M3_TAB_IMAD 0
#endif
#ifndef HB_M3_ASM_EMIT
#define HB_M3_ASM_EMIT 0
#endif
#ifndef HB_M3_SHARED_ROWSUM
#define HB_M3_SHARED_ROWSUM 1  // x-row sorts of the two outputs share r1 + r2 (one IMAD fewer per row)
#endif
#ifndef HB_M3_ALU_EVERY
#define HB_M3_ALU_EVERY 0  // merge exchanges in ALU form: 1, 2, 3 measured 226, 238, 240 vs 244 Gvox/s at 0
#endif
constexpr int TXO = 64, TYO = 8;       // outputs per CTA slice (32 x-pairs x 8 rows)
constexpr int SW = 72, SH = TYO + 2;   // staged box: columns x0-4 .. x0+67, rows y0-1 .. y0+8
constexpr int NST = 6;                 // TMA stages
constexpr int STAGE_FLOATS = SW * SH;  // 2880 B (a multiple of 128 B? no: padded below)
constexpr int STAGE_PITCH = (STAGE_FLOATS * 4 + 127) / 128 * 128 / 4;

__device__ __forceinline__ int imad(int a, int b, int c) {
  int d;
  asm("mad.lo.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
__device__ __forceinline__ int fmn(int a, int b) {
  return __float_as_int(fminf(__int_as_float(a), __int_as_float(b)));
}
__device__ __forceinline__ int fmx(int a, int b) {
  return __float_as_int(fmaxf(__int_as_float(a), __int_as_float(b)));
}
__device__ __forceinline__ int fmn3(int a, int b, int c) {
  float r;
  asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(__int_as_float(a)), "f"(__int_as_float(b)), "f"(__int_as_float(c)));
  return __float_as_int(r);
}
__device__ __forceinline__ int fmx3(int a, int b, int c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(__int_as_float(a)), "f"(__int_as_float(b)), "f"(__int_as_float(c)));
  return __float_as_int(r);
}

// networks on float bit patterns held in int registers
struct NetF {
  int one, mone;  // runtime 1 / -1: IMAD, not IADD3 (the ALU pipe is the scarce one)
  __device__ __forceinline__ void ce(int& a, int& b) const {
    const int lo = fmn(a, b);
    const int s = imad(a, one, b);
    b = imad(lo, mone, s);
    a = lo;
  }
  // compare-exchange entirely on the ALU pipe (2 issue slots instead of 3):
  // the kernel is issue-bound with ALU-pipe headroom (ncu: issue 84%, ALU
  // 67%), so a share of the exchanges use this form
  __device__ __forceinline__ void ce_alu(int& a, int& b) const {
    const int lo = fmn(a, b);
    b = fmx(a, b);
    a = lo;
  }
  __device__ __forceinline__ void sort3(int& a, int& b, int& c) const {
    const int lo = fmn3(a, b, c);
    const int hi = fmx3(a, b, c);
    int t = imad(a, one, b);
    t = imad(c, one, t);
    t = imad(lo, mone, t);
    b = imad(hi, mone, t);
    a = lo;
    c = hi;
  }
  // 3x3 matrix sorted along both axes -> ascending s[0..8] (7 CE)
  __device__ __forceinline__ void tableau(const int (&m)[3][3], int (&s)[9]) const {
    s[0] = m[0][0]; s[1] = m[0][1]; s[2] = m[1][0]; s[3] = m[0][2]; s[4] = m[1][1];
    s[5] = m[2][0]; s[6] = m[1][2]; s[7] = m[2][1]; s[8] = m[2][2];
    // the first HB_M3_TAB_IMAD exchanges in min + IMAD form, the rest ALU-only
    // (balances the ALU pipe against issue)
#define HB_TCE(n, i, j) if ((n) < HB_M3_TAB_IMAD) ce(s[i], s[j]); else ce_alu(s[i], s[j]);
    HB_TCE(0, 3, 5) HB_TCE(1, 1, 2) HB_TCE(2, 2, 3) HB_TCE(3, 6, 7)
    HB_TCE(4, 5, 6) HB_TCE(5, 3, 4) HB_TCE(6, 4, 5)
#undef HB_TCE
  }
  // sorted planes of the two x-adjacent outputs from r[row][x-1 .. x+2]
  __device__ __forceinline__ void planes2(int (&r)[3][4], int (&pa)[9], int (&pb)[9]) const {
#pragma unroll
    for (int j = 0; j < 4; ++j) sort3(r[0][j], r[1][j], r[2][j]);
    int a[3][3], b[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
#if HB_M3_SHARED_ROWSUM
      // the two rows share r1, r2: their sum once, each middle = total - min - max
      const int s12 = imad(r[i][1], one, r[i][2]);
      a[i][0] = fmn3(r[i][0], r[i][1], r[i][2]);
      a[i][2] = fmx3(r[i][0], r[i][1], r[i][2]);
      a[i][1] = imad(a[i][2], mone, imad(a[i][0], mone, imad(r[i][0], one, s12)));
      b[i][0] = fmn3(r[i][1], r[i][2], r[i][3]);
      b[i][2] = fmx3(r[i][1], r[i][2], r[i][3]);
      b[i][1] = imad(b[i][2], mone, imad(b[i][0], mone, imad(r[i][3], one, s12)));
#else
      a[i][0] = r[i][0]; a[i][1] = r[i][1]; a[i][2] = r[i][2];
      b[i][0] = r[i][1]; b[i][1] = r[i][2]; b[i][2] = r[i][3];
      sort3(a[i][0], a[i][1], a[i][2]);
      sort3(b[i][0], b[i][1], b[i][2]);
#endif
    }
    tableau(a, pa);
    tableau(b, pb);
  }
  // ranks 4..13 of cur ∪ nxt (two sorted 9-lists)
  __device__ __forceinline__ void merge(const int (&cur)[9], const int (&nxt)[9], int (&m)[10]) const {
    int w[18];
#pragma unroll
    for (int i = 0; i < 9; ++i) {
      w[i] = cur[i];
      w[9 + i] = nxt[i];
    }
    int nce = 0;  // compile-time after unrolling: every HB_M3_ALU_EVERY-th exchange in ALU form
#define HB_CE(i, j) \
  if (HB_M3_ALU_EVERY > 0 && (nce++ % HB_M3_ALU_EVERY) == 0) ce_alu(w[i], w[j]); else ce(w[i], w[j]);
#define HB_MN(i, j) w[i] = fmn(w[i], w[j]);
#define HB_MX(i, j) w[j] = fmx(w[i], w[j]);
    HB_MERGE9_RANK4_13(HB_CE, HB_MN, HB_MX)
#undef HB_CE
#undef HB_MN
#undef HB_MX
#pragma unroll
    for (int i = 0; i < 10; ++i) m[i] = w[4 + i];
  }
  // rank 13 of M ∪ P: min over j of max(M[13-j], P[j-1])
  __device__ __forceinline__ int select(const int (&m)[10], const int (&p)[9]) const {
    const int t1 = fmx(m[8], p[0]), t2 = fmx(m[7], p[1]), t3 = fmx(m[6], p[2]);
    const int t4 = fmx(m[5], p[3]), t5 = fmx(m[4], p[4]), t6 = fmx(m[3], p[5]);
    const int t7 = fmx(m[2], p[6]), t8 = fmx(m[1], p[7]), t9 = fmx(m[0], p[8]);
    int r = fmn3(m[9], t1, t2);
    r = fmn3(r, t3, t4);
    r = fmn3(r, t5, t6);
    r = fmn3(r, t7, t8);
    return fmn(r, t9);
  }
};

struct M3Args {
  int nz, ny, nx, zo, nzo, zchunk;
  int one, mone;
};

template <bool LCLAMP>
__global__ void __launch_bounds__(256, 3)
k_median3_f32(const __grid_constant__ CUtensorMap tin, float* __restrict__ out,
              const __grid_constant__ M3Args a) {
  __shared__ __align__(128) float stage[NST][STAGE_PITCH];
  __shared__ __align__(8) uint64_t bar[NST];
  const NetF net{a.one, a.mone};
  const int tid = threadIdx.x;
  const int tx = tid & 31, ty = tid >> 5;
  const int x0 = blockIdx.x * TXO, y0 = blockIdx.y * TYO;
  const int zs = blockIdx.z * a.zchunk;
  const int ze = min(zs + a.zchunk, a.nzo);
  const int cnt = ze - zs + 2;  // input slices: block z (zo + zs - 1) .. (zo + ze)
  const int zb0 = a.zo + zs - 1;
  auto zin = [&](int k) { return min(max(zb0 + k, 0), a.nz - 1); };
  constexpr uint32_t kBytes = SW * SH * 4;
  if (tid == 0) {
#pragma unroll
    for (int i = 0; i < NST; ++i) mbar_init(&bar[i], 1);
    fence_mbar_init();
    prefetch_tmap(&tin);
#pragma unroll
    for (int i = 0; i < NST; ++i)
      if (i < cnt) {
        mbar_expect_tx(&bar[i], kBytes);
        tma_load_3d(stage[i], &tin, x0 - 4, y0 - 1, zin(i), &bar[i]);
      }
  }
  __syncthreads();
  const int gx = x0 + 2 * tx, gy = y0 + ty;
  // clamp-to-edge folded into the staging offsets a border thread reads: the
  // rows y-1 / y+1 and columns x-1 / x+2 are clamped into the volume, so the
  // zero-filled out-of-volume parts of a border tile's TMA box are never read
  // and no smem fix-up pass (two loops + two CTA barriers per slice on ~14% of
  // the 1024^2 tiles) is needed; interior tiles read at fixed offsets.
  // Threads past the volume's edge (not stored) read in-box garbage.
  const bool border = x0 - 1 < 0 || x0 + TXO + 1 > a.nx || y0 - 1 < 0 || y0 + TYO + 1 > a.ny;
  const bool st_y = gy < a.ny, st_x0 = gx < a.nx, st_x1 = gx + 1 < a.nx;
  const int64_t plane = (int64_t)a.ny * a.nx;
  float* optr = out + (int64_t)zs * plane + (int64_t)min(gy, a.ny - 1) * a.nx + min(gx, a.nx - 1);
  const bool pair_store = st_y && st_x1 && ((reinterpret_cast<uintptr_t>(optr) & 7) == 0);
  int k = 0, st = 0;
  uint32_t ph = 0;
  // the plane pair of input slice k (consumes one stage, refills it)
  auto next_plane = [&](int (&pa)[9], int (&pb)[9]) {
    float* sp = stage[st];
    mbar_wait(&bar[st], ph);
    if (!LCLAMP && border) {
      // (A/B: HB_M3_SMEM_CLAMP=1) clamp-to-edge by fixing up the staged box:
      // rows then columns of the zero-filled out-of-volume parts
      const int r_lo = max(0, -(y0 - 1)), r_hi = min(SH, a.ny - (y0 - 1));
      const int c_lo = max(0, -(x0 - 4)), c_hi = min(SW, a.nx - (x0 - 4));
      for (int e = tid; e < SH * SW; e += 256) {
        const int r = e / SW, c = e - r * SW;
        if (r < r_lo || r >= r_hi) sp[r * SW + c] = sp[min(max(r, r_lo), r_hi - 1) * SW + c];
      }
      __syncthreads();
      for (int e = tid; e < SH * SW; e += 256) {
        const int r = e / SW, c = e - r * SW;
        if (c < c_lo || c >= c_hi) sp[r * SW + c] = sp[r * SW + min(max(c, c_lo), c_hi - 1)];
      }
      __syncthreads();
    }
    int r[3][4];
    if (!LCLAMP || !border) {
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const float* row = sp + (ty + i) * SW + 2 * tx;
        const float2 q1 = *reinterpret_cast<const float2*>(row + 4);  // x, x+1
        r[i][0] = __float_as_int(row[3]);                              // x-1
        r[i][1] = __float_as_int(q1.x);
        r[i][2] = __float_as_int(q1.y);
        r[i][3] = __float_as_int(row[6]);                              // x+2
      }
    } else {
      // recomputed per slice from %tid (volatile: not hoisted into registers
      // the interior path would have to carry)
      int t;
      asm volatile("mov.u32 %0, %%tid.x;" : "=r"(t));
      const int bx = 2 * (t & 31), by = t >> 5;
      const int c0 = min(max(x0 + bx - 1, 0), a.nx - 1) - (x0 - 4);
      const int c3 = min(max(x0 + bx + 2, 0), a.nx - 1) - (x0 - 4);
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const float* row = sp + (min(max(y0 + by - 1 + i, 0), a.ny - 1) - (y0 - 1)) * SW;
        const float2 q1 = *reinterpret_cast<const float2*>(row + bx + 4);
        r[i][0] = __float_as_int(row[c0]);
        r[i][1] = __float_as_int(q1.x);
        r[i][2] = __float_as_int(q1.y);
        r[i][3] = __float_as_int(row[c3]);
      }
    }
    __syncthreads();  // every thread has read stage st
    if (tid == 0 && k + NST < cnt) {
      fence_proxy_async();
      mbar_expect_tx(&bar[st], kBytes);
      tma_load_3d(sp, &tin, x0 - 4, y0 - 1, zin(k + NST), &bar[st]);
    }
    if (++st == NST) { st = 0; ph ^= 1u; }
    ++k;
    net.planes2(r, pa, pb);
  };
  // predicated stores (no divergent branch around them)
  const bool single0 = !pair_store && st_y && st_x0, single1 = !pair_store && st_y && st_x1;
  auto emit = [&](int m0, int m1) {
#if HB_M3_ASM_EMIT
    asm volatile(
        "{\n.reg .pred p, q, r;\n"
        "setp.ne.b32 p, %3, 0;\n setp.ne.b32 q, %4, 0;\n setp.ne.b32 r, %5, 0;\n"
        "@p st.global.v2.b32 [%0], {%1, %2};\n"
        "@q st.global.b32 [%0], %1;\n"
        "@r st.global.b32 [%0+4], %2;\n}\n" ::"l"(optr),
        "r"(m0), "r"(m1), "r"((int)pair_store), "r"((int)single0), "r"((int)single1)
        : "memory");
#else
    // loop-invariant predicates (the asm form re-derived them per store)
    if (pair_store) {
      *reinterpret_cast<int2*>(optr) = make_int2(m0, m1);
    } else {
      if (single0) reinterpret_cast<int*>(optr)[0] = m0;
      if (single1) reinterpret_cast<int*>(optr)[1] = m1;
    }
#endif
    optr += plane;
  };
  int X[2][9], Y[2][9], Z[2][9], W[2][9], M[2][10];
  next_plane(X[0], X[1]);  // P(zs - 1)
  next_plane(Y[0], Y[1]);  // P(zs)
  int left = ze - zs;
  while (true) {
    // state: X = P(z-1), Y = P(z)
    next_plane(Z[0], Z[1]);
    net.merge(Y[0], Z[0], M[0]);
    net.merge(Y[1], Z[1], M[1]);
    emit(net.select(M[0], X[0]), net.select(M[1], X[1]));
    if (--left == 0) break;
    next_plane(W[0], W[1]);
    emit(net.select(M[0], W[0]), net.select(M[1], W[1]));
    if (--left == 0) break;
    // state: Z = P(z-1), W = P(z)
    next_plane(X[0], X[1]);
    net.merge(W[0], X[0], M[0]);
    net.merge(W[1], X[1], M[1]);
    emit(net.select(M[0], Z[0]), net.select(M[1], Z[1]));
    if (--left == 0) break;
    next_plane(Y[0], Y[1]);
    emit(net.select(M[0], Y[0]), net.select(M[1], Y[1]));
    if (--left == 0) break;
  }
}

}  // namespace

// NotSupported outside the envelope (the caller keeps k_median3_plane):
// TMA-compatible layout (16-B aligned base, nx % 4 == 0), extents < 2^31.
// HB_MEDIAN3_PLANE=1 skips this kernel (A/B).
cudaError_t median3_f32(const DevIn& in, int64_t zo, int64_t nzo, float* out, cudaStream_t s,
                        int64_t* launches) {
  if (std::getenv("HB_MEDIAN3_PLANE") || in.dt != HB_F32 || nzo <= 0 || in.nx < 8 || in.ny < 2 ||
      in.nz >= (1 << 30) || in.nx >= (1 << 30) || in.ny >= (1 << 30) || (in.nx % 4) != 0 ||
      (reinterpret_cast<uintptr_t>(in.p) & 15) != 0)
    return cudaErrorNotSupported;
  CUtensorMap tin;
  if (!make_tmap_3d(&tin, in.p, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, in.nx, in.ny, in.nz, SW, SH))
    return cudaErrorNotSupported;
  M3Args a;
  a.nz = (int)in.nz;
  a.ny = (int)in.ny;
  a.nx = (int)in.nx;
  a.zo = (int)zo;
  a.nzo = (int)nzo;
  a.one = 1;
  a.mone = -1;
  dim3 grid((unsigned)((in.nx + TXO - 1) / TXO), (unsigned)((in.ny + TYO - 1) / TYO), 1);
  const int64_t tiles = (int64_t)grid.x * grid.y;
  // z-chunk: enough CTAs for a small wave tail (3 CTAs/SM), long enough that
  // the 2-plane prologue per chunk stays small
  const int64_t slots = 3 * kNumSMs;
  int zchunk = (int)std::min<int64_t>(nzo, 16);
  double best = 1e300;
  for (int64_t zc = std::max<int64_t>(16, nzo / 64); zc <= std::max<int64_t>(16, nzo); zc += 16) {
    const int64_t ctas = tiles * ((nzo + zc - 1) / zc);
    const double cost = (double)((ctas + slots - 1) / slots) * (double)(zc + 2);
    if (cost < best * 0.995) {
      best = cost;
      zchunk = (int)zc;
    }
  }
  a.zchunk = zchunk;
  grid.z = (unsigned)((nzo + zchunk - 1) / zchunk);
  if (std::getenv("HB_M3_SMEM_CLAMP"))
    k_median3_f32<false><<<grid, 256, 0, s>>>(tin, out, a);
  else
    k_median3_f32<true><<<grid, 256, 0, s>>>(tin, out, a);
  if (launches) *launches += 1;
  return cudaGetLastError();
}

}  // namespace hb
