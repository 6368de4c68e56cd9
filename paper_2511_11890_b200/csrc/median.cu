// median.cu — (2r+1)^3 median filter, rank = size//2, clamp-to-edge
// (filters.py:78-82 -> scipy median_filter -> rank_filter).  Output dtype is
// the input dtype; the order statistic is exact, so results are bit-exact.
//
// r = 1:    plane formulation with shared sorted planes (k_median3_plane).
// r = 2:    forgetful selection in registers (working set N/2+2, each round
//           discards the min and max of the set and admits one new sample).
// r >= 3:   per-voxel radix (bit-by-bit) selection over order-preserving keys.
#include <algorithm>
#include <type_traits>
#include <cstdlib>

#include "ops.cuh"
#include "median_nets.h"
#include "median5_nets.h"

namespace hb {
namespace {

constexpr int kThreads = 256;

template <typename K> struct MinMax;
template <> struct MinMax<float> {
  static __device__ __forceinline__ float mn(float a, float b) { return fminf(a, b); }
  static __device__ __forceinline__ float mx(float a, float b) { return fmaxf(a, b); }
};
template <> struct MinMax<uint32_t> {
  static __device__ __forceinline__ uint32_t mn(uint32_t a, uint32_t b) { return min(a, b); }
  static __device__ __forceinline__ uint32_t mx(uint32_t a, uint32_t b) { return max(a, b); }
};

template <typename K>
__device__ __forceinline__ void cs(K& a, K& b) {
  K t = MinMax<K>::mn(a, b);
  b = MinMax<K>::mx(a, b);
  a = t;
}

// Move the minimum of a[0..m) to a[0] and the maximum to a[m-1], keeping the
// set.  Pairs (i, m-1-i) split the candidates, then two tournaments (depth
// log2 m, same m-2 compare-exchanges as a linear scan, but independent ones
// the scheduler can issue back to back).  With m odd the middle slot is in
// both halves; it is always the upper index of its min-tournament pairs, so a
// maximum parked there stays for the max tournament.
template <int m, typename K>
__device__ __forceinline__ void minmax_to_ends(K* a) {
#pragma unroll
  for (int i = 0; i < m / 2; ++i) cs(a[i], a[m - 1 - i]);
#pragma unroll
  for (int len = (m + 1) / 2; len > 1; len = (len + 1) / 2) {
    const int h = (len + 1) / 2;
#pragma unroll
    for (int i = 0; i < len - h; ++i) cs(a[i], a[i + h]);
  }
#pragma unroll
  for (int len = m - m / 2; len > 1; len = (len + 1) / 2) {
    const int h = (len + 1) / 2;
#pragma unroll
    for (int i = 0; i < len - h; ++i) cs(a[m - 1 - i - h], a[m - 1 - i]);
  }
}

template <typename T, typename K> struct Key;
template <> struct Key<float, float> {
  static __device__ __forceinline__ float to(float v) { return v; }
  static __device__ __forceinline__ float from(float k) { return k; }
};
template <typename T> struct Key<T, uint32_t> {
  static __device__ __forceinline__ uint32_t to(T v) { return (uint32_t)v; }
  static __device__ __forceinline__ T from(uint32_t k) { return (T)k; }
};

// Clamped window addressing: W slice pointers + W in-plane row offsets + W
// column indices (~4W registers, not the W*W 64-bit row table).
template <int W, typename T>
struct Window {
  const T* __restrict__ sl[W];
  int yo[W];
  int xc[W];
  __device__ __forceinline__ T get(int e) const {
    const int a = e / (W * W), b = (e / W) % W, c = e % W;
    return __ldg(sl[a] + yo[b] + xc[c]);
  }
};

// Two x-adjacent outputs of 8/16-bit data in one register: lo half = output x,
// hi half = output x+1; the (data-oblivious) selection network runs on both
// with VIMNMX.U16x2, halving its cost.
struct U2 {
  unsigned v;
};
template <> struct MinMax<U2> {
  static __device__ __forceinline__ U2 mn(U2 a, U2 b) { return U2{__vminu2(a.v, b.v)}; }
  static __device__ __forceinline__ U2 mx(U2 a, U2 b) { return U2{__vmaxu2(a.v, b.v)}; }
};
template <int W, typename T>
struct Window2 {
  const T* __restrict__ sl[W];
  int yo[W];
  int xa[W], xb[W];
  __device__ __forceinline__ U2 get(int e) const {
    const int a = e / (W * W), b = (e / W) % W, c = e % W;
    const T* r = sl[a] + yo[b];
    return U2{(unsigned)__ldg(r + xa[c]) | ((unsigned)__ldg(r + xb[c]) << 16)};
  }
};

template <int m, int next, int N, int W, typename T>
__device__ __forceinline__ U2 forgetful2(U2* a, const Window2<W, T>& win) {
  minmax_to_ends<m>(a);
  if constexpr (next < N) {
    a[0] = win.get(next);
    return forgetful2<m - 1, next + 1, N, W, T>(a, win);
  } else {
    static_assert(m == 3, "forgetful selection must end with three candidates");
    return a[1];
  }
}

// ---- 5x5x5, two z-outputs per thread ---------------------------------------
// Windows of outputs z and z+1 share C = slices z-1..z+2 (100 samples) and add
// Ua = slice z-2 or Ub = slice z+3 (25 each).  A sample whose rank in C is
// below 37 (above 62) has rank below (above) 62 in either window of 125, so
// only C's middle band of ranks 37..62 (26 samples) can be a median: the band
// comes from a forgetful trim of C (set of 64, discard min and max, admit one;
// valid while the unseen count stays below the discards still owed on each
// side), and each output is then the median of band ∪ U (51 samples) by the
// usual forgetful selection.  ~1840 compare-exchanges per output instead of
// ~3100 for the direct 125-sample selection.
template <typename K>
struct Get5 {  // element e of slice s (0..5 = z-2..z+3) of the 5x5 (y, x) plane
  const void* sl[6];
  int yo[5];
  int xa[5], xb[5];
};

template <typename T, typename K> __device__ __forceinline__ K load5(const Get5<K>& g, int s, int e);
template <> __device__ __forceinline__ U2 load5<uint8_t, U2>(const Get5<U2>& g, int s, int e) {
  const uint8_t* r = (const uint8_t*)g.sl[s] + g.yo[e / 5];
  return U2{(unsigned)__ldg(r + g.xa[e % 5]) | ((unsigned)__ldg(r + g.xb[e % 5]) << 16)};
}
template <> __device__ __forceinline__ U2 load5<uint16_t, U2>(const Get5<U2>& g, int s, int e) {
  const uint16_t* r = (const uint16_t*)g.sl[s] + g.yo[e / 5];
  return U2{(unsigned)__ldg(r + g.xa[e % 5]) | ((unsigned)__ldg(r + g.xb[e % 5]) << 16)};
}
template <> __device__ __forceinline__ float load5<float, float>(const Get5<float>& g, int s, int e) {
  return __ldg((const float*)g.sl[s] + g.yo[e / 5] + g.xa[e % 5]);
}
template <> __device__ __forceinline__ uint32_t load5<uint32_t, uint32_t>(const Get5<uint32_t>& g, int s, int e) {
  return __ldg((const uint32_t*)g.sl[s] + g.yo[e / 5] + g.xa[e % 5]);
}

// trim C (elements 0..99 = slices 1..4) to its middle 26 at a[1..26]
template <int m, int next, typename T, typename K>
__device__ __forceinline__ void trim5(K* a, const Get5<K>& g) {
  minmax_to_ends<m>(a);
  if constexpr (next < 100) {
    a[0] = load5<T, K>(g, 1 + next / 25, next % 25);
    trim5<m - 1, next + 1, T, K>(a, g);
  } else {
    static_assert(m == 28, "band trim must end with 28 candidates");
  }
}
// median of band (26, in w[0..25]) ∪ slice s (25): w[26] = slice element 0 on entry
template <int m, int next, typename T, typename K>
__device__ __forceinline__ K sel51(K* a, const Get5<K>& g, int s) {
  minmax_to_ends<m>(a);
  if constexpr (next < 25) {
    a[0] = load5<T, K>(g, s, next);
    return sel51<m - 1, next + 1, T, K>(a, g, s);
  } else {
    static_assert(m == 3, "forgetful selection must end with three candidates");
    return a[1];
  }
}

template <typename T, typename K, bool PACKED>
__global__ void __launch_bounds__(kThreads)
k_median5_pair(const T* __restrict__ in, int64_t nz, int64_t ny, int64_t nx, int64_t zo,
               int64_t nzo, T* __restrict__ out) {
  const int64_t plane = ny * nx;
  const int64_t px = PACKED ? (nx + 1) / 2 : nx;
  const int64_t pz = (nzo + 1) / 2;
  const int64_t total = pz * ny * px;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / px;
    const int x = (int)(i - row * px) * (PACKED ? 2 : 1);
    const int64_t zp = row / ny;
    const int y = (int)(row - zp * ny);
    const int64_t zl = 2 * zp, z = zl + zo;
    Get5<K> g;
#pragma unroll
    for (int k = 0; k < 6; ++k) g.sl[k] = in + clamp64(z - 2 + k, 0, nz - 1) * plane;
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      g.yo[k] = clampi(y + k - 2, 0, (int)ny - 1) * (int)nx;
      g.xa[k] = clampi(x + k - 2, 0, (int)nx - 1);
      g.xb[k] = clampi(x + 1 + k - 2, 0, (int)nx - 1);
    }
    K band[64];
#pragma unroll
    for (int e = 0; e < 64; ++e) band[e] = load5<T, K>(g, 1 + e / 25, e % 25);
    trim5<64, 64, T, K>(band, g);
    K res[2];
#pragma unroll
    for (int o = 0; o < 2; ++o) {
      const int sl = o == 0 ? 0 : 5;
      K w[27];
#pragma unroll
      for (int j = 0; j < 26; ++j) w[j] = band[1 + j];
      w[26] = load5<T, K>(g, sl, 0);
      res[o] = sel51<27, 1, T, K>(w, g, sl);
    }
#pragma unroll
    for (int o = 0; o < 2; ++o) {
      if (zl + o >= nzo) break;
      T* op = out + (zl + o) * plane + (int64_t)y * nx + x;
      if constexpr (PACKED) {
        const unsigned v = reinterpret_cast<const U2&>(res[o]).v;
        op[0] = (T)(v & 0xffffu);
        if (x + 1 < nx) op[1] = (T)(v >> 16);
      } else {
        op[0] = (T)res[o];
      }
    }
  }
}

// ---- 5x5x5 by comparator networks, marching z (k_median5_net) --------------
// Same band argument as k_median5_pair (C = the 4 planes shared by outputs z
// and z+1, only C's ranks 37..62 can be either median), but with sorted planes
// and data-oblivious networks (tools/netgen/median125.py) instead of
// forgetful selection, and every plane sorted once per column as the thread
// marches z (two outputs per step):
//   S(p)  = the 25 samples of plane p sorted (SORT25, 152 CE);
//   M     = merge(S(z-1), S(z)) carried from the previous step, M' =
//           merge(S(z+1), S(z+2)) (MERGE25, 119 CE);
//   band  = ranks 37..62 of M u M' (BAND, 85 CE + 74 single min/max);
//   out z = rank 26 of band u S(z-2), out z+1 = rank 26 of band u S(z+3):
//           min_j max(band[25-j], S[j-1]) (25 max + 13 three-input min).
// ~2 x 152 + 119 + 85 CE per output pair instead of ~3700 forgetful
// exchanges.  Sorted planes and M wait in shared memory ([slot][rank][thread]:
// conflict-free, every index static), which keeps the registers at the band
// merge's 100 wires: 3 CTAs (12 warps) per SM.  8/16-bit data
// runs the networks on two x-adjacent outputs per register (U2).
constexpr int M5_NT = 128;
#ifndef HB_M5_MINB_PACKED
#define HB_M5_MINB_PACKED 3  // u8/u16: 3 CTAs/SM spill ~80 B of the packed loads and still win (u16 49.6 vs 47.5 Gvox/s at 2)
#endif
#ifndef HB_M5_ALU_EVERY
#define HB_M5_ALU_EVERY 2  // every n-th exchange in min+max (ALU) form, the rest min + IMAD pair (1024^2x256 f32: 0 23.7, 1 24.3, 2 27.1, 3 27.0 Gvox/s)
#endif

// compare-exchange with the partner maximum as a + b - min on the raw bits
// (IMAD on the FMA pipe; exact mod 2^32 since min is one of the inputs, and
// lane-wise exact for the packed u16x2 keys)
__device__ __forceinline__ int m5_imad(int a, int b, int c) {
  int d;
  asm("mad.lo.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
template <typename K> __device__ __forceinline__ int m5_bits(K v) { return (int)v; }
template <> __device__ __forceinline__ int m5_bits<float>(float v) { return __float_as_int(v); }
template <> __device__ __forceinline__ int m5_bits<U2>(U2 v) { return (int)v.v; }
template <typename K> __device__ __forceinline__ K m5_from(int b) { return (K)b; }
template <> __device__ __forceinline__ float m5_from<float>(int b) { return __int_as_float(b); }
template <> __device__ __forceinline__ U2 m5_from<U2>(int b) { return U2{(unsigned)b}; }
template <typename K>
__device__ __forceinline__ void m5_ce(K& a, K& b, int one, int mone) {
  const K lo = MinMax<K>::mn(a, b);
  const int s = m5_imad(m5_bits(a), one, m5_bits(b));
  b = m5_from<K>(m5_imad(m5_bits(lo), mone, s));
  a = lo;
}

template <typename K> __device__ __forceinline__ K m5_min3(K a, K b, K c) {
  return MinMax<K>::mn(MinMax<K>::mn(a, b), c);  // ptxas: VIMNMX3 for the integer keys
}
template <> __device__ __forceinline__ float m5_min3<float>(float a, float b, float c) {
  float r;
  asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
// rank 26 of band (26, sorted) u the 25 sorted samples u(0..24):
// min over j of max(band[25-j], u[j-1]) — 25 max, 13 three-input min
template <typename K, typename U>
__device__ __forceinline__ K m5_select(const K (&band)[26], U u) {
  K t[27];
  t[0] = band[25];
#pragma unroll
  for (int j = 1; j <= 25; ++j) t[j] = MinMax<K>::mx(band[25 - j], u(j - 1));
  t[26] = t[25];
#pragma unroll
  for (int w = 27; w > 1; w /= 3) {
#pragma unroll
    for (int i = 0; i < w / 3; ++i) t[i] = m5_min3<K>(t[3 * i], t[3 * i + 1], t[3 * i + 2]);
  }
  return t[0];
}

template <typename T, typename K, bool PACKED>
__global__ void __launch_bounds__(M5_NT, PACKED ? HB_M5_MINB_PACKED : 3)
k_median5_net(const T* __restrict__ in, int64_t nz, int64_t ny, int64_t nx, int64_t zo, int64_t nzo,
              int zchunk, T* __restrict__ out, int one, int mone) {
  extern __shared__ unsigned char m5_smem[];
  K* sm = reinterpret_cast<K*>(m5_smem);  // [3 plane slots][25 ranks] + [M: 50 ranks], x M5_NT
  const int tid = threadIdx.x;
  const int64_t px = PACKED ? (nx + 1) / 2 : nx;
  const int64_t col = (int64_t)blockIdx.x * M5_NT + tid;
  if (col >= ny * px) return;  // no CTA-wide synchronisation below
  const int y = (int)(col / px);
  const int x = (int)(col - (int64_t)y * px) * (PACKED ? 2 : 1);
  const int64_t plane = ny * nx;
  const int z0 = blockIdx.y * zchunk, z1 = (int)min((int64_t)z0 + zchunk, nzo);
  Get5<K> g;
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    g.yo[k] = clampi(y + k - 2, 0, (int)ny - 1) * (int)nx;
    g.xa[k] = clampi(x + k - 2, 0, (int)nx - 1);
    g.xb[k] = clampi(x + 1 + k - 2, 0, (int)nx - 1);
  }
  // sorted plane of (output-relative) slice zr, in rank order in a[]
  // columns x-2 .. x+2 (+1 packed) all inside the volume: the 25 loads of a
  // plane are 5 row pointers + immediate offsets (the clamped per-element
  // address path costs ~3 integer ops per load)
  const bool xin = x >= 2 && x + 2 + (PACKED ? 1 : 0) < nx;
  auto sortplane = [&](int zr, K (&a)[25]) {
    g.sl[0] = in + clamp64(zo + zr, 0, nz - 1) * plane;
    K w[25];
    if (xin) {
#pragma unroll
      for (int dy = 0; dy < 5; ++dy) {
        const T* r = (const T*)g.sl[0] + g.yo[dy] + (x - 2);
#pragma unroll
        for (int dx = 0; dx < 5; ++dx) {
          if constexpr (PACKED) {
            w[dy * 5 + dx] = m5_from<K>((int)((unsigned)__ldg(r + dx) | ((unsigned)__ldg(r + dx + 1) << 16)));
          } else {
            w[dy * 5 + dx] = (K)__ldg(r + dx);
          }
        }
      }
    } else {
#pragma unroll
      for (int e = 0; e < 25; ++e) w[e] = load5<T, K>(g, 0, e);
    }
  int nce = 0;  // compile-time after unrolling
#define HB_CE(i, j) \
  if (HB_M5_ALU_EVERY > 0 && (nce++ % HB_M5_ALU_EVERY) == 0) cs(w[i], w[j]); else m5_ce(w[i], w[j], one, mone);
#define HB_MN(i, j) w[i] = MinMax<K>::mn(w[i], w[j]);
#define HB_MX(i, j) w[j] = MinMax<K>::mx(w[i], w[j]);
    HB_SORT25(HB_CE, HB_MN, HB_MX)
    constexpr int o[25] = HB_SORT25_OUT;
#pragma unroll
    for (int k = 0; k < 25; ++k) a[k] = w[o[k]];
  };
  auto put = [&](int slot, const K (&a)[25]) {
#pragma unroll
    for (int k = 0; k < 25; ++k) sm[(slot * 25 + k) * M5_NT + tid] = a[k];
  };
  auto putm = [&](const K (&m)[50]) {
#pragma unroll
    for (int k = 0; k < 50; ++k) sm[(3 * 25 + k) * M5_NT + tid] = m[k];
  };
  auto get = [&](int slot, K (&a)[25]) {
#pragma unroll
    for (int k = 0; k < 25; ++k) a[k] = sm[(slot * 25 + k) * M5_NT + tid];
  };
  auto merge = [&](const K (&a)[25], const K (&b)[25], K (&m)[50]) {
    K w[50];
#pragma unroll
    for (int k = 0; k < 25; ++k) w[k] = a[k], w[25 + k] = b[k];
    int nce = 0;
    HB_MERGE25(HB_CE, HB_MN, HB_MX)
    constexpr int o[50] = HB_MERGE25_OUT;
#pragma unroll
    for (int k = 0; k < 50; ++k) m[k] = w[o[k]];
  };
  K A[25], B[25];
  int lo = 0, kk = 1, nn = 2;  // plane slots: S(z-2), S(z), S(z+1)
  {
    K M[50];
    sortplane(z0 - 2, A);
    put(lo, A);
    sortplane(z0 - 1, A);
    sortplane(z0, B);
    put(kk, B);
    merge(A, B, M);
    putm(M);
    sortplane(z0 + 1, A);
    put(nn, A);
  }
  for (int z = z0; z < z1; z += 2) {
    K band[26];
    {
      sortplane(z + 2, A);
      get(nn, B);  // S(z+1)
      put(nn, A);  // S(z+2) takes its slot (the next step's S(z'))
      K w[100];
      {
        K Mn[50];
        merge(B, A, Mn);  // M(z+1, z+2)
#pragma unroll
        for (int k = 0; k < 50; ++k) w[50 + k] = Mn[k];
      }
#pragma unroll
      for (int k = 0; k < 50; ++k) {
        w[k] = sm[(3 * 25 + k) * M5_NT + tid];  // M(z-1, z)
        sm[(3 * 25 + k) * M5_NT + tid] = w[50 + k];
      }
      int nce = 0;
      HB_BAND(HB_CE, HB_MN, HB_MX)
      constexpr int o[26] = HB_BAND_OUT;
#pragma unroll
      for (int k = 0; k < 26; ++k) band[k] = w[o[k]];
    }
#undef HB_CE
#undef HB_MN
#undef HB_MX
    const K* ulo = sm + lo * 25 * M5_NT + tid;
    const K r0 = m5_select<K>(band, [&](int j) { return ulo[j * M5_NT]; });
    sortplane(z + 3, A);
    put(lo, A);  // S(z+3): the next step's S(z'+1)
    const K r1 = m5_select<K>(band, [&](int j) { return A[j]; });  // S(z+3) still in registers
    const K res[2] = {r0, r1};
#pragma unroll
    for (int o = 0; o < 2; ++o) {
      if (z + o >= z1) break;
      T* op = out + (int64_t)(z + o) * plane + (int64_t)y * nx + x;
      if constexpr (PACKED) {
        const unsigned v = reinterpret_cast<const U2&>(res[o]).v;
        op[0] = (T)(v & 0xffffu);
        if (x + 1 < nx) op[1] = (T)(v >> 16);
      } else {
        op[0] = (T)res[o];
      }
    }
    // S(z') = S(z+2) sits in nn, S(z'+1) = S(z+3) in lo, S(z'-2) = S(z) in kk
    const int t = lo;
    lo = kk;
    kk = nn;
    nn = t;
  }
}

template <typename T, typename K, bool PACKED>
cudaError_t launch_median5_net(const T* src, const DevIn& in, int64_t zo, int64_t nzo, T* dst,
                               cudaStream_t s) {
  const int64_t px = PACKED ? (in.nx + 1) / 2 : in.nx;
  const int64_t cols = in.ny * px;
  if (cols <= 0 || nzo <= 0 || in.nz >= (1LL << 30) || in.ny * in.nx >= (1LL << 31)) return cudaErrorNotSupported;
  const int64_t nblk = (cols + M5_NT - 1) / M5_NT;
  if (nblk > 0x7fffffffLL) return cudaErrorNotSupported;
  // z-chunks: >= ~4 waves of 3 CTAs/SM; each chunk pays a 4-plane prologue
  const int64_t want = std::max<int64_t>(1, (12 * kNumSMs + nblk - 1) / nblk);
  int64_t zc = std::max<int64_t>(16, (nzo + want - 1) / want);
  zc = std::min<int64_t>(zc + (zc & 1), std::max<int64_t>(2, nzo + (nzo & 1)));
  const int64_t nch = (nzo + zc - 1) / zc;
  if (nch > 65535) return cudaErrorNotSupported;
  const int smem = (3 * 25 + 50) * M5_NT * (int)sizeof(K);
  auto kern = k_median5_net<T, K, PACKED>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
    return cudaErrorNotSupported;
  kern<<<dim3((unsigned)nblk, (unsigned)nch), M5_NT, smem, s>>>(src, in.nz, in.ny, in.nx, zo, nzo, (int)zc, dst, 1, -1);
  return cudaGetLastError();
}

template <int R, typename T>
__global__ void __launch_bounds__(kThreads)
k_median_forgetful2(const T* __restrict__ in, int64_t nz, int64_t ny, int64_t nx, int64_t zo,
                    int64_t nzo, T* __restrict__ out) {
  constexpr int W = 2 * R + 1;
  constexpr int N = W * W * W;
  constexpr int M0 = N / 2 + 2;
  const int64_t plane = ny * nx;
  const int64_t px = (nx + 1) / 2;
  const int64_t total = nzo * ny * px;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / px;
    const int x = (int)(i - row * px) * 2;
    const int64_t zl = row / ny;
    const int y = (int)(row - zl * ny);
    const int64_t z = zl + zo;
    Window2<W, T> win;
#pragma unroll
    for (int a = 0; a < W; ++a) {
      win.sl[a] = in + clamp64(z + a - R, 0, nz - 1) * plane;
      win.yo[a] = clampi(y + a - R, 0, (int)ny - 1) * (int)nx;
      win.xa[a] = clampi(x + a - R, 0, (int)nx - 1);
      win.xb[a] = clampi(x + 1 + a - R, 0, (int)nx - 1);
    }
    U2 a[M0];
#pragma unroll
    for (int e = 0; e < M0; ++e) a[e] = win.get(e);
    const unsigned med = forgetful2<M0, M0, N, W, T>(a, win).v;
    T* o = out + zl * plane + (int64_t)y * nx + x;
    o[0] = (T)(med & 0xffffu);
    if (x + 1 < nx) o[1] = (T)(med >> 16);
  }
}

template <int m, int next, int N, int W, typename T, typename K>
__device__ __forceinline__ K forgetful_step(K* a, const Window<W, T>& win) {
  minmax_to_ends<m>(a);
  if constexpr (next < N) {
    a[0] = Key<T, K>::to(win.get(next));
    return forgetful_step<m - 1, next + 1, N, W, T, K>(a, win);
  } else {
    static_assert(m == 3, "forgetful selection must end with three candidates");
    return a[1];
  }
}

template <int R, typename T, typename K>
__global__ void __launch_bounds__(kThreads)
k_median_forgetful(const T* __restrict__ in, int64_t nz, int64_t ny, int64_t nx, int64_t zo,
                   int64_t nzo, T* __restrict__ out) {
  constexpr int W = 2 * R + 1;
  constexpr int N = W * W * W;
  constexpr int M0 = N / 2 + 2;
  const int64_t plane = ny * nx;
  const int64_t total = nzo * plane;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t zl = i / plane;
    int64_t rr = i - zl * plane;
    int64_t y = rr / nx;
    int64_t x = rr - y * nx;
    int64_t z = zl + zo;
    Window<W, T> win;
#pragma unroll
    for (int a = 0; a < W; ++a) {
      win.sl[a] = in + clamp64(z + a - R, 0, nz - 1) * plane;
      win.yo[a] = (int)clamp64(y + a - R, 0, ny - 1) * (int)nx;
      win.xc[a] = (int)clamp64(x + a - R, 0, nx - 1);
    }
    K a[M0];
#pragma unroll
    for (int e = 0; e < M0; ++e) a[e] = Key<T, K>::to(win.get(e));
    K med = forgetful_step<M0, M0, N, W, T, K>(a, win);
    out[i] = Key<T, K>::from(med);
  }
}

template <typename T> __device__ __forceinline__ uint32_t okey(T v) { return (uint32_t)v; }
template <> __device__ __forceinline__ uint32_t okey<float>(float v) { return f32_key(v); }
template <typename T> __device__ __forceinline__ T unkey(uint32_t k) { return (T)k; }
template <> __device__ __forceinline__ float unkey<float>(uint32_t k) { return key_f32(k); }

// Radix selection of the k-th smallest key, one bit per pass, any radius.
template <typename T, int BITS>
__global__ void __launch_bounds__(kThreads)
k_median_radix(const T* __restrict__ in, int64_t nz, int64_t ny, int64_t nx, int64_t zo,
               int64_t nzo, T* __restrict__ out, int R) {
  const int W = 2 * R + 1;
  const int N = W * W * W;
  const int64_t plane = ny * nx;
  const int64_t total = nzo * plane;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t zl = i / plane;
    int64_t rr = i - zl * plane;
    int64_t y = rr / nx;
    int64_t x = rr - y * nx;
    int64_t z = zl + zo;
    uint32_t prefix = 0;
    int k = N / 2;
    for (int bit = BITS - 1; bit >= 0; --bit) {
      const uint32_t hi_mask = (bit == 31) ? 0u : (0xffffffffu << (bit + 1));
      int cnt0 = 0;
      for (int dz = -R; dz <= R; ++dz) {
        int64_t zc = clamp64(z + dz, 0, nz - 1);
        for (int dy = -R; dy <= R; ++dy) {
          const T* row = in + (zc * ny + clamp64(y + dy, 0, ny - 1)) * nx;
          for (int dx = -R; dx <= R; ++dx) {
            uint32_t key = okey<T>(__ldg(row + clamp64(x + dx, 0, nx - 1)));
            cnt0 += (((key ^ prefix) & hi_mask) == 0u) & (((key >> bit) & 1u) == 0u);
          }
        }
      }
      if (k >= cnt0) {
        k -= cnt0;
        prefix |= (1u << bit);
      }
    }
    out[i] = unkey<T>(prefix);
  }
}


// ---------------------------------------------------------------------------
// 3x3x3 median, plane formulation (the fast path for r = 1)
//
// Output (z, y, x) = rank 13 of P(z-1) ∪ P(z) ∪ P(z+1), where P(s) is the sorted
// 3x3 XY neighbourhood of slice s.  Each thread owns two adjacent x columns and
// marches down z, so every plane is sorted once and used by three outputs:
//   plane sort : rows sort3 -> columns sort3 (3x3 Young tableau) -> 7 comparators
//   merge      : P(z) ∪ P(z+1) pruned to ranks 4..13 (27 comparators, generated)
//   select     : rank13 = min_{i+j=14} max(M[i-1], P(z-1)[j-1])
// All comparisons run on order-preserving int32 keys so that half of every
// compare-exchange runs on the FMA pipe: max(a,b) = (a + b) - min(a,b) (exact
// mod 2^32) via IMAD with a runtime multiplier ptxas cannot fold.
// ---------------------------------------------------------------------------
struct ImadOnes {
  int one, mone;  // runtime 1 and -1 (kernel params) -> IMAD, not IADD3
};

__device__ __forceinline__ int imad(int a, int b, int c) {
  int d;
  asm("mad.lo.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

template <typename T> __device__ __forceinline__ int to_key(T v) { return (int)v; }
template <> __device__ __forceinline__ int to_key<uint32_t>(uint32_t v) { return (int)(v ^ 0x80000000u); }
template <> __device__ __forceinline__ int to_key<float>(float v) {
  const int u = __float_as_int(v);
  return u ^ ((u >> 31) & 0x7fffffff);
}
template <typename T> __device__ __forceinline__ T from_key(int k) { return (T)k; }
template <> __device__ __forceinline__ uint32_t from_key<uint32_t>(int k) { return (uint32_t)k ^ 0x80000000u; }
template <> __device__ __forceinline__ float from_key<float>(int k) {
  return __int_as_float(k ^ ((k >> 31) & 0x7fffffff));
}

struct Net {
  ImadOnes c;
  // compare-exchange: a <- min, b <- max (max from the sum on the FMA pipe)
  __device__ __forceinline__ void ce(int& a, int& b) const {
    const int lo = min(a, b);
    const int s = imad(a, c.one, b);
    b = imad(lo, c.mone, s);
    a = lo;
  }
  __device__ __forceinline__ void sort3(int& a, int& b, int& cc) const {
    const int lo = min(a, min(b, cc));
    const int hi = max(a, max(b, cc));
    int t = imad(a, c.one, b);
    t = imad(cc, c.one, t);
    t = imad(lo, c.mone, t);
    b = imad(hi, c.mone, t);
    a = lo;
    cc = hi;
  }
  // 3x3 matrix sorted along both axes (Young tableau) -> ascending s[0..8];
  // wire order (0,0),(0,1),(1,0),(0,2),(1,1),(2,0),(1,2),(2,1),(2,2) + 7 CE
  // (tools/netgen: exhaustive over the 20 monotone 0/1 tableaux)
  __device__ __forceinline__ void tableau(const int (&m)[3][3], int (&s)[9]) const {
    s[0] = m[0][0]; s[1] = m[0][1]; s[2] = m[1][0]; s[3] = m[0][2]; s[4] = m[1][1];
    s[5] = m[2][0]; s[6] = m[1][2]; s[7] = m[2][1]; s[8] = m[2][2];
    ce(s[3], s[5]); ce(s[1], s[2]); ce(s[2], s[3]); ce(s[6], s[7]);
    ce(s[5], s[6]); ce(s[3], s[4]); ce(s[4], s[5]);
  }
  // the sorted planes of two x-adjacent outputs from r[row][x-1..x+2]: the four
  // vertical triples are sorted once and shared, then each plane sorts across
  // its three columns per rank (rows and columns sorted -> tableau)
  __device__ __forceinline__ void planes2(int (&r)[3][4], int (&pa)[9], int (&pb)[9]) const {
#pragma unroll
    for (int j = 0; j < 4; ++j) sort3(r[0][j], r[1][j], r[2][j]);
    int a[3][3], b[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      a[i][0] = r[i][0]; a[i][1] = r[i][1]; a[i][2] = r[i][2];
      b[i][0] = r[i][1]; b[i][1] = r[i][2]; b[i][2] = r[i][3];
      sort3(a[i][0], a[i][1], a[i][2]);
      sort3(b[i][0], b[i][1], b[i][2]);
    }
    tableau(a, pa);
    tableau(b, pb);
  }
  // ranks 4..13 of cur ∪ nxt (two sorted 9-lists) -> m[0..9]
  __device__ __forceinline__ void merge(const int (&cur)[9], const int (&nxt)[9], int (&m)[10]) const {
    int w[18];
#pragma unroll
    for (int i = 0; i < 9; ++i) {
      w[i] = cur[i];
      w[9 + i] = nxt[i];
    }
#define HB_CE(i, j) ce(w[i], w[j]);
#define HB_MN(i, j) w[i] = min(w[i], w[j]);
#define HB_MX(i, j) w[j] = max(w[i], w[j]);
    HB_MERGE9_RANK4_13(HB_CE, HB_MN, HB_MX)
#undef HB_CE
#undef HB_MN
#undef HB_MX
#pragma unroll
    for (int i = 0; i < 10; ++i) m[i] = w[4 + i];
  }
  // rank 13 of M ∪ P where M holds ranks 4..13 of two planes and P is the
  // third sorted plane: min over j=0..9 of max(M[13-j], P[j-1])
  __device__ __forceinline__ int select(const int (&m)[10], const int (&p)[9]) const {
    const int t0 = m[9];
    const int t1 = max(m[8], p[0]);
    const int t2 = max(m[7], p[1]);
    const int t3 = max(m[6], p[2]);
    const int t4 = max(m[5], p[3]);
    const int t5 = max(m[4], p[4]);
    const int t6 = max(m[3], p[5]);
    const int t7 = max(m[2], p[6]);
    const int t8 = max(m[1], p[7]);
    const int t9 = max(m[0], p[8]);
    // chained 3-input mins (VIMNMX3): 5 ALU ops instead of 9
    int r = min(t0, min(t1, t2));
    r = min(r, min(t3, t4));
    r = min(r, min(t5, t6));
    r = min(r, min(t7, t8));
    return min(r, t9);
  }
};

constexpr int M3_TX = 64, M3_TY = 8;  // outputs per CTA slice (32 x-pairs x 8 rows)
constexpr int M3_W = M3_TX + 2, M3_H = M3_TY + 2;

template <typename T>
__global__ void __launch_bounds__(256, 3)
k_median3_plane(const T* __restrict__ in, int64_t nz, int64_t ny, int64_t nx, int64_t zo,
                int64_t nzo, int zchunk, T* __restrict__ out, ImadOnes ones) {
  __shared__ __align__(16) int tile[3][M3_H][M3_W];
  const Net net{ones};
  const int tid = threadIdx.x;
  const int tx = tid & 31, ty = tid >> 5;
  const int64_t x0 = (int64_t)blockIdx.x * M3_TX, y0 = (int64_t)blockIdx.y * M3_TY;
  // 32-bit z bookkeeping (slices < 2^30): 64-bit compares/selects in the step
  // loop cost ~10 uniform-datapath issue slots per output
  const int zs = (int)blockIdx.z * zchunk;
  const int ze = min(zs + zchunk, (int)nzo);
  // cooperative slice loader: element e of the halo'd tile -> (ly, lx)
  constexpr int NE = M3_H * M3_W;
  constexpr int PER = (NE + 255) / 256;
  int goff[PER];  // in-plane offsets (a plane has < 2^31 voxels)
  bool gval[PER];
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int e = tid + 256 * k;
    gval[k] = e < NE;
    const int ly = gval[k] ? e / M3_W : 0, lx = gval[k] ? e % M3_W : 0;
    const int64_t gy = clamp64(y0 - 1 + ly, 0, ny - 1), gx = clamp64(x0 - 1 + lx, 0, nx - 1);
    goff[k] = (int)(gy * nx + gx);
  }
  const int64_t plane = ny * nx;
  // fetch keeps the raw samples; the key conversion happens in stash, one
  // step later, so the global-load latency overlaps a whole step of sorting.
  // Slices are addressed by a running pointer (clamped only at the volume faces).
  const int zlast = (int)nz - 1;
  auto slice_ptr = [&](int zb) { return in + (int64_t)min(max(zb, 0), zlast) * plane; };
  auto fetch = [&](const T* src, T (&v)[PER]) {
#pragma unroll
    for (int k = 0; k < PER; ++k) v[k] = gval[k] ? __ldg(src + goff[k]) : T(0);
  };
  auto stash = [&](int* buf, const T (&v)[PER]) {
#pragma unroll
    for (int k = 0; k < PER; ++k)
      if (gval[k]) buf[tid + 256 * k] = to_key<T>(v[k]);
  };
  // this thread's two planes of a tile buffer
  auto planes = [&](const int* buf, int (&pa)[9], int (&pb)[9]) {
    int r[3][4];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const int2 lo = *reinterpret_cast<const int2*>(buf + (ty + i) * M3_W + 2 * tx);
      const int2 hi = *reinterpret_cast<const int2*>(buf + (ty + i) * M3_W + 2 * tx + 2);
      r[i][0] = lo.x; r[i][1] = lo.y; r[i][2] = hi.x; r[i][3] = hi.y;
    }
    net.planes2(r, pa, pb);
  };
  const int64_t gy = y0 + ty, gx = x0 + 2 * tx;
  const bool st_y = gy < ny, st_x0 = gx < nx, st_x1 = gx + 1 < nx;
  T* optr = out + (int64_t)zs * plane + gy * nx + gx;  // output slice zs, advanced per step
  auto emit = [&](int k0, int k1) {
    if (st_y) {
      if (st_x0) optr[0] = from_key<T>(k0);
      if (st_x1) optr[1] = from_key<T>(k1);
    }
    optr += plane;
  };

  // One merge serves two outputs: out(z) = sel(M, P(z-1)), out(z+1) = sel(M, P(z+2))
  // with M = ranks 4..13 of P(z) ∪ P(z+1).  Four steps cycle the plane names.
  int X[2][9], Y[2][9], Z[2][9], W[2][9], M[2][10];
  T v[PER];
  // slice zs-1+k lives in tile[k % 3]; a buffer is rewritten three steps after
  // it was read, so one barrier per step orders all reads before the rewrite
  int* const tb0 = &tile[0][0][0];
  constexpr int TPITCH = M3_H * M3_W;
  const int zb0 = (int)zo + zs;
  fetch(slice_ptr(zb0 - 1), v);
  stash(tb0, v);
  fetch(slice_ptr(zb0), v);
  stash(tb0 + TPITCH, v);
  // next slice to fetch: block z = zb0 + 1, then + 1 per step; a running
  // pointer that stops advancing at the last slice (the clamp at the face)
  int zf = zb0 + 1;
  const T* pf = slice_ptr(zf);
  fetch(pf, v);
  __syncthreads();
  planes(tb0, X[0], X[1]);           // P(zs-1)
  planes(tb0 + TPITCH, Y[0], Y[1]);  // P(zs)
  int z = zs;
  int* tb = tb0 + 2 * TPITCH;  // buffer that receives slice z+1
  auto next_plane = [&](int (&pa)[9], int (&pb)[9]) {
    stash(tb, v);
    ++zf;
    if (zf <= zlast && zf > 0) pf += plane;
    fetch(pf, v);
    __syncthreads();
    planes(tb, pa, pb);
    tb = (tb == tb0 + 2 * TPITCH) ? tb0 : tb + TPITCH;
  };
  auto emit2 = [&](int m0, int m1) {
    emit(m0, m1);
    ++z;
  };
  while (z < ze) {
    // state: X = P(z-1), Y = P(z)
    next_plane(Z[0], Z[1]);  // P(z+1)
    net.merge(Y[0], Z[0], M[0]);
    net.merge(Y[1], Z[1], M[1]);
    emit2(net.select(M[0], X[0]), net.select(M[1], X[1]));
    if (z >= ze) break;
    next_plane(W[0], W[1]);  // P(z+2)  (z already advanced)
    emit2(net.select(M[0], W[0]), net.select(M[1], W[1]));
    if (z >= ze) break;
    // state: Z = P(z-1), W = P(z)
    next_plane(X[0], X[1]);
    net.merge(W[0], X[0], M[0]);
    net.merge(W[1], X[1], M[1]);
    emit2(net.select(M[0], Z[0]), net.select(M[1], Z[1]));
    if (z >= ze) break;
    next_plane(Y[0], Y[1]);
    emit2(net.select(M[0], Y[0]), net.select(M[1], Y[1]));
    // state: X = P(z-1), Y = P(z)
  }
}

// ---------------------------------------------------------------------------
// 3x3x3 median of 8/16-bit data: the same plane / merge / select networks on
// two x-adjacent outputs packed per 32-bit register (lo half = x, hi half =
// x+1): min/max are VIMNMX(3).U16x2, and the max = a + b - min identity stays
// exact lane-wise (the 32-bit result is the packed maxima mod 2^32).  One
// plane network per output pair instead of planes2's shared-triple pair, one
// merge and one select per pair.
// ---------------------------------------------------------------------------
struct NetP {
  ImadOnes c;
  static __device__ __forceinline__ int mn(int a, int b) { return (int)__vminu2((unsigned)a, (unsigned)b); }
  static __device__ __forceinline__ int mx(int a, int b) { return (int)__vmaxu2((unsigned)a, (unsigned)b); }
  __device__ __forceinline__ void ce(int& a, int& b) const {
    const int lo = mn(a, b);
    const int s = imad(a, c.one, b);
    b = imad(lo, c.mone, s);
    a = lo;
  }
  __device__ __forceinline__ void sort3(int& a, int& b, int& cc) const {
    const int lo = mn(a, mn(b, cc));
    const int hi = mx(a, mx(b, cc));
    int t = imad(a, c.one, b);
    t = imad(cc, c.one, t);
    t = imad(lo, c.mone, t);
    b = imad(hi, c.mone, t);
    a = lo;
    cc = hi;
  }
  __device__ __forceinline__ void tableau(const int (&m)[3][3], int (&s)[9]) const {
    s[0] = m[0][0]; s[1] = m[0][1]; s[2] = m[1][0]; s[3] = m[0][2]; s[4] = m[1][1];
    s[5] = m[2][0]; s[6] = m[1][2]; s[7] = m[2][1]; s[8] = m[2][2];
    ce(s[3], s[5]); ce(s[1], s[2]); ce(s[2], s[3]); ce(s[6], s[7]);
    ce(s[5], s[6]); ce(s[3], s[4]); ce(s[4], s[5]);
  }
  // packed plane of the output pair from r[row][x-1..x+2] (16-bit keys)
  __device__ __forceinline__ void plane(const int (&r)[3][4], int (&p)[9]) const {
    int m[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) m[i][j] = (int)__byte_perm((unsigned)r[i][j], (unsigned)r[i][j + 1], 0x5410);
#pragma unroll
    for (int j = 0; j < 3; ++j) sort3(m[0][j], m[1][j], m[2][j]);
#pragma unroll
    for (int i = 0; i < 3; ++i) sort3(m[i][0], m[i][1], m[i][2]);
    tableau(m, p);
  }
  __device__ __forceinline__ void merge(const int (&cur)[9], const int (&nxt)[9], int (&m)[10]) const {
    int w[18];
#pragma unroll
    for (int i = 0; i < 9; ++i) {
      w[i] = cur[i];
      w[9 + i] = nxt[i];
    }
#define HB_CE(i, j) ce(w[i], w[j]);
#define HB_MN(i, j) w[i] = mn(w[i], w[j]);
#define HB_MX(i, j) w[j] = mx(w[i], w[j]);
    HB_MERGE9_RANK4_13(HB_CE, HB_MN, HB_MX)
#undef HB_CE
#undef HB_MN
#undef HB_MX
#pragma unroll
    for (int i = 0; i < 10; ++i) m[i] = w[4 + i];
  }
  __device__ __forceinline__ int select(const int (&m)[10], const int (&p)[9]) const {
    const int t0 = m[9];
    const int t1 = mx(m[8], p[0]);
    const int t2 = mx(m[7], p[1]);
    const int t3 = mx(m[6], p[2]);
    const int t4 = mx(m[5], p[3]);
    const int t5 = mx(m[4], p[4]);
    const int t6 = mx(m[3], p[5]);
    const int t7 = mx(m[2], p[6]);
    const int t8 = mx(m[1], p[7]);
    const int t9 = mx(m[0], p[8]);
    int r = mn(t0, mn(t1, t2));
    r = mn(r, mn(t3, t4));
    r = mn(r, mn(t5, t6));
    r = mn(r, mn(t7, t8));
    return mn(r, t9);
  }
};

template <typename T>
__global__ void __launch_bounds__(256, 3)
k_median3_packed(const T* __restrict__ in, int64_t nz, int64_t ny, int64_t nx, int64_t zo,
                 int64_t nzo, int zchunk, T* __restrict__ out, ImadOnes ones) {
  __shared__ __align__(16) int tile[3][M3_H][M3_W];
  const NetP net{ones};
  const int tid = threadIdx.x;
  const int tx = tid & 31, ty = tid >> 5;
  const int64_t x0 = (int64_t)blockIdx.x * M3_TX, y0 = (int64_t)blockIdx.y * M3_TY;
  const int zs = (int)blockIdx.z * zchunk;
  const int ze = min(zs + zchunk, (int)nzo);
  constexpr int NE = M3_H * M3_W;
  constexpr int PER = (NE + 255) / 256;
  int goff[PER];
  bool gval[PER];
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int e = tid + 256 * k;
    gval[k] = e < NE;
    const int ly = gval[k] ? e / M3_W : 0, lx = gval[k] ? e % M3_W : 0;
    const int64_t gy = clamp64(y0 - 1 + ly, 0, ny - 1), gx = clamp64(x0 - 1 + lx, 0, nx - 1);
    goff[k] = (int)(gy * nx + gx);
  }
  const int64_t plane = ny * nx;
  const int zlast = (int)nz - 1;
  auto slice_ptr = [&](int zb) { return in + (int64_t)min(max(zb, 0), zlast) * plane; };
  auto fetch = [&](const T* src, T (&v)[PER]) {
#pragma unroll
    for (int k = 0; k < PER; ++k) v[k] = gval[k] ? __ldg(src + goff[k]) : T(0);
  };
  auto stash = [&](int* buf, const T (&v)[PER]) {
#pragma unroll
    for (int k = 0; k < PER; ++k)
      if (gval[k]) buf[tid + 256 * k] = (int)v[k];
  };
  auto planes = [&](const int* buf, int (&p)[9]) {
    int r[3][4];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const int2 lo = *reinterpret_cast<const int2*>(buf + (ty + i) * M3_W + 2 * tx);
      const int2 hi = *reinterpret_cast<const int2*>(buf + (ty + i) * M3_W + 2 * tx + 2);
      r[i][0] = lo.x; r[i][1] = lo.y; r[i][2] = hi.x; r[i][3] = hi.y;
    }
    net.plane(r, p);
  };
  const int64_t gy = y0 + ty, gx = x0 + 2 * tx;
  const bool st_y = gy < ny, st_x0 = gx < nx, st_x1 = gx + 1 < nx;
  T* optr = out + (int64_t)zs * plane + gy * nx + gx;
  auto emit = [&](int k) {
    if (st_y) {
      if (st_x0) optr[0] = (T)(k & 0xffff);
      if (st_x1) optr[1] = (T)((unsigned)k >> 16);
    }
    optr += plane;
  };
  int X[9], Y[9], Z[9], W[9], M[10];
  T v[PER];
  int* const tb0 = &tile[0][0][0];
  constexpr int TPITCH = M3_H * M3_W;
  const int zb0 = (int)zo + zs;
  fetch(slice_ptr(zb0 - 1), v);
  stash(tb0, v);
  fetch(slice_ptr(zb0), v);
  stash(tb0 + TPITCH, v);
  int zf = zb0 + 1;
  const T* pf = slice_ptr(zf);
  fetch(pf, v);
  __syncthreads();
  planes(tb0, X);
  planes(tb0 + TPITCH, Y);
  int z = zs;
  int* tb = tb0 + 2 * TPITCH;
  auto next_plane = [&](int (&p)[9]) {
    stash(tb, v);
    ++zf;
    if (zf <= zlast && zf > 0) pf += plane;
    fetch(pf, v);
    __syncthreads();
    planes(tb, p);
    tb = (tb == tb0 + 2 * TPITCH) ? tb0 : tb + TPITCH;
  };
  while (z < ze) {
    next_plane(Z);
    net.merge(Y, Z, M);
    emit(net.select(M, X));
    if (++z >= ze) break;
    next_plane(W);
    emit(net.select(M, W));
    if (++z >= ze) break;
    next_plane(X);
    net.merge(W, X, M);
    emit(net.select(M, Z));
    if (++z >= ze) break;
    next_plane(Y);
    emit(net.select(M, Y));
    ++z;
  }
}

inline int grid_for(int64_t n) {
  int64_t b = (n + kThreads - 1) / kThreads;
  int64_t cap = (int64_t)kNumSMs * 16;
  return (int)(b < cap ? (b < 1 ? 1 : b) : cap);
}

template <typename T, typename K, int BITS>
cudaError_t run_median(const DevIn& in, int64_t zo, int64_t nzo, void* out, int r,
                       cudaStream_t s, int64_t* launches) {
  int64_t n = nzo * in.ny * in.nx;
  int g = grid_for(n);
  const T* src = (const T*)in.p;
  T* dst = (T*)out;
  if (r == 1) {
    if constexpr (std::is_same<T, float>::value) {
      const cudaError_t e = median3_f32(in, zo, nzo, (float*)out, s, launches);
      if (e != cudaErrorNotSupported) return e;
      cudaGetLastError();
    }
    dim3 grid((unsigned)((in.nx + M3_TX - 1) / M3_TX), (unsigned)((in.ny + M3_TY - 1) / M3_TY), 1);
    const int64_t tiles = (int64_t)grid.x * grid.y;
    // z-chunk: enough CTAs that the wave tail is small (3 CTAs/SM resident),
    // long enough that the 2-plane prologue per chunk stays ~1%
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
    grid.z = (unsigned)((nzo + zchunk - 1) / zchunk);
    if constexpr (sizeof(T) <= 2) {
      if (!std::getenv("HB_MEDIAN3_UNPACKED")) {
        k_median3_packed<T><<<grid, 256, 0, s>>>(src, in.nz, in.ny, in.nx, zo, nzo, zchunk, dst,
                                                 ImadOnes{1, -1});
        if (launches) *launches += 1;
        return cudaGetLastError();
      }
    }
    k_median3_plane<T><<<grid, 256, 0, s>>>(src, in.nz, in.ny, in.nx, zo, nzo, zchunk, dst,
                                            ImadOnes{1, -1});
  } else if (r == 2) {
    if (!std::getenv("HB_MEDIAN5_FORGETFUL") && !std::getenv("HB_MEDIAN5_SINGLE")) {
      cudaError_t e;
      if constexpr (sizeof(T) <= 2) e = launch_median5_net<T, U2, true>(src, in, zo, nzo, dst, s);
      else e = launch_median5_net<T, K, false>(src, in, zo, nzo, dst, s);
      if (e != cudaErrorNotSupported) {
        if (launches) *launches += 1;
        return e;
      }
      cudaGetLastError();
    }
    if (!std::getenv("HB_MEDIAN5_SINGLE")) {
      const int64_t pairs = ((nzo + 1) / 2) * in.ny * (sizeof(T) <= 2 ? (in.nx + 1) / 2 : in.nx);
      const int gp = grid_for(pairs);
      if constexpr (sizeof(T) <= 2)
        k_median5_pair<T, U2, true><<<gp, kThreads, 0, s>>>(src, in.nz, in.ny, in.nx, zo, nzo, dst);
      else
        k_median5_pair<T, K, false><<<gp, kThreads, 0, s>>>(src, in.nz, in.ny, in.nx, zo, nzo, dst);
      if (launches) *launches += 1;
      return cudaGetLastError();
    }
    if constexpr (sizeof(T) <= 2) {
      if (!std::getenv("HB_MEDIAN5_SCALAR")) {
        const int g2 = grid_for(nzo * in.ny * ((in.nx + 1) / 2));
        k_median_forgetful2<2, T><<<g2, kThreads, 0, s>>>(src, in.nz, in.ny, in.nx, zo, nzo, dst);
        if (launches) *launches += 1;
        return cudaGetLastError();
      }
    }
    k_median_forgetful<2, T, K><<<g, kThreads, 0, s>>>(src, in.nz, in.ny, in.nx, zo, nzo, dst);
  } else {
    k_median_radix<T, BITS><<<g, kThreads, 0, s>>>(src, in.nz, in.ny, in.nx, zo, nzo, dst, r);
  }
  if (launches) *launches += 1;
  return cudaGetLastError();
}

}  // namespace

cudaError_t median(const DevIn& in, int64_t zo, int64_t nzo, void* out, int r,
                   cudaStream_t s, int64_t* launches) {
  if (nzo <= 0) return cudaSuccess;
  switch (in.dt) {
    case HB_U8: return run_median<uint8_t, uint32_t, 8>(in, zo, nzo, out, r, s, launches);
    case HB_U16: return run_median<uint16_t, uint32_t, 16>(in, zo, nzo, out, r, s, launches);
    case HB_U32: return run_median<uint32_t, uint32_t, 32>(in, zo, nzo, out, r, s, launches);
    case HB_F32: return run_median<float, float, 32>(in, zo, nzo, out, r, s, launches);
  }
  return cudaErrorInvalidValue;
}

}  // namespace hb
