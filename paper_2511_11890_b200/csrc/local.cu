// local.cu — local adaptive thresholds (threshold.py:174-217, registry.py:
// 257-272): labels = data > T as uint32, T per voxel from the clamped
// (2w+1)^3 window of the reference's padded chunk.
//
//   mean     T = m - c            niblack  T = m + k*sqrt(var)
//   sauvola  T = m*(1 + k*(sqrt(var)/R - 1))
//       m = s1/n, var = max(s2/n - m*m, 0), s1 = sum v, s2 = sum v^2 over the
//       window (threshold.py:133-146); k_local_box.
//   median   T = f64(median_filter(data, 2w+1)) - c: the median stage
//       (median.cu) into scratch, then k_local_cmp.
//   gaussian T = correlate1d^3(f64(data), kern) - c with f64 between the
//       passes (threshold.py:198-206, no float32 rounding, unlike
//       filters.gaussian): k_corr64 passes, the X pass compares.
// The comparison is NumPy's: data (any dtype) vs a float64 array -> float64.
//
// Window sums.  Integer data: the reference sums in int64 (threshold.py:
// 133-145, _box_sum / _box_sum_precast); integer addition mod 2^64 is
// associative, so any order is exact — here u32/u64 accumulators chosen per
// dtype and radius so nothing can wrap differently (u32 data squares wrap
// mod 2^64 exactly as NumPy's int64 do).  Float32 data: the reference's
// float64 sums are differences of running cumsums along each axis of the
// whole padded chunk, so their last bits depend on the chunk plan; here they
// are direct float64 window sums (at least as accurate), and a label can only
// differ where data is within a few ulp of T (tested with that tolerance).
//
// k_local_box streams one 32 x 8 (x, y) tile of output columns down a z range:
// per input slice the (8+2w) x (32+2w) tile is staged in shared memory, an X
// pass and a Y pass give the slice's 2D sums (s1, s2), which go into a ring of
// 2w+1 slices (shared memory, private per thread); each output sums its ring.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <type_traits>

#include "ops.cuh"

namespace hb {
namespace {

constexpr int LT_X = 32, LT_Y = 8, LT_NT = LT_X * LT_Y;

struct LocalArgs {
  int nz, ny, nx;  // input block
  int zo, nzo;     // output slices (block z)
  int w, zchunk;
  int kind;        // HB_LT_*
  double n, k, r, c;
};

template <typename T> struct Stage { using t = uint32_t; };
template <> struct Stage<float> { using t = float; };

template <typename A, typename S>
__device__ __forceinline__ A sqr(S v) {
  if constexpr (std::is_same<A, double>::value) return __dmul_rn((double)v, (double)v);
  else return (A)v * (A)v;  // unsigned: wraps mod 2^width like NumPy's int64
}

template <typename A>
__device__ __forceinline__ double to_f64(A s) {
  if constexpr (std::is_same<A, double>::value) return s;
  else if constexpr (std::is_same<A, uint64_t>::value) return __ll2double_rn((long long)s);  // int64 view
  else return (double)s;
}

template <typename A>
__device__ __forceinline__ A addA(A a, A b) {
  if constexpr (std::is_same<A, double>::value) return __dadd_rn(a, b);
  else return a + b;
}

// threshold from the window statistics (threshold.py:193-216 order)
__device__ __forceinline__ double box_threshold(double s1, double s2, const LocalArgs& a) {
  const double m = __ddiv_rn(s1, a.n);
  if (a.kind == HB_LT_MEAN) return __dsub_rn(m, a.c);
  double var = __dsub_rn(__ddiv_rn(s2, a.n), __dmul_rn(m, m));
  var = (var >= 0.0 || var != var) ? var : 0.0;  // np.maximum(var, 0.0)
  const double sd = __dsqrt_rn(var);
  if (a.kind == HB_LT_NIBLACK) return __dadd_rn(m, __dmul_rn(a.k, sd));
  return __dmul_rn(m, __dadd_rn(1.0, __dmul_rn(a.k, __dsub_rn(__ddiv_rn(sd, a.r), 1.0))));
}

template <typename T, typename A1, typename A2>
__global__ void __launch_bounds__(LT_NT)
k_local_box(const T* __restrict__ in, uint32_t* __restrict__ out, const LocalArgs a) {
  using S = typename Stage<T>::t;
  extern __shared__ __align__(16) unsigned char smem[];
  const int w = a.w, W = 2 * w + 1, HT = LT_Y + 2 * w, WT = LT_X + 2 * w;
  // layout: ring1 [W][256] A1 | ring2 [W][256] A2 | sx1 [HT][32] A1 | sx2 [HT][32] A2 | tile [HT][WT] S
  A2* ring2 = reinterpret_cast<A2*>(smem);
  A2* sx2 = ring2 + W * LT_NT;
  A1* ring1 = reinterpret_cast<A1*>(sx2 + HT * LT_X);
  A1* sx1 = ring1 + W * LT_NT;
  S* tile = reinterpret_cast<S*>(sx1 + HT * LT_X);
  const int tid = threadIdx.x, tx = tid & (LT_X - 1), ty = tid >> 5;
  const int x0 = blockIdx.x * LT_X, y0 = blockIdx.y * LT_Y;
  const int o0 = blockIdx.z * a.zchunk, o1 = min(o0 + a.zchunk, a.nzo);  // output-local
  const int64_t plane = (int64_t)a.ny * a.nx;
  const int gx = x0 + tx, gy = y0 + ty;
  const bool live = gx < a.nx && gy < a.ny;
  int step = 0;
  for (int zi = a.zo + o0 - w; zi < a.zo + o1 + w; ++zi, ++step) {
    const T* sl = in + (int64_t)clampi(zi, 0, a.nz - 1) * plane;
    for (int i = tid; i < HT * WT; i += LT_NT) {
      const int r = i / WT, c = i - r * WT;
      const int yy = clampi(y0 - w + r, 0, a.ny - 1), xx = clampi(x0 - w + c, 0, a.nx - 1);
      tile[i] = (S)__ldg(sl + (int64_t)yy * a.nx + xx);
    }
    __syncthreads();
    for (int i = tid; i < HT * LT_X; i += LT_NT) {
      const int r = i >> 5, c = i & (LT_X - 1);
      const S* t = tile + r * WT + c;
      A1 p1 = (A1)t[0];
      A2 p2 = sqr<A2>(t[0]);
      for (int d = 1; d < W; ++d) {
        p1 = addA(p1, (A1)t[d]);
        p2 = addA(p2, sqr<A2>(t[d]));
      }
      sx1[i] = p1;
      sx2[i] = p2;
    }
    __syncthreads();
    A1 q1 = sx1[ty * LT_X + tx];
    A2 q2 = sx2[ty * LT_X + tx];
    for (int d = 1; d < W; ++d) {
      q1 = addA(q1, sx1[(ty + d) * LT_X + tx]);
      q2 = addA(q2, sx2[(ty + d) * LT_X + tx]);
    }
    const int slot = step % W;
    ring1[slot * LT_NT + tid] = q1;
    ring2[slot * LT_NT + tid] = q2;
    if (step >= 2 * w && live) {
      // output slice zi - w; its window is the whole ring (oldest first)
      A1 s1 = ring1[((step + 1) % W) * LT_NT + tid];
      A2 s2 = ring2[((step + 1) % W) * LT_NT + tid];
      for (int d = 2; d <= W; ++d) {
        const int sl2 = (step + d) % W;
        s1 = addA(s1, ring1[sl2 * LT_NT + tid]);
        s2 = addA(s2, ring2[sl2 * LT_NT + tid]);
      }
      const double t = box_threshold(to_f64(s1), to_f64(s2), a);
      const int zc = zi - w;
      const int64_t off = (int64_t)gy * a.nx + gx;
      const double v = (double)__ldg(in + (int64_t)zc * plane + off);
      out[(int64_t)(zc - a.zo) * plane + off] = v > t ? 1u : 0u;
    }
  }
}

// Compile-time window (w <= 4): per-thread tile offsets hoisted out of the z
// loop, the next slice's tile prefetched into registers while the current one
// is summed, unrolled X / Y passes; integer data keeps running z sums
// (S += new - oldest: exact mod 2^64), float data sums the ring directly.
template <typename T, typename A1, typename A2, int WR>
__global__ void __launch_bounds__(LT_NT)
k_local_box_w(const T* __restrict__ in, uint32_t* __restrict__ out, const LocalArgs a) {
  using S = typename Stage<T>::t;
  constexpr int W = 2 * WR + 1, HT = LT_Y + 2 * WR, WT = LT_X + 2 * WR;
  constexpr int NL = (HT * WT + LT_NT - 1) / LT_NT;  // tile loads per thread
  constexpr int NXI = (HT + LT_Y - 1) / LT_Y;        // X-pass rows per thread
  constexpr bool RUN = !std::is_same<A1, double>::value;
  __shared__ S tile[HT * WT];
  __shared__ A1 sx1[HT * LT_X];
  __shared__ A2 sx2[HT * LT_X];
  __shared__ A1 ring1[W * LT_NT];
  __shared__ A2 ring2[W * LT_NT];
  const int tid = threadIdx.x, tx = tid & (LT_X - 1), ty = tid >> 5;
  const int x0 = blockIdx.x * LT_X, y0 = blockIdx.y * LT_Y;
  const int o0 = blockIdx.z * a.zchunk, o1 = min(o0 + a.zchunk, a.nzo);
  const int64_t plane = (int64_t)a.ny * a.nx;
  int off[NL];
#pragma unroll
  for (int j = 0; j < NL; ++j) {
    const int i = min(tid + j * LT_NT, HT * WT - 1);
    const int r = i / WT, c = i - r * WT;
    off[j] = clampi(y0 - WR + r, 0, a.ny - 1) * a.nx + clampi(x0 - WR + c, 0, a.nx - 1);
  }
  const int gx = x0 + tx, gy = y0 + ty;
  const bool live = gx < a.nx && gy < a.ny;
  const int zbeg = a.zo + o0 - WR, zend = a.zo + o1 + WR;
  S pre[NL];
  {
    const T* sl = in + (int64_t)clampi(zbeg, 0, a.nz - 1) * plane;
#pragma unroll
    for (int j = 0; j < NL; ++j) pre[j] = (S)__ldg(sl + off[j]);
  }
#pragma unroll
  for (int d = 0; d < W; ++d) {
    ring1[d * LT_NT + tid] = A1(0);
    ring2[d * LT_NT + tid] = A2(0);
  }
  A1 run1 = A1(0);
  A2 run2 = A2(0);
  int slot = 0;
  for (int zi = zbeg, step = 0; zi < zend; ++zi, ++step) {
#pragma unroll
    for (int j = 0; j < NL; ++j)
      if (j < NL - 1 || tid + j * LT_NT < HT * WT) tile[tid + j * LT_NT] = pre[j];
    __syncthreads();
    if (zi + 1 < zend) {
      const T* sl = in + (int64_t)clampi(zi + 1, 0, a.nz - 1) * plane;
#pragma unroll
      for (int j = 0; j < NL; ++j) pre[j] = (S)__ldg(sl + off[j]);
    }
#pragma unroll
    for (int k = 0; k < NXI; ++k) {
      const int r = ty + k * LT_Y;
      if (k < NXI - 1 || r < HT) {
        const S* t = tile + r * WT + tx;
        A1 p1 = (A1)t[0];
        A2 p2 = sqr<A2>(t[0]);
#pragma unroll
        for (int d = 1; d < W; ++d) {
          p1 = addA(p1, (A1)t[d]);
          p2 = addA(p2, sqr<A2>(t[d]));
        }
        sx1[r * LT_X + tx] = p1;
        sx2[r * LT_X + tx] = p2;
      }
    }
    __syncthreads();
    A1 q1 = sx1[ty * LT_X + tx];
    A2 q2 = sx2[ty * LT_X + tx];
#pragma unroll
    for (int d = 1; d < W; ++d) {
      q1 = addA(q1, sx1[(ty + d) * LT_X + tx]);
      q2 = addA(q2, sx2[(ty + d) * LT_X + tx]);
    }
    if constexpr (RUN) {
      run1 += q1 - ring1[slot * LT_NT + tid];
      run2 += q2 - ring2[slot * LT_NT + tid];
    }
    ring1[slot * LT_NT + tid] = q1;
    ring2[slot * LT_NT + tid] = q2;
    slot = slot + 1 == W ? 0 : slot + 1;
    if (step >= 2 * WR && live) {
      A1 s1;
      A2 s2;
      if constexpr (RUN) {
        s1 = run1;
        s2 = run2;
      } else {  // oldest first: slots slot, slot+1, ... (mod W)
        int sl2 = slot;
        s1 = ring1[sl2 * LT_NT + tid];
        s2 = ring2[sl2 * LT_NT + tid];
#pragma unroll
        for (int d = 1; d < W; ++d) {
          sl2 = sl2 + 1 == W ? 0 : sl2 + 1;
          s1 = addA(s1, ring1[sl2 * LT_NT + tid]);
          s2 = addA(s2, ring2[sl2 * LT_NT + tid]);
        }
      }
      const double t = box_threshold(to_f64(s1), to_f64(s2), a);
      const int zc = zi - WR;
      const int64_t o = (int64_t)gy * a.nx + gx;
      const double v = (double)__ldg(in + (int64_t)zc * plane + o);
      __stcs(out + (int64_t)(zc - a.zo) * plane + o, v > t ? 1u : 0u);
    }
  }
}

template <typename T, typename A1, typename A2, int WR>
cudaError_t run_box_w(const DevIn& in, int64_t nzo, uint32_t* out, LocalArgs a, cudaStream_t s,
                      int64_t* launches) {
  auto k = k_local_box_w<T, A1, A2, WR>;
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, LT_NT, 0) != cudaSuccess || per_sm < 1)
    per_sm = 1;
  const int gx = (int)((in.nx + LT_X - 1) / LT_X), gy = (int)((in.ny + LT_Y - 1) / LT_Y);
  const int64_t tiles = (int64_t)gx * gy, slots = (int64_t)kNumSMs * per_sm;
  int64_t split = std::max<int64_t>(1, (2 * slots + tiles - 1) / tiles);
  split = std::min<int64_t>(split, std::max<int64_t>(1, nzo / std::max(8 * WR, 8)));
  split = std::min<int64_t>(split, 65535);
  a.zchunk = (int)((nzo + split - 1) / split);
  dim3 grid(gx, gy, (unsigned)((nzo + a.zchunk - 1) / a.zchunk));
  k<<<grid, LT_NT, 0, s>>>((const T*)in.p, out, a);
  if (launches) *launches += 1;
  return cudaGetLastError();
}

template <typename T, typename A1, typename A2>
size_t box_smem(int w) {
  const int W = 2 * w + 1, HT = LT_Y + 2 * w, WT = LT_X + 2 * w;
  return (size_t)W * LT_NT * (sizeof(A1) + sizeof(A2)) + (size_t)HT * LT_X * (sizeof(A1) + sizeof(A2)) +
         (size_t)HT * WT * 4;
}

template <typename T, typename A1, typename A2>
cudaError_t run_box(const DevIn& in, int64_t zo, int64_t nzo, uint32_t* out, LocalArgs a, cudaStream_t s,
                    int64_t* launches) {
  if (!std::getenv("HB_LOCAL_GENERIC")) {
    switch (a.w) {
      case 1: return run_box_w<T, A1, A2, 1>(in, nzo, out, a, s, launches);
      case 2: return run_box_w<T, A1, A2, 2>(in, nzo, out, a, s, launches);
      case 3: return run_box_w<T, A1, A2, 3>(in, nzo, out, a, s, launches);
      case 4: return run_box_w<T, A1, A2, 4>(in, nzo, out, a, s, launches);
    }
  }
  const size_t smem = box_smem<T, A1, A2>(a.w);
  if (smem > 220 * 1024) return cudaErrorNotSupported;
  auto k = k_local_box<T, A1, A2>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, LT_NT, smem) != cudaSuccess || per_sm < 1)
    per_sm = 1;
  const int gx = (int)((in.nx + LT_X - 1) / LT_X), gy = (int)((in.ny + LT_Y - 1) / LT_Y);
  // z split: >= 2 waves of CTAs while each CTA's 2w priming slices stay < 1/4
  const int64_t tiles = (int64_t)gx * gy, slots = (int64_t)kNumSMs * per_sm;
  int64_t split = std::max<int64_t>(1, (2 * slots + tiles - 1) / tiles);
  split = std::min<int64_t>(split, std::max<int64_t>(1, nzo / std::max(8 * a.w, 8)));
  split = std::min<int64_t>(split, 65535);
  a.zchunk = (int)((nzo + split - 1) / split);
  dim3 grid(gx, gy, (unsigned)((nzo + a.zchunk - 1) / a.zchunk));
  k<<<grid, LT_NT, smem, s>>>((const T*)in.p, out, a);
  if (launches) *launches += 1;
  return cudaGetLastError();
}

// ---- gaussian kind: three float64 correlate1d passes (mode nearest) --------
struct CorrArgs {
  double w[2 * kMaxLocalRadius + 1];
  int R;
  int sym;
};

// one output voxel per thread-iteration, rows (z, y) x columns x.
// AXIS 0 reads the block input (T) at block slices zo+z; AXIS 1/2 read the
// previous pass (f64, nzo slices).  AXIS 2 compares: out = data > acc - c.
template <int AXIS, typename Tin, typename T>
__global__ void __launch_bounds__(256)
k_corr64(const Tin* __restrict__ src, double* __restrict__ dst, const T* __restrict__ data,
         uint32_t* __restrict__ labels, int nz, int ny, int nx, int zo, int nzo, double c,
         const CorrArgs a) {
  const int R = a.R;
  const int len = AXIS == 0 ? nz : (AXIS == 1 ? ny : nx);
  const int64_t plane = (int64_t)ny * nx;
  for (int64_t row = blockIdx.x; row < (int64_t)nzo * ny; row += gridDim.x) {
    const int z = (int)(row / ny), y = (int)(row - (int64_t)z * ny);
    for (int x = threadIdx.x; x < nx; x += 256) {
      int pos;
      const Tin* base;
      int64_t stride;
      if (AXIS == 0) {
        pos = zo + z;
        base = src + (int64_t)y * nx + x;
        stride = plane;
      } else if (AXIS == 1) {
        pos = y;
        base = src + (int64_t)z * plane + x;
        stride = nx;
      } else {
        pos = x;
        base = src + (int64_t)z * plane + (int64_t)y * nx;
        stride = 1;
      }
      auto at = [&](int q) { return (double)__ldg(base + (int64_t)clampi(q, 0, len - 1) * stride); };
      double acc;
      if (a.sym) {  // NI_Correlate1D symmetric fold
        acc = __dmul_rn(at(pos), a.w[R]);
        for (int d = R; d >= 1; --d)
          acc = __dadd_rn(acc, __dmul_rn(__dadd_rn(at(pos - d), at(pos + d)), a.w[R - d]));
      } else {
        acc = __dmul_rn(at(pos + R), a.w[2 * R]);
        for (int j = -R; j < R; ++j) acc = __dadd_rn(acc, __dmul_rn(at(pos + j), a.w[R + j]));
      }
      const int64_t o = (int64_t)z * plane + (int64_t)y * nx + x;
      if (AXIS < 2) {
        dst[o] = acc;
      } else {
        const double v = (double)__ldg(data + (int64_t)zo * plane + o);
        labels[o] = v > __dsub_rn(acc, c) ? 1u : 0u;
      }
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(256)
k_local_cmp(const T* __restrict__ data, const T* __restrict__ med, int64_t n, double c,
            uint32_t* __restrict__ labels) {
  for (int64_t i = blockIdx.x * 256ll + threadIdx.x; i < n; i += (int64_t)gridDim.x * 256)
    labels[i] = (double)__ldg(data + i) > __dsub_rn((double)__ldg(med + i), c) ? 1u : 0u;
}

inline int rows_grid(int64_t rows) { return (int)std::min<int64_t>(std::max<int64_t>(rows, 1), (int64_t)kNumSMs * 16); }

// Fused gaussian kind: a 32 x 8 tile of outputs streams down z with a ring of
// the last 2w+1 raw slices (halo'd, exact 4-byte staging) in shared memory; per
// output slice the Z pass runs once per (y, x) of the halo'd tile, the Y pass
// once per (y, x'), then the X pass and the comparison — the same three f64
// folds per voxel as k_corr64 (identical operation order), without the two
// float64 intermediate volumes (40 -> ~6 B/voxel of HBM traffic).
template <typename T, int RC>  // RC > 0: compile-time radius (unrolled folds)
__global__ void __launch_bounds__(LT_NT)
k_local_gauss_tile(const T* __restrict__ in, uint32_t* __restrict__ out, int nz, int ny, int nx, int zo,
                   int nzo, int zchunk, double c, const CorrArgs a) {
  using S = typename Stage<T>::t;
  extern __shared__ __align__(16) unsigned char smem[];
  const int R = RC > 0 ? RC : a.R, W = 2 * R + 1, HT = LT_Y + 2 * R, WT = LT_X + 2 * R;
  double* zt = reinterpret_cast<double*>(smem);  // [HT][WT]
  double* yt = zt + HT * WT;                      // [LT_Y][WT]
  S* ring = reinterpret_cast<S*>(yt + LT_Y * WT); // [W][HT][WT]
  const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
  const int x0 = blockIdx.x * LT_X, y0 = blockIdx.y * LT_Y;
  const int o0 = blockIdx.z * zchunk, o1 = min(o0 + zchunk, nzo);
  const int64_t plane = (int64_t)ny * nx;
  const int TS = HT * WT;
  auto fold = [&](auto at) {  // NI_Correlate1D order over window at(0..2R)
    double acc;
    if (a.sym) {
      acc = __dmul_rn(at(R), a.w[R]);
#pragma unroll
      for (int d = R; d >= 1; --d) acc = __dadd_rn(acc, __dmul_rn(__dadd_rn(at(R - d), at(R + d)), a.w[R - d]));
    } else {
      acc = __dmul_rn(at(2 * R), a.w[2 * R]);
#pragma unroll
      for (int j = 0; j < 2 * R; ++j) acc = __dadd_rn(acc, __dmul_rn(at(j), a.w[j]));
    }
    return acc;
  };
  auto load = [&](int zb, S* dst) {
    const T* sl = in + (int64_t)min(max(zb, 0), nz - 1) * plane;
    for (int i = tid; i < TS; i += LT_NT) {
      const int r = i / WT, cc = i - r * WT;
      dst[i] = (S)__ldg(sl + (int64_t)min(max(y0 - R + r, 0), ny - 1) * nx + min(max(x0 - R + cc, 0), nx - 1));
    }
  };
  // prime slices zo+o0-R .. zo+o0+R-1 into ring slots 0 .. 2R-1
  for (int k = 0; k < 2 * R; ++k) load(zo + o0 - R + k, ring + k * TS);
  int head = 2 * R;  // slot receiving the newest slice
  const int gx = x0 + tx, gy = y0 + ty;
  for (int o = o0; o < o1; ++o) {
    load(zo + o + R, ring + head * TS);
    __syncthreads();
    const int oldest = head + 1 == W ? 0 : head + 1;  // slice zo+o-R
    for (int i = tid; i < TS; i += LT_NT) {
      zt[i] = fold([&](int k) {
        int sl = oldest + k;
        sl -= sl >= W ? W : 0;
        return (double)ring[sl * TS + i];
      });
    }
    __syncthreads();
    for (int i = tid; i < LT_Y * WT; i += LT_NT) {
      const int r = i / WT, cc = i - r * WT;
      yt[i] = fold([&](int k) { return zt[(r + k) * WT + cc]; });
    }
    __syncthreads();
    if (gx < nx && gy < ny) {
      const double acc = fold([&](int k) { return yt[ty * WT + tx + k]; });
      int ctr = oldest + R;
      ctr -= ctr >= W ? W : 0;
      const double v = (double)ring[ctr * TS + (ty + R) * WT + tx + R];
      __stcs(out + (int64_t)o * plane + (int64_t)gy * nx + gx, v > __dsub_rn(acc, c) ? 1u : 0u);
    }
    head = oldest;
    __syncthreads();
  }
}

template <typename T>
size_t gauss_tile_smem(int w) {
  const int W = 2 * w + 1, HT = LT_Y + 2 * w, WT = LT_X + 2 * w;
  return (size_t)HT * WT * 8 + (size_t)LT_Y * WT * 8 + (size_t)W * HT * WT * 4;
}
inline bool gauss_fused_ok(int w) {
  return gauss_tile_smem<float>(w) <= 200 * 1024 && !std::getenv("HB_LOCAL_GAUSS_3PASS");
}

template <typename T>
cudaError_t run_gauss(const DevIn& in, int64_t zo, int64_t nzo, uint32_t* out, const double* kern, int w,
                      double c, double* t0, double* t1, cudaStream_t s, int64_t* launches) {
  CorrArgs a;
  a.R = w;
  for (int i = 0; i < 2 * w + 1; ++i) a.w[i] = kern[i];
  a.sym = 1;  // NI_Correlate1D's symmetry test (DBL_EPSILON tolerance)
  for (int i = 1; i <= w; ++i)
    if (std::fabs(kern[w + i] - kern[w - i]) > 2.220446049250313e-16) a.sym = 0;
  const int nz = (int)in.nz, ny = (int)in.ny, nx = (int)in.nx;
  const T* data = (const T*)in.p;
  const size_t smem = gauss_tile_smem<T>(w);
  if (gauss_fused_ok(w)) {
    auto k = w == 1 ? k_local_gauss_tile<T, 1> : w == 2 ? k_local_gauss_tile<T, 2>
           : w == 3 ? k_local_gauss_tile<T, 3> : w == 4 ? k_local_gauss_tile<T, 4> : k_local_gauss_tile<T, 0>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, LT_NT, smem) != cudaSuccess || per_sm < 1)
      per_sm = 1;
    const int gx = (nx + LT_X - 1) / LT_X, gy = (ny + LT_Y - 1) / LT_Y;
    const int64_t tiles = (int64_t)gx * gy, slots = (int64_t)kNumSMs * per_sm;
    int64_t split = std::max<int64_t>(1, (2 * slots + tiles - 1) / tiles);
    split = std::min<int64_t>(std::min<int64_t>(split, std::max<int64_t>(1, nzo / std::max(8 * w, 8))), 65535);
    const int zc = (int)((nzo + split - 1) / split);
    k<<<dim3(gx, gy, (unsigned)((nzo + zc - 1) / zc)), LT_NT, smem, s>>>(data, out, nz, ny, nx, (int)zo,
                                                                        (int)nzo, zc, c, a);
    if (launches) *launches += 1;
    return cudaGetLastError();
  }
  const int g = rows_grid(nzo * in.ny);
  k_corr64<0, T, T><<<g, 256, 0, s>>>(data, t0, data, out, nz, ny, nx, (int)zo, (int)nzo, c, a);
  k_corr64<1, double, T><<<g, 256, 0, s>>>(t0, t1, data, out, nz, ny, nx, (int)zo, (int)nzo, c, a);
  k_corr64<2, double, T><<<g, 256, 0, s>>>(t1, nullptr, data, out, nz, ny, nx, (int)zo, (int)nzo, c, a);
  if (launches) *launches += 3;
  return cudaGetLastError();
}

template <typename T>
cudaError_t run_median_cmp(const DevIn& in, int64_t zo, int64_t nzo, uint32_t* out, int w, double c,
                           void* med, cudaStream_t s, int64_t* launches) {
  cudaError_t e = median(in, zo, nzo, med, w, s, launches);
  if (e != cudaSuccess) return e;
  const int64_t n = nzo * in.ny * in.nx;
  const int g = (int)std::min<int64_t>((n + 255) / 256, (int64_t)kNumSMs * 32);
  k_local_cmp<T><<<g, 256, 0, s>>>((const T*)in.p + zo * in.ny * in.nx, (const T*)med, n, c, out);
  if (launches) *launches += 1;
  return cudaGetLastError();
}

template <typename T>
cudaError_t dispatch(const DevIn& in, int64_t zo, int64_t nzo, uint32_t* out, const LocalParams& p,
                     void* scratch, cudaStream_t s, int64_t* launches) {
  if (p.kind == HB_LT_MEDIAN) return run_median_cmp<T>(in, zo, nzo, out, p.w, p.c, scratch, s, launches);
  if (p.kind == HB_LT_GAUSSIAN) {
    double* t0 = (double*)scratch;
    double* t1 = t0 + nzo * in.ny * in.nx;
    return run_gauss<T>(in, zo, nzo, out, p.kern, p.w, p.c, t0, t1, s, launches);
  }
  LocalArgs a;
  a.nz = (int)in.nz;
  a.ny = (int)in.ny;
  a.nx = (int)in.nx;
  a.zo = (int)zo;
  a.nzo = (int)nzo;
  a.w = p.w;
  a.kind = p.kind;
  const double W = 2.0 * p.w + 1.0;
  a.n = W * W * W;  // (2w+1)**3 as an exact float64
  a.k = p.k;
  a.r = p.r;
  a.c = p.c;
  const bool small = p.w <= 19;  // (2w+1)^3 * 65535 < 2^32
  if constexpr (std::is_same<T, uint8_t>::value) {
    return small ? run_box<T, uint32_t, uint32_t>(in, zo, nzo, out, a, s, launches)
                 : run_box<T, uint32_t, uint64_t>(in, zo, nzo, out, a, s, launches);
  } else if constexpr (std::is_same<T, uint16_t>::value) {
    return small ? run_box<T, uint32_t, uint64_t>(in, zo, nzo, out, a, s, launches)
                 : run_box<T, uint64_t, uint64_t>(in, zo, nzo, out, a, s, launches);
  } else if constexpr (std::is_same<T, uint32_t>::value) {
    return run_box<T, uint64_t, uint64_t>(in, zo, nzo, out, a, s, launches);
  } else {
    return run_box<T, double, double>(in, zo, nzo, out, a, s, launches);
  }
}

}  // namespace

size_t local_threshold_scratch(int kind, int dt, int w, int64_t slices, int64_t plane) {
  if (kind == HB_LT_GAUSSIAN) return gauss_fused_ok(w) ? 0 : (size_t)(2 * slices * plane * 8);
  if (kind == HB_LT_MEDIAN) return (size_t)(slices * plane * dtype_size(dt));
  return 0;
}

int local_threshold_max_radius(int kind, int dt) {
  if (kind == HB_LT_GAUSSIAN) return kMaxLocalRadius;
  if (kind == HB_LT_MEDIAN) return 50;
  int w = 1;
  auto fits = [&](int r) {
    switch (dt) {
      case HB_U8: return box_smem<uint8_t, uint32_t, uint64_t>(r) <= 220 * 1024;
      case HB_U16: return box_smem<uint16_t, uint64_t, uint64_t>(r) <= 220 * 1024;
      default: return box_smem<float, double, double>(r) <= 220 * 1024;
    }
  };
  while (w < 50 && fits(w + 1)) ++w;
  return w;
}

cudaError_t local_threshold(const DevIn& in, int64_t zo, int64_t nzo, uint32_t* out, const LocalParams& p,
                            void* scratch, cudaStream_t s, int64_t* launches) {
  if (nzo <= 0) return cudaSuccess;
  switch (in.dt) {
    case HB_U8: return dispatch<uint8_t>(in, zo, nzo, out, p, scratch, s, launches);
    case HB_U16: return dispatch<uint16_t>(in, zo, nzo, out, p, scratch, s, launches);
    case HB_U32: return dispatch<uint32_t>(in, zo, nzo, out, p, scratch, s, launches);
    case HB_F32: return dispatch<float>(in, zo, nzo, out, p, scratch, s, launches);
  }
  return cudaErrorInvalidValue;
}

}  // namespace hb
