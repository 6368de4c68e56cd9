// box.cu — streaming 3D box mean (filters.py:66-75, scipy uniform_filter with
// mode="nearest"), fast fp32 mode, radius 1..2.
//
// The mean is pure HBM traffic (6 adds + 1 divide per voxel), so this kernel is
// built for bytes in flight, not for arithmetic: no shared memory, no barriers,
// no TMA single-thread issue.  A warp owns a 128-column x strip (4 columns per
// lane, one 128-bit load per row) of RY output rows and marches down a z-chunk:
//   per input slice: RY+2R rows are loaded with vector LDG (the next slice's
//   loads are in flight while the current one is summed), column (Y) sums run
//   in registers, the x neighbours come from the adjacent lanes by shuffle
//   (lanes 0/31 read the strip's edge columns directly, clamped), and the 2D
//   sums are accumulated into 2R running z accumulators — output o completes
//   when slice o+2R arrives and is stored with one streaming 128-bit store.
// Rows shared by vertically adjacent warps hit L1/L2; DRAM sees each input
// byte about once.  Summation order is identical to k_sep3d_fused (Y, then X,
// then Z, each left to right, z ascending), so results are bit-identical to it
// and independent of the chunk plan; the division is correctly rounded
// (FMA-refined reciprocal, checked exhaustively against __fdiv_rn for integer
// sums and on 2^30 sampled floats: tools/microbench/divtest.cu).
#include <cuda_runtime.h>

#include "ops.cuh"

namespace hb {
namespace {

constexpr int BX = 128;  // x columns per warp

template <typename T> struct V4;
template <> struct V4<float> { using t = float4; };
template <> struct V4<uint16_t> { using t = ushort4; };
template <> struct V4<uint8_t> { using t = uchar4; };

template <typename T>
__device__ __forceinline__ void ld4(const T* p, float (&f)[4]) {
  const typename V4<T>::t v = __ldg(reinterpret_cast<const typename V4<T>::t*>(p));
  f[0] = (float)v.x;
  f[1] = (float)v.y;
  f[2] = (float)v.z;
  f[3] = (float)v.w;
}

struct BoxArgs {
  int nz, ny, nx;   // input block
  int zo;           // block z of output slice 0
  int nzo;          // output slices
  int zchunk;       // output slices per CTA
  float count;      // (2r+1)^3
  float inv;        // RN(1/count)
};

template <typename T, int R, int RY>
struct Slice {
  float v[RY + 2 * R][4];  // own 4 columns of every loaded row
  float e[RY + 2 * R][R];  // edge columns (lane 0: left of the strip, lane 31: right)
};

template <typename T, int R, int RY>
__device__ __forceinline__ void load_slice(Slice<T, R, RY>& s, const T* __restrict__ plane,
                                           const int (&rowoff)[RY + 2 * R], int xc,
                                           const int (&ecol)[R], bool edge_lane) {
#pragma unroll
  for (int j = 0; j < RY + 2 * R; ++j) ld4(plane + rowoff[j] + xc, s.v[j]);
  if (edge_lane) {
#pragma unroll
    for (int j = 0; j < RY + 2 * R; ++j)
#pragma unroll
      for (int k = 0; k < R; ++k) s.e[j][k] = (float)__ldg(plane + rowoff[j] + ecol[k]);
  }
}

template <typename T, int R, int RY, int W>
__global__ void __launch_bounds__(32 * W) k_box_stream(const T* __restrict__ in,
                                                       float* __restrict__ out, const BoxArgs a) {
  constexpr int NR = RY + 2 * R;
  constexpr int P = 2 * R;  // live z accumulators
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int x0 = blockIdx.x * BX;
  const int xl = x0 + 4 * lane;
  const int y0 = (blockIdx.y * W + warp) * RY;
  if (y0 >= a.ny) return;  // no block-level synchronisation below
  const int oz0 = blockIdx.z * a.zchunk;
  const int oz1 = min(oz0 + a.zchunk, a.nzo);
  if (oz0 >= oz1) return;
  const int nsl = oz1 - oz0 + 2 * R;
  const bool act = xl < a.nx;
  const int xc = act ? xl : a.nx - 4;  // idle lanes read a valid vector
  const bool clamp_right = xl + 4 >= a.nx;  // right neighbours clamp to my column 3
  const bool edge_lane = lane == 0 || lane == 31;
  int ecol[R];
#pragma unroll
  for (int k = 0; k < R; ++k)
    ecol[k] = lane == 0 ? max(x0 - R + k, 0) : min(x0 + BX + k, a.nx - 1);
  int rowoff[NR];
#pragma unroll
  for (int j = 0; j < NR; ++j) rowoff[j] = min(max(y0 - R + j, 0), a.ny - 1) * a.nx;
  const int64_t plane = (int64_t)a.ny * a.nx;
  auto plane_of = [&](int i) {
    const int z = min(max(a.zo + oz0 - R + i, 0), a.nz - 1);
    return in + (int64_t)z * plane;
  };
  float* obase = out + (int64_t)oz0 * plane + (int64_t)y0 * a.nx + xl;
  const bool st_ok = act;

  float acc[P][RY][4];
#pragma unroll
  for (int p = 0; p < P; ++p)
#pragma unroll
    for (int r = 0; r < RY; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[p][r][c] = 0.f;

  Slice<T, R, RY> cur;
  load_slice<T, R, RY>(cur, plane_of(0), rowoff, xc, ecol, edge_lane);

  for (int i0 = 0; i0 < nsl; i0 += P) {
#pragma unroll
    for (int u = 0; u < P; ++u) {
      const int i = i0 + u;
      if (i < nsl) {
        Slice<T, R, RY> nxt;
        if (i + 1 < nsl) load_slice<T, R, RY>(nxt, plane_of(i + 1), rowoff, xc, ecol, edge_lane);
        // ---- Y pass: column sums of own and edge columns
        float ys[RY][4], ye[RY][R];
#pragma unroll
        for (int r = 0; r < RY; ++r) {
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            float t = cur.v[r][c];
#pragma unroll
            for (int k = 1; k <= 2 * R; ++k) t += cur.v[r + k][c];
            ys[r][c] = t;
          }
#pragma unroll
          for (int c = 0; c < R; ++c) {
            float t = cur.e[r][c];
#pragma unroll
            for (int k = 1; k <= 2 * R; ++k) t += cur.e[r + k][c];
            ye[r][c] = t;
          }
        }
        // ---- X pass over [left R | own 4 | right R]
        float s2[RY][4];
#pragma unroll
        for (int r = 0; r < RY; ++r) {
          float ext[4 + 2 * R];
#pragma unroll
          for (int k = 0; k < R; ++k) {
            const float l = __shfl_up_sync(0xffffffffu, ys[r][4 - R + k], 1);
            const float rr = __shfl_down_sync(0xffffffffu, ys[r][k], 1);
            ext[k] = lane == 0 ? ye[r][k] : l;
            ext[R + 4 + k] = lane == 31 ? ye[r][k] : (clamp_right ? ys[r][3] : rr);
          }
#pragma unroll
          for (int c = 0; c < 4; ++c) ext[R + c] = ys[r][c];
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            float t = ext[c];
#pragma unroll
            for (int k = 1; k <= 2 * R; ++k) t += ext[c + k];
            s2[r][c] = t;
          }
        }
        // ---- Z: slot (o mod 2R) accumulates output o over slices o..o+2R
        // (u == i mod 2R because i0 is a multiple of 2R)
        if (i >= 2 * R) {
          const int o = i - 2 * R;
          float* dst = obase + (int64_t)o * plane;
#pragma unroll
          for (int r = 0; r < RY; ++r) {
            float q[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              const float sum = acc[u][r][c] + s2[r][c];
              const float q0 = sum * a.inv;
              q[c] = fmaf(fmaf(-q0, a.count, sum), a.inv, q0);
            }
            if (st_ok && y0 + r < a.ny)
              __stcs(reinterpret_cast<float4*>(dst + r * a.nx), make_float4(q[0], q[1], q[2], q[3]));
          }
        }
#pragma unroll
        for (int d = 1; d < P; ++d) {
#pragma unroll
          for (int r = 0; r < RY; ++r)
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[(u + d) % P][r][c] += s2[r][c];
        }
#pragma unroll
        for (int r = 0; r < RY; ++r)
#pragma unroll
          for (int c = 0; c < 4; ++c) acc[u][r][c] = s2[r][c];
        cur = nxt;
      }
    }
  }
}

template <typename T, int R>
cudaError_t launch_box(const DevIn& in, int64_t zo, int64_t nzo, float* out, float count,
                       cudaStream_t s) {
  constexpr int RY = 4, W = 4;
  BoxArgs a;
  a.nz = (int)in.nz;
  a.ny = (int)in.ny;
  a.nx = (int)in.nx;
  a.zo = (int)zo;
  a.nzo = (int)nzo;
  a.count = count;
  a.inv = 1.0f / count;
  auto kern = k_box_stream<T, R, RY, W>;
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * W, 0) != cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
  int dev = 0, nsm = kNumSMs;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int gx = (int)((in.nx + BX - 1) / BX);
  const int gy = (int)((in.ny + RY * W - 1) / (RY * W));
  // z-chunking: balance waves of resident CTAs against each chunk's 2R priming slices
  const int64_t tiles = (int64_t)gx * gy, slots = (int64_t)nsm * per_sm;
  double best = 1e300;
  int64_t best_zc = nzo;
  for (int split = 1; split <= 512; ++split) {
    const int64_t zc = (nzo + split - 1) / split;
    if (split > 1 && zc < 8 * R + 8) break;
    const int64_t ctas = tiles * ((nzo + zc - 1) / zc);
    const int64_t waves = (ctas + slots - 1) / slots;
    const double cost = (double)waves * (double)(zc + 2 * R);
    if (cost < best * 0.98) {
      best = cost;
      best_zc = zc;
    }
  }
  a.zchunk = (int)best_zc;
  dim3 grid(gx, gy, (unsigned)((nzo + best_zc - 1) / best_zc));
  kern<<<grid, 32 * W, 0, s>>>(static_cast<const T*>(in.p), out, a);
  return cudaGetLastError();
}

template <typename T>
cudaError_t box_r(int r, const DevIn& in, int64_t zo, int64_t nzo, float* out, float count,
                  cudaStream_t s) {
  switch (r) {
    case 1: return launch_box<T, 1>(in, zo, nzo, out, count, s);
    case 2: return launch_box<T, 2>(in, zo, nzo, out, count, s);
  }
  return cudaErrorNotSupported;
}

}  // namespace

cudaError_t mean_stream(const DevIn& in, int64_t zo, int64_t nzo, float* out, int r,
                        cudaStream_t s, int64_t* launches) {
  if (nzo <= 0 || r < 1 || r > 2) return cudaErrorNotSupported;
  if (in.nx < 4 || in.nx % 4 != 0) return cudaErrorNotSupported;
  if (in.nz >= (1 << 30) || in.ny >= (1 << 30) || in.nx >= (1 << 30) ||
      in.ny * in.nx >= (1ll << 31))
    return cudaErrorNotSupported;
  const int es = dtype_size(in.dt);
  if ((reinterpret_cast<uintptr_t>(in.p) % (4 * es)) != 0 ||
      (reinterpret_cast<uintptr_t>(out) % 16) != 0)
    return cudaErrorNotSupported;
  const float size = (float)(2 * r + 1);
  const float count = size * size * size;
  cudaError_t e = cudaErrorNotSupported;
  switch (in.dt) {
    case HB_F32: e = box_r<float>(r, in, zo, nzo, out, count, s); break;
    case HB_U16: e = box_r<uint16_t>(r, in, zo, nzo, out, count, s); break;
    case HB_U8: e = box_r<uint8_t>(r, in, zo, nzo, out, count, s); break;
  }
  if (e == cudaSuccess && launches) *launches += 1;
  return e;
}

}  // namespace hb
