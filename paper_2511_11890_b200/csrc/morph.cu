// morph.cu — flat grey erosion / dilation with an arbitrary structuring element
// (morphology.py:103-121): out(p) = min_b I(clamp(p + b)) for erosion and
// max_b I(clamp(p - b)) for dilation (the host passes the reflected SE).
// Clamp-to-edge equals np.pad(mode="edge") followed by the offset views.
//
// The SE is decomposed on the host into (dz, dy) rows of contiguous dx runs
// [lo, lo+len).  The kernel stages a halo'd XY tile of each input slice in
// shared memory, computes the sliding window min/max of every run length
// once per slice (x direction), and folds the rows (y, z directions) for each
// output — for ball:3 that is 29 row terms instead of 123 offsets.
#include <vector>
#include <cstdlib>
#include <algorithm>
#include <array>
#include <map>

#include "ops.cuh"
#include "tma.cuh"

namespace hb {
namespace {

constexpr int kMaxRows = 256;
constexpr int kMaxLens = 8;

struct SeRows {
  int n_rows;
  int n_lens;
  int ez, ey, ex;          // extents (max |d|) per axis
  int lens[kMaxLens];      // distinct run lengths
  // packed row: dz (8b, +128) | dy (8b, +128) | lo (8b, +128) | len index (8b)
  uint32_t row[kMaxRows];
};

template <typename T, bool MAX>
__device__ __forceinline__ T op2(T a, T b) {
  return MAX ? (a > b ? a : b) : (a < b ? a : b);
}

// One CTA = TX x TY outputs, marching over z slices [z0, z1) of the output.
// Shared memory per slice of the ring (2*ez+1 slices):
//   runs[len_idx][TY + 2*ey][TX] = window reduce over [x+lo, x+lo+len) for the
//   row's lo; lo varies per row, so we store the run reduction for all x in
//   [x0 - ex, x0 + TX + ex) and index with lo.
template <typename T, bool MAX, int TX, int TY>
__global__ void __launch_bounds__(256)
k_morph(const T* __restrict__ in, int64_t nz, int64_t ny, int64_t nx, int64_t zo,
        int64_t nzo, int zchunk, T* __restrict__ out, SeRows se) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int nthreads = blockDim.x;
  const int tid = threadIdx.x;
  const int64_t x0 = (int64_t)blockIdx.x * TX;
  const int64_t y0 = (int64_t)blockIdx.y * TY;
  const int64_t zs = zo + (int64_t)blockIdx.z * zchunk;
  const int64_t ze = min(zs + zchunk, zo + nzo);
  if (zs >= ze) return;
  const int ring = 2 * se.ez + 1;
  const int WX = TX + 2 * se.ex;   // width of the halo'd raw row
  const int HY = TY + 2 * se.ey;   // rows per slice
  // layout: raw[HY][WX] scratch, then runs[ring][n_lens][HY][WX]
  T* raw = reinterpret_cast<T*>(smem_raw);
  T* runs = raw + HY * WX;
  const int slice_elems = se.n_lens * HY * WX;

  auto load_slice = [&](int64_t zin, int slot) {
    const int64_t zc = clamp64(zin, 0, nz - 1);
    const T* src = in + zc * ny * nx;
    for (int e = tid; e < HY * WX; e += nthreads) {
      int yy = e / WX, xx = e - yy * WX;
      int64_t gy = clamp64(y0 - se.ey + yy, 0, ny - 1);
      int64_t gx = clamp64(x0 - se.ex + xx, 0, nx - 1);
      raw[e] = src[gy * nx + gx];
    }
    __syncthreads();
    T* dst = runs + slot * slice_elems;
    for (int li = 0; li < se.n_lens; ++li) {
      const int len = se.lens[li];
      for (int e = tid; e < HY * WX; e += nthreads) {
        int yy = e / WX, xx = e - yy * WX;
        const T* r = raw + yy * WX;
        T acc = r[xx];
        for (int t = 1; t < len; ++t) acc = op2<T, MAX>(acc, r[min(xx + t, WX - 1)]);
        dst[li * HY * WX + e] = acc;
      }
    }
    __syncthreads();
  };

  // prime the ring with slices zs - ez .. zs + ez - 1
  for (int64_t zi = zs - se.ez; zi < zs + se.ez; ++zi) {
    int slot = (int)(((zi % ring) + ring) % ring);
    load_slice(zi, slot);
  }
  for (int64_t z = zs; z < ze; ++z) {
    {
      int64_t zi = z + se.ez;
      int slot = (int)(((zi % ring) + ring) % ring);
      load_slice(zi, slot);
    }
    for (int e = tid; e < TX * TY; e += nthreads) {
      int ty = e / TX, tx = e - ty * TX;
      int64_t gy = y0 + ty, gx = x0 + tx;
      if (gy >= ny || gx >= nx) continue;
      T acc = MAX ? (T)0 : (T)0;
      bool first = true;
      for (int k = 0; k < se.n_rows; ++k) {
        uint32_t pk = se.row[k];
        int dz = (int)((pk >> 24) & 0xff) - 128;
        int dy = (int)((pk >> 16) & 0xff) - 128;
        int lo = (int)((pk >> 8) & 0xff) - 128;
        int li = (int)(pk & 0xff);
        int64_t zi = z + dz;
        int slot = (int)(((zi % ring) + ring) % ring);
        // x index in the halo'd row: tx + ex + lo (>= 0 since lo >= -ex)
        T v = runs[slot * slice_elems + li * HY * WX + (ty + se.ey + dy) * WX + tx + se.ex + lo];
        acc = first ? v : op2<T, MAX>(acc, v);
        first = false;
      }
      out[((z - zo) * ny + gy) * nx + gx] = acc;
    }
    __syncthreads();
  }
}

bool build_rows(const int32_t* off, int n, SeRows& se) {
  if (n < 1) return false;
  std::map<std::pair<int, int>, std::vector<int>> rows;
  int ez = 0, ey = 0, ex = 0;
  for (int k = 0; k < n; ++k) {
    int dz = off[3 * k], dy = off[3 * k + 1], dx = off[3 * k + 2];
    if (std::abs(dz) > 100 || std::abs(dy) > 100 || std::abs(dx) > 100) return false;
    rows[{dz, dy}].push_back(dx);
    ez = std::max(ez, std::abs(dz));
    ey = std::max(ey, std::abs(dy));
    ex = std::max(ex, std::abs(dx));
  }
  se.ez = ez; se.ey = ey; se.ex = ex;
  se.n_rows = 0;
  se.n_lens = 0;
  for (auto& kv : rows) {
    std::vector<int>& v = kv.second;
    std::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
    size_t i = 0;
    while (i < v.size()) {
      size_t j = i;
      while (j + 1 < v.size() && v[j + 1] == v[j] + 1) ++j;
      int lo = v[i], len = v[j] - v[i] + 1;
      int li = -1;
      for (int q = 0; q < se.n_lens; ++q) if (se.lens[q] == len) li = q;
      if (li < 0) {
        if (se.n_lens >= kMaxLens) return false;
        li = se.n_lens;
        se.lens[se.n_lens++] = len;
      }
      if (se.n_rows >= kMaxRows) return false;
      se.row[se.n_rows++] = ((uint32_t)(kv.first.first + 128) << 24) |
                            ((uint32_t)(kv.first.second + 128) << 16) |
                            ((uint32_t)(lo + 128) << 8) | (uint32_t)li;
      i = j + 1;
    }
  }
  return true;
}

template <typename T>
cudaError_t run_morph(const DevIn& in, int64_t zo, int64_t nzo, void* out, const SeRows& se,
                      bool is_max, cudaStream_t s, int64_t* launches) {
  constexpr int TX = 32, TY = 16;
  const int threads = 256;
  const int WX = TX + 2 * se.ex, HY = TY + 2 * se.ey;
  size_t smem = sizeof(T) * (size_t)HY * WX * (1 + (size_t)(2 * se.ez + 1) * se.n_lens);
  if (smem > 200 * 1024) return cudaErrorNotSupported;
  dim3 grid((unsigned)((in.nx + TX - 1) / TX), (unsigned)((in.ny + TY - 1) / TY), 1);
  int64_t tiles = (int64_t)grid.x * grid.y;
  int64_t want_z = std::max<int64_t>(1, (4 * kNumSMs + tiles - 1) / tiles);
  int zchunk = (int)std::max<int64_t>(8, (nzo + want_z - 1) / want_z);
  grid.z = (unsigned)((nzo + zchunk - 1) / zchunk);
  auto kern = is_max ? k_morph<T, true, TX, TY> : k_morph<T, false, TX, TY>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  kern<<<grid, threads, smem, s>>>((const T*)in.p, in.nz, in.ny, in.nx, zo, nzo, zchunk,
                                   (T*)out, se);
  if (launches) *launches += 1;
  return cudaGetLastError();
}


// ===========================================================================
// v2: TMA-fed, shape-shared erosion/dilation for u8/u16 with odd centred runs
// ---------------------------------------------------------------------------
// The SE's dz-layers are 2D shapes; identical shapes (e.g. +dz and -dz of a
// ball) are evaluated once per slice.  Per input slice:
//   H: every halo'd row computes run-min/max of each needed odd length L
//      (run_{L+2}(c) = op(run_L(c+1), raw[c], raw[c+L+1]) -> one 3-input op per
//      length) and stores packed u16x2 pairs (run(c), run(c+1)) in smem;
//   V: each thread folds the rows of every distinct shape for its output pair
//      with min/max.u16x2 (two voxels per instruction);
//   Z: the shape values are pushed into a (2*EZ+1)-deep register ring of
//      pending outputs; the oldest output is complete and stored.
// ===========================================================================
constexpr int M2_TX = 64, M2_TY = 16, M2_NT = 256, M2_NST = 3;
constexpr int M2_MAXL = 8, M2_MAXSH = 9, M2_MAXROWS = 96;

struct Morph2Args {
  int nzi, zo, nzo, zchunk, nx, ny;
  int ez, ey, ex;
  int xa, wbox, hy, wc;          // smem geometry of the raw stage
  int n_lens;
  int lens[M2_MAXL];             // ascending odd run lengths (1 = raw)
  int n_shapes;
  int shape_of_dz[17];           // dz + ez -> shape id
  int row_begin[M2_MAXSH + 1];   // rows of shape k: [row_begin[k], row_begin[k+1])
  int row_off[M2_MAXROWS];       // (dy + ey) * wc + ex + lo  (index into a run array)
  int row_len[M2_MAXROWS];       // index into lens
  int off_runs, stage_pitch, off_bar;
};

template <bool MAX>
__device__ __forceinline__ uint32_t op2x2(uint32_t a, uint32_t b) {
  uint32_t d;
  if (MAX) asm("max.u16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  else asm("min.u16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
template <bool MAX>
__device__ __forceinline__ uint32_t op1(uint32_t a, uint32_t b) { return MAX ? max(a, b) : min(a, b); }

template <typename T, bool MAX, int EZ>
__global__ void __launch_bounds__(M2_NT, 2)
k_morph2(const __grid_constant__ CUtensorMap tin, T* __restrict__ out, const Morph2Args a) {
  constexpr int RING = 2 * EZ + 1;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem =
      smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u)  /* stays in .shared */;
  T* sraw = reinterpret_cast<T*>(smem);
  uint32_t* runs = reinterpret_cast<uint32_t*>(smem + a.off_runs);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + a.off_bar);
  const int tid = threadIdx.x;
  const int x0 = blockIdx.x * M2_TX, y0 = blockIdx.y * M2_TY;
  const int z0 = blockIdx.z * a.zchunk;
  const int z1 = min(z0 + a.zchunk, a.nzo);
  const int nsl = (z1 - z0) + 2 * EZ;
  const bool border = (x0 - a.ex < 0) || (x0 + M2_TX + a.ex > a.nx) || (y0 - a.ey < 0) ||
                      (y0 + M2_TY + a.ey > a.ny);
  const int xoff = a.xa - a.ex;
  const int stage_elems = a.stage_pitch / (int)sizeof(T);
  const uint32_t box_bytes = (uint32_t)(a.hy * a.wbox * sizeof(T));
  const int run_plane = a.hy * a.wc;  // uint32 entries per run length
  auto zin_of = [&](int s) { return min(max(a.zo + z0 - EZ + s, 0), a.nzi - 1); };

  if (tid == 0) {
    prefetch_tmap(&tin);
    for (int i = 0; i < M2_NST; ++i) mbar_init(&bar[i], 1);
    fence_mbar_init();
    for (int i = 0; i < M2_NST && i < nsl; ++i) {
      mbar_expect_tx(&bar[i], box_bytes);
      tma_load_3d(sraw + i * stage_elems, &tin, x0 - a.xa, y0 - a.ey, zin_of(i), &bar[i]);
    }
  }
  __syncthreads();

  const int px = tid & 31, ty = tid >> 5;  // output pair px (x = 2px), rows ty, ty+8
  uint32_t acc[2][RING];
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int u = 0; u < RING; ++u) acc[r][u] = MAX ? 0u : 0xffffffffu;
  const int lmax = a.lens[a.n_lens - 1];
  const int nseg = (a.wc + 7) / 8;

  for (int s = 0; s < nsl; ++s) {
    const int st = s % M2_NST;
    T* stage = sraw + st * stage_elems;
    mbar_wait(&bar[st], (uint32_t)((s / M2_NST) & 1));
    if (border) {
      for (int e = tid; e < a.hy * a.wc; e += M2_NT) {
        const int ly = e / a.wc, lx = e - ly * a.wc;
        const int gy = y0 - a.ey + ly, gx = x0 - a.ex + lx;
        const int cy = min(max(gy, 0), a.ny - 1), cx = min(max(gx, 0), a.nx - 1);
        if (cy != gy || cx != gx)
          stage[ly * a.wbox + xoff + lx] = stage[(cy - (y0 - a.ey)) * a.wbox + xoff + (cx - (x0 - a.ex))];
      }
      fence_proxy_async();
      __syncthreads();
    }
    // ---- H: runs of every length for 8 consecutive columns per item -------
    for (int item = tid; item < a.hy * nseg; item += M2_NT) {
      const int r = item / nseg, c0 = (item - r * nseg) * 8;
      const T* row = stage + r * a.wbox + xoff;
      uint32_t raw[8 + 2 * 8 + 2];  // c0 .. c0 + 9 + lmax (clamped to the row)
      const int need = 9 + lmax;
#pragma unroll
      for (int i = 0; i < 26; ++i)
        if (i < need) raw[i] = (uint32_t)row[min(c0 + i, a.wc - 1)];
      // run_L(c0 + i) for i = 0..17; position i at step t needs i+1 at step t-1,
      // so 18 entries keep i <= 8 exact for up to 8 steps (L <= 17)
      uint32_t run[18];
#pragma unroll
      for (int i = 0; i < 18; ++i) run[i] = raw[i];
      int li = 0;
#pragma unroll
      for (int step = 0; step <= 8; ++step) {
        const int L = 2 * step + 1;
        if (li < a.n_lens && a.lens[li] == L) {
          uint32_t* dst = runs + li * run_plane + r * a.wc + c0;
#pragma unroll
          for (int i = 0; i < 8; ++i)
            if (c0 + i < a.wc) dst[i] = run[i] | (run[i + 1] << 16);
          ++li;
        }
        if (L >= lmax) break;
        // run_{L+2}(c) = op(run_L(c+1), raw[c], raw[c+L+1])
#pragma unroll
        for (int i = 0; i < 18; ++i) {
          const uint32_t inner = run[i < 17 ? i + 1 : 17];
          run[i] = op1<MAX>(op1<MAX>(inner, raw[i]), raw[(i + L + 1) < 26 ? (i + L + 1) : 25]);
        }
      }
    }
    __syncthreads();
    if (tid == 0 && s + M2_NST < nsl) {
      fence_proxy_async();
      mbar_expect_tx(&bar[st], box_bytes);
      tma_load_3d(stage, &tin, x0 - a.xa, y0 - a.ey, zin_of(s + M2_NST), &bar[st]);
    }
    // ---- V + Z --------------------------------------------------------------
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
      const int yo = ty + 8 * rr;
      const int base = yo * a.wc + 2 * px;
      uint32_t shape_val[M2_MAXSH];
#pragma unroll
      for (int k = 0; k < M2_MAXSH; ++k) {
        if (k < a.n_shapes) {
          uint32_t v = MAX ? 0u : 0xffffffffu;
          for (int q = a.row_begin[k]; q < a.row_begin[k + 1]; ++q)
            v = op2x2<MAX>(v, runs[a.row_len[q] * run_plane + base + a.row_off[q]]);
          shape_val[k] = v;
        }
      }
      // slice s sits at dz = s - z from pending output z (z = s - EZ .. s + EZ)
      switch (s % RING) {
#define HB_M2_CASE(U)                                                              \
  case U:                                                                          \
    if constexpr (U < RING) {                                                      \
      _Pragma("unroll") for (int d = -EZ; d <= EZ; ++d) {                          \
        /* output z = s - d lives in ring slot (U - d) mod RING */                 \
        const int sh = a.shape_of_dz[d + EZ];                                      \
        uint32_t sv = shape_val[0];                                                \
        _Pragma("unroll") for (int k = 1; k < M2_MAXSH; ++k) if (k == sh) sv = shape_val[k]; \
        if (sh >= 0) acc[rr][((U - d) % RING + RING) % RING] =                     \
            op2x2<MAX>(acc[rr][((U - d) % RING + RING) % RING], sv);               \
      }                                                                            \
      {                                                                            \
        const int o = s - 2 * EZ; /* output (chunk-local) completed now */        \
        const int slot = ((U - EZ) % RING + RING) % RING;                          \
        if (o >= 0) {                                                              \
          const int gy = y0 + yo, gx = x0 + 2 * px;                                \
          if (gy < a.ny && gx < a.nx) {                                            \
            T* dst = out + ((int64_t)(z0 + o) * a.ny + gy) * (int64_t)a.nx + gx;    \
            const uint32_t v = acc[rr][slot];                                      \
            dst[0] = (T)(v & 0xffffu);                                             \
            if (gx + 1 < a.nx) dst[1] = (T)(v >> 16);                              \
          }                                                                        \
        }                                                                          \
        acc[rr][slot] = MAX ? 0u : 0xffffffffu;                                    \
      }                                                                            \
    }                                                                              \
    break;
        HB_M2_CASE(0) HB_M2_CASE(1) HB_M2_CASE(2) HB_M2_CASE(3) HB_M2_CASE(4)
        HB_M2_CASE(5) HB_M2_CASE(6) HB_M2_CASE(7) HB_M2_CASE(8)
#undef HB_M2_CASE
        default: break;
      }
    }
    __syncthreads();  // runs are rewritten by the next slice's H phase
  }
}

// host-side builder for Morph2Args; false if the SE is outside v2's envelope
bool build_morph2(const int32_t* off, int n, Morph2Args& a) {
  std::map<int, std::map<int, std::vector<int>>> layers;  // dz -> dy -> dx list
  int ez = 0, ey = 0, ex = 0;
  for (int k = 0; k < n; ++k) {
    const int dz = off[3 * k], dy = off[3 * k + 1], dx = off[3 * k + 2];
    layers[dz][dy].push_back(dx);
    ez = std::max(ez, std::abs(dz));
    ey = std::max(ey, std::abs(dy));
    ex = std::max(ex, std::abs(dx));
  }
  if (ez > 4 || ey > 8 || ex > 8) return false;
  a.ez = ez; a.ey = ey; a.ex = ex;
  // rows: each (dz, dy) must be one contiguous dx run of odd length centred at 0
  std::vector<std::vector<std::pair<int, int>>> shapes;  // list of (dy, len)
  for (int i = 0; i < 17; ++i) a.shape_of_dz[i] = -1;
  std::vector<int> lens;
  for (auto& L : layers) {
    std::vector<std::pair<int, int>> rows;
    for (auto& R : L.second) {
      std::vector<int> v = R.second;
      std::sort(v.begin(), v.end());
      v.erase(std::unique(v.begin(), v.end()), v.end());
      const int lo = v.front(), hi = v.back();
      if ((int)v.size() != hi - lo + 1 || lo != -hi) return false;  // contiguous, centred
      rows.push_back({R.first, hi - lo + 1});
      lens.push_back(hi - lo + 1);
    }
    int id = -1;
    for (size_t k = 0; k < shapes.size(); ++k)
      if (shapes[k] == rows) id = (int)k;
    if (id < 0) {
      id = (int)shapes.size();
      shapes.push_back(rows);
    }
    a.shape_of_dz[L.first + ez] = id;
  }
  std::sort(lens.begin(), lens.end());
  lens.erase(std::unique(lens.begin(), lens.end()), lens.end());
  if ((int)lens.size() > M2_MAXL || (int)shapes.size() > M2_MAXSH) return false;
  a.n_lens = (int)lens.size();
  for (int i = 0; i < a.n_lens; ++i) a.lens[i] = lens[i];
  a.n_shapes = (int)shapes.size();
  a.wc = M2_TX + 2 * ex;
  int q = 0;
  for (int k = 0; k < a.n_shapes; ++k) {
    a.row_begin[k] = q;
    for (auto& rl : shapes[k]) {
      if (q >= M2_MAXROWS) return false;
      const int li = (int)(std::find(lens.begin(), lens.end(), rl.second) - lens.begin());
      const int half = (rl.second - 1) / 2;
      a.row_off[q] = (rl.first + ey) * a.wc + ex - half;
      a.row_len[q] = li;
      ++q;
    }
  }
  a.row_begin[a.n_shapes] = q;
  return true;
}

template <typename T, bool MAX, int EZ>
cudaError_t launch_morph2(const DevIn& in, int64_t zo, int64_t nzo, void* out, Morph2Args a,
                          cudaStream_t s) {
  const int align = 16 / (int)sizeof(T);
  a.xa = (a.ex + align - 1) / align * align;
  a.wbox = (a.xa + M2_TX + a.ex + align - 1) / align * align;
  a.hy = M2_TY + 2 * a.ey;
  CUtensorMap tin;
  const CUtensorMapDataType dt = sizeof(T) == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_UINT16;
  if (!make_tmap_3d(&tin, in.p, dt, sizeof(T), in.nx, in.ny, in.nz, a.wbox, a.hy))
    return cudaErrorNotSupported;
  a.stage_pitch = (a.hy * a.wbox * (int)sizeof(T) + 127) / 128 * 128;
  a.off_runs = M2_NST * a.stage_pitch;
  a.off_bar = a.off_runs + a.n_lens * a.hy * a.wc * 4;
  a.off_bar = (a.off_bar + 15) / 16 * 16;
  const int smem = a.off_bar + M2_NST * 8 + 128;
  if (smem > 110 * 1024) return cudaErrorNotSupported;
  a.nzi = (int)in.nz;
  a.zo = (int)zo;
  a.nzo = (int)nzo;
  a.nx = (int)in.nx;
  a.ny = (int)in.ny;
  const int gx = (int)((in.nx + M2_TX - 1) / M2_TX), gy = (int)((in.ny + M2_TY - 1) / M2_TY);
  const int64_t tiles = (int64_t)gx * gy;
  const int64_t want = std::max<int64_t>(1, (2 * 2 * kNumSMs + tiles - 1) / tiles);
  a.zchunk = (int)std::max<int64_t>(std::min<int64_t>(nzo, 8 * EZ + 8), (nzo + want - 1) / want);
  dim3 grid(gx, gy, (unsigned)((nzo + a.zchunk - 1) / a.zchunk));
  auto kern = k_morph2<T, MAX, EZ>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  kern<<<grid, M2_NT, smem, s>>>(tin, (T*)out, a);
  return cudaGetLastError();
}

template <typename T, bool MAX>
cudaError_t dispatch_morph2(const DevIn& in, int64_t zo, int64_t nzo, void* out,
                            const Morph2Args& a, cudaStream_t s) {
  switch (a.ez) {
    case 0: return launch_morph2<T, MAX, 0>(in, zo, nzo, out, a, s);
    case 1: return launch_morph2<T, MAX, 1>(in, zo, nzo, out, a, s);
    case 2: return launch_morph2<T, MAX, 2>(in, zo, nzo, out, a, s);
    case 3: return launch_morph2<T, MAX, 3>(in, zo, nzo, out, a, s);
    case 4: return launch_morph2<T, MAX, 4>(in, zo, nzo, out, a, s);
  }
  return cudaErrorNotSupported;
}


// ===========================================================================
// v3: compile-time structuring elements (ball / box / cross, r <= 3) — the fast
// path for the reference's factory shapes (morphology.py:49-82).
// ---------------------------------------------------------------------------
// Layer |dz| of the SE is a 2D shape of centred x-runs with half-width
// hw(dz, dy) (-1 = row absent), known at compile time.  Per input slice:
//   H: each (row, 4-wide x block) item builds the run reductions h_k, k<=R,
//      as packed u16x2 pairs: h_k = op(h_{k-1}, shift(-k), shift(+k)), one
//      3-input VIMNMX per k, odd shifts via PRMT; stored to smem.
//   V: each thread folds the rows of every layer for its 4 outputs (two
//      u16x2 words); identical smem loads across layers are CSE'd.
//   Z: layer values are pushed into a (2R+1)-slot register ring of pending
//      outputs (output z takes layer |dz| of slice z+dz); the oldest is stored.
// u8 volumes are widened into u16 lanes on load and narrowed on store.
// ===========================================================================
enum { SE_BALL = 0, SE_BOX = 1, SE_CROSS = 2 };

template <int KIND, int R>
struct SeShape {
  static constexpr __host__ __device__ int isqrt(int v) {
    int r = 0;
    while ((r + 1) * (r + 1) <= v) ++r;
    return r;
  }
  // half-width of the x-run at (dz, dy), -1 if the row is absent
  static constexpr __host__ __device__ int hw(int dz, int dy) {
    if (dz < 0) dz = -dz;
    if (dy < 0) dy = -dy;
    if (dz > R || dy > R) return -1;
    if (KIND == SE_BOX) return R;
    if (KIND == SE_CROSS) return (dz == 0 && dy == 0) ? R : ((dz == 0 || dy == 0) ? 0 : -1);
    const int rem = R * R - dz * dz - dy * dy;
    return rem < 0 ? -1 : isqrt(rem);
  }
  // number of rows (dy) of layer |dz| = L, and its dy extent
  static constexpr __host__ __device__ int nterms(int L) {
    int n = 0;
    for (int dy = -R; dy <= R; ++dy) n += hw(L, dy) >= 0;
    return n;
  }
  static constexpr __host__ __device__ int dyext(int L) {
    int e = -1;
    for (int dy = 0; dy <= R; ++dy)
      if (hw(L, dy) >= 0) e = dy;
    return e;
  }
  static constexpr __host__ __device__ bool needs(int k) {  // is run half-width k used anywhere?
    for (int dz = 0; dz <= R; ++dz)
      for (int dy = 0; dy <= R; ++dy)
        if (hw(dz, dy) == k) return true;
    return false;
  }
};

constexpr int M3X_TX = 64, M3X_TY = 32, M3X_NT = 512, M3X_NST = 3;
constexpr int M3X_Q = M3X_TX / 4;  // 4-wide x blocks per row (16)
// output rows per V/Z thread: 2 for grey data — each staged H row a thread
// loads serves two output rows, cutting the shared-memory reads of the layer
// folds that bounded the kernel (ncu: LSU 66%, LDS barrier/mio stalls) —
// and 1 for the binary AND/OR variant
#ifndef HB_M3X_MINB
#define HB_M3X_MINB 3
#endif
#ifndef HB_M3X_VR
#define HB_M3X_VR 2  // u16 ball:3 2048^2: VR 1 576, 2 598 (at 3 CTAs/SM), 4 spills (518)
#endif
template <bool BIN> struct M3XV {
  static constexpr int VR = BIN ? 1 : HB_M3X_VR;
  static constexpr int NT = M3X_Q * (M3X_TY / VR);
  static constexpr int MINB = BIN ? 2 : HB_M3X_MINB;  // resident CTAs the register budget is sized for
};

struct Morph3Args {
  int nzi, zo, nzo, zchunk, nx, ny;
};

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
  return d;
}
template <bool MAX>
__device__ __forceinline__ uint32_t op3x2(uint32_t a, uint32_t b, uint32_t c) {
  return op2x2<MAX>(op2x2<MAX>(a, b), c);  // ptxas fuses into VIMNMX3.U16x2
}

// BIN (uint8 only): a {0,1} volume, where min/max are AND/OR of whole words —
// four voxels per 32-bit op (LOP3 folds three), no u16 widening.  `gate`
// (device): 0 = the block is binary, 1 = grey; the BIN and grey u8 kernels
// are both enqueued and each returns at once unless the gate selects it.
template <bool MAX, bool BIN>
__device__ __forceinline__ uint32_t mop2(uint32_t a, uint32_t b) {
  if constexpr (BIN) return MAX ? (a | b) : (a & b);
  else return op2x2<MAX>(a, b);
}
template <bool MAX, bool BIN>
__device__ __forceinline__ uint32_t mop3(uint32_t a, uint32_t b, uint32_t c) {
  if constexpr (BIN) return MAX ? (a | b | c) : (a & b & c);
  else return op3x2<MAX>(a, b, c);
}

template <typename T, bool MAX, int KIND, int R, bool BIN>
__global__ void __launch_bounds__(M3XV<BIN>::NT, M3XV<BIN>::MINB)
k_morph3(const __grid_constant__ CUtensorMap tin, T* __restrict__ out, const Morph3Args a,
         const int* __restrict__ gate) {
  static_assert(!BIN || sizeof(T) == 1, "the binary path is uint8 only");
  if (gate != nullptr && ((*gate != 0) == BIN)) return;  // the other variant runs
  using S = SeShape<KIND, R>;
  constexpr int NW = BIN ? 1 : 2;  // 32-bit words per thread (4 voxels)
  constexpr int ALIGN = 16 / (int)sizeof(T);
  constexpr int XA = (R + ALIGN - 1) / ALIGN * ALIGN < 4 ? 4 : (R + ALIGN - 1) / ALIGN * ALIGN;
  constexpr int XA2 = (XA + ALIGN - 1) / ALIGN * ALIGN;   // box start offset (>= 4, 16-B aligned)
  constexpr int WBOX = (XA2 + M3X_TX + XA2 + ALIGN - 1) / ALIGN * ALIGN;
  constexpr int HY = M3X_TY + 2 * R;
  constexpr int STAGE_BYTES = HY * WBOX * (int)sizeof(T);
  constexpr int STAGE_PITCH = (STAGE_BYTES + 127) / 128 * 128;
  constexpr int RING = 2 * R + 1;
  constexpr int WPR = BIN ? M3X_TX / 4 : M3X_TX / 2;  // words per H row
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem =
      smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u)  /* stays in .shared */;
  T* sraw = reinterpret_cast<T*>(smem);
  uint32_t* sH = reinterpret_cast<uint32_t*>(smem + M3X_NST * STAGE_PITCH);  // [R][HY][WPR]
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + M3X_NST * STAGE_PITCH + (R > 0 ? R : 1) * HY * WPR * 4);
  const int tid = threadIdx.x;
  const int x0 = blockIdx.x * M3X_TX, y0 = blockIdx.y * M3X_TY;
  const int z0 = blockIdx.z * a.zchunk;
  const int z1 = min(z0 + a.zchunk, a.nzo);
  const int nsl = (z1 - z0) + 2 * R;
  const bool border = (x0 - R < 0) || (x0 + M3X_TX + R > a.nx) || (y0 - R < 0) || (y0 + M3X_TY + R > a.ny);
  constexpr uint32_t BOX_BYTES = HY * WBOX * sizeof(T);
  auto zin_of = [&](int s) { return min(max(a.zo + z0 - R + s, 0), a.nzi - 1); };

  if (tid == 0) {
    prefetch_tmap(&tin);
    for (int i = 0; i < M3X_NST; ++i) mbar_init(&bar[i], 1);
    fence_mbar_init();
    for (int i = 0; i < M3X_NST && i < nsl; ++i) {
      mbar_expect_tx(&bar[i], BOX_BYTES);
      tma_load_3d(sraw + i * (STAGE_PITCH / sizeof(T)), &tin, x0 - XA2, y0 - R, zin_of(i), &bar[i]);
    }
  }
  __syncthreads();

  // V/Z ownership: rows vy .. vy+VR-1, 4-wide x block vq (two u16x2 words:
  // pairs 2vq, 2vq+1)
  constexpr int VR = M3XV<BIN>::VR, NTK = M3XV<BIN>::NT;
  const int vq = tid % M3X_Q, vy = (tid / M3X_Q) * VR;  // vy in [0, 32)
  uint32_t acc[RING][VR][NW];
  constexpr uint32_t IDENT = MAX ? 0u : 0xffffffffu;
#pragma unroll
  for (int u = 0; u < RING; ++u)
#pragma unroll
    for (int t = 0; t < VR; ++t)
#pragma unroll
      for (int j = 0; j < NW; ++j) acc[u][t][j] = IDENT;

  // load the u16x2 word covering x = (tile) 2p, 2p+1 of stage row r
  auto word = [&](const T* row, int p) -> uint32_t {
    if constexpr (sizeof(T) == 2) {
      return *reinterpret_cast<const uint32_t*>(row + XA2 + 2 * p);
    } else {
      const uint16_t b2 = *reinterpret_cast<const uint16_t*>(row + XA2 + 2 * p);
      return (uint32_t)(b2 & 0xff) | ((uint32_t)(b2 >> 8) << 16);
    }
  };

  // output pointer of local output slice 0 and this thread's store shape
  const int gy = y0 + vy, gx = x0 + 4 * vq;
  const bool st_x = gx + 3 < a.nx, st_xp = gx < a.nx && !st_x;
  T* const obase = out + ((int64_t)z0 * a.ny + min(gy, a.ny - 1)) * (int64_t)a.nx + min(gx, a.nx - 1);
  const int64_t oplane = (int64_t)a.ny * a.nx;
  auto store_out = [&](int o, int t, uint32_t v0, uint32_t v1) {
    const bool st_full = gy + t < a.ny && st_x;
    const bool st_part = gy + t < a.ny && st_xp;
    T* dst = obase + o * oplane + (gy + t < a.ny ? t : 0) * (int64_t)a.nx;
    if constexpr (BIN) {
      if (st_full) *reinterpret_cast<uint32_t*>(dst) = v0;
      else if (st_part)
        for (int i = 0; i < 4 && gx + i < a.nx; ++i) dst[i] = (T)((v0 >> (8 * i)) & 0xffu);
    } else {
      if (st_full) {
        if constexpr (sizeof(T) == 2) *reinterpret_cast<uint2*>(dst) = make_uint2(v0, v1);
        else *reinterpret_cast<uint32_t*>(dst) = prmt(v0, v1, 0x6420);
      } else if (st_part) {
        const uint32_t vv[2] = {v0, v1};
        for (int i = 0; i < 4 && gx + i < a.nx; ++i) dst[i] = (T)((vv[i >> 1] >> (16 * (i & 1))) & 0xffffu);
      }
    }
  };

  for (int s = 0; s < nsl; ++s) {
    const int st = s % M3X_NST;
    T* stage = sraw + st * (STAGE_PITCH / sizeof(T));
    mbar_wait(&bar[st], (uint32_t)((s / M3X_NST) & 1));
    if (border) {
      clamp_tile<T, NTK>(stage, WBOX, HY, M3X_TX + 2 * XA2, y0 - R, x0 - XA2, a.ny, a.nx, tid);
      fence_proxy_async();
      __syncthreads();
    }
    // ---- H: run reductions for every halo'd row -----------------------------
    if constexpr (R > 0) {
      // a compile-time trip count lets the per-item index math hoist out of the slice loop
#pragma unroll
      for (int it = 0; it < (HY * M3X_Q + NTK - 1) / NTK; ++it) {
        const int item = tid + it * NTK;
        if (item >= HY * M3X_Q) break;
        const int r = item / M3X_Q, q = item % M3X_Q;
        const T* row = stage + r * WBOX;
        if constexpr (BIN) {
          // words of 4 voxels: w[0] = voxels 4q-4..4q-1, w[1] = 4q..4q+3, w[2] = 4q+4..4q+7;
          // shift(d) picks bytes across word boundaries with one PRMT
          uint32_t wb[3];
#pragma unroll
          for (int i = 0; i < 3; ++i) wb[i] = *reinterpret_cast<const uint32_t*>(row + XA2 + 4 * q - 4 + 4 * i);
          auto shb = [&](int d) -> uint32_t {
            if (d == 0) return wb[1];
            // bytes (4 + d) .. (7 + d) of the 12-byte window wb[0..2]
            const int b0 = 4 + d;
            const uint32_t lo = b0 < 4 ? wb[0] : wb[1], hi = b0 < 4 ? wb[1] : wb[2];
            const int o = b0 & 3;
            const uint32_t sel = (uint32_t)(o | ((o + 1) << 4) | ((o + 2) << 8) | ((o + 3) << 12));
            return prmt(lo, hi, sel);
          };
          uint32_t h = wb[1];
#pragma unroll
          for (int k = 1; k <= R; ++k) {
            h = mop3<MAX, BIN>(h, shb(-k), shb(k));
            if (S::needs(k)) sH[((k - 1) * HY + r) * WPR + q] = h;
          }
        } else {
        uint32_t w[6];  // pairs 2q-2 .. 2q+3
#pragma unroll
        for (int i = 0; i < 6; ++i) {
          if constexpr (sizeof(T) == 2) {
            w[i] = word(row, 2 * q - 2 + i);
          } else {
            // u8: three aligned 32-bit loads cover voxels 4q-4 .. 4q+7; each
            // byte pair is widened into u16 lanes with one PRMT
            const uint32_t b4 = *reinterpret_cast<const uint32_t*>(row + XA2 + 4 * q - 4 + 4 * (i >> 1));
            w[i] = prmt(b4, 0u, (i & 1) ? 0x4342u : 0x4140u);
          }
        }
#pragma unroll
        for (int j = 0; j < 2; ++j) {  // pair 2q + j -> w[2 + j]
          const uint32_t c = w[2 + j];
          // shift(d): the pair of voxels (2j+d, 2j+d+1) relative to x = 4q; word i
          // holds voxels (2i-4, 2i-3); odd starts straddle two words
          auto sh = [&](int d) -> uint32_t {
            const int v = 2 * j + d;
            if ((v & 1) == 0) return w[(v + 4) / 2];
            const int k = (v + 3) / 2;
            return prmt(w[k], w[k + 1], 0x5432);
          };
          uint32_t h = c;
#pragma unroll
          for (int k = 1; k <= R; ++k) {
            h = op3x2<MAX>(h, sh(-k), sh(k));
            if (S::needs(k)) sH[((k - 1) * HY + r) * WPR + 2 * q + j] = h;
          }
        }
        }  // !BIN
      }
    }
    __syncthreads();
    // ---- V: every layer's 2D shape for this thread's 4 outputs ----------------
    // rows of one layer are folded three at a time (VIMNMX3.U16x2); the two
    // words of a row come from one LDS.64; identical loads across layers CSE
    uint32_t layer[VR][R + 1][NW];
#pragma unroll
    for (int t = 0; t < VR; ++t) {
      const uint32_t* hb = sH + (vy + t + R) * WPR + NW * vq;  // H_k row r: hb[((k-1)*HY + r-vy-R)*WPR]
      const T* rb = stage + (vy + t + R) * WBOX + XA2 + 4 * vq;
      auto term = [&](int k, int dy, int j) -> uint32_t {
        if (k == 0) {
          if constexpr (BIN) {
            return *reinterpret_cast<const uint32_t*>(rb + dy * WBOX);
          } else if constexpr (sizeof(T) == 2) {
            return *reinterpret_cast<const uint32_t*>(rb + dy * WBOX + 2 * j);
          } else {
            const uint32_t b4 = *reinterpret_cast<const uint32_t*>(rb + dy * WBOX);
            return prmt(b4, 0u, j ? 0x4342u : 0x4140u);
          }
        }
        return hb[((k - 1) * HY + dy) * WPR + j];
      };
#pragma unroll
      for (int L = 0; L <= R; ++L) {
#pragma unroll
        for (int j = 0; j < NW; ++j) {
          uint32_t v = 0;
          int nt = 0;
          uint32_t pend = 0;
          bool has_pend = false;
#pragma unroll
          for (int dy = -R; dy <= R; ++dy) {
            const int k = S::hw(L, dy);
            if (k < 0) continue;
            const uint32_t t = term(k, dy, j);
            if (nt == 0) {
              v = t;
            } else if (!has_pend) {
              pend = t;
              has_pend = true;
            } else {
              v = mop3<MAX, BIN>(v, pend, t);
              has_pend = false;
            }
            ++nt;
          }
          if (has_pend) v = mop2<MAX, BIN>(v, pend);
          layer[t][L][j] = v;
        }
      }
    }
    // ---- Z: slice s feeds outputs o = s-2R .. s (offset dz = s - o - R, layer
    // |dz|); output o lives in acc slot o % RING and completes at s = o + 2R
    switch (s % RING) {
#define HB_M3_CASE(U)                                                                   \
  case U:                                                                               \
    if constexpr (U < RING) {                                                           \
      _Pragma("unroll") for (int d = -R; d <= R; ++d) {                                 \
        const int slot = ((U - d - R) % RING + RING) % RING; /* o = s - d - R */        \
        const int L = d < 0 ? -d : d;                                                   \
        _Pragma("unroll") for (int t = 0; t < VR; ++t) {                                \
        if (d == R) {                                                                   \
          const uint32_t v0 = mop2<MAX, BIN>(acc[slot][t][0], layer[t][L][0]);          \
          const uint32_t v1 = NW > 1 ? mop2<MAX, BIN>(acc[slot][t][NW - 1], layer[t][L][NW - 1]) : 0u; \
          if (s >= 2 * R) store_out(s - 2 * R, t, v0, v1);                              \
          _Pragma("unroll") for (int j = 0; j < NW; ++j) acc[slot][t][j] = IDENT;       \
        } else {                                                                        \
          _Pragma("unroll") for (int j = 0; j < NW; ++j)                                \
            acc[slot][t][j] = mop2<MAX, BIN>(acc[slot][t][j], layer[t][L][j]);          \
        }                                                                               \
        }                                                                               \
      }                                                                                 \
    }                                                                                   \
    break;
      HB_M3_CASE(0) HB_M3_CASE(1) HB_M3_CASE(2) HB_M3_CASE(3) HB_M3_CASE(4) HB_M3_CASE(5) HB_M3_CASE(6)
#undef HB_M3_CASE
      default: break;
    }
    __syncthreads();  // sH and this stage (raw rows read by V) are free again
    if (tid == 0 && s + M3X_NST < nsl) {
      fence_proxy_async();
      mbar_expect_tx(&bar[st], BOX_BYTES);
      tma_load_3d(stage, &tin, x0 - XA2, y0 - R, zin_of(s + M3X_NST), &bar[st]);
    }
  }
}

// Recognise the factory shapes from an offset list (exact set equality).
bool classify_se(const int32_t* off, int n, int& kind, int& r) {
  std::vector<std::array<int, 3>> v(n);
  int ext = 0;
  for (int k = 0; k < n; ++k) {
    v[k] = {off[3 * k], off[3 * k + 1], off[3 * k + 2]};
    ext = std::max({ext, std::abs(v[k][0]), std::abs(v[k][1]), std::abs(v[k][2])});
  }
  std::sort(v.begin(), v.end());
  v.erase(std::unique(v.begin(), v.end()), v.end());
  if (ext < 1 || ext > 3) return false;
  for (int kd = 0; kd < 3; ++kd) {
    std::vector<std::array<int, 3>> w;
    for (int dz = -ext; dz <= ext; ++dz)
      for (int dy = -ext; dy <= ext; ++dy)
        for (int dx = -ext; dx <= ext; ++dx) {
          bool in;
          if (kd == SE_BOX) in = true;
          else if (kd == SE_BALL) in = dz * dz + dy * dy + dx * dx <= ext * ext;
          else in = (dz == 0 && dy == 0) || (dz == 0 && dx == 0) || (dy == 0 && dx == 0);
          if (in) w.push_back({dz, dy, dx});
        }
    if (w == v) {
      kind = kd;
      r = ext;
      return true;
    }
  }
  return false;
}

template <typename T, bool MAX, int KIND, int R, bool BIN>
cudaError_t launch_morph3_v(const DevIn& in, int64_t zo, int64_t nzo, void* out, const int* gate,
                            cudaStream_t s) {
  constexpr int ALIGN = 16 / (int)sizeof(T);
  constexpr int XA = (R + ALIGN - 1) / ALIGN * ALIGN < 4 ? 4 : (R + ALIGN - 1) / ALIGN * ALIGN;
  constexpr int XA2 = (XA + ALIGN - 1) / ALIGN * ALIGN;
  constexpr int WBOX = (XA2 + M3X_TX + XA2 + ALIGN - 1) / ALIGN * ALIGN;
  constexpr int HY = M3X_TY + 2 * R;
  constexpr int STAGE_PITCH = (HY * WBOX * (int)sizeof(T) + 127) / 128 * 128;
  const int smem = M3X_NST * STAGE_PITCH + R * HY * (M3X_TX / 2) * 4 + M3X_NST * 8 + 128;  // BIN uses half the sH
  CUtensorMap tin;
  const CUtensorMapDataType dt = sizeof(T) == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_UINT16;
  if (!make_tmap_3d(&tin, in.p, dt, sizeof(T), in.nx, in.ny, in.nz, WBOX, HY)) return cudaErrorNotSupported;
  Morph3Args a;
  a.nzi = (int)in.nz;
  a.zo = (int)zo;
  a.nzo = (int)nzo;
  a.nx = (int)in.nx;
  a.ny = (int)in.ny;
  const int gx = (int)((in.nx + M3X_TX - 1) / M3X_TX), gy = (int)((in.ny + M3X_TY - 1) / M3X_TY);
  const int64_t tiles = (int64_t)gx * gy;
  const int64_t want = std::max<int64_t>(1, (4 * kNumSMs + tiles - 1) / tiles);
  a.zchunk = (int)std::max<int64_t>(std::min<int64_t>(nzo, 8 * R + 8), (nzo + want - 1) / want);
  dim3 grid(gx, gy, (unsigned)((nzo + a.zchunk - 1) / a.zchunk));
  auto kern = k_morph3<T, MAX, KIND, R, BIN>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  kern<<<grid, M3XV<BIN>::NT, smem, s>>>(tin, (T*)out, a, gate);
  return cudaGetLastError();
}

#ifndef HB_MB_MINB
#define HB_MB_MINB 2  // resident CTAs per SM the register budget is sized for
#endif
#ifndef HB_MB_PD
#define HB_MB_PD 3  // slices prefetched ahead into L2
#endif
#ifndef HB_MB_TY
#define HB_MB_TY 8  // output rows per thread (4/6/8 at 3-4 CTAs/SM: all 1030-1100 Gvox/s)
#endif
// ---------------------------------------------------------------------------
// Binary {0,1} uint8 volumes (configs[2]'s binary case), ONE BIT per voxel in
// registers: erosion is AND and dilation OR over the SE, so 32 voxels go
// through every logic op.  A thread owns one 32-voxel word column x MB_TY
// output rows and marches z:
//   * each staged row is loaded as 32 bytes (2 x LDG.128, a warp reads 1 KB
//     contiguous) and packed to a word with (v * 0x204081) >> 21 (the bytes
//     are 0/1, so the products cannot carry into the nibble);
//   * x-runs |dx| <= w: funnel shifts against the neighbouring words (lane
//     shuffles; the segment-edge lanes load theirs; row ends replicate the
//     edge voxel = the clamp), H_w = OP(H_{w-1}, x-w, x+w);
//   * every (dz, dy) row of the SE is one AND/OR of H_{hw(dz,dy)} into the
//     accumulator of its output slice: A[j] collects output (s - 2R + j) from
//     input slice s, A[0] is complete after s and leaves unpacked
//     ((nibble * 0x204081) & 0x01010101) as 2 x STG.128.
// ~3 logic/pack instructions per voxel: the kernel is bound by HBM (1 B in,
// 1 B out per voxel), not by the ALU.  Gated on the device grey check like
// the byte-wise AND/OR kernel it replaces (nx % 32 == 0).
// ---------------------------------------------------------------------------
constexpr int MB_TY = HB_MB_TY, MB_WARPS = 8, MB_PD = HB_MB_PD;

__device__ __forceinline__ uint32_t mb_pack(const uint4& a, const uint4& b) {
  const uint32_t c = 0x204081u;
  const uint32_t b0 = (((a.x * c) >> 21) & 0x0Fu) | (((a.y * c) >> 17) & 0xF0u);
  const uint32_t b1 = (((a.z * c) >> 21) & 0x0Fu) | (((a.w * c) >> 17) & 0xF0u);
  const uint32_t b2 = (((b.x * c) >> 21) & 0x0Fu) | (((b.y * c) >> 17) & 0xF0u);
  const uint32_t b3 = (((b.z * c) >> 21) & 0x0Fu) | (((b.w * c) >> 17) & 0xF0u);
  return __byte_perm(__byte_perm(b0, b1, 0x0040), __byte_perm(b2, b3, 0x0040), 0x5410);
}
__device__ __forceinline__ void mb_unpack(uint32_t w, uint4& a, uint4& b) {
  const uint32_t c = 0x204081u, m = 0x01010101u;
  a.x = ((w & 0xFu) * c) & m;
  a.y = (((w >> 4) & 0xFu) * c) & m;
  a.z = (((w >> 8) & 0xFu) * c) & m;
  a.w = (((w >> 12) & 0xFu) * c) & m;
  b.x = (((w >> 16) & 0xFu) * c) & m;
  b.y = (((w >> 20) & 0xFu) * c) & m;
  b.z = (((w >> 24) & 0xFu) * c) & m;
  b.w = ((w >> 28) * c) & m;
}
// packs 32 bytes; `grey` collects any bit a {0,1} byte cannot have
__device__ __forceinline__ uint32_t mb_word(const uint8_t* p, uint32_t& grey) {
  const uint4 a = __ldg(reinterpret_cast<const uint4*>(p));
  const uint4 b = __ldg(reinterpret_cast<const uint4*>(p) + 1);
  grey |= (a.x | a.y | a.z | a.w | b.x | b.y | b.z | b.w);
  return mb_pack(a, b);
}

template <bool MAX, int KIND, int R>
__global__ void __launch_bounds__(MB_WARPS * 32, HB_MB_MINB)
k_morph_bits(const uint8_t* __restrict__ in, int nz, int ny, int nx, int zo, int nzo, int zchunk,
             uint8_t* __restrict__ out, int* __restrict__ grey_flag) {
  using S = SeShape<KIND, R>;
  constexpr int L = MB_TY + 2 * R;            // staged rows per thread
  constexpr uint32_t ID = MAX ? 0u : ~0u;     // identity of the fold
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = nx >> 5;                     // words per row
  const int wc = blockIdx.x * 32 + lane;      // this lane's word column
  const bool active = wc < nw;
  const int wcl = min(wc, nw - 1);
  const int y0 = (blockIdx.y * MB_WARPS + warp) * MB_TY;
  const int zs = blockIdx.z * zchunk, ze = min(zs + zchunk, nzo);
  const int nsl = ze - zs + 2 * R;
  const int64_t plane = (int64_t)ny * nx;
  int64_t roff[L];
#pragma unroll
  for (int r = 0; r < L; ++r) roff[r] = (int64_t)min(max(y0 - R + r, 0), ny - 1) * nx;
  uint32_t A[2 * R + 1][MB_TY];
#pragma unroll
  for (int j = 0; j < 2 * R + 1; ++j)
#pragma unroll
    for (int t = 0; t < MB_TY; ++t) A[j][t] = ID;
  uint32_t grey = 0;
  // L2 prefetch of the rows MB_PD slices ahead: lanes 0..L-1 issue one bulk
  // prefetch per staged row of this warp's segment (the loads were latency-
  // bound: long-scoreboard stalls on the packs, 21% warps active)
  const int seg0 = blockIdx.x * 32 * 32;  // first byte of this segment in a row
  const uint32_t seg_bytes = (uint32_t)min(32 * 32, nx - seg0);
  const int prow = min(max(y0 - R + lane, 0), ny - 1);
  auto prefetch = [&](int sp) {
    if (lane < L && sp < nsl) {
      const int zp = min(max(zo + zs - R + sp, 0), nz - 1);
      const uint8_t* a = in + (int64_t)zp * plane + (int64_t)prow * nx + seg0;
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(seg_bytes) : "memory");
    }
  };
#pragma unroll
  for (int sp = 0; sp < MB_PD; ++sp) prefetch(sp);
  for (int s = 0; s < nsl; ++s) {
    prefetch(s + MB_PD);
    const int zi = min(max(zo + zs - R + s, 0), nz - 1);
    const uint8_t* sl = in + (int64_t)zi * plane + (int64_t)wcl * 32;
#pragma unroll
    for (int r = 0; r < L; ++r) {
      const uint8_t* rp = sl + roff[r];
      const uint32_t p = mb_word(rp, grey);
      uint32_t prv = __shfl_up_sync(0xffffffffu, p, 1);
      uint32_t nxt = __shfl_down_sync(0xffffffffu, p, 1);
      if (lane == 0) prv = wc == 0 ? 0u - (p & 1u) : mb_word(rp - 32, grey);
      if (wc == nw - 1) nxt = 0u - (p >> 31);
      else if (lane == 31 && wc + 1 < nw) nxt = mb_word(rp + 32, grey);  // lanes past the row end are idle
      uint32_t h[R + 1];
      h[0] = p;
#pragma unroll
      for (int w = 1; w <= R; ++w) {
        const uint32_t lo = __funnelshift_l(prv, p, w), hi = __funnelshift_r(p, nxt, w);
        h[w] = MAX ? (h[w - 1] | lo | hi) : (h[w - 1] & lo & hi);
      }
#pragma unroll
      for (int t = 0; t < MB_TY; ++t) {
        const int dy = r - R - t;
        if (dy < -R || dy > R) continue;
#pragma unroll
        for (int j = 0; j < 2 * R + 1; ++j) {
          const int w = S::hw(R - j, dy);
          if (w >= 0) A[j][t] = MAX ? (A[j][t] | h[w]) : (A[j][t] & h[w]);
        }
      }
    }
    const int o = s - 2 * R;  // output slice completed by this input slice
    if (o >= 0 && active) {
      uint8_t* op = out + (int64_t)(zs + o) * plane + (int64_t)wc * 32;
#pragma unroll
      for (int t = 0; t < MB_TY; ++t)
        if (y0 + t < ny) {
          uint4 a, b;
          mb_unpack(A[0][t], a, b);
          uint4* q = reinterpret_cast<uint4*>(op + (int64_t)(y0 + t) * nx);
          q[0] = a;
          q[1] = b;
        }
    }
#pragma unroll
    for (int j = 0; j < 2 * R; ++j)
#pragma unroll
      for (int t = 0; t < MB_TY; ++t) A[j][t] = A[j + 1][t];
#pragma unroll
    for (int t = 0; t < MB_TY; ++t) A[2 * R][t] = ID;
  }
  // a byte > 1 anywhere in what this CTA read: the block is grey, this
  // output is void and the u16-lane kernel queued behind rewrites it
  if (__syncthreads_or((grey & 0xfefefefeu) != 0u) && threadIdx.x == 0) atomicOr(grey_flag, 1);
}

// ---------------------------------------------------------------------------
// k_morph_bits2: the same one-bit-per-voxel erosion / dilation with the input
// staged by TMA (k_morph_bits above was load-latency-bound: each thread
// loaded and packed its 8 + 2R rows itself, long-scoreboard 67%).  CTA tile =
// 64 output rows x 8 words (256 voxels); per slice two TMA boxes (160 B x
// (64 + 2R) rows: the 256 columns plus one halo word each side) land in a
// 3-deep ring; every staged row word is packed ONCE into a shared bit plane
// (double-buffered), then a thread (one word x 2 output rows) builds its
// x-runs from the packed words of its 2 + 2R rows and folds the SE rows into
// per-output-slice accumulators exactly as k_morph_bits does.  Border tiles
// replicate the edge bytes (the clamp) before packing.
// ---------------------------------------------------------------------------
constexpr int MB2_TXW = 8, MB2_TYO = 64, MB2_NT = 256, MB2_NST = 3;
constexpr int MB2_BOXW = 160;  // bytes per TMA box row (half of 32 + 256 + 32)

template <int R>
struct MB2Geo {
  static constexpr int ROWS = MB2_TYO + 2 * R;
  static constexpr int BOX = MB2_BOXW * ROWS;              // bytes per box
  static constexpr int BOXP = (BOX + 127) / 128 * 128;     // TMA destinations are 128-B aligned
  static constexpr int STAGE = 2 * BOXP;
  static constexpr int PW = MB2_TXW + 2;                    // packed words per row (1 halo each side)
  static constexpr int PLANE = ROWS * PW;                   // packed words per slice
  static constexpr int OFF_P = MB2_NST * STAGE;
  static constexpr int OFF_BAR = OFF_P + 2 * PLANE * 4;
  static constexpr int SMEM = OFF_BAR + MB2_NST * 8 + 128;
};

template <bool MAX, int KIND, int R>
__global__ void __launch_bounds__(MB2_NT, 2)
k_morph_bits2(const __grid_constant__ CUtensorMap tin, uint8_t* __restrict__ out, int nz, int ny,
              int nx, int zo, int nzo, int zchunk, int* __restrict__ grey_flag) {
  using S = SeShape<KIND, R>;
  using G = MB2Geo<R>;
  constexpr uint32_t ID = MAX ? 0u : ~0u;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  uint32_t* sP = reinterpret_cast<uint32_t*>(smem + G::OFF_P);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + G::OFF_BAR);
  const int tid = threadIdx.x;
  const int x0 = blockIdx.x * (MB2_TXW * 32), y0 = blockIdx.y * MB2_TYO;
  const int zs = blockIdx.z * zchunk, ze = min(zs + zchunk, nzo);
  const int nsl = ze - zs + 2 * R;
  auto zin = [&](int k) { return min(max(zo + zs - R + k, 0), nz - 1); };
  auto load = [&](int k, int stg) {
    unsigned char* d = smem + stg * G::STAGE;
    mbar_expect_tx(&bar[stg], 2 * G::BOX);
    tma_load_3d(d, &tin, x0 - 32, y0 - R, zin(k), &bar[stg]);
    tma_load_3d(d + G::BOXP, &tin, x0 - 32 + MB2_BOXW, y0 - R, zin(k), &bar[stg]);
  };
  // a block already flagged grey by an earlier CTA: its output is void (the
  // u16-lane kernel queued behind rewrites all of it), so later CTAs leave
  // at once — decided by thread 0 before any TMA is issued, so the exit is
  // CTA-uniform and leaves no copy in flight (grey u8 2048^2 x 256: the bits
  // pass shrinks to ~its first wave)
  __shared__ int s_skip;
  if (tid == 0) {
    s_skip = *reinterpret_cast<volatile const int*>(grey_flag);
    if (!s_skip) {
#pragma unroll
      for (int i = 0; i < MB2_NST; ++i) mbar_init(&bar[i], 1);
      fence_mbar_init();
      prefetch_tmap(&tin);
      for (int i = 0; i < MB2_NST && i < nsl; ++i) load(i, i);
    }
  }
  __syncthreads();
  if (s_skip) return;
  const bool border = x0 - 32 < 0 || x0 + MB2_TXW * 32 + 32 > nx || y0 - R < 0 || y0 + MB2_TYO + R > ny;
  // this thread: word w of the tile, output rows y0 + 2g, y0 + 2g + 1
  const int w = tid % MB2_TXW, g = tid / MB2_TXW;
  const int gw = (x0 >> 5) + w;  // global word column
  const bool active = gw < (nx >> 5);
  const int64_t plane = (int64_t)ny * nx;
  uint32_t A[2 * R + 1][2];
#pragma unroll
  for (int j = 0; j < 2 * R + 1; ++j) A[j][0] = A[j][1] = ID;
  uint32_t grey = 0;
  int st = 0;
  uint32_t ph = 0;
  for (int s = 0; s < nsl; ++s) {
    unsigned char* stage = smem + st * G::STAGE;
    mbar_wait(&bar[st], ph);
    // pack every staged row word once (buffer s & 1)
    uint32_t* P = sP + (s & 1) * G::PLANE;
    for (int e = tid; e < G::PLANE; e += MB2_NT) {
      const int r = e / G::PW, c = e - r * G::PW;  // c: word 0..9 of the staged row
      const unsigned char* src = stage + (c < 5 ? 0 : G::BOXP) + r * MB2_BOXW + (c % 5) * 32;
      const uint4 a = *reinterpret_cast<const uint4*>(src);
      const uint4 b = *reinterpret_cast<const uint4*>(src + 16);
      grey |= (a.x | a.y | a.z | a.w | b.x | b.y | b.z | b.w);
      P[e] = mb_pack(a, b);
    }
    __syncthreads();  // P complete; stage st fully read
    if (border) {
      // clamp-to-edge in the bit domain (TMA zero-filled the out-of-volume
      // bytes): halo words beyond a row end take the edge voxel's bit, then
      // rows beyond the volume copy the nearest valid row
      const int r_lo = max(0, -(y0 - R)), r_hi = min(G::ROWS, ny - (y0 - R));
      const int w_lo = max(0, -((x0 >> 5) - 1)), w_hi = min(G::PW, (nx >> 5) - ((x0 >> 5) - 1));
      if (tid < G::ROWS && tid >= r_lo && tid < r_hi) {
        uint32_t* row = P + tid * G::PW;
        const uint32_t left = 0u - (row[w_lo] & 1u), right = 0u - (row[w_hi - 1] >> 31);
        for (int c = 0; c < w_lo; ++c) row[c] = left;
        for (int c = w_hi; c < G::PW; ++c) row[c] = right;
      }
      __syncthreads();
      for (int e = tid; e < G::PLANE; e += MB2_NT) {
        const int r = e / G::PW, c = e - r * G::PW;
        if (r < r_lo || r >= r_hi) P[e] = P[min(max(r, r_lo), r_hi - 1) * G::PW + c];
      }
      __syncthreads();
    }
    if (tid == 0 && s + MB2_NST < nsl) {
      fence_proxy_async();
      load(s + MB2_NST, st);
    }
    if (++st == MB2_NST) { st = 0; ph ^= 1u; }
    // x-runs of the 2 + 2R rows this thread needs, folded per SE row
#pragma unroll
    for (int r = 0; r < 2 + 2 * R; ++r) {
      const uint32_t* row = P + (2 * g + r) * G::PW + w;  // words w-1, w, w+1 at +0, +1, +2
      const uint32_t prv = row[0], p = row[1], nxt = row[2];
      uint32_t h[R + 1];
      h[0] = p;
#pragma unroll
      for (int k = 1; k <= R; ++k) {
        const uint32_t lo = __funnelshift_l(prv, p, k), hi = __funnelshift_r(p, nxt, k);
        h[k] = MAX ? (h[k - 1] | lo | hi) : (h[k - 1] & lo & hi);
      }
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const int dy = r - R - t;
        if (dy < -R || dy > R) continue;
#pragma unroll
        for (int j = 0; j < 2 * R + 1; ++j) {
          const int hw = S::hw(R - j, dy);
          if (hw >= 0) A[j][t] = MAX ? (A[j][t] | h[hw]) : (A[j][t] & h[hw]);
        }
      }
    }
    const int o = s - 2 * R;
    if (o >= 0 && active) {
      uint8_t* op = out + (int64_t)(zs + o) * plane + (int64_t)gw * 32;
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const int y = y0 + 2 * g + t;
        if (y < ny) {
          uint4 a, b;
          mb_unpack(A[0][t], a, b);
          uint4* q = reinterpret_cast<uint4*>(op + (int64_t)y * nx);
          q[0] = a;
          q[1] = b;
        }
      }
    }
#pragma unroll
    for (int j = 0; j < 2 * R; ++j) A[j][0] = A[j + 1][0], A[j][1] = A[j + 1][1];
    A[2 * R][0] = A[2 * R][1] = ID;
  }
  if (__syncthreads_or((grey & 0xfefefefeu) != 0u) && tid == 0) atomicOr(grey_flag, 1);
}

template <bool MAX, int KIND, int R>
cudaError_t launch_morph_bits2(const DevIn& in, int64_t zo, int64_t nzo, void* out, int* gate,
                               cudaStream_t s) {
  using G = MB2Geo<R>;
  if (in.nx % 32 != 0 || (reinterpret_cast<uintptr_t>(in.p) & 15) != 0 ||
      (reinterpret_cast<uintptr_t>(out) & 15) != 0 || in.nz >= (1 << 30) || in.ny >= (1 << 30) ||
      in.nx >= (1 << 30) || std::getenv("HB_MORPH_BITS1"))
    return cudaErrorNotSupported;
  CUtensorMap tin;
  if (!make_tmap_3d(&tin, in.p, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, in.nx, in.ny, in.nz, MB2_BOXW, G::ROWS))
    return cudaErrorNotSupported;
  auto kern = k_morph_bits2<MAX, KIND, R>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM) != cudaSuccess)
    return cudaErrorNotSupported;
  dim3 grid((unsigned)((in.nx + MB2_TXW * 32 - 1) / (MB2_TXW * 32)),
            (unsigned)((in.ny + MB2_TYO - 1) / MB2_TYO), 1);
  const int64_t tiles = (int64_t)grid.x * grid.y, slots = 2 * (int64_t)kNumSMs;
  // z-chunks capped (HB_MB2_ZCAP, default 48 slices; 32-48: 2645, 64-128: 2340 Gvox/s) so neighbouring tiles,
  // which re-read each other's halo rows and words, stay close in z and hit
  // in L2 (uncapped runs drifted apart: 1.41x DRAM reads)
  const char* zv = std::getenv("HB_MB2_ZCAP");
  const int64_t zcap = zv ? std::max(16, std::atoi(zv)) : 48;
  int zchunk = (int)std::min<int64_t>(nzo, 16);
  double best = 1e300;
  for (int64_t zc = 16; zc <= std::max<int64_t>(16, std::min<int64_t>(nzo, zcap)); zc += 8) {
    const int64_t ctas = tiles * ((nzo + zc - 1) / zc);
    const double cost = (double)((ctas + slots - 1) / slots) * (double)(zc + 2 * R);
    if (cost < best * 0.995) {
      best = cost;
      zchunk = (int)zc;
    }
  }
  grid.z = (unsigned)((nzo + zchunk - 1) / zchunk);
  kern<<<grid, MB2_NT, G::SMEM, s>>>(tin, (uint8_t*)out, (int)in.nz, (int)in.ny, (int)in.nx, (int)zo,
                                      (int)nzo, zchunk, gate);
  return cudaGetLastError();
}

template <bool MAX, int KIND, int R>
cudaError_t launch_morph_bits(const DevIn& in, int64_t zo, int64_t nzo, void* out, int* gate,
                              cudaStream_t s) {
  if (in.nx % 32 != 0 || (reinterpret_cast<uintptr_t>(in.p) & 15) != 0 ||
      (reinterpret_cast<uintptr_t>(out) & 15) != 0 || in.nz >= (1 << 30) || in.ny >= (1 << 30) ||
      in.nx >= (1 << 30) || std::getenv("HB_MORPH_NOBITS"))
    return cudaErrorNotSupported;
  const int nw = (int)(in.nx / 32);
  dim3 grid((unsigned)((nw + 31) / 32), (unsigned)((in.ny + MB_WARPS * MB_TY - 1) / (MB_WARPS * MB_TY)), 1);
  const int64_t tiles = (int64_t)grid.x * grid.y, slots = 2 * (int64_t)kNumSMs;
  int zchunk = (int)std::min<int64_t>(nzo, 32);
  double best = 1e300;
  for (int64_t zc = std::max<int64_t>(32, nzo / 128); zc <= std::max<int64_t>(32, nzo); zc += 16) {
    const int64_t ctas = tiles * ((nzo + zc - 1) / zc);
    const double cost = (double)((ctas + slots - 1) / slots) * (double)(zc + 2 * R);
    if (cost < best * 0.995) {
      best = cost;
      zchunk = (int)zc;
    }
  }
  grid.z = (unsigned)((nzo + zchunk - 1) / zchunk);
  k_morph_bits<MAX, KIND, R><<<grid, MB_WARPS * 32, 0, s>>>(
      (const uint8_t*)in.p, (int)in.nz, (int)in.ny, (int)in.nx, (int)zo, (int)nzo, zchunk, (uint8_t*)out, gate);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// k_morph_u16s: grey u16 erosion / dilation (configs[2]'s u16 volumes) with
// k_morph_bits2's register-streaming structure on u16x2 words instead of bits
// (k_morph3 above stages every x-run in shared memory and re-reads it per
// layer: LSU/barrier-bound at ~0.37 of HBM).  CTA tile = 128 columns x 32
// rows, 8 warps; a thread owns 2 words (4 voxels) x 4 output rows and marches
// z.  Per input slice (TMA box 144 x 38 u16, x0-8 .. x0+135, into a 4-deep
// mbarrier ring):
//   * each of its 4 + 2R rows is read as 3 LDS.64 (words w-2 .. w+3), the
//     odd-start pairs come from 5 PRMTs shared by both words, and the x-runs
//     h_k = op(h_{k-1}, x-k, x+k) are one VIMNMX3.U16x2 each;
//   * rows are taken two at a time; the dz = 0 rows of the SE are folded
//     straight into their accumulator (two SE rows per VIMNMX3, the
//     accumulator is the third operand), the rows of each layer |dz| = L > 0
//     are reduced to the 2D layer once and that is folded into both the +L
//     and the -L accumulator (ball:3: 14 instead of 18 VIMNMX per output
//     word; HB_MU_DIRECT=1 builds the all-direct form);
//   * accumulators live in a (2R+1)-slot register ring indexed by the slice
//     number mod 2R+1 (the slice loop is unrolled 2R+1 times, so completing
//     an output is a store + reset, never a register shift).
// Border tiles clamp the staged box (clamp_tile) before reading it.  Grey
// u8 volumes run the same kernel on a 160-byte box, each staged byte pair
// widened into u16 lanes by one PRMT (queued behind k_morph_bits2, which
// flags the grey blocks; HB_MORPH_U8_SMEM=1 keeps k_morph3 for them).
// ---------------------------------------------------------------------------
#ifndef HB_MU_DIRECT
#define HB_MU_DIRECT 0  // 1: every SE row folded straight into its accumulators (no shared +/-dz layers)
#endif
constexpr int MU_TX = 128, MU_RO = 4, MU_WARPS = 8, MU_TY = MU_RO * MU_WARPS, MU_NST = 4;
// the box starts 16 B left of the tile: 8 u16 / 16 u8 voxels; staged rows
// are 144 u16 (288 B) / 160 u8 (160 B)
template <typename T> struct MUT {
  static constexpr int XA = 16 / (int)sizeof(T);
  static constexpr int WBOX = MU_TX + 2 * XA;
  static constexpr int PB = WBOX * (int)sizeof(T);  // bytes per staged row
};
#ifndef HB_MU_MINB
#define HB_MU_MINB 2
#endif

template <typename T, int R>
struct MUGeo {
  static constexpr int HY = MU_TY + 2 * R;
  static constexpr int BOX = MUT<T>::PB * HY;            // bytes
  static constexpr int PITCH = (BOX + 127) / 128 * 128;
  static constexpr int SMEM = MU_NST * PITCH + MU_NST * 8 + 128;
};

template <int V>
struct IC {
  static constexpr int value = V;
};

template <typename T, bool MAX, int KIND, int R>
__global__ void __launch_bounds__(MU_WARPS * 32, HB_MU_MINB)
k_morph_u16s(const __grid_constant__ CUtensorMap tin, T* __restrict__ out, const Morph3Args a,
             const int* __restrict__ gate) {
  // u8: queued behind k_morph_bits2, which flags grey blocks; a binary block
  // is already done
  if (gate != nullptr && *gate == 0) return;
  using S = SeShape<KIND, R>;
  using G = MUGeo<T, R>;
  constexpr int MU_XA = MUT<T>::XA, MU_WBOX = MUT<T>::WBOX, PB = MUT<T>::PB;
  constexpr int RING = 2 * R + 1, NROW = MU_RO + 2 * R;
  constexpr uint32_t ID = MAX ? 0u : 0xffffffffu;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + MU_NST * G::PITCH);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int x0 = blockIdx.x * MU_TX, y0 = blockIdx.y * MU_TY;
  const int z0 = blockIdx.z * a.zchunk, z1 = min(z0 + a.zchunk, a.nzo);
  const int nsl = (z1 - z0) + 2 * R;
  auto zin = [&](int k) { return min(max(a.zo + z0 - R + k, 0), a.nzi - 1); };
  if (tid == 0) {
#pragma unroll
    for (int i = 0; i < MU_NST; ++i) mbar_init(&bar[i], 1);
    fence_mbar_init();
    prefetch_tmap(&tin);
    for (int i = 0; i < MU_NST && i < nsl; ++i) {
      mbar_expect_tx(&bar[i], G::BOX);
      tma_load_3d(smem + i * G::PITCH, &tin, x0 - MU_XA, y0 - R, zin(i), &bar[i]);
    }
  }
  __syncthreads();
  const bool border = x0 - MU_XA < 0 || x0 + MU_TX + MU_XA > a.nx || y0 - R < 0 || y0 + MU_TY + R > a.ny;
  // this thread: voxels x0 + 4*lane .. +3 (words W[2], W[3]) of rows y0 + 4*warp .. +3
  const int gx = x0 + 4 * lane, gy = y0 + MU_RO * warp;
  // staged row r (0 .. NROW-1) of this thread = box row MU_RO*warp + r; words
  // w-2 .. w+3 start at box column 4*lane + MU_XA - 4 (8-B aligned)
  const int roff = (MU_RO * warp) * PB + (4 * lane + MU_XA - 4) * (int)sizeof(T);
  const int64_t plane = (int64_t)a.ny * a.nx;
  const bool st_full = gx + 3 < a.nx;
  const bool st_part = gx < a.nx && !st_full;
  T* obase = out + (int64_t)z0 * plane + (int64_t)min(gy, a.ny - 1) * a.nx + min(gx, a.nx - 1);
  uint32_t A[RING][MU_RO][2];
#pragma unroll
  for (int u = 0; u < RING; ++u)
#pragma unroll
    for (int t = 0; t < MU_RO; ++t) A[u][t][0] = A[u][t][1] = ID;

  int st = 0;
  uint32_t ph = 0;
  // x-runs h[k][j] (k = 0..R) of staged row r for words j = 0, 1
  auto runs = [&](const unsigned char* stage, int r, uint32_t (&h)[R + 1][2]) {
    uint32_t W[6];  // u16x2 pairs 2w-2 .. 2w+3
    if constexpr (sizeof(T) == 2) {
      const uint2* p = reinterpret_cast<const uint2*>(stage + roff + r * PB);
      const uint2 q0 = p[0], q1 = p[1], q2 = p[2];
      W[0] = q0.x, W[1] = q0.y, W[2] = q1.x, W[3] = q1.y, W[4] = q2.x, W[5] = q2.y;
    } else {
      // u8: three aligned words (voxels x-4 .. x+7), each byte pair widened
      // into u16 lanes with one PRMT
      const uint32_t* p = reinterpret_cast<const uint32_t*>(stage + roff + r * PB);
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const uint32_t b4 = p[i];
        W[2 * i] = prmt(b4, 0u, 0x4140u);
        W[2 * i + 1] = prmt(b4, 0u, 0x4342u);
      }
    }
    uint32_t P[5];  // P[i] = (hi of W[i], lo of W[i+1]): odd-start pairs
    // (IMAD.HI + IMAD on the idle FMA pipe instead of the PRMT measured 784
    // vs 831 Gvox/s: the IMAD.HI rate)
#pragma unroll
    for (int i = 0; i < 5; ++i) P[i] = prmt(W[i], W[i + 1], 0x5432);
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      h[0][j] = W[2 + j];
      if constexpr (R >= 1) h[1][j] = op3x2<MAX>(W[2 + j], P[1 + j], P[2 + j]);
      if constexpr (R >= 2) h[2][j] = op3x2<MAX>(h[1][j], W[1 + j], W[3 + j]);
      if constexpr (R >= 3) h[3][j] = op3x2<MAX>(h[2][j], P[j], P[3 + j]);
    }
  };
  auto step = [&](auto Uc, int s) {
    constexpr int U = decltype(Uc)::value;  // s % RING
    unsigned char* stage = smem + st * G::PITCH;
    mbar_wait(&bar[st], ph);
    if (border) {
      clamp_tile<T, MU_WARPS * 32>(reinterpret_cast<T*>(stage), MU_WBOX, G::HY, MU_WBOX,
                                          y0 - R, x0 - MU_XA, a.ny, a.nx, tid);
      __syncthreads();
    }
    uint32_t LP[MU_RO][R + 1][2];  // 2D layers |dz| = L in construction
#pragma unroll
    for (int r = 0; r < NROW; r += 2) {
      uint32_t hA[R + 1][2], hB[R + 1][2];
      runs(stage, r, hA);
      const bool two = r + 1 < NROW;
      if (two) runs(stage, r + 1, hB);
#pragma unroll
      for (int t = 0; t < MU_RO; ++t) {
        const int dyA = r - R - t, dyB = dyA + 1;
#pragma unroll
        for (int L = 0; L <= R; ++L) {
          const int kA = (dyA >= -R && dyA <= R) ? S::hw(L, dyA) : -1;
          const int kB = (two && dyB >= -R && dyB <= R) ? S::hw(L, dyB) : -1;
          if (kA < 0 && kB < 0) continue;
          // input slice s feeds output o = s - 2R + j at dz = R - j; its ring
          // slot is o mod RING = (U + 1 + j) mod RING.  Layer |dz| = L.
          const int sp = (U + 1 + R - L) % RING, sm = (U + 1 + R + L) % RING;
          if (HB_MU_DIRECT || L == 0 || S::nterms(L) == 1) {
            // straight into the accumulator(s): the accumulator is the third
            // operand of every VIMNMX3
#pragma unroll
            for (int g = 0; g < (L == 0 ? 1 : 2); ++g) {
              const int slot = g == 0 ? sp : sm;
#pragma unroll
              for (int w = 0; w < 2; ++w) {
                if (kA >= 0 && kB >= 0) A[slot][t][w] = op3x2<MAX>(A[slot][t][w], hA[kA][w], hB[kB][w]);
                else if (kA >= 0) A[slot][t][w] = op2x2<MAX>(A[slot][t][w], hA[kA][w]);
                else A[slot][t][w] = op2x2<MAX>(A[slot][t][w], hB[kB][w]);
              }
            }
          } else {
            // dz = +L and -L take the same 2D layer: build it once (rows
            // t+R+dymin .. t+R+dymax), then fold it into both accumulators
            const int rf = t + R - S::dyext(L), rl = t + R + S::dyext(L);
#pragma unroll
            for (int w = 0; w < 2; ++w) {
              uint32_t& lp = LP[t][L][w];
              if (rf >= r) {  // the layer starts in this row pair
                if (kA >= 0 && kB >= 0) lp = op2x2<MAX>(hA[kA][w], hB[kB][w]);
                else lp = kA >= 0 ? hA[kA][w] : hB[kB][w];
              } else {
                if (kA >= 0 && kB >= 0) lp = op3x2<MAX>(lp, hA[kA][w], hB[kB][w]);
                else lp = op2x2<MAX>(lp, kA >= 0 ? hA[kA][w] : hB[kB][w]);
              }
              if (rl <= r + 1) {  // complete
                A[sp][t][w] = op2x2<MAX>(A[sp][t][w], lp);
                A[sm][t][w] = op2x2<MAX>(A[sm][t][w], lp);
              }
            }
          }
        }
      }
    }
    __syncthreads();  // every thread has read stage st
    if (tid == 0 && s + MU_NST < nsl) {
      fence_proxy_async();
      mbar_expect_tx(&bar[st], G::BOX);
      tma_load_3d(stage, &tin, x0 - MU_XA, y0 - R, zin(s + MU_NST), &bar[st]);
    }
    if (++st == MU_NST) { st = 0; ph ^= 1u; }
    // output o = s - 2R is complete (slot (U + 1) mod RING)
    constexpr int cs = (U + 1) % RING;
    if (s >= 2 * R) {
      T* op = obase + (int64_t)(s - 2 * R) * plane;
#pragma unroll
      for (int t = 0; t < MU_RO; ++t) {
        if (gy + t < a.ny) {
          T* d = op + (int64_t)t * a.nx;
          if (st_full) {
            if constexpr (sizeof(T) == 2) *reinterpret_cast<uint2*>(d) = make_uint2(A[cs][t][0], A[cs][t][1]);
            else *reinterpret_cast<uint32_t*>(d) = prmt(A[cs][t][0], A[cs][t][1], 0x6420);
          } else if (st_part) {
            for (int i = 0; i < 4 && gx + i < a.nx; ++i)
              d[i] = (T)((A[cs][t][i >> 1] >> (16 * (i & 1))) & 0xffffu);
          }
        }
      }
    }
#pragma unroll
    for (int t = 0; t < MU_RO; ++t) A[cs][t][0] = A[cs][t][1] = ID;
  };
  for (int s = 0; s < nsl; s += RING) {
    step(IC<0>{}, s);
    if constexpr (RING > 1) { if (s + 1 >= nsl) break; step(IC<1 % RING>{}, s + 1); }
    if constexpr (RING > 2) { if (s + 2 >= nsl) break; step(IC<2 % RING>{}, s + 2); }
    if constexpr (RING > 3) { if (s + 3 >= nsl) break; step(IC<3 % RING>{}, s + 3); }
    if constexpr (RING > 4) { if (s + 4 >= nsl) break; step(IC<4 % RING>{}, s + 4); }
    if constexpr (RING > 5) { if (s + 5 >= nsl) break; step(IC<5 % RING>{}, s + 5); }
    if constexpr (RING > 6) { if (s + 6 >= nsl) break; step(IC<6 % RING>{}, s + 6); }
  }
}

// NotSupported outside the envelope (k_morph3 takes those): TMA layout (16-B
// aligned base, nx * sizeof(T) % 16 == 0), extents < 2^30.
// HB_MORPH_U16_SMEM=1 / HB_MORPH_U8_SMEM=1 keep k_morph3 (A/B).
template <typename T, bool MAX, int KIND, int R>
cudaError_t launch_morph_u16s(const DevIn& in, int64_t zo, int64_t nzo, void* out, cudaStream_t s,
                              const int* gate = nullptr) {
  using G = MUGeo<T, R>;
  constexpr int dt = sizeof(T) == 2 ? HB_U16 : HB_U8;
  if (in.dt != dt || (in.nx % (16 / (int)sizeof(T))) != 0 || (reinterpret_cast<uintptr_t>(in.p) & 15) != 0 ||
      in.nz >= (1 << 30) || in.ny >= (1 << 30) || in.nx >= (1 << 30) ||
      std::getenv(sizeof(T) == 2 ? "HB_MORPH_U16_SMEM" : "HB_MORPH_U8_SMEM"))
    return cudaErrorNotSupported;
  CUtensorMap tin;
  if (!make_tmap_3d(&tin, in.p, sizeof(T) == 2 ? CU_TENSOR_MAP_DATA_TYPE_UINT16 : CU_TENSOR_MAP_DATA_TYPE_UINT8,
                    (int)sizeof(T), in.nx, in.ny, in.nz, MUT<T>::WBOX, G::HY))
    return cudaErrorNotSupported;
  auto kern = k_morph_u16s<T, MAX, KIND, R>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM) != cudaSuccess)
    return cudaErrorNotSupported;
  Morph3Args a;
  a.nzi = (int)in.nz;
  a.zo = (int)zo;
  a.nzo = (int)nzo;
  a.nx = (int)in.nx;
  a.ny = (int)in.ny;
  dim3 grid((unsigned)((in.nx + MU_TX - 1) / MU_TX), (unsigned)((in.ny + MU_TY - 1) / MU_TY), 1);
  const int64_t tiles = (int64_t)grid.x * grid.y, slots = (int64_t)HB_MU_MINB * kNumSMs;
  // z-chunks: wave-quantised cost, capped (HB_MU_ZCAP, default 128; 2048^2
  // x 256 ball:3: 16 691, 32 781, 64 832, 128 836, 256 839 Gvox/s)
  const char* zv = std::getenv("HB_MU_ZCAP");
  const int64_t zcap = zv ? std::max(8, std::atoi(zv)) : 128;
  int zchunk = (int)std::min<int64_t>(nzo, 16);
  double best = 1e300;
  for (int64_t zc = 16; zc <= std::max<int64_t>(16, std::min<int64_t>(nzo, zcap)); zc += 8) {
    const int64_t ctas = tiles * ((nzo + zc - 1) / zc);
    const double cost = (double)((ctas + slots - 1) / slots) * (double)(zc + 2 * R);
    if (cost < best * 0.995) {
      best = cost;
      zchunk = (int)zc;
    }
  }
  a.zchunk = (int)std::min<int64_t>(zchunk, std::max<int64_t>(1, nzo));
  grid.z = (unsigned)((nzo + a.zchunk - 1) / a.zchunk);
  kern<<<grid, MU_WARPS * 32, G::SMEM, s>>>(tin, (T*)out, a, gate);
  return cudaGetLastError();
}

__global__ void k_u8_grey_check(const uint8_t* __restrict__ p, int64_t n, int* __restrict__ grey) {
  const int64_t n16 = n / 16;
  bool any = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x) {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(p) + i);
    any |= ((v.x | v.y | v.z | v.w) & 0xfefefefeu) != 0u;
  }
  for (int64_t i = n16 * 16 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    any |= p[i] > 1;
  if (__syncthreads_or(any) && threadIdx.x == 0) *grey = 1;
}

// u16: the grey kernel.  u8: a device check of the block (any byte > 1?)
// gates the binary (AND/OR, 4 voxels per op) and the grey kernel; both are
// enqueued and the unselected one exits at once — no host round trip.
template <typename T, bool MAX, int KIND, int R>
cudaError_t launch_morph3(const DevIn& in, int64_t zo, int64_t nzo, void* out, cudaStream_t s,
                          int* gate_scratch) {
  if constexpr (sizeof(T) == 2) {
    const cudaError_t e = launch_morph_u16s<uint16_t, MAX, KIND, R>(in, zo, nzo, out, s);
    if (e != cudaErrorNotSupported) return e;
    cudaGetLastError();
    return launch_morph3_v<T, MAX, KIND, R, false>(in, zo, nzo, out, nullptr, s);
  } else {
    if ((reinterpret_cast<uintptr_t>(in.p) & 15) != 0 || std::getenv("HB_MORPH_NOBIN"))
      return launch_morph3_v<T, MAX, KIND, R, false>(in, zo, nzo, out, nullptr, s);
    int* gate = gate_scratch;
    cudaError_t e = cudaSuccess;
    if (!gate) {
      e = cudaMallocAsync(&gate, sizeof(int), s);
      if (e != cudaSuccess) return e;
    }
    cudaMemsetAsync(gate, 0, sizeof(int), s);
    auto release = [&]() {
      if (!gate_scratch) cudaFreeAsync(gate, s);
    };
    // whole-word rows: the one-bit-per-voxel kernel runs first and flags a
    // grey block itself (no separate read pass); the u16-lane kernel behind
    // it exits unless flagged
    e = launch_morph_bits2<MAX, KIND, R>(in, zo, nzo, out, gate, s);
    if (e == cudaErrorNotSupported) {
      cudaGetLastError();
      e = launch_morph_bits<MAX, KIND, R>(in, zo, nzo, out, gate, s);
    }
    if (e == cudaSuccess) {
      // grey blocks (flagged by the bits kernel): the u16-lane streaming
      // kernel, else k_morph3
      e = launch_morph_u16s<uint8_t, MAX, KIND, R>(in, zo, nzo, out, s, gate);
      if (e == cudaErrorNotSupported) {
        cudaGetLastError();
        e = launch_morph3_v<T, MAX, KIND, R, false>(in, zo, nzo, out, gate, s);
      }
      release();
      return e;
    }
    cudaGetLastError();
    // else: device grey check gating the byte-wise AND/OR and the grey kernel
    k_u8_grey_check<<<kNumSMs * 4, 256, 0, s>>>((const uint8_t*)in.p, in.nz * in.ny * in.nx, gate);
    e = launch_morph3_v<T, MAX, KIND, R, true>(in, zo, nzo, out, gate, s);
    if (e == cudaSuccess) e = launch_morph3_v<T, MAX, KIND, R, false>(in, zo, nzo, out, gate, s);
    release();
    return e;
  }
}

template <typename T, bool MAX>
cudaError_t dispatch_morph3(int kind, int r, const DevIn& in, int64_t zo, int64_t nzo, void* out,
                            cudaStream_t s, int* gate = nullptr) {
#define HB_M3_K(K)                                                              \
  if (kind == K) {                                                              \
    if (r == 1) return launch_morph3<T, MAX, K, 1>(in, zo, nzo, out, s, gate);  \
    if (r == 2) return launch_morph3<T, MAX, K, 2>(in, zo, nzo, out, s, gate);  \
    if (r == 3) return launch_morph3<T, MAX, K, 3>(in, zo, nzo, out, s, gate);  \
  }
  HB_M3_K(SE_BALL) HB_M3_K(SE_BOX) HB_M3_K(SE_CROSS)
#undef HB_M3_K
  return cudaErrorNotSupported;
}

}  // namespace

cudaError_t morph(const DevIn& in, int64_t zo, int64_t nzo, void* out, const int32_t* offsets,
                  int n, bool is_max, cudaStream_t s, int64_t* launches, int* gate) {
  if (nzo <= 0) return cudaSuccess;
  if ((in.dt == HB_U16 || in.dt == HB_U8) && in.nx >= 8 && in.ny >= 8) {
    int kind = 0, rr = 0;
    if (classify_se(offsets, n, kind, rr)) {
      cudaError_t e;
      if (in.dt == HB_U16)
        e = is_max ? dispatch_morph3<uint16_t, true>(kind, rr, in, zo, nzo, out, s)
                   : dispatch_morph3<uint16_t, false>(kind, rr, in, zo, nzo, out, s);
      else
        e = is_max ? dispatch_morph3<uint8_t, true>(kind, rr, in, zo, nzo, out, s, gate)
                   : dispatch_morph3<uint8_t, false>(kind, rr, in, zo, nzo, out, s, gate);
      if (e != cudaErrorNotSupported) {
        if (e == cudaSuccess && launches) *launches += 1;
        return e;
      }
      cudaGetLastError();
    }
    Morph2Args a2;
    if (build_morph2(offsets, n, a2)) {
      cudaError_t e;
      if (in.dt == HB_U16)
        e = is_max ? dispatch_morph2<uint16_t, true>(in, zo, nzo, out, a2, s)
                   : dispatch_morph2<uint16_t, false>(in, zo, nzo, out, a2, s);
      else
        e = is_max ? dispatch_morph2<uint8_t, true>(in, zo, nzo, out, a2, s)
                   : dispatch_morph2<uint8_t, false>(in, zo, nzo, out, a2, s);
      if (e != cudaErrorNotSupported) {
        if (e == cudaSuccess && launches) *launches += 1;
        return e;
      }
      cudaGetLastError();
    }
  }
  SeRows se;
  if (!build_rows(offsets, n, se)) return cudaErrorNotSupported;
  switch (in.dt) {
    case HB_U8: return run_morph<uint8_t>(in, zo, nzo, out, se, is_max, s, launches);
    case HB_U16: return run_morph<uint16_t>(in, zo, nzo, out, se, is_max, s, launches);
    case HB_U32: return run_morph<uint32_t>(in, zo, nzo, out, se, is_max, s, launches);
    case HB_F32: return run_morph<float>(in, zo, nzo, out, se, is_max, s, launches);
  }
  return cudaErrorInvalidValue;
}

}  // namespace hb
