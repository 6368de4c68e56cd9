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
#include <algorithm>
#include <map>

#include "ops.cuh"

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

}  // namespace

cudaError_t morph(const DevIn& in, int64_t zo, int64_t nzo, void* out, const int32_t* offsets,
                  int n, bool is_max, cudaStream_t s, int64_t* launches) {
  if (nzo <= 0) return cudaSuccess;
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
