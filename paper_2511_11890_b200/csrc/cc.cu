// cc.cu — connected-components labelling (quantify.py:60-111) on the device.
//
// The reference labels a binary mask (ndimage.label, 6- or 26-connectivity)
// and compacts the ids to 1..count in first-voxel scan order (quantify.py:
// 48-57), so its output is canonical: any correct partition into components,
// numbered by first occurrence, reproduces it exactly.  Here:
//   init     : every foreground voxel is its own root (label = linear index)
//   union    : each foreground voxel unions with its already-scanned
//              neighbours (smaller linear index) through a lock-free
//              union-find whose links always point to the smaller root
//              (atomicMin), so a component's final root is its smallest index
//              = its first voxel in scan order
//   flatten  : root of every voxel (path halving) into the output buffer
//   compact  : roots flagged, exclusive prefix sum (CUB) -> 1..count in root
//              order = first-occurrence order; every voxel takes its root's id
// Volumes up to 2^31 - 1 voxels (int32 labels), resident in HBM.
#include <cuda_runtime.h>

#include <algorithm>

#include <cub/device/device_scan.cuh>

#include "ops.cuh"

namespace hb {
namespace {

constexpr int kCT = 256;

inline int cgrid(int64_t n) {
  const int64_t b = (n + kCT - 1) / kCT, cap = (int64_t)kNumSMs * 16;
  return (int)(b < 1 ? 1 : (b < cap ? b : cap));
}

// modes: CC_NONZERO (components of nonzero voxels), CC_ZERO (components of
// the zero voxels: fill_holes' background), CC_SAME (nonzero voxels connect
// only to equal values: remove_islands' per-label components)
enum { CC_NONZERO = 0, CC_ZERO = 1, CC_SAME = 2 };

template <typename T, int MODE>
__device__ __forceinline__ bool cc_fg(T v) {
  return MODE == CC_ZERO ? v == T(0) : v != T(0);
}

// init with the x-runs already linked: a warp covers 32 consecutive voxels;
// a voxel joined to its left neighbour (same row, both foreground, equal
// values for CC_SAME) points to its run's first voxel inside the warp, or to
// the voxel left of the warp when the run enters from the previous warp.
// Links point to smaller indices and run starts are roots, so the union-find
// invariants hold and no x-direction union is left to do.
template <typename T, int MODE>
__global__ void __launch_bounds__(kCT) k_cc_init(const T* __restrict__ in, int nx, int n, int* __restrict__ lab) {
  const int lane = threadIdx.x & 31;
  const int warps = gridDim.x * (kCT / 32);
  for (int base = (blockIdx.x * (kCT / 32) + (threadIdx.x >> 5)) * 32; base < n; base += warps * 32) {
    const int i = base + lane;
    bool fg = false, join = false;
    if (i < n) {
      const T v = in[i];
      fg = cc_fg<T, MODE>(v);
      if (fg && i % nx != 0) {
        const T u = in[i - 1];
        join = cc_fg<T, MODE>(u) && (MODE != CC_SAME || u == v);
      }
    }
    const unsigned starts = __ballot_sync(0xffffffffu, !join);
    const unsigned upto = starts & (0xffffffffu >> (31 - lane));  // lanes <= this one
    if (i < n) {
      if (!fg) lab[i] = -1;
      else if (!join) lab[i] = i;
      else lab[i] = upto ? base + (31 - __clz(upto)) : base - 1;
    }
  }
}

// find with path halving: a link is only ever rewritten while its node is a
// non-root, and always to an ancestor, so racing (even stale) halving stores
// keep the partition and never touch a root — the smallest index of every
// component stays its root
__device__ __forceinline__ int cc_find(int* lab, int x) {
  int p = lab[x];
  while (p != x) {
    const int gp = lab[p];
    if (gp != p) lab[x] = gp;
    x = p;
    p = gp;
  }
  return x;
}

// link the larger root under the smaller one; retry when another thread moved it
__device__ __forceinline__ void cc_union(int* lab, int a, int b) {
  while (true) {
    a = cc_find(lab, a);
    b = cc_find(lab, b);
    if (a == b) return;
    if (a > b) {
      const int t = a;
      a = b;
      b = t;
    }
    const int old = atomicMin(&lab[b], a);
    if (old == b) return;
    b = old;
  }
}

// backward (scan-order preceding) 26-neighbours, most-connected first
__device__ constexpr int kB26[13][3] = {
    {-1, 0, 0}, {0, -1, 0}, {0, 0, -1}, {-1, 1, 0}, {-1, -1, 0}, {-1, 0, -1}, {-1, 0, 1},
    {0, -1, -1}, {0, -1, 1}, {-1, 1, 1}, {-1, 1, -1}, {-1, -1, 1}, {-1, -1, -1}};
__device__ constexpr unsigned b26_adj(int k) {  // neighbours 26-adjacent to k, and k
  unsigned m = 0;
  for (int j = 0; j < 13; ++j) {
    const int a = kB26[k][0] - kB26[j][0], b = kB26[k][1] - kB26[j][1], c = kB26[k][2] - kB26[j][2];
    if (a >= -1 && a <= 1 && b >= -1 && b <= 1 && c >= -1 && c <= 1) m |= 1u << j;
  }
  return m;
}

template <int CONN, typename T, int MODE>
__global__ void __launch_bounds__(kCT)
k_cc_union(int* __restrict__ lab, const T* __restrict__ in, int nz, int ny, int nx) {
  const int plane = ny * nx;
  // one (z, y) row per block iteration: no per-voxel integer division
  for (int row = blockIdx.x; row < nz * ny; row += gridDim.x)
  for (int x = threadIdx.x; x < nx; x += kCT) {
    const int i = row * nx + x;
    if (lab[i] < 0) continue;
    const int z = row / ny, y = row - z * ny;
    const T vi = MODE == CC_SAME ? in[i] : T(0);
    auto linked = [&](int j) { return lab[j] >= 0 && (MODE != CC_SAME || in[j] == vi); };
    if (CONN == 6) {
      // x-edges are linked by k_cc_init.  A y (z) edge is implied when the left
      // neighbours are joined the same way: i ~ i-1 ~ i-1-nx ~ i-nx, the middle
      // edge being some voxel's own y (z) edge further left in the run.
      const bool left = x > 0 && linked(i - 1);
      if (y > 0 && linked(i - nx) && !(left && linked(i - 1 - nx))) cc_union(lab, i, i - nx);
      if (z > 0 && linked(i - plane) && !(left && linked(i - 1 - plane))) cc_union(lab, i, i - plane);
    } else {
      // The 13 neighbours that precede i in scan order, greedily: once i is
      // linked to a neighbour A, every other neighbour B that is 26-adjacent to
      // A needs no union of its own — A and B are linked by whichever of the
      // two comes later in scan order (the relation is transitive for all
      // modes: nonzero, zero, equal value).  The centre below (first in the
      // list) is adjacent to all twelve others.
      // Neighbours are loaded lazily, in priority order, only while some are
      // still uncovered (the centre below alone covers all twelve others).
      unsigned todo = (1u << 13) - 1;
      // the x-1 neighbour is already joined by k_cc_init: a free link
      if (x > 0 && linked(i - 1)) todo &= ~b26_adj(2);
      todo &= ~(1u << 2);
#pragma unroll
      for (int k = 0; k < 13; ++k) {
        if (k == 2 || !(todo & (1u << k))) continue;
        const int dz = kB26[k][0], dy = kB26[k][1], dx = kB26[k][2];
        const int zz = z + dz, yy = y + dy, xx = x + dx;
        const int j = i + dz * plane + dy * nx + dx;
        if (zz >= 0 && yy >= 0 && yy < ny && xx >= 0 && xx < nx && linked(j)) {
          cc_union(lab, i, j);
          todo &= ~b26_adj(k);
        } else {
          todo &= ~(1u << k);
        }
        if (!todo) break;
      }
    }
  }
}

// each voxel's root goes to `root` (the output buffer), not back into `lab`:
// another thread's stale halving store could overwrite it there
__global__ void __launch_bounds__(kCT)
k_cc_flatten(int* __restrict__ lab, int* __restrict__ flag, int n, int* __restrict__ root) {
  for (int i = blockIdx.x * kCT + threadIdx.x; i < n; i += gridDim.x * kCT) {
    const int l = lab[i];
    const int r = l >= 0 ? cc_find(lab, i) : -1;
    flag[i] = (l >= 0 && r == i) ? 1 : 0;
    root[i] = r;
  }
}

__global__ void __launch_bounds__(kCT)
k_cc_relabel(const int* root, const int* __restrict__ ids, int n, uint32_t* out) {
  for (int i = blockIdx.x * kCT + threadIdx.x; i < n; i += gridDim.x * kCT) {
    const int r = root[i];
    out[i] = r >= 0 ? (uint32_t)(ids[r] + 1) : 0u;  // in place over root (same index)
  }
}

// fill_holes: mark the roots of zero components that touch a volume face
__global__ void __launch_bounds__(kCT)
k_mark_border(const int* __restrict__ root, int nz, int ny, int nx, int* __restrict__ mark) {
  const int plane = ny * nx, n = nz * plane;
  for (int i = blockIdx.x * kCT + threadIdx.x; i < n; i += gridDim.x * kCT) {
    const int r = root[i];
    if (r < 0) continue;
    const int z = i / plane, rr = i - z * plane, y = rr / nx, x = rr - y * nx;
    if (z == 0 || z == nz - 1 || y == 0 || y == ny - 1 || x == 0 || x == nx - 1) mark[r] = 1;
  }
}

template <typename T>
__global__ void __launch_bounds__(kCT)
k_fill(const T* __restrict__ in, const int* __restrict__ root, const int* __restrict__ mark, int n,
       T* __restrict__ out) {
  for (int i = blockIdx.x * kCT + threadIdx.x; i < n; i += gridDim.x * kCT) {
    const int r = root[i];
    out[i] = (r >= 0 && !mark[r]) ? T(1) : in[i];
  }
}

// component sizes by root; neighbouring voxels mostly share a root, so the
// lanes of a warp with equal roots add once (__match_any_sync) instead of
// serialising on one address (a giant component made this 2.3 Gvox/s)
// — and the block's "hot" root (its first voxel's, usually the giant
// component's) is counted in shared memory and added once per block
__global__ void __launch_bounds__(kCT) k_sizes(const int* __restrict__ root, int n, int* __restrict__ size) {
  __shared__ int hot, cnt;
  if (threadIdx.x == 0) {
    hot = blockIdx.x * kCT < n ? root[blockIdx.x * kCT] : -1;
    cnt = 0;
  }
  __syncthreads();
  const int h = hot;
  for (int i0 = blockIdx.x * kCT; i0 < n; i0 += gridDim.x * kCT) {
    const int i = i0 + threadIdx.x;
    const int r = i < n ? root[i] : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, r);
    const int leader = __ffs(peers) - 1;
    if (r >= 0 && (int)(threadIdx.x & 31) == leader) {
      if (r == h) atomicAdd(&cnt, __popc(peers));
      else atomicAdd(&size[r], __popc(peers));
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && h >= 0 && cnt) atomicAdd(&size[h], cnt);
}

template <typename T>
__global__ void __launch_bounds__(kCT)
k_drop_small(const T* __restrict__ in, const int* __restrict__ root, const int* __restrict__ size,
             int n, int64_t min_size, T* __restrict__ out) {
  for (int i = blockIdx.x * kCT + threadIdx.x; i < n; i += gridDim.x * kCT) {
    const int r = root[i];
    out[i] = (r >= 0 && (int64_t)size[r] < min_size) ? T(0) : in[i];
  }
}

// union-find labelling: root[i] = smallest index of i's component, -1 off it
template <typename T, int MODE>
void cc_label_t(const T* in, int nz, int ny, int nx, int conn, int* lab, int* root, int* flag,
                cudaStream_t s) {
  const int n = nz * ny * nx;
  const int g = cgrid(n);
  k_cc_init<T, MODE><<<g, kCT, 0, s>>>(in, nx, n, lab);
  const int gr = (int)std::min<int64_t>((int64_t)nz * ny, (int64_t)kNumSMs * 64);
  if (conn == 6) k_cc_union<6, T, MODE><<<gr, kCT, 0, s>>>(lab, in, nz, ny, nx);
  else k_cc_union<26, T, MODE><<<gr, kCT, 0, s>>>(lab, in, nz, ny, nx);
  k_cc_flatten<<<g, kCT, 0, s>>>(lab, flag, n, root);
}

template <int MODE>
cudaError_t cc_label(const void* in, int dt, int nz, int ny, int nx, int conn, int* lab, int* root,
                     int* flag, cudaStream_t s) {
  switch (dt) {
    case HB_U8: cc_label_t<uint8_t, MODE>((const uint8_t*)in, nz, ny, nx, conn, lab, root, flag, s); break;
    case HB_U16: cc_label_t<uint16_t, MODE>((const uint16_t*)in, nz, ny, nx, conn, lab, root, flag, s); break;
    case HB_U32: cc_label_t<uint32_t, MODE>((const uint32_t*)in, nz, ny, nx, conn, lab, root, flag, s); break;
    case HB_F32: cc_label_t<float, MODE>((const float*)in, nz, ny, nx, conn, lab, root, flag, s); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace

cudaError_t connected_components(const void* in, int dt, int64_t nz, int64_t ny, int64_t nx,
                                 int conn, uint32_t* out, int* lab, int* flag, int* ids,
                                 void* scan_tmp, size_t scan_bytes, int64_t* count, cudaStream_t s) {
  const int64_t n64 = nz * ny * nx;
  if (n64 <= 0) {
    if (count) *count = 0;
    return cudaSuccess;
  }
  if (n64 >= (1ll << 31) - 1) return cudaErrorNotSupported;
  const int n = (int)n64;
  const int g = cgrid(n64);
  int* root = reinterpret_cast<int*>(out);  // roots first, compacted ids in place after
  cudaError_t e = cc_label<CC_NONZERO>(in, dt, (int)nz, (int)ny, (int)nx, conn, lab, root, flag, s);
  if (e != cudaSuccess) return e;
  size_t need = scan_bytes;
  e = cub::DeviceScan::ExclusiveSum(scan_tmp, need, flag, ids, n, s);
  if (e != cudaSuccess) return e;
  k_cc_relabel<<<g, kCT, 0, s>>>(root, ids, n, out);
  if (count) {
    int last_id = 0, last_flag = 0;
    cudaMemcpyAsync(&last_id, ids + n - 1, 4, cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(&last_flag, flag + n - 1, 4, cudaMemcpyDeviceToHost, s);
    e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return e;
    *count = (int64_t)last_id + last_flag;
  }
  return cudaGetLastError();
}

// chunked labelling, pass 1 / 2 helpers: rank[i] = position of i's root among
// the chunk's roots (ascending index = scan order), -1 off the mask
__global__ void __launch_bounds__(kCT)
k_cc_rank(const int* __restrict__ root, const int* __restrict__ ids, int n, int* __restrict__ rank) {
  for (int i = blockIdx.x * kCT + threadIdx.x; i < n; i += gridDim.x * kCT) {
    const int r = root[i];
    rank[i] = r >= 0 ? ids[r] : -1;
  }
}

__global__ void __launch_bounds__(kCT)
k_cc_table(const int* __restrict__ rank, int n, const uint32_t* __restrict__ table, uint32_t* __restrict__ out) {
  for (int i = blockIdx.x * kCT + threadIdx.x; i < n; i += gridDim.x * kCT) {
    const int r = rank[i];
    out[i] = r >= 0 ? table[r] : 0u;
  }
}

cudaError_t cc_chunk_ranks(const void* in, int dt, int cz, int ny, int nx, int conn, int* lab, int* root,
                           int* flag, int* ids, void* scan_tmp, size_t scan_bytes, int* rank,
                           int64_t* nroots, cudaStream_t s) {
  const int n = cz * ny * nx;
  const int g = cgrid(n);
  cudaError_t e = cc_label<CC_NONZERO>(in, dt, cz, ny, nx, conn, lab, root, flag, s);
  if (e != cudaSuccess) return e;
  size_t need = scan_bytes;
  e = cub::DeviceScan::ExclusiveSum(scan_tmp, need, flag, ids, n, s);
  if (e != cudaSuccess) return e;
  k_cc_rank<<<g, kCT, 0, s>>>(root, ids, n, rank);
  int last_id = 0, last_flag = 0;
  cudaMemcpyAsync(&last_id, ids + n - 1, 4, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(&last_flag, flag + n - 1, 4, cudaMemcpyDeviceToHost, s);
  e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return e;
  *nroots = (int64_t)last_id + last_flag;
  return cudaGetLastError();
}

cudaError_t cc_apply_table(const int* rank, int n, const uint32_t* table, uint32_t* out, cudaStream_t s) {
  k_cc_table<<<cgrid(n), kCT, 0, s>>>(rank, n, table, out);
  return cudaGetLastError();
}

cudaError_t label_filter(const void* in, int dt, int64_t nz, int64_t ny, int64_t nx, int conn,
                         int op, int64_t min_size, void* out, int* lab, int* root, int* aux,
                         cudaStream_t s) {
  const int64_t n64 = nz * ny * nx;
  if (n64 <= 0) return cudaSuccess;
  if (n64 >= (1ll << 31) - 1) return cudaErrorNotSupported;
  const int n = (int)n64;
  const int g = cgrid(n64);
  cudaError_t e = op == 0 ? cc_label<CC_ZERO>(in, dt, (int)nz, (int)ny, (int)nx, conn, lab, root, aux, s)
                          : cc_label<CC_SAME>(in, dt, (int)nz, (int)ny, (int)nx, conn, lab, root, aux, s);
  if (e != cudaSuccess) return e;
  cudaMemsetAsync(aux, 0, (size_t)n * 4, s);  // border marks / component sizes, by root
  if (op == 0) k_mark_border<<<g, kCT, 0, s>>>(root, (int)nz, (int)ny, (int)nx, aux);
  else k_sizes<<<g, kCT, 0, s>>>(root, n, aux);
  switch (dt) {
#define HB_LF(T)                                                                                  \
  if (op == 0) k_fill<T><<<g, kCT, 0, s>>>((const T*)in, root, aux, n, (T*)out);                  \
  else k_drop_small<T><<<g, kCT, 0, s>>>((const T*)in, root, aux, n, min_size, (T*)out);          \
  break;
    case HB_U8: HB_LF(uint8_t)
    case HB_U16: HB_LF(uint16_t)
    case HB_U32: HB_LF(uint32_t)
    case HB_F32: HB_LF(float)
#undef HB_LF
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

size_t connected_components_scan_bytes(int64_t n) {
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, (int*)nullptr, (int*)nullptr, (int)n);
  return bytes;
}

}  // namespace hb
