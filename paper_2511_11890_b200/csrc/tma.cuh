// tma.cuh — TMA (cp.async.bulk.tensor) + mbarrier helpers for sm_100a, and the
// host-side tensor-map encoder obtained through the runtime's driver entry point
// (no -lcuda needed).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace hb {

// ---------------------------------------------------------------------------
// device side
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
}

// 3D tile load: box at (x, y, z) -> smem dst, completion on bar.
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y, int z,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}

// 3D tile store smem -> global (out-of-range parts of the box are dropped).
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int x, int y,
                                             int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(smem_u32(src)), "r"(x), "r"(y), "r"(z)
      : "memory");
}

__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }

template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// Clamp-to-edge fix-up of a TMA-staged halo'd tile whose out-of-volume parts
// TMA zero-filled: out-of-range rows are copied whole from the nearest valid
// row, then out-of-range columns of every row from the nearest valid column.
// Touches only the halo strips (the per-element loop over the whole tile it
// replaces was ~20% of k_morph3's instructions at 1024^3).  The caller fences
// and synchronises afterwards.
template <typename T, int NT>
__device__ __forceinline__ void clamp_tile(T* st, int pitch, int h, int w, int gy0, int gx0, int ny,
                                           int nx, int tid) {
  const int r_lo = max(0, -gy0), r_hi = min(h, ny - gy0);
  if (r_lo > 0 || r_hi < h) {
    const int nbad = r_lo + (h - r_hi);
    for (int e = tid; e < nbad * w; e += NT) {
      const int i = e / w, c = e - i * w;
      const int r = i < r_lo ? i : r_hi + (i - r_lo);
      const int src = i < r_lo ? r_lo : r_hi - 1;
      st[r * pitch + c] = st[src * pitch + c];
    }
    __syncthreads();
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

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
// Encodes a 3D (x fastest) tiled map over a C-contiguous (nz, ny, nx) volume.
// Returns false if the layout violates TMA constraints (16-B aligned base and
// strides, box <= 256 per dim) — callers then use a non-TMA kernel.
bool make_tmap_3d(CUtensorMap* map, const void* base, CUtensorMapDataType dt, int elem_bytes,
                  int64_t nx, int64_t ny, int64_t nz, int box_x, int box_y);

}  // namespace hb
