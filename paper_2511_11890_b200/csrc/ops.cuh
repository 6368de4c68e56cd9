// ops.cuh — internal launch API of the hot-path kernels (host side).
//
// Every kernel evaluates one map operator on a device block whose local z runs
// over [0, in.nz) with clamp-to-edge at all six faces (exactly the padded-chunk
// semantics of chunking.execute_chunked, chunking.py:248-257), and writes the
// output slices [zo, zo + nzo) of that block.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace hb {

constexpr int kMaxTaps = 129;  // R <= 64  (sigma <= 16)

struct Taps {
  float w[kMaxTaps];  // 2R+1 f32 weights (filters.py:26-30), w[R] is the centre
  int R;
};

struct DevIn {
  const void* p;
  int dt;  // hb_dtype
  int64_t nz, ny, nx;
};

// Epilogue of the last separable pass.
enum Epi { EPI_NONE = 0, EPI_UNSHARP = 1, EPI_BOX_MEAN = 2 };

struct EpiArgs {
  int kind = EPI_NONE;
  // unsharp: base = f32(orig[z + orig_zo]) (filters.py:136-139)
  const void* orig = nullptr;
  int orig_dt = HB_F32;
  int64_t orig_zo = 0;
  float amount = 0.f;
  float inv_count = 1.f;  // box mean: divide by (2r+1)^3
  float count = 1.f;
};

// --- separable stencils (sep.cu) ------------------------------------------
// Gaussian (fast: fp32 FMA; exact: fp64 fold per pass, f32 round per pass,
// axis order Z, Y, X as filters.py:38-40).  `tmp` must hold nzo*ny*nx floats.
cudaError_t gaussian_generic(const DevIn& in, int64_t zo, int64_t nzo, float* out,
                             const Taps& taps, bool exact, const EpiArgs& epi,
                             float* tmp, cudaStream_t s, int64_t* launches);
// Box mean of (2r+1)^3 (filters.py:66-75).
cudaError_t mean_generic(const DevIn& in, int64_t zo, int64_t nzo, float* out, int r,
                         float* tmp, cudaStream_t s, int64_t* launches);
// LoG second stage: out = (cd_x cd_x g + cd_y cd_y g) + cd_z cd_z g, where the
// smoothed block g covers local slices [gz0, gz0+ngz) of a block of `nz`
// slices (clamps at [0, nz)) — filters.py:234-253.
cudaError_t log_diff(const float* g, int64_t gz0, int64_t ngz, int64_t nz, int64_t ny,
                     int64_t nx, int64_t zo, int64_t nzo, float* out, cudaStream_t s,
                     int64_t* launches);
// streaming form of log_diff (logd.cu); NotSupported unless nx % 4 == 0
cudaError_t log_diff_stream(const float* g, int64_t gz0, int64_t nz, int64_t ny, int64_t nx,
                            int64_t zo, int64_t nzo, float* out, cudaStream_t s,
                            int64_t* launches);
// next local map ops (extra.cu): one Hessian component cd_b(cd_a(g)) of a
// smoothed block g laid out like log_diff's; Sobel/Prewitt gradient
// magnitude; apply_threshold -> uint32 labels
cudaError_t hessian_stage(const float* g, int64_t gz0, int64_t nz, int64_t ny, int64_t nx,
                          int64_t zo, int64_t nzo, int axis_a, int axis_b, float* out,
                          cudaStream_t s, int64_t* launches);
cudaError_t gradmag(const DevIn& in, int64_t zo, int64_t nzo, float* out, bool sobel,
                    cudaStream_t s, int64_t* launches);
cudaError_t threshold(const DevIn& in, int64_t zo, int64_t nzo, uint32_t* out, double t,
                      cudaStream_t s, int64_t* launches);
cudaError_t lbp2d(const DevIn& in, int64_t zo, int64_t nzo, uint8_t* out, cudaStream_t s,
                  int64_t* launches);
// anisotropic diffusion over the whole block (closed faces, as the reference's
// padded chunk), then slices [zo, zo+nzo) -> out; b0/b1: nz*ny*nx floats each
cudaError_t diffusion(const DevIn& in, int64_t zo, int64_t nzo, float* out, int iterations,
                      float kappa, float dt, bool rational, float* b0, float* b1, cudaStream_t s,
                      int64_t* launches);
// local adaptive thresholds (local.cu, threshold.py:174-217) -> uint32 labels;
// scratch: local_threshold_scratch bytes
constexpr int kMaxLocalRadius = 50;
struct LocalParams {
  int kind = HB_LT_MEAN, w = 1;
  double k = 0.2, r = 0.5, c = 0.0;
  const double* kern = nullptr;  // gaussian kind: 2w+1 float64 taps (host)
};
size_t local_threshold_scratch(int kind, int dt, int w, int64_t slices, int64_t plane);
int local_threshold_max_radius(int kind, int dt);
cudaError_t local_threshold(const DevIn& in, int64_t zo, int64_t nzo, uint32_t* out, const LocalParams& p,
                            void* scratch, cudaStream_t s, int64_t* launches);
// dtype conversion / copy (identity op, registry.py:127-133)
cudaError_t copy_slices(const DevIn& in, int64_t zo, int64_t nzo, void* out,
                        cudaStream_t s, int64_t* launches);

// --- fused fast Gaussian family (gauss_fused.cu) --------------------------
// Returns cudaErrorNotSupported when the shape/radius is outside the fused
// kernel's envelope; the caller then uses the generic path.
// warp-specialised Gaussian / unsharp (gauss_ws.cu), 2 <= R <= 8, nx % 4 == 0
cudaError_t gaussian_small(const DevIn& in, int64_t zo, int64_t nzo, float* out, const Taps& taps,
                           const EpiArgs& epi, float* tmp, cudaStream_t s, int64_t* launches);
cudaError_t gaussian_tri(const DevIn& in, int64_t zo, int64_t nzo, float* out, const Taps& taps,
                        const EpiArgs& epi, cudaStream_t s, int64_t* launches);
cudaError_t gaussian_ws(const DevIn& in, int64_t zo, int64_t nzo, float* out, const Taps& taps,
                        const EpiArgs& epi, cudaStream_t s, int64_t* launches);
cudaError_t gaussian_fused(const DevIn& in, int64_t zo, int64_t nzo, float* out,
                           const Taps& taps, const EpiArgs& epi, cudaStream_t s,
                           int64_t* launches);

// bit-exact Gaussian in two kernels (gauss_exact.cu); tmp: nzo*ny*nx floats
cudaError_t gaussian_exact_fused(const DevIn& in, int64_t zo, int64_t nzo, float* out,
                                 const Taps& taps, const EpiArgs& epi, float* tmp,
                                 cudaStream_t s, int64_t* launches);

cudaError_t mean_fused(const DevIn& in, int64_t zo, int64_t nzo, float* out, int r,
                       cudaStream_t s, int64_t* launches);
// streaming box mean, r <= 2, nx % 4 == 0 (box.cu); NotSupported outside that
cudaError_t mean_stream(const DevIn& in, int64_t zo, int64_t nzo, float* out, int r,
                        cudaStream_t s, int64_t* launches);

// --- two-pass global operators, pass 1 (reduce.cu) ---------------------------
// acc: 3 unsigned on the device, initialised {~0u, 0, 0}: ordered-key min,
// max, NaN flag
cudaError_t minmax_f32(const float* p, int64_t n, unsigned* acc, cudaStream_t s);
// np.histogram counts (accumulated into counts[bins]); edges: bins+1 doubles
// on the device
cudaError_t histogram(const void* p, int dt, int64_t n, int bins, double lo, double hi,
                      const double* edges, bool edges_f32, unsigned long long* counts,
                      cudaStream_t s);

// --- connected components (cc.cu) --------------------------------------------
cudaError_t connected_components(const void* in, int dt, int64_t nz, int64_t ny, int64_t nx,
                                 int conn, uint32_t* out, int* lab, int* flag, int* ids,
                                 void* scan_tmp, size_t scan_bytes, int64_t* count, cudaStream_t s);
size_t connected_components_scan_bytes(int64_t n);
// chunked labelling (volumes beyond one device pass): per chunk, the rank of
// every voxel's root among the chunk's roots, and the final table lookup
cudaError_t cc_chunk_ranks(const void* in, int dt, int cz, int ny, int nx, int conn, int* lab, int* root,
                           int* flag, int* ids, void* scan_tmp, size_t scan_bytes, int* rank,
                           int64_t* nroots, cudaStream_t s);
cudaError_t cc_apply_table(const int* rank, int n, const uint32_t* table, uint32_t* out, cudaStream_t s);
// exact EDT (edt.cu): d2a/d2b: n doubles each; work: edt_workspace_bytes
size_t edt_workspace_bytes(int64_t nz, int64_t ny, int64_t nx);
cudaError_t edt(const void* in, int dt, int64_t nz, int64_t ny, int64_t nx, const double* spacing,
                bool squared, void* out, double* d2a, double* d2b, void* work, cudaStream_t s);
// geodesic reconstruction (extra.cu); cudaErrorInvalidValue = marker ordering violated
cudaError_t geodesic(const void* marker, const void* mask, int dt, int64_t nz, int64_t ny, int64_t nx,
                     bool dilation, void* out, int* flags, cudaStream_t s, int64_t* sweeps);
// op 0 fill_holes, op 1 remove_islands; lab/root/aux: n ints each
cudaError_t label_filter(const void* in, int dt, int64_t nz, int64_t ny, int64_t nx, int conn,
                         int op, int64_t min_size, void* out, int* lab, int* root, int* aux,
                         cudaStream_t s);

// --- median (median.cu) ----------------------------------------------------
// r = 1 on float32 through the TMA-fed kernel (median3f.cu); NotSupported
// outside its envelope
cudaError_t median3_f32(const DevIn& in, int64_t zo, int64_t nzo, float* out, cudaStream_t s,
                        int64_t* launches);
cudaError_t median(const DevIn& in, int64_t zo, int64_t nzo, void* out, int r,
                   cudaStream_t s, int64_t* launches);

// --- flat grey morphology (morph.cu) --------------------------------------
// offsets: 3*n ints (dz,dy,dx) host array; is_max selects dilation, in which
// case the caller has already reflected the SE (morphology.py:119-121).
// `gate` (optional): a device int of scratch for the u8 binary/grey gate
// (from the executor's pool); null -> a stream-ordered allocation per call.
cudaError_t morph(const DevIn& in, int64_t zo, int64_t nzo, void* out,
                  const int32_t* offsets, int n, bool is_max, cudaStream_t s,
                  int64_t* launches, int* gate = nullptr);

}  // namespace hb
