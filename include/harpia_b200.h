/*
 * harpia_b200.h — C ABI of the B200-native Harpia map-operator hot path.
 *
 * The reference (a pure-Python package, /root/reference/pkg/src/harpia) has no
 * FFI; its hot path is the Python call chain
 *
 *     registry.run_operator            (registry.py:82-103)
 *       -> chunking.execute_chunked    (chunking.py:215-279)
 *         -> fn(block, params, aux)    (chunking.py:257), e.g. filters.gaussian
 *
 * Each entry point below replaces one piece of that chain; the Python mirror in
 * paper_2511_11890_b200/ binds them with ctypes:
 *
 *   hb_run            replaces execute_chunked's chunk loop + every per-chunk fn
 *                     (chunking.py:242-274) for a chain of map operators, on
 *                     caller-owned HOST buffers (C-contiguous Z,Y,X).
 *   hb_apply_device   replaces one fn(block, ...) call (chunking.py:257) on a
 *                     DEVICE-resident block (torch tensors, sharded slabs).
 *   hb_device_info    replaces probe_free_bytes (chunking.py:57-61): free bytes
 *                     come from cudaMemGetInfo instead of psutil.
 *   hb_plan           restates plan_chunks (chunking.py:135-174) for C callers.
 *   hb_gaussian_weights restates _gaussian_kernel (filters.py:26-30).
 *   hb_minmax / hb_histogram, hb_connected_components, hb_label_filter,
 *   hb_geodesic, hb_edt  replace the global operators' run functions
 *                     (registry.py:312-417).
 *
 * Status codes map 1:1 onto the reference exception hierarchy (errors.py:4-41);
 * see hb_status.  No torch types cross this boundary: plain pointers and sizes.
 */
#ifndef HARPIA_B200_H
#define HARPIA_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HB_ABI_VERSION 1

/* errors.py:4-41 */
typedef enum {
  HB_OK = 0,
  HB_EPARAM = 1,              /* ParameterError            errors.py:8        */
  HB_EBUDGET_SMALL = 2,       /* BudgetTooSmallError       errors.py:24-29    */
  HB_EBUDGET_UNAVAILABLE = 3, /* BudgetUnavailableError    errors.py:20       */
  HB_ECHUNK = 4,              /* ChunkExecutionError       errors.py:32-37    */
  HB_ECANCELLED = 5,          /* JobCancelled              errors.py:40-41    */
  HB_ECUDA = 6,               /* ChunkExecutionError (device fault) / no GPU  */
  HB_EUNSUPPORTED = 7         /* UnsupportedFormatError    errors.py:16       */
} hb_status;

/* volume.py:17-23 SUPPORTED_DTYPES + LABEL_DTYPE */
typedef enum {
  HB_U8 = 0, HB_U16 = 1, HB_U32 = 2, HB_F32 = 3,
  HB_F64 = 4 /* output only: hb_edt's squared distances */
} hb_dtype;

typedef enum { HB_HOST = 0, HB_DEVICE = 1 } hb_location;

/* A C-contiguous (Z, Y, X) volume, x fastest (volume.py:1-5). */
typedef struct {
  void* data;
  int32_t dtype;     /* hb_dtype */
  int32_t location;  /* hb_location */
  int64_t nz, ny, nx;
} hb_volume;

/* Map operators on the hot path (registry.py:135-191, 234-246, 274-285). */
typedef enum {
  HB_OP_IDENTITY = 0, /* registry.py:127-133 */
  HB_OP_GAUSSIAN = 1, /* filters.py:33-41    */
  HB_OP_MEAN = 2,     /* filters.py:66-75    */
  HB_OP_MEDIAN = 3,   /* filters.py:78-82    */
  HB_OP_UNSHARP = 4,  /* filters.py:136-139  */
  HB_OP_LOG = 5,      /* hessian trace, filters.py:234-264 */
  HB_OP_ERODE = 6,    /* morphology.py:114-116 */
  HB_OP_DILATE = 7,   /* morphology.py:119-121 (caller passes the SE; the
                         library reflects it, as the reference does) */
  /* SURVEY.md §8(f) row 2, the next local map ops on the same machinery: */
  HB_OP_HESSIAN = 8,  /* one component, filters.py:246-253; radius = component
                         index 0..5 = xx, yy, zz, xy, xz, yz (filters.py:228) */
  HB_OP_SOBEL = 9,    /* filters.py:200-202 */
  HB_OP_PREWITT = 10, /* filters.py:205-207 */
  HB_OP_THRESHOLD = 11, /* threshold.py:110-112; amount = t; uint32 labels */
  HB_OP_LBP2D = 12,   /* filters.py:213-227; uint8 per-slice codes */
  HB_OP_DIFFUSION = 13, /* anisotropic_diffusion, filters.py:142-184: radius =
                          iterations, sigma = kappa, amount = dt, precision =
                          mode (0 exponential, 1 rational) */
  HB_OP_LOCAL_THRESHOLD = 14 /* threshold.local_threshold, threshold.py:174-217
                          (registry.py:257-272): radius = window, precision =
                          hb_local_kind, sigma = k, amount = c (mean / median /
                          gaussian) or R (sauvola; NaN = half the
                          input dtype's range, 0.5 for float32); gaussian: weights64 = the
                          2*window+1 float64 taps (threshold.py:199-202), NULL =
                          computed by the library; uint32 labels */
} hb_op;

/* local_threshold kinds, in threshold.LOCAL_KINDS order (threshold.py:21) */
typedef enum {
  HB_LT_MEAN = 0,
  HB_LT_MEDIAN = 1,
  HB_LT_GAUSSIAN = 2,
  HB_LT_NIBLACK = 3,
  HB_LT_SAUVOLA = 4
} hb_local_kind;

typedef enum {
  HB_PREC_FAST = 0,  /* fp32 accumulation, within 1e-5 of the reference */
  HB_PREC_EXACT = 1  /* fp64 per pass + f32 round: bit-exact Gaussian */
} hb_precision;

/* One stage of a (possibly chained) map pipeline.  open/close/iterations are
 * expressed as chains of erode/dilate stages (morphology.py:124-140). */
typedef struct {
  int32_t op;          /* hb_op */
  int32_t precision;   /* hb_precision (gaussian/unsharp/log/hessian) */
  double sigma;        /* gaussian/unsharp/log/hessian */
  double amount;       /* unsharp: amount; threshold: t */
  int32_t radius;      /* mean/median: radius; hessian: component index */
  int32_t n_offsets;   /* erode/dilate: number of (dz,dy,dx) triples */
  const int32_t* offsets; /* erode/dilate: 3*n_offsets ints, must contain origin */
  int32_t n_weights;   /* gaussian/unsharp/log: 2*ceil(4 sigma)+1, or 0 */
  const float* weights; /* optional f32 taps from the caller's _gaussian_kernel
                           (filters.py:26-30); NULL = computed by the library */
  const double* weights64; /* local_threshold gaussian: n_weights float64 taps */
} hb_stage;

/* One chunk of a ChunkPlan (chunking.py:93-111): interior [z_start, z_stop),
 * halos already truncated at the volume faces. */
typedef struct {
  int64_t z_start, z_stop, halo_lo, halo_hi;
} hb_chunk;

typedef int32_t (*hb_cancel_fn)(void* ctx); /* nonzero => cancel */

typedef struct {
  int32_t device;            /* CUDA ordinal */
  int32_t pipeline_depth;    /* chunks in flight (1 = serial, 2 = double buffer; 0 = auto) */
  int64_t device_budget;     /* cap on executor device bytes (0 = no cap) */
  hb_cancel_fn cancel;       /* polled before every chunk (chunking.py:245-246) */
  void* cancel_ctx;
  double* chunk_seconds;     /* optional out array [nchunks] (chunking.py:274) */
  int32_t fault_chunk;       /* test hook: fail chunk i with HB_ECHUNK (-1 = off) */
  int32_t host_threads;      /* threads for pageable<->pinned staging (0 = auto) */
} hb_exec;

typedef struct {
  int64_t chunk_count;
  int64_t failed_chunk;        /* ChunkExecutionError.chunk_index, -1 if none */
  int64_t minimum_bytes;       /* BudgetTooSmallError.minimum_bytes */
  int64_t device_peak_bytes;   /* executor high-water mark of device bytes */
  int64_t device_residual_bytes; /* executor bytes still held at return (must be 0) */
  int64_t h2d_bytes, d2h_bytes;
  double h2d_ms, kernel_ms, d2h_ms, wall_ms;
  int64_t kernel_launches;
  char message[512];
} hb_report;

/* Library / device introspection ----------------------------------------- */
int32_t hb_abi_version(void);
const char* hb_version(void);
/* hb_status; free/total bytes of device `dev` (chunking.py:57-61 analogue). */
int32_t hb_device_info(int32_t dev, int64_t* free_bytes, int64_t* total_bytes);
int32_t hb_device_count(void);

/* Chunk planning for C callers: plan_chunks (chunking.py:135-174), same
 * formula and error.  t = floor(usable / (scratch_factor * slice_bytes))
 * padded slices; t <= 2*halo -> HB_EBUDGET_SMALL with *minimum_bytes =
 * ceil((2*halo + 1) * scratch_factor * slice_bytes); else interior n = t - 2*halo
 * and chunks [k*n, min((k+1)*n, nz)) with halos min(halo, z_start),
 * min(halo, nz - z_stop).  *nchunks receives the count; chunks (capacity
 * entries, may be NULL) receives them when it is large enough. */
int32_t hb_plan(int64_t nz, int64_t ny, int64_t nx, int32_t itemsize, int64_t halo,
                double scratch_factor, int64_t usable_bytes, hb_chunk* chunks, int64_t capacity,
                int64_t* nchunks, int64_t* minimum_bytes);

/* Parameter helpers ------------------------------------------------------- */
/* ceil(4*sigma) (filters.py:21-23) */
int32_t hb_gaussian_radius(double sigma);
/* Writes 2r+1 float32 weights of _gaussian_kernel (filters.py:26-30). */
int32_t hb_gaussian_weights(double sigma, float* out, int32_t capacity);
/* Z dependence radius of a stage chain (sum of per-stage halos, registry.py). */
int64_t hb_chain_halo(const hb_stage* stages, int32_t nstages);

/* Execution --------------------------------------------------------------- */
/* Chunked streaming executor over HOST volumes: for every chunk, upload the
 * padded slab, run the stage chain on the device, download the interior.
 * `out` must be a host volume of the chain's output dtype and in's shape. */
int32_t hb_run(const hb_volume* in, hb_volume* out,
               const hb_stage* stages, int32_t nstages,
               const hb_chunk* chunks, int64_t nchunks,
               const hb_exec* ex, hb_report* rep);

/* Apply a stage chain to a DEVICE block `in` (clamp-to-edge at all its faces)
 * and write output slices [z_begin, z_begin + out->nz) of the block into `out`
 * (a device volume with out->ny == in->ny, out->nx == in->nx).  Runs on
 * `stream` (cudaStream_t, NULL = legacy default); asynchronous unless
 * `synchronize` is nonzero.  Device temporaries come from a library-private
 * pool that is trimmed to zero before return. */
int32_t hb_apply_device(const hb_volume* in, hb_volume* out,
                        const hb_stage* stages, int32_t nstages,
                        int64_t z_begin, void* stream, int32_t synchronize,
                        hb_report* rep);

/* Multi-device streaming executor (SURVEY.md §8(b) "ndev, devices[]"): the
 * plan's chunks are split into ndev contiguous z-slab groups (balanced by
 * interior slices) and each group is streamed by hb_run's loop on its own
 * device from its own host thread — one PCIe link per device, no device-to-
 * device exchange (halos at group faces are read from the host volume, plan
 * invariance keeps the stitched result identical to hb_run's).  `ex` is used
 * for every group (its `device` is ignored; `cancel` must be thread-safe);
 * failed_chunk is the global chunk index; `per_device` (optional, ndev
 * entries) receives each group's report.  Replaces the sequential chunk loop
 * of execute_chunked (chunking.py:242-274) when several B200s share a host. */
int32_t hb_run_multi(const hb_volume* in, hb_volume* out,
                     const hb_stage* stages, int32_t nstages,
                     const hb_chunk* chunks, int64_t nchunks,
                     const hb_exec* ex, int32_t ndev, const int32_t* devices,
                     hb_report* rep, hb_report* per_device);

/* Library-pool device buffers (extension): stream-ordered allocation from the
 * same private cudaMemPool the executor uses, so z-slab buffers of a sharded
 * job (ghost slices + interior) are reported by hb_device_pool_bytes and
 * released by hb_trim_device / hb_session_end — never PyTorch's caching
 * allocator.  HB_EBUDGET_SMALL when the device is out of memory. */
int32_t hb_device_alloc(int32_t dev, int64_t bytes, void* stream, void** ptr);
int32_t hb_device_free(int32_t dev, void* ptr, void* stream);

/* Output dtype of a chain for a given input dtype (hb_dtype), or -1. */
int32_t hb_chain_out_dtype(const hb_stage* stages, int32_t nstages, int32_t in_dtype);

/* Trim the library's private device pool of `dev` to zero bytes (after
 * asynchronous hb_apply_device calls; synchronous jobs trim themselves). */
int32_t hb_trim_device(int32_t dev);
/* Device-arena session (extension; no reference counterpart): between
 * hb_session_begin(dev) and the matching hb_session_end(dev), jobs on `dev`
 * return their buffers to the library pool without trimming it, so repeated
 * jobs skip the driver's map/unmap; hb_session_end trims the pool to zero.
 * Nested sessions are counted.  Outside a session every job trims itself
 * (chunking.py's job-scoped reservation, chunking.py:243). */
int32_t hb_session_begin(int32_t dev);
int32_t hb_session_end(int32_t dev);
/* Bytes currently reserved by the library's private pool on `dev`. */
int64_t hb_device_pool_bytes(int32_t dev);

/* Pass 1 of the two-pass global operators (chunking.py:282-306
 * chunked_reduce) on the device, for Otsu (threshold.py:90-107).  `in` may be
 * host (pinned or pageable; streamed in slabs) or device memory.
 * hb_minmax: float32 volumes only (threshold.py:49-55); EPARAM if a NaN is
 * present (the reference's range check raises).
 * hb_histogram: np.histogram(data, bins, range=(lo, hi)) counts, bit-exact:
 * values outside [lo, hi] are dropped, index = int(((v - lo) / (hi - lo)) *
 * bins) with NumPy's edge corrections against `edges` (bins + 1 values of
 * np.linspace(lo, hi, bins + 1, dtype=bin_type)); edges_f32 = 1 when bin_type
 * is float32 (float32 data), else float64.  counts: bins int64, overwritten. */
int32_t hb_minmax(const hb_volume* in, int32_t device, double* lo, double* hi);
int32_t hb_histogram(const hb_volume* in, int32_t device, int32_t bins, double lo, double hi,
                     const double* edges, int32_t edges_f32, int64_t* counts);

/* Connected-components labelling (quantify.py:60-111): labels 1..count in
 * first-voxel scan order (uint32, `out`), background 0; connectivity 6 or 26;
 * the volume must fit in device memory (< 2^31 voxels).  `in`/`out` host or
 * device; any nonzero voxel is foreground. */
int32_t hb_connected_components(const hb_volume* in, hb_volume* out, int32_t connectivity,
                                int32_t device, int64_t* count);
/* Label-volume filters built on the same labelling (out: the input's dtype and
 * shape): op 0 = fill_holes (morphology.py:176-194: zero components not
 * touching a volume face become 1), op 1 = remove_islands (morphology.py:
 * 209-229: components of equal nonzero value smaller than min_size become 0). */
int32_t hb_label_filter(const hb_volume* in, hb_volume* out, int32_t op, int32_t connectivity,
                        int64_t min_size, int32_t device);
/* Geodesic reconstruction (morphology.py:143-165): fixed point of
 * min(dilate(m, cross(1)), mask) (dilation = 1) or max(erode(m, cross(1)),
 * mask) (dilation = 0) from `marker`; marker, mask and out share dtype and
 * shape; EPARAM if marker > mask (dilation) / marker < mask (erosion)
 * anywhere.  `sweeps` (optional) receives the number of in-place passes. */
int32_t hb_geodesic(const hb_volume* marker, const hb_volume* mask, hb_volume* out,
                    int32_t dilation, int32_t device, int64_t* sweeps);
/* Exact Euclidean distance transform (quantify.py:115-175): distance of every
 * nonzero voxel to the nearest zero voxel with per-axis `spacing` (z, y, x).
 * out dtype HB_F32: sqrt(d^2) cast to float32 (the reference's default);
 * out dtype HB_F64 (squared=True): d^2.  No zero voxel -> +inf. */
int32_t hb_edt(const hb_volume* in, hb_volume* out, const double* spacing, int32_t device);

/* Pinned-host helpers (cudaHostRegister for the duration of a job). */
int32_t hb_pin(void* ptr, int64_t bytes);
int32_t hb_unpin(void* ptr);

/* Last error message of the calling thread. */
const char* hb_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* HARPIA_B200_H */
