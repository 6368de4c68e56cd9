// executor.cu — C ABI (include/harpia_b200.h): stage-chain planning, the device
// memory manager, and the chunked streaming executor that replaces
// chunking.execute_chunked (chunking.py:215-279) for map operators.
//
// Memory model (SURVEY.md §5 "Memory release"): every device byte a job uses
// comes from a library-private cudaMemPool per device; at the end of every
// synchronous job the pool is trimmed to zero, so the job's device residual is
// exactly 0 and PyTorch's caching allocator is never involved.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: ranges for ncu --nvtx / nsys (no-ops without a tool)

#include <algorithm>
#include <atomic>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "ops.cuh"

using namespace hb;

namespace {
// NVTX range (job / chunk-piece / device-apply) on the calling host thread
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace

namespace {

thread_local std::string g_last_error;

void set_err(hb_report* rep, const std::string& m) {
  g_last_error = m;
  if (rep) {
    std::snprintf(rep->message, sizeof(rep->message), "%s", m.c_str());
  }
}

// ---------------------------------------------------------------------------
// Stage normalisation
// ---------------------------------------------------------------------------
struct StageDesc {
  int op = HB_OP_IDENTITY;
  int precision = HB_PREC_FAST;
  int64_t halo = 0;
  int radius = 0;
  float amount = 0.f;
  Taps taps{};
  std::vector<int32_t> offsets;  // reflected for dilation
  double threshold = 0.0;        // apply_threshold's t (kept in f64, NumPy semantics)
  float kappa = 0.f;             // anisotropic diffusion
  LocalParams lt;                // local_threshold (kern set at run time)
  std::vector<double> lt_kern;
  int in_dt = HB_F32, out_dt = HB_F32;
};

int gaussian_radius(double sigma) { return (int)std::ceil(4.0 * sigma); }

// numpy pairwise_sum for n <= 128 (see oracle/harpia_oracle.c for the citation)
double pairwise_sum(const double* a, int n) {
  if (n < 8) {
    double r = 0.;
    for (int i = 0; i < n; i++) r += a[i];
    return r;
  }
  double r[8];
  int i;
  for (i = 0; i < 8; i++) r[i] = a[i];
  for (i = 8; i < n - (n % 8); i += 8)
    for (int j = 0; j < 8; j++) r[j] += a[i + j];
  double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
  for (; i < n; i++) res += a[i];
  return res;
}

int fill_weights(double sigma, float* out, int cap) {
  int r = gaussian_radius(sigma);
  int n = 2 * r + 1;
  if (n > cap) return -1;
  std::vector<double> k(n);
  for (int i = 0; i < n; i++) {
    double q = (double)(i - r) / sigma;
    k[i] = std::exp(-0.5 * (q * q));
  }
  double s = pairwise_sum(k.data(), n);
  for (int i = 0; i < n; i++) out[i] = (float)(k[i] / s);
  return n;
}

int z_extent(const std::vector<int32_t>& off) {
  int e = 0;
  for (size_t k = 0; k < off.size(); k += 3) e = std::max(e, std::abs(off[k]));
  return e;
}

hb_status normalise(const hb_stage* st, int nst, int in_dt, std::vector<StageDesc>& out,
                    std::string& msg) {
  if (nst < 1) {
    msg = "empty stage chain";
    return HB_EPARAM;
  }
  int dt = in_dt;
  for (int i = 0; i < nst; i++) {
    const hb_stage& s = st[i];
    StageDesc d;
    d.op = s.op;
    d.precision = s.precision;
    d.in_dt = dt;
    switch (s.op) {
      case HB_OP_IDENTITY:
        d.out_dt = dt;
        break;
      case HB_OP_GAUSSIAN:
      case HB_OP_UNSHARP:
      case HB_OP_LOG:
      case HB_OP_HESSIAN: {
        if (!(s.sigma > 0) || !std::isfinite(s.sigma)) {
          msg = "sigma must be positive, got " + std::to_string(s.sigma);
          return HB_EPARAM;
        }
        int r = gaussian_radius(s.sigma);
        if (2 * r + 1 > kMaxTaps) {
          msg = "sigma too large for the device stencil (ceil(4 sigma) must be <= 64)";
          return HB_EUNSUPPORTED;
        }
        d.taps.R = r;
        if (s.weights && s.n_weights > 0) {
          if (s.n_weights != 2 * r + 1) {
            msg = "weights length does not match 2*ceil(4*sigma)+1";
            return HB_EPARAM;
          }
          std::memcpy(d.taps.w, s.weights, sizeof(float) * s.n_weights);
        } else {
          fill_weights(s.sigma, d.taps.w, kMaxTaps);
        }
        for (int k = 1; k <= r; k++)
          if (d.taps.w[r + k] != d.taps.w[r - k]) {
            msg = "gaussian weights must be symmetric";
            return HB_EPARAM;
          }
        d.halo = r + (s.op == HB_OP_LOG || s.op == HB_OP_HESSIAN ? 2 : 0);
        d.amount = (float)s.amount;
        if (s.op == HB_OP_HESSIAN) {
          if (s.radius < 0 || s.radius > 5) {
            msg = "hessian component index must be 0..5 (xx, yy, zz, xy, xz, yz)";
            return HB_EPARAM;
          }
          d.radius = s.radius;
        }
        d.out_dt = HB_F32;
        break;
      }
      case HB_OP_SOBEL:
      case HB_OP_PREWITT:
        d.halo = 1;
        d.out_dt = HB_F32;
        break;
      case HB_OP_THRESHOLD:
        d.threshold = s.amount;  // NaN compares false everywhere, as in NumPy
        d.out_dt = HB_U32;
        break;
      case HB_OP_LBP2D:
        d.out_dt = HB_U8;
        break;
      case HB_OP_DIFFUSION:  // filters.py:152-159 validation
        if (s.radius < 1) {
          msg = "iterations must be >= 1, got " + std::to_string(s.radius);
          return HB_EPARAM;
        }
        if (!(s.amount > 0) || s.amount > 1.0 / 6.0 + 1e-12) {
          msg = "dt must be in (0, 1/6], got " + std::to_string(s.amount);
          return HB_EPARAM;
        }
        if (!(s.sigma > 0)) {
          msg = "kappa must be positive, got " + std::to_string(s.sigma);
          return HB_EPARAM;
        }
        d.radius = s.radius;
        d.halo = s.radius;  // each explicit step widens the stencil by one slice
        d.kappa = (float)s.sigma;
        d.amount = (float)s.amount;
        d.precision = s.precision;
        d.out_dt = HB_F32;
        break;
      case HB_OP_LOCAL_THRESHOLD: {  // threshold.py:188-216 validation
        if (s.precision < HB_LT_MEAN || s.precision > HB_LT_SAUVOLA) {
          msg = "kind must be one of ('mean', 'median', 'gaussian', 'niblack', 'sauvola'), got code " +
                std::to_string(s.precision);
          return HB_EPARAM;
        }
        if (s.radius < 1) {
          msg = "window radius must be >= 1, got " + std::to_string(s.radius);
          return HB_EPARAM;
        }
        if (s.radius > local_threshold_max_radius(s.precision, dt)) {
          msg = "window radius " + std::to_string(s.radius) + " exceeds the device limit " +
                std::to_string(local_threshold_max_radius(s.precision, dt)) + " for this kind and dtype";
          return HB_EUNSUPPORTED;
        }
        double sauvola_r = s.amount;
        if (s.precision == HB_LT_SAUVOLA && std::isnan(sauvola_r))  // default_sauvola_r, threshold.py:166-171
          sauvola_r = dt == HB_U8 ? 127.5 : dt == HB_U16 ? 32767.5 : dt == HB_U32 ? 2147483647.5 : 0.5;
        if (s.precision == HB_LT_SAUVOLA && !(sauvola_r > 0)) {
          msg = "sauvola R must be positive, got " + std::to_string(sauvola_r);
          return HB_EPARAM;
        }
        d.lt.kind = s.precision;
        d.lt.w = s.radius;
        d.lt.k = s.sigma;
        d.lt.c = s.precision == HB_LT_SAUVOLA ? 0.0 : s.amount;
        d.lt.r = s.precision == HB_LT_SAUVOLA ? sauvola_r : 1.0;
        if (s.precision == HB_LT_GAUSSIAN) {
          const int n = 2 * s.radius + 1;
          d.lt_kern.resize(n);
          if (s.weights64 && s.n_weights > 0) {
            if (s.n_weights != n) {
              msg = "weights64 length must be 2*window+1";
              return HB_EPARAM;
            }
            std::memcpy(d.lt_kern.data(), s.weights64, sizeof(double) * n);
          } else {  // threshold.py:199-202 (std::exp; the Python layer passes NumPy's)
            const double sg = s.radius / 2.0;
            for (int i = 0; i < n; i++) {
              const double x = (double)(i - s.radius) / sg;
              d.lt_kern[i] = std::exp(-0.5 * (x * x));
            }
            const double sum = pairwise_sum(d.lt_kern.data(), n);
            for (int i = 0; i < n; i++) d.lt_kern[i] /= sum;
          }
        }
        d.halo = s.radius;
        d.out_dt = HB_U32;
        break;
      }
      case HB_OP_MEAN:
      case HB_OP_MEDIAN:
        if (s.radius < 1) {
          msg = "radius must be >= 1, got " + std::to_string(s.radius);
          return HB_EPARAM;
        }
        if (s.radius > 50) {
          msg = "radius too large";
          return HB_EUNSUPPORTED;
        }
        d.radius = s.radius;
        d.halo = s.radius;
        d.out_dt = s.op == HB_OP_MEAN ? HB_F32 : dt;
        break;
      case HB_OP_ERODE:
      case HB_OP_DILATE: {
        if (s.n_offsets < 1 || !s.offsets) {
          msg = "structuring element must not be empty";
          return HB_EPARAM;
        }
        bool has_origin = false;
        d.offsets.resize(3 * (size_t)s.n_offsets);
        int sgn = s.op == HB_OP_DILATE ? -1 : 1;  // dilate uses the reflected SE
        for (int k = 0; k < s.n_offsets; k++) {
          int dz = s.offsets[3 * k], dy = s.offsets[3 * k + 1], dx = s.offsets[3 * k + 2];
          if (dz == 0 && dy == 0 && dx == 0) has_origin = true;
          d.offsets[3 * k] = sgn * dz;
          d.offsets[3 * k + 1] = sgn * dy;
          d.offsets[3 * k + 2] = sgn * dx;
        }
        if (!has_origin) {
          msg = "structuring element must contain the origin";
          return HB_EPARAM;
        }
        d.halo = z_extent(d.offsets);
        d.out_dt = dt;
        break;
      }
      default:
        msg = "unknown operator code " + std::to_string(s.op);
        return HB_EPARAM;
    }
    dt = d.out_dt;
    out.push_back(std::move(d));
  }
  return HB_OK;
}

// ---------------------------------------------------------------------------
// Device memory: private pool per device, trimmed to zero after each job.
// ---------------------------------------------------------------------------
struct DeviceCtx {
  std::mutex mu;
  cudaMemPool_t pool = nullptr;
  bool init = false;
  // hb_session_begin/end nesting depth: while > 0, jobs return their buffers
  // to the pool without trimming it, so back-to-back jobs skip the driver's
  // map/unmap (measured 2-400 ms per job on the B200 box); the session's end
  // trims to zero.
  std::atomic<int> session{0};
};
DeviceCtx g_dev[64];

cudaError_t ensure_pool(int dev) {
  DeviceCtx& d = g_dev[dev];
  if (d.init) return cudaSuccess;
  cudaMemPoolProps props{};
  props.allocType = cudaMemAllocationTypePinned;
  props.location.type = cudaMemLocationTypeDevice;
  props.location.id = dev;
  cudaError_t e = cudaMemPoolCreate(&d.pool, &props);
  if (e != cudaSuccess) return e;
  uint64_t keep = UINT64_MAX;  // hold memory between async calls; jobs trim explicitly
  cudaMemPoolSetAttribute(d.pool, cudaMemPoolAttrReleaseThreshold, &keep);
  d.init = true;
  return cudaSuccess;
}

void pool_reset_peak(int dev) {
  uint64_t z = 0;
  cudaMemPoolSetAttribute(g_dev[dev].pool, cudaMemPoolAttrUsedMemHigh, &z);
  cudaMemPoolSetAttribute(g_dev[dev].pool, cudaMemPoolAttrReservedMemHigh, &z);
}
int64_t pool_attr(int dev, cudaMemPoolAttr a) {
  uint64_t v = 0;
  cudaMemPoolGetAttribute(g_dev[dev].pool, a, &v);
  return (int64_t)v;
}

struct PoolAlloc {
  cudaMemPool_t pool;
  cudaStream_t s;
  std::vector<void*> ptrs;
  cudaError_t err = cudaSuccess;
  void* get(size_t bytes) {
    if (bytes == 0) bytes = 256;
    void* p = nullptr;
    cudaError_t e = cudaMallocFromPoolAsync(&p, bytes, pool, s);
    if (e != cudaSuccess) {
      err = e;
      return nullptr;
    }
    ptrs.push_back(p);
    return p;
  }
  void release() {
    for (void* p : ptrs) cudaFreeAsync(p, s);
    ptrs.clear();
  }
};

// ---------------------------------------------------------------------------
// Chain evaluation on a device block
// ---------------------------------------------------------------------------
struct Range {
  int64_t a, b;  // [a, b) in block-local z
};

// Output range each stage must produce so that the last stage can produce
// [zo, zo+nzo): stage s covers [zo - H_s, zo + nzo + H_s) ∩ [0, nz) where H_s
// is the sum of the halos of the stages after s.
std::vector<Range> stage_ranges(const std::vector<StageDesc>& st, int64_t nz, int64_t zo,
                                int64_t nzo) {
  std::vector<Range> r(st.size());
  int64_t h = 0;
  for (int s = (int)st.size() - 1; s >= 0; --s) {
    r[s].a = std::max<int64_t>(0, zo - h);
    r[s].b = std::min<int64_t>(nz, zo + nzo + h);
    h += st[s].halo;
  }
  return r;
}

// Scratch bytes needed to evaluate the chain (excluding the final output).
bool widen_eligible(const StageDesc& d, const DevIn& in);
int64_t widened_nx(int64_t nx, int dt);

size_t chain_scratch(const std::vector<StageDesc>& st, int64_t nz, int64_t ny, int64_t nx,
                     int64_t zo, int64_t nzo) {
  auto rg = stage_ranges(st, nz, zo, nzo);
  size_t plane = (size_t)ny * nx, total = 0;
  for (size_t s = 0; s < st.size(); ++s) {
    size_t n = (size_t)(rg[s].b - rg[s].a);
    if (s + 1 < st.size()) total += n * plane * dtype_size(st[s].out_dt);  // stage output
    // per-op temporaries (generic gaussian: one f32 buffer; LoG: g + tmp)
    if (st[s].op == HB_OP_GAUSSIAN || st[s].op == HB_OP_UNSHARP || st[s].op == HB_OP_MEAN)
      total += n * plane * 4;
    if (st[s].op == HB_OP_DIFFUSION) {
      int64_t in_n = s == 0 ? nz : (rg[s - 1].b - rg[s - 1].a);
      total += 2 * (size_t)in_n * plane * 4;
    }
    {  // row-pitch widening (run_stage): widened input + output of the stage
      StageDesc tmp = st[s];
      DevIn probe{nullptr, st[s].in_dt, 1, ny, nx};
      if (tmp.op == HB_OP_LOG || tmp.op == HB_OP_HESSIAN) tmp.op = HB_OP_GAUSSIAN;  // their smoothing
      if (widen_eligible(tmp, probe)) {
        const int64_t nxp = widened_nx(nx, st[s].in_dt);
        const int64_t in_n = s == 0 ? nz : (rg[s - 1].b - rg[s - 1].a);
        // LoG / hessian widen their smoothing, which produces up to n + 4 slices
        const bool smooth = st[s].op == HB_OP_LOG || st[s].op == HB_OP_HESSIAN;
        const int64_t wn = smooth ? std::min<int64_t>(in_n, (int64_t)n + 4) : (int64_t)n;
        total += (size_t)(in_n * ny * nxp) * dtype_size(st[s].in_dt) + (size_t)(wn * ny * nxp) * 4 + 512;
        total += (size_t)(wn * ny * nxp) * 4;  // the stage's own temporaries at the wider pitch
      }
    }
    if (st[s].op == HB_OP_LOCAL_THRESHOLD)
      total += local_threshold_scratch(st[s].lt.kind, st[s].in_dt, st[s].lt.w, n, (int64_t)plane) + 256;
    if (st[s].op == HB_OP_LOG || st[s].op == HB_OP_HESSIAN) {
      int64_t in_n = s == 0 ? nz : (rg[s - 1].b - rg[s - 1].a);
      size_t gn = (size_t)std::min<int64_t>(in_n, n + 4);
      total += 2 * gn * plane * 4;
    }
  }
  return total + 4096 * st.size();
}

cudaError_t run_stage(const StageDesc& d, const DevIn& in, int64_t zo, int64_t nzo, void* out,
                      PoolAlloc& pa, cudaStream_t s, int64_t* launches);

cudaError_t run_stage_impl(const StageDesc& d, const DevIn& in, int64_t zo, int64_t nzo, void* out,
                           PoolAlloc& pa, cudaStream_t s, int64_t* launches) {
  const size_t plane = (size_t)in.ny * in.nx;
  switch (d.op) {
    case HB_OP_IDENTITY:
      return copy_slices(in, zo, nzo, out, s, launches);
    case HB_OP_GAUSSIAN:
    case HB_OP_UNSHARP: {
      EpiArgs epi;
      if (d.op == HB_OP_UNSHARP) {
        epi.kind = EPI_UNSHARP;
        epi.orig = in.p;
        epi.orig_dt = in.dt;
        epi.orig_zo = zo;
        epi.amount = d.amount;
      }
      if (d.precision == HB_PREC_FAST && epi.kind == EPI_NONE && in.dt == HB_F32 &&
          (in.nx < 384 || in.ny < 384)) {
        // small planes: split passes (gauss_small.cu) instead of z-streaming
        float* tmp = (float*)pa.get((size_t)nzo * plane * 4);
        if (tmp) {
          cudaError_t e = gaussian_small(in, zo, nzo, (float*)out, d.taps, epi, tmp, s, launches);
          if (e != cudaErrorNotSupported) return e;
        } else {
          pa.err = cudaSuccess;
        }
        cudaGetLastError();
      }
      if (d.precision == HB_PREC_FAST) {
        cudaError_t e = gaussian_fused(in, zo, nzo, (float*)out, d.taps, epi, s, launches);
        if (e != cudaErrorNotSupported) return e;
        cudaGetLastError();  // clear the NotSupported marker
      }
      float* tmp = (float*)pa.get((size_t)nzo * plane * 4);
      if (!tmp) return pa.err;
      if (d.precision == HB_PREC_EXACT) {
        cudaError_t e = gaussian_exact_fused(in, zo, nzo, (float*)out, d.taps, epi, tmp, s, launches);
        if (e != cudaErrorNotSupported) return e;
        cudaGetLastError();
      }
      return gaussian_generic(in, zo, nzo, (float*)out, d.taps,
                              d.precision == HB_PREC_EXACT, epi, tmp, s, launches);
    }
    case HB_OP_MEAN: {
      cudaError_t e = cudaErrorNotSupported;
      if (!std::getenv("HB_MEAN_TMA")) {
        e = mean_stream(in, zo, nzo, (float*)out, d.radius, s, launches);
        if (e != cudaErrorNotSupported) return e;
        cudaGetLastError();
      }
      e = mean_fused(in, zo, nzo, (float*)out, d.radius, s, launches);
      if (e != cudaErrorNotSupported) return e;
      cudaGetLastError();
      float* tmp = (float*)pa.get((size_t)nzo * plane * 4);
      if (!tmp) return pa.err;
      return mean_generic(in, zo, nzo, (float*)out, d.radius, tmp, s, launches);
    }
    case HB_OP_SOBEL:
    case HB_OP_PREWITT:
      return gradmag(in, zo, nzo, (float*)out, d.op == HB_OP_SOBEL, s, launches);
    case HB_OP_THRESHOLD:
      return threshold(in, zo, nzo, (uint32_t*)out, d.threshold, s, launches);
    case HB_OP_LBP2D:
      return lbp2d(in, zo, nzo, (uint8_t*)out, s, launches);
    case HB_OP_LOCAL_THRESHOLD: {
      LocalParams p = d.lt;
      p.kern = d.lt_kern.data();
      const size_t sb = local_threshold_scratch(p.kind, in.dt, p.w, nzo, (int64_t)plane);
      void* scr = sb ? pa.get(sb) : nullptr;
      if (sb && !scr) return pa.err;
      return local_threshold(in, zo, nzo, (uint32_t*)out, p, scr, s, launches);
    }
    case HB_OP_DIFFUSION: {
      float* b0 = (float*)pa.get((size_t)in.nz * plane * 4);
      float* b1 = (float*)pa.get((size_t)in.nz * plane * 4);
      if (!b0 || !b1) return pa.err;
      return diffusion(in, zo, nzo, (float*)out, d.radius, d.kappa, d.amount,
                       d.precision == 1, b0, b1, s, launches);
    }
    case HB_OP_LOG:
    case HB_OP_HESSIAN: {
      // smoothed g over [zo-2, zo+nzo+2) ∩ [0, nz) then the cd∘cd stage
      int64_t g0 = std::max<int64_t>(0, zo - 2), g1 = std::min<int64_t>(in.nz, zo + nzo + 2);
      float* g = (float*)pa.get((size_t)(g1 - g0) * plane * 4);
      if (!g) return pa.err;
      // the smoothing is a plain gaussian stage (same taps and precision), so
      // ragged rows get the widening of run_stage; g itself stays at nx
      StageDesc gd = d;
      gd.op = HB_OP_GAUSSIAN;
      gd.out_dt = HB_F32;
      gd.amount = 0.f;
      cudaError_t e = run_stage(gd, in, g0, g1 - g0, g, pa, s, launches);
      if (e != cudaSuccess) return e;
      if (d.op == HB_OP_HESSIAN) {
        // component index -> (a, b) axes, x = 2, y = 1, z = 0 (filters.py:228-231)
        static const int ax[6][2] = {{2, 2}, {1, 1}, {0, 0}, {2, 1}, {2, 0}, {1, 0}};
        return hessian_stage(g, g0, in.nz, in.ny, in.nx, zo, nzo, ax[d.radius][0],
                             ax[d.radius][1], (float*)out, s, launches);
      }
      return log_diff(g, g0, g1 - g0, in.nz, in.ny, in.nx, zo, nzo, (float*)out, s, launches);
    }
    case HB_OP_MEDIAN:
      return median(in, zo, nzo, out, d.radius, s, launches);
    case HB_OP_ERODE:
    case HB_OP_DILATE:
    {
      // the u8 binary/grey gate word comes from the job's pool (a per-call
      // stream-ordered allocation measured noisy: +/-30% on 2 ms launches)
      int* gate = in.dt == HB_U8 ? (int*)pa.get(256) : nullptr;
      if (in.dt == HB_U8 && !gate) {  // no room: morph() allocates its own word
        pa.err = cudaSuccess;
        cudaGetLastError();
      }
      return morph(in, zo, nzo, out, d.offsets.data(), (int)(d.offsets.size() / 3),
                   d.op == HB_OP_DILATE, s, launches, gate);
    }
  }
  return cudaErrorInvalidValue;
}

// Evaluate the chain on block `in`, writing [zo, zo+nzo) into `out`.
// Row pitch widening.  The TMA / vector kernels need 16-byte rows; a volume
// whose x extent is not a multiple of 16 / itemsize would fall to the generic
// per-pass kernels (10-40x slower).  For the single-window operators (each
// output depends on its clamped input window only: gaussian, unsharp, mean,
// erode, dilate) replicating the last column out to the aligned width gives
// exactly the clamp-to-edge values, so the stage runs on the widened block
// and its first nx columns are the result, bit for bit.
template <typename E>
__global__ void k_widen_rows(const E* __restrict__ src, E* __restrict__ dst, int64_t rows, int nx, int nxp) {
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    const E* a = src + r * nx;
    E* b = dst + r * nxp;
    for (int x = threadIdx.x; x < nxp; x += blockDim.x) b[x] = a[x < nx ? x : nx - 1];
  }
}

bool widen_eligible(const StageDesc& d, const DevIn& in) {
  const bool op = d.op == HB_OP_GAUSSIAN || d.op == HB_OP_UNSHARP || d.op == HB_OP_MEAN ||
                  d.op == HB_OP_ERODE || d.op == HB_OP_DILATE;
  const int64_t al = 16 / dtype_size(in.dt);
  return op && in.nx % al != 0 && in.nx > 1 && !std::getenv("HB_NO_WIDEN");
}

int64_t widened_nx(int64_t nx, int dt) {
  const int64_t al = 16 / dtype_size(dt);
  return (nx + al - 1) / al * al;
}

cudaError_t run_stage(const StageDesc& d, const DevIn& in, int64_t zo, int64_t nzo, void* out,
                      PoolAlloc& pa, cudaStream_t s, int64_t* launches) {
  if (!widen_eligible(d, in)) return run_stage_impl(d, in, zo, nzo, out, pa, s, launches);
  const int64_t nxp = widened_nx(in.nx, in.dt);
  const size_t ies = dtype_size(in.dt), oes = dtype_size(d.out_dt);
  // widen only the slices the stage reads: [zo - halo, zo + nzo + halo) clipped
  // to the block (faces inside the block are never reached by a clamp, so the
  // sub-block evaluates exactly as the whole block does)
  const int64_t za = std::max<int64_t>(0, zo - d.halo);
  const int64_t zb = std::min<int64_t>(in.nz, zo + nzo + d.halo);
  void* wi = pa.get((size_t)((zb - za) * in.ny * nxp) * ies);
  void* wo = wi ? pa.get((size_t)(nzo * in.ny * nxp) * oes) : nullptr;
  if (!wi || !wo) {
    // no room for the widened copies (e.g. hb_apply_device on a device-resident
    // volume without a budget): the generic kernels run on the block as is
    if (wi) {
      cudaFreeAsync(wi, s);
      pa.ptrs.pop_back();
    }
    pa.err = cudaSuccess;
    cudaGetLastError();
    return run_stage_impl(d, in, zo, nzo, out, pa, s, launches);
  }
  const int64_t rows = (zb - za) * in.ny;
  const size_t off = (size_t)(za * in.ny * in.nx) * ies;
  const void* src = static_cast<const char*>(in.p) + off;
  const int g = (int)std::min<int64_t>(rows, (int64_t)kNumSMs * 32);
  switch (ies) {
    case 1: k_widen_rows<uint8_t><<<g, 128, 0, s>>>((const uint8_t*)src, (uint8_t*)wi, rows, (int)in.nx, (int)nxp); break;
    case 2: k_widen_rows<uint16_t><<<g, 128, 0, s>>>((const uint16_t*)src, (uint16_t*)wi, rows, (int)in.nx, (int)nxp); break;
    default: k_widen_rows<uint32_t><<<g, 128, 0, s>>>((const uint32_t*)src, (uint32_t*)wi, rows, (int)in.nx, (int)nxp); break;
  }
  if (launches) *launches += 1;
  DevIn win{wi, in.dt, zb - za, in.ny, nxp};
  cudaError_t e = run_stage_impl(d, win, zo - za, nzo, wo, pa, s, launches);
  if (e != cudaSuccess) return e;
  return cudaMemcpy2DAsync(out, (size_t)in.nx * oes, wo, (size_t)nxp * oes, (size_t)in.nx * oes,
                           (size_t)(nzo * in.ny), cudaMemcpyDeviceToDevice, s);
}

cudaError_t run_chain(const std::vector<StageDesc>& st, const DevIn& in, int64_t zo,
                      int64_t nzo, void* out, PoolAlloc& pa, cudaStream_t s,
                      int64_t* launches) {
  auto rg = stage_ranges(st, in.nz, zo, nzo);
  DevIn cur = in;
  int64_t cur_a = 0;  // block-local z of cur's slice 0
  const size_t plane = (size_t)in.ny * in.nx;
  for (size_t k = 0; k < st.size(); ++k) {
    const bool last = k + 1 == st.size();
    void* dst;
    if (last) {
      dst = out;
    } else {
      dst = pa.get((size_t)(rg[k].b - rg[k].a) * plane * dtype_size(st[k].out_dt));
      if (!dst) return pa.err;
    }
    // in cur-local coordinates
    int64_t lzo = rg[k].a - cur_a;
    cudaError_t e = run_stage(st[k], cur, lzo, rg[k].b - rg[k].a, dst, pa, s, launches);
    if (e != cudaSuccess) return e;
    if (!last) {
      cur.p = dst;
      cur.dt = st[k].out_dt;
      cur.nz = rg[k].b - rg[k].a;
      cur_a = rg[k].a;
    }
  }
  return cudaSuccess;
}

// ---------------------------------------------------------------------------
// Host staging: parallel memcpy + cached pinned bounce ring
// ---------------------------------------------------------------------------
void par_memcpy(void* dst, const void* src, size_t bytes, int threads) {
  if (bytes < (8u << 20) || threads <= 1) {
    std::memcpy(dst, src, bytes);
    return;
  }
  std::vector<std::thread> th;
  size_t per = (bytes + threads - 1) / threads;
  per = (per + 4095) & ~(size_t)4095;
  for (int t = 0; t < threads; t++) {
    size_t o = (size_t)t * per;
    if (o >= bytes) break;
    size_t n = std::min(per, bytes - o);
    th.emplace_back([=] { std::memcpy((char*)dst + o, (const char*)src + o, n); });
  }
  for (auto& t : th) t.join();
}

struct PinnedRing {
  static constexpr int kSlots = 4;
  static constexpr size_t kPiece = 64u << 20;
  void* buf[kSlots] = {};
  cudaEvent_t ev[kSlots] = {};
  bool used[kSlots] = {};
  int next = 0;
  bool ok = false;
  cudaError_t init() {
    if (ok) return cudaSuccess;
    for (int i = 0; i < kSlots; i++) {
      cudaError_t e = cudaMallocHost(&buf[i], kPiece);
      if (e != cudaSuccess) return e;
      cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming);
    }
    ok = true;
    return cudaSuccess;
  }
};
PinnedRing g_ring[64];

bool is_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// H2D of `bytes` from pageable host memory through the pinned ring.
cudaError_t h2d_staged(PinnedRing& ring, void* dst, const void* src, size_t bytes,
                       cudaStream_t s, int threads) {
  size_t off = 0;
  while (off < bytes) {
    int i = ring.next;
    ring.next = (ring.next + 1) % PinnedRing::kSlots;
    if (ring.used[i]) cudaEventSynchronize(ring.ev[i]);
    size_t n = std::min(PinnedRing::kPiece, bytes - off);
    par_memcpy(ring.buf[i], (const char*)src + off, n, threads);
    cudaError_t e = cudaMemcpyAsync((char*)dst + off, ring.buf[i], n, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return e;
    cudaEventRecord(ring.ev[i], s);
    ring.used[i] = true;
    off += n;
  }
  return cudaSuccess;
}

// D2H into pageable host memory through the pinned ring (synchronous for the
// host thread; `s` must already be ordered after the producing work).
cudaError_t d2h_staged(PinnedRing& ring, void* dst, const void* src, size_t bytes,
                       cudaStream_t s, int threads) {
  struct Pending { int slot; size_t off, n; };
  std::vector<Pending> q;
  size_t off = 0;
  auto drain_one = [&]() {
    Pending p = q.front();
    q.erase(q.begin());
    cudaEventSynchronize(ring.ev[p.slot]);
    par_memcpy((char*)dst + p.off, ring.buf[p.slot], p.n, threads);
    ring.used[p.slot] = false;
  };
  while (off < bytes) {
    if ((int)q.size() >= PinnedRing::kSlots - 1) drain_one();
    int i = ring.next;
    ring.next = (ring.next + 1) % PinnedRing::kSlots;
    if (ring.used[i]) cudaEventSynchronize(ring.ev[i]);
    size_t n = std::min(PinnedRing::kPiece, bytes - off);
    cudaError_t e = cudaMemcpyAsync(ring.buf[i], (const char*)src + off, n, cudaMemcpyDeviceToHost, s);
    if (e != cudaSuccess) return e;
    cudaEventRecord(ring.ev[i], s);
    ring.used[i] = true;
    q.push_back({i, off, n});
    off += n;
  }
  while (!q.empty()) drain_one();
  return cudaSuccess;
}

int auto_threads(int req) {
  if (req > 0) return req;
  unsigned n = std::thread::hardware_concurrency();  // measured best: all cores, <= 16
  return (int)std::max(1u, std::min(16u, n ? n : 1u));
}

// Whole-volume copies of the global operators: direct DMA for pinned host
// memory, the pinned ring with parallel staging for pageable memory (a plain
// cudaMemcpy from pageable memory ran at a few GB/s: 90% of an EDT's time).
cudaError_t h2d_any(int dev, void* dst, const void* src, size_t bytes, cudaStream_t s) {
  if (is_pinned(src)) return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s);
  PinnedRing& ring = g_ring[dev];
  cudaError_t e = ring.init();
  return e != cudaSuccess ? e : h2d_staged(ring, dst, src, bytes, s, auto_threads(0));
}
// returns after the data is in `dst` when it is pageable; `s` must be ordered
// after the producing work
cudaError_t d2h_any(int dev, void* dst, const void* src, size_t bytes, cudaStream_t s) {
  if (is_pinned(dst)) return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s);
  PinnedRing& ring = g_ring[dev];
  cudaError_t e = ring.init();
  return e != cudaSuccess ? e : d2h_staged(ring, dst, src, bytes, s, auto_threads(0));
}

double now_ms() {
  return std::chrono::duration<double, std::milli>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================
// ---------------------------------------------------------------------------
// Two-pass global operators, pass 1 (chunking.py:282-306 chunked_reduce): the
// volume streams through the device in bounded slabs (host volumes: pinned
// DMA or the pinned ring) and `fn(device_ptr, n_voxels, stream)` folds each.
// ---------------------------------------------------------------------------
namespace {
template <typename F>
int32_t for_each_slab(const hb_volume* in, int32_t dev, F&& fn) {
  if (!in || !in->data || in->nz < 0 || in->ny < 0 || in->nx < 0) {
    set_err(nullptr, "bad volume");
    return HB_EPARAM;
  }
  if (dev < 0 || dev >= hb_device_count()) {
    set_err(nullptr, "no CUDA device " + std::to_string(dev));
    return HB_EBUDGET_UNAVAILABLE;
  }
  std::lock_guard<std::mutex> lk(g_dev[dev].mu);
  cudaSetDevice(dev);
  cudaError_t e = ensure_pool(dev);
  if (e != cudaSuccess) {
    set_err(nullptr, cudaGetErrorString(e));
    return HB_ECUDA;
  }
  const int64_t es = dtype_size(in->dtype);
  const int64_t total = in->nz * in->ny * in->nx;
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  PoolAlloc pa{g_dev[dev].pool, s};
  if (in->location == HB_DEVICE) {
    e = fn(in->data, total, s);
  } else {
    const int64_t slab = std::max<int64_t>(1, (256ll << 20) / es);
    void* buf = pa.get((size_t)std::min(total, slab) * es);
    if (!buf) {
      e = pa.err;
    } else {
      const bool pinned_in = is_pinned(in->data);
      PinnedRing& ring = g_ring[dev];
      if (!pinned_in) e = ring.init();
      for (int64_t off = 0; off < total && e == cudaSuccess; off += slab) {
        const int64_t n = std::min(slab, total - off);
        const char* src = (const char*)in->data + off * es;
        e = pinned_in ? cudaMemcpyAsync(buf, src, (size_t)(n * es), cudaMemcpyHostToDevice, s)
                      : h2d_staged(ring, buf, src, (size_t)(n * es), s, auto_threads(0));
        if (e == cudaSuccess) e = fn(buf, n, s);
        // the single buffer is reused: the next copy is ordered after this
        // fold on the same stream
      }
    }
  }
  cudaError_t se = cudaStreamSynchronize(s);
  if (e == cudaSuccess) e = se;
  pa.release();
  cudaStreamSynchronize(s);
  cudaStreamDestroy(s);
  if (g_dev[dev].session.load() == 0) cudaMemPoolTrimTo(g_dev[dev].pool, 0);
  if (e != cudaSuccess) {
    set_err(nullptr, cudaGetErrorString(e));
    cudaGetLastError();
    return HB_ECUDA;
  }
  return HB_OK;
}
}  // namespace

// ---------------------------------------------------------------------------
// Chunked connected components (quantify.py:73-111): volumes beyond one
// device pass are labelled z-chunk by z-chunk.  Pass 1 labels each chunk on
// the device (roots numbered in scan order -> "candidates", globally ordered
// by chunk then rank) and unions candidates that touch across each chunk
// boundary (the reference's boundary union-find, smaller candidate wins);
// the final ids number the surviving candidates in order, which is the
// global first-voxel order.  Pass 2 relabels each chunk through the table.
// ---------------------------------------------------------------------------
namespace {
int64_t dsu_find(std::vector<int64_t>& p, int64_t x) {
  while (p[x] != x) {
    p[x] = p[p[x]];
    x = p[x];
  }
  return x;
}

int32_t cc_chunked(const hb_volume* in, hb_volume* out, int conn, int dev, int64_t cs, int64_t* count) {
  const int64_t nz = in->nz, ny = in->ny, nx = in->nx, plane = ny * nx;
  const size_t es = (size_t)dtype_size(in->dtype);
  const int64_t nchunks = (nz + cs - 1) / cs;
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  PoolAlloc pa{g_dev[dev].pool, s};
  const size_t cn = (size_t)(cs * plane);
  const size_t scan_bytes = connected_components_scan_bytes((int64_t)cn) + 256;
  void* d_in = pa.get(cn * es);
  int* lab = (int*)pa.get(cn * 4);
  int* root = (int*)pa.get(cn * 4);
  int* flag = (int*)pa.get(cn * 4);
  int* ids = (int*)pa.get(cn * 4);
  int* rank = (int*)pa.get(cn * 4);
  void* tmp = pa.get(scan_bytes);
  uint32_t* table = (uint32_t*)pa.get(cn * 4);
  uint32_t* d_out = (uint32_t*)pa.get(cn * 4);
  cudaError_t e = (!d_in || !lab || !root || !flag || !ids || !rank || !tmp || !table || !d_out)
                      ? (pa.err != cudaSuccess ? pa.err : cudaErrorMemoryAllocation)
                      : cudaSuccess;
  std::vector<int64_t> offs(nchunks + 1, 0), parent;
  std::vector<int> prev_last((size_t)plane), first((size_t)plane), last((size_t)plane);
  auto load_chunk = [&](int64_t c, int64_t& cz) -> cudaError_t {
    const int64_t z0 = c * cs;
    cz = std::min(cs, nz - z0);
    const size_t bytes = (size_t)(cz * plane) * es;
    const char* src = (const char*)in->data + (size_t)(z0 * plane) * es;
    return in->location == HB_DEVICE ? cudaMemcpyAsync(d_in, src, bytes, cudaMemcpyDeviceToDevice, s)
                                     : h2d_any(dev, d_in, src, bytes, s);
  };
  // pass 1: per-chunk candidates + boundary unions
  for (int64_t c = 0; c < nchunks && e == cudaSuccess; ++c) {
    int64_t cz = 0, nr = 0;
    e = load_chunk(c, cz);
    if (e == cudaSuccess)
      e = cc_chunk_ranks(d_in, in->dtype, (int)cz, (int)ny, (int)nx, conn, lab, root, flag, ids, tmp,
                         scan_bytes, rank, &nr, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(first.data(), rank, (size_t)plane * 4, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(last.data(), rank + (cz - 1) * plane, (size_t)plane * 4, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) break;
    offs[c + 1] = offs[c] + nr;
    parent.resize((size_t)offs[c + 1]);
    for (int64_t k = offs[c]; k < offs[c + 1]; ++k) parent[(size_t)k] = k;
    if (c > 0) {
      for (int64_t y = 0; y < ny; ++y)
        for (int64_t x = 0; x < nx; ++x) {
          const int b = first[(size_t)(y * nx + x)];
          if (b < 0) continue;
          for (int dy = -1; dy <= 1; ++dy)
            for (int dx = -1; dx <= 1; ++dx) {
              if (conn == 6 && (dy != 0 || dx != 0)) continue;
              const int64_t yy = y + dy, xx = x + dx;
              if (yy < 0 || yy >= ny || xx < 0 || xx >= nx) continue;
              const int a = prev_last[(size_t)(yy * nx + xx)];
              if (a < 0) continue;
              int64_t ra = dsu_find(parent, offs[c - 1] + a), rb = dsu_find(parent, offs[c] + b);
              if (ra == rb) continue;
              if (ra < rb) parent[(size_t)rb] = ra;
              else parent[(size_t)ra] = rb;
            }
        }
    }
    prev_last.swap(last);
  }
  // final ids in candidate order (= first-voxel scan order); roots precede members
  std::vector<uint32_t> fin(parent.size());
  int64_t cnt = 0;
  for (size_t k = 0; e == cudaSuccess && k < parent.size(); ++k) {
    const int64_t r = dsu_find(parent, (int64_t)k);
    fin[k] = r == (int64_t)k ? (uint32_t)(++cnt) : fin[(size_t)r];
  }
  // pass 2: relabel every chunk through its slice of the table
  for (int64_t c = 0; c < nchunks && e == cudaSuccess; ++c) {
    int64_t cz = 0, nr = 0;
    e = load_chunk(c, cz);
    if (e == cudaSuccess)
      e = cc_chunk_ranks(d_in, in->dtype, (int)cz, (int)ny, (int)nx, conn, lab, root, flag, ids, tmp,
                         scan_bytes, rank, &nr, s);
    if (e == cudaSuccess && nr > 0)
      e = cudaMemcpyAsync(table, fin.data() + offs[c], (size_t)nr * 4, cudaMemcpyHostToDevice, s);
    uint32_t* dst = out->location == HB_DEVICE ? (uint32_t*)out->data + c * cs * plane : d_out;
    if (e == cudaSuccess) e = cc_apply_table(rank, (int)(cz * plane), table, dst, s);
    if (e == cudaSuccess && out->location != HB_DEVICE)
      e = d2h_any(dev, (uint32_t*)out->data + c * cs * plane, d_out, (size_t)(cz * plane) * 4, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);  // the host table slice / d_out are reused
  }
  cudaStreamSynchronize(s);
  pa.release();
  cudaStreamSynchronize(s);
  cudaStreamDestroy(s);
  if (g_dev[dev].session.load() == 0) cudaMemPoolTrimTo(g_dev[dev].pool, 0);
  if (e != cudaSuccess) {
    set_err(nullptr, std::string("connected components (chunked): ") + cudaGetErrorString(e));
    cudaGetLastError();
    return e == cudaErrorMemoryAllocation ? HB_EBUDGET_UNAVAILABLE : HB_ECUDA;
  }
  if (count) *count = cnt;
  return HB_OK;
}
}  // namespace

extern "C" {

int32_t hb_abi_version(void) { return HB_ABI_VERSION; }

const char* hb_version(void) { return "harpia-b200 0.1.0 (sm_100a)"; }

const char* hb_last_error(void) { return g_last_error.c_str(); }

int32_t hb_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int32_t hb_plan(int64_t nz, int64_t ny, int64_t nx, int32_t itemsize, int64_t halo,
                double scratch_factor, int64_t usable_bytes, hb_chunk* chunks, int64_t capacity,
                int64_t* nchunks, int64_t* minimum_bytes) {
  if (nz < 0 || ny < 0 || nx < 0 || itemsize <= 0 || halo < 0 || !(scratch_factor > 0) ||
      usable_bytes < 0 || !nchunks) {
    set_err(nullptr, "hb_plan: bad arguments");
    return HB_EPARAM;
  }
  const double slice_bytes = (double)(ny * nx * (int64_t)itemsize);
  const double denom = scratch_factor * slice_bytes;
  // Python's float floor division: the floor of the exact quotient
  int64_t t = denom > 0 ? (int64_t)std::floor((double)usable_bytes / denom) : INT64_MAX / 4;
  if (denom > 0) {  // the quotient is within one step of the floor; bounded fix-ups
    for (int i = 0; i < 4 && (double)(t + 1) * denom <= (double)usable_bytes; ++i) ++t;
    for (int i = 0; i < 4 && t > 0 && (double)t * denom > (double)usable_bytes; ++i) --t;
  }
  if (t <= 2 * halo) {
    const int64_t minimum = (int64_t)std::ceil((double)(2 * halo + 1) * scratch_factor * slice_bytes);
    if (minimum_bytes) *minimum_bytes = minimum;
    set_err(nullptr, "budget of " + std::to_string(usable_bytes) + " usable bytes holds only " +
                         std::to_string(t) + " padded slices but the operator needs more than " +
                         std::to_string(2 * halo) + "; minimum usable budget is " +
                         std::to_string(minimum) + " bytes");
    return HB_EBUDGET_SMALL;
  }
  const int64_t n = std::max<int64_t>(t - 2 * halo, 1);
  const int64_t count = (nz + n - 1) / n;
  *nchunks = count;
  if (chunks && capacity >= count) {
    for (int64_t k = 0; k < count; ++k) {
      const int64_t z0 = k * n, z1 = std::min(z0 + n, nz);
      chunks[k] = hb_chunk{z0, z1, std::min(halo, z0), std::min(halo, nz - z1)};
    }
  }
  return HB_OK;
}

int32_t hb_device_info(int32_t dev, int64_t* free_bytes, int64_t* total_bytes) {
  int n = hb_device_count();
  if (dev < 0 || dev >= n) {
    set_err(nullptr, "no CUDA device " + std::to_string(dev));
    return HB_EBUDGET_UNAVAILABLE;
  }
  cudaSetDevice(dev);
  size_t f = 0, t = 0;
  cudaError_t e = cudaMemGetInfo(&f, &t);
  if (e != cudaSuccess) {
    set_err(nullptr, cudaGetErrorString(e));
    return HB_EBUDGET_UNAVAILABLE;
  }
  if (free_bytes) *free_bytes = (int64_t)f;
  if (total_bytes) *total_bytes = (int64_t)t;
  return HB_OK;
}

int32_t hb_gaussian_radius(double sigma) { return gaussian_radius(sigma); }

int32_t hb_gaussian_weights(double sigma, float* out, int32_t capacity) {
  if (!(sigma > 0)) return -1;
  return fill_weights(sigma, out, capacity);
}

int64_t hb_chain_halo(const hb_stage* stages, int32_t nstages) {
  std::vector<StageDesc> st;
  std::string msg;
  if (normalise(stages, nstages, HB_F32, st, msg) != HB_OK) return -1;
  int64_t h = 0;
  for (auto& d : st) h += d.halo;
  return h;
}

int32_t hb_chain_out_dtype(const hb_stage* stages, int32_t nstages, int32_t in_dtype) {
  std::vector<StageDesc> st;
  std::string msg;
  if (in_dtype < HB_U8 || in_dtype > HB_F32) return -1;
  if (normalise(stages, nstages, in_dtype, st, msg) != HB_OK) return -1;
  return st.back().out_dt;
}

int32_t hb_pin(void* ptr, int64_t bytes) {
  cudaError_t e = cudaHostRegister(ptr, (size_t)bytes, cudaHostRegisterDefault);
  if (e != cudaSuccess) {
    set_err(nullptr, cudaGetErrorString(e));
    cudaGetLastError();
    return HB_ECUDA;
  }
  return HB_OK;
}

int32_t hb_unpin(void* ptr) {
  cudaError_t e = cudaHostUnregister(ptr);
  if (e != cudaSuccess) {
    set_err(nullptr, cudaGetErrorString(e));
    cudaGetLastError();
    return HB_ECUDA;
  }
  return HB_OK;
}

int32_t hb_trim_device(int32_t dev) {
  if (dev < 0 || dev >= hb_device_count()) return HB_EPARAM;
  std::lock_guard<std::mutex> lk(g_dev[dev].mu);
  if (!g_dev[dev].init) return HB_OK;
  cudaSetDevice(dev);
  cudaDeviceSynchronize();
  cudaMemPoolTrimTo(g_dev[dev].pool, 0);
  return HB_OK;
}

int32_t hb_session_begin(int32_t dev) {
  if (dev < 0 || dev >= hb_device_count()) return HB_EPARAM;
  g_dev[dev].session.fetch_add(1);
  return HB_OK;
}

int32_t hb_session_end(int32_t dev) {
  if (dev < 0 || dev >= hb_device_count()) return HB_EPARAM;
  if (g_dev[dev].session.fetch_sub(1) <= 1) {
    g_dev[dev].session.store(0);
    return hb_trim_device(dev);
  }
  return HB_OK;
}

int32_t hb_minmax(const hb_volume* in, int32_t device, double* lo, double* hi) {
  if (!in || in->dtype != HB_F32) {
    set_err(nullptr, "hb_minmax: float32 volumes only (integer ranges are the dtype range)");
    return HB_EUNSUPPORTED;
  }
  unsigned* acc = nullptr;
  unsigned host[3] = {0xffffffffu, 0u, 0u};
  int32_t rc = for_each_slab(in, device, [&](const void* p, int64_t n, cudaStream_t s) {
    if (!acc) {
      cudaError_t e = cudaMallocAsync(&acc, sizeof(host), s);
      if (e != cudaSuccess) return e;
      cudaMemcpyAsync(acc, host, sizeof(host), cudaMemcpyHostToDevice, s);
    }
    cudaError_t e = minmax_f32((const float*)p, n, acc, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(host, acc, sizeof(host), cudaMemcpyDeviceToHost, s);
    return e;
  });
  if (acc) cudaFree(acc);
  if (rc != HB_OK) return rc;
  if (host[2] || host[0] > host[1]) {
    set_err(nullptr, "autodetected histogram range is not finite (NaN or empty volume)");
    return HB_EPARAM;
  }
  auto unkey = [](unsigned k) {
    const unsigned u = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
    float f;
    std::memcpy(&f, &u, 4);
    return (double)f;
  };
  if (lo) *lo = unkey(host[0]);
  if (hi) *hi = unkey(host[1]);
  return HB_OK;
}

int32_t hb_connected_components(const hb_volume* in, hb_volume* out, int32_t connectivity,
                                int32_t device, int64_t* count) {
  if (!in || !out || !in->data || !out->data || out->dtype != HB_U32 || in->nz != out->nz ||
      in->ny != out->ny || in->nx != out->nx) {
    set_err(nullptr, "hb_connected_components: uint32 output of the input's shape required");
    return HB_EPARAM;
  }
  if (connectivity != 6 && connectivity != 26) {
    set_err(nullptr, "connectivity must be 6 or 26, got " + std::to_string(connectivity));
    return HB_EPARAM;
  }
  if (device < 0 || device >= hb_device_count()) {
    set_err(nullptr, "no CUDA device " + std::to_string(device));
    return HB_EBUDGET_UNAVAILABLE;
  }
  const int64_t n = in->nz * in->ny * in->nx;
  std::lock_guard<std::mutex> lk(g_dev[device].mu);
  cudaSetDevice(device);
  cudaError_t e = ensure_pool(device);
  if (e != cudaSuccess) {
    set_err(nullptr, cudaGetErrorString(e));
    return HB_ECUDA;
  }
  {
    // one device pass when the volume fits (int32 indices, ~22 B/voxel of
    // scratch); otherwise z-chunks with the boundary union-find.
    // HB_CC_CHUNK_SLICES forces a chunk height (tests).
    const int64_t plane = std::max<int64_t>(1, in->ny * in->nx);
    const size_t es = (size_t)dtype_size(in->dtype);
    size_t fr = 0, tot = 0;
    cudaMemGetInfo(&fr, &tot);
    const double per_voxel = 22.0 + (double)es;
    int64_t cs = 0;
    if (const char* env = std::getenv("HB_CC_CHUNK_SLICES")) cs = std::atoll(env);
    if (cs <= 0 && (n >= (1ll << 31) - 1 || (double)n * per_voxel > 0.8 * (double)fr)) {
      const int64_t by_index = ((1ll << 31) - 2) / plane;
      const int64_t by_mem = (int64_t)(0.6 * (double)fr / (per_voxel * (double)plane));
      cs = std::max<int64_t>(1, std::min(by_index, by_mem));
    }
    if (cs > 0 && cs < in->nz) {
      if (cs * plane >= (1ll << 31) - 1) {
        set_err(nullptr, "connected components: one slice exceeds 2^31 voxels");
        return HB_EUNSUPPORTED;
      }
      return cc_chunked(in, out, connectivity, device, cs, count);
    }
  }
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  PoolAlloc pa{g_dev[device].pool, s};
  const size_t es = (size_t)dtype_size(in->dtype), nn = (size_t)std::max<int64_t>(n, 1);
  const size_t scan_bytes = connected_components_scan_bytes(n) + 256;
  const void* d_in = in->data;
  uint32_t* d_out = (uint32_t*)out->data;
  int* lab = (int*)pa.get(nn * 4);
  int* flag = (int*)pa.get(nn * 4);
  int* ids = (int*)pa.get(nn * 4);
  void* tmp = pa.get(scan_bytes);
  if (in->location != HB_DEVICE && lab) {
    void* buf = pa.get(nn * es);
    if (buf) {
      e = h2d_any(device, buf, in->data, (size_t)n * es, s);
      d_in = buf;
    }
  }
  if (out->location != HB_DEVICE && lab) d_out = (uint32_t*)pa.get(nn * 4);
  if (!lab || !flag || !ids || !tmp || !d_out || pa.err != cudaSuccess) e = pa.err != cudaSuccess ? pa.err : cudaErrorMemoryAllocation;
  int64_t cnt = 0;
  if (e == cudaSuccess)
    e = connected_components(d_in, in->dtype, in->nz, in->ny, in->nx, connectivity, d_out, lab,
                             flag, ids, tmp, scan_bytes, &cnt, s);
  if (e == cudaSuccess && out->location != HB_DEVICE)
    e = d2h_any(device, out->data, d_out, (size_t)n * 4, s);
  cudaError_t se = cudaStreamSynchronize(s);
  if (e == cudaSuccess) e = se;
  pa.release();
  cudaStreamSynchronize(s);
  cudaStreamDestroy(s);
  if (g_dev[device].session.load() == 0) cudaMemPoolTrimTo(g_dev[device].pool, 0);
  if (e != cudaSuccess) {
    set_err(nullptr, std::string("connected components: ") + cudaGetErrorString(e));
    cudaGetLastError();
    return e == cudaErrorMemoryAllocation ? HB_EBUDGET_UNAVAILABLE : HB_ECUDA;
  }
  if (count) *count = cnt;
  return HB_OK;
}

int32_t hb_label_filter(const hb_volume* in, hb_volume* out, int32_t op, int32_t connectivity,
                        int64_t min_size, int32_t device) {
  if (!in || !out || !in->data || !out->data || out->dtype != in->dtype || in->nz != out->nz ||
      in->ny != out->ny || in->nx != out->nx || (op != 0 && op != 1)) {
    set_err(nullptr, "hb_label_filter: op 0/1 and an output of the input's dtype and shape");
    return HB_EPARAM;
  }
  if (connectivity != 6 && connectivity != 26) {
    set_err(nullptr, "connectivity must be 6 or 26, got " + std::to_string(connectivity));
    return HB_EPARAM;
  }
  if (op == 1 && min_size < 1) {
    set_err(nullptr, "min_size must be >= 1, got " + std::to_string(min_size));
    return HB_EPARAM;
  }
  if (device < 0 || device >= hb_device_count()) {
    set_err(nullptr, "no CUDA device " + std::to_string(device));
    return HB_EBUDGET_UNAVAILABLE;
  }
  const int64_t n = in->nz * in->ny * in->nx;
  if (n >= (1ll << 31) - 1) {
    set_err(nullptr, "label filters: volumes of 2^31 voxels or more are not supported");
    return HB_EUNSUPPORTED;
  }
  std::lock_guard<std::mutex> lk(g_dev[device].mu);
  cudaSetDevice(device);
  cudaError_t e = ensure_pool(device);
  if (e != cudaSuccess) {
    set_err(nullptr, cudaGetErrorString(e));
    return HB_ECUDA;
  }
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  PoolAlloc pa{g_dev[device].pool, s};
  const size_t es = (size_t)dtype_size(in->dtype), nn = (size_t)std::max<int64_t>(n, 1);
  int* lab = (int*)pa.get(nn * 4);
  int* root = (int*)pa.get(nn * 4);
  int* aux = (int*)pa.get(nn * 4);
  const void* d_in = in->data;
  void* d_out = out->data;
  if (in->location != HB_DEVICE && aux) {
    void* buf = pa.get(nn * es);
    if (buf) {
      e = h2d_any(device, buf, in->data, (size_t)n * es, s);
      d_in = buf;
    }
  }
  if (out->location != HB_DEVICE && aux) d_out = pa.get(nn * es);
  if (!lab || !root || !aux || !d_out || pa.err != cudaSuccess)
    e = pa.err != cudaSuccess ? pa.err : cudaErrorMemoryAllocation;
  if (e == cudaSuccess)
    e = label_filter(d_in, in->dtype, in->nz, in->ny, in->nx, connectivity, op, min_size, d_out,
                     lab, root, aux, s);
  if (e == cudaSuccess && out->location != HB_DEVICE)
    e = d2h_any(device, out->data, d_out, (size_t)n * es, s);
  cudaError_t se = cudaStreamSynchronize(s);
  if (e == cudaSuccess) e = se;
  pa.release();
  cudaStreamSynchronize(s);
  cudaStreamDestroy(s);
  if (g_dev[device].session.load() == 0) cudaMemPoolTrimTo(g_dev[device].pool, 0);
  if (e != cudaSuccess) {
    set_err(nullptr, std::string("label filter: ") + cudaGetErrorString(e));
    cudaGetLastError();
    return e == cudaErrorMemoryAllocation ? HB_EBUDGET_UNAVAILABLE : HB_ECUDA;
  }
  return HB_OK;
}

int32_t hb_geodesic(const hb_volume* marker, const hb_volume* mask, hb_volume* out,
                    int32_t dilation, int32_t device, int64_t* sweeps) {
  if (!marker || !mask || !out || !marker->data || !mask->data || !out->data ||
      marker->dtype != mask->dtype || out->dtype != mask->dtype || marker->nz != mask->nz ||
      marker->ny != mask->ny || marker->nx != mask->nx || out->nz != mask->nz ||
      out->ny != mask->ny || out->nx != mask->nx) {
    set_err(nullptr, "hb_geodesic: marker, mask and out must share dtype and shape");
    return HB_EPARAM;
  }
  if (device < 0 || device >= hb_device_count()) {
    set_err(nullptr, "no CUDA device " + std::to_string(device));
    return HB_EBUDGET_UNAVAILABLE;
  }
  std::lock_guard<std::mutex> lk(g_dev[device].mu);
  cudaSetDevice(device);
  cudaError_t e = ensure_pool(device);
  if (e != cudaSuccess) {
    set_err(nullptr, cudaGetErrorString(e));
    return HB_ECUDA;
  }
  const int64_t n = mask->nz * mask->ny * mask->nx;
  const size_t es = (size_t)dtype_size(mask->dtype), nn = (size_t)std::max<int64_t>(n, 1);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  PoolAlloc pa{g_dev[device].pool, s};
  int* flags = (int*)pa.get(64);
  auto dev_copy = [&](const hb_volume* v) -> const void* {
    if (v->location == HB_DEVICE) return v->data;
    void* b = pa.get(nn * es);
    if (b && e == cudaSuccess) e = h2d_any(device, b, v->data, (size_t)n * es, s);
    return b;
  };
  const void* d_marker = dev_copy(marker);
  const void* d_mask = dev_copy(mask);
  void* d_out = out->location == HB_DEVICE ? out->data : pa.get(nn * es);
  if (!flags || !d_marker || !d_mask || !d_out || pa.err != cudaSuccess)
    e = pa.err != cudaSuccess ? pa.err : cudaErrorMemoryAllocation;
  int64_t k = 0;
  if (e == cudaSuccess)
    e = geodesic(d_marker, d_mask, mask->dtype, mask->nz, mask->ny, mask->nx, dilation != 0, d_out,
                 flags, s, &k);
  const bool order_bad = e == cudaErrorInvalidValue;
  if (e == cudaSuccess && out->location != HB_DEVICE)
    e = d2h_any(device, out->data, d_out, (size_t)n * es, s);
  cudaStreamSynchronize(s);
  pa.release();
  cudaStreamSynchronize(s);
  cudaStreamDestroy(s);
  if (g_dev[device].session.load() == 0) cudaMemPoolTrimTo(g_dev[device].pool, 0);
  cudaGetLastError();
  if (order_bad) {
    set_err(nullptr, dilation ? "reconstruction by dilation requires marker <= mask"
                              : "reconstruction by erosion requires marker >= mask");
    return HB_EPARAM;
  }
  if (e != cudaSuccess) {
    set_err(nullptr, std::string("geodesic reconstruction: ") + cudaGetErrorString(e));
    return e == cudaErrorMemoryAllocation ? HB_EBUDGET_UNAVAILABLE : HB_ECUDA;
  }
  if (sweeps) *sweeps = k;
  return HB_OK;
}

int32_t hb_edt(const hb_volume* in, hb_volume* out, const double* spacing, int32_t device) {
  if (!in || !out || !in->data || !out->data || !spacing || (out->dtype != HB_F32 && out->dtype != HB_F64) ||
      in->nz != out->nz || in->ny != out->ny || in->nx != out->nx || in->dtype < HB_U8 || in->dtype > HB_F32) {
    set_err(nullptr, "hb_edt: float32 (or float64 squared) output of the input's shape required");
    return HB_EPARAM;
  }
  if (in->nz >= (1 << 30) || in->ny >= (1 << 30) || in->nx >= (1 << 30)) {
    set_err(nullptr, "hb_edt: axis too long");
    return HB_EUNSUPPORTED;
  }
  if (device < 0 || device >= hb_device_count()) {
    set_err(nullptr, "no CUDA device " + std::to_string(device));
    return HB_EBUDGET_UNAVAILABLE;
  }
  std::lock_guard<std::mutex> lk(g_dev[device].mu);
  cudaSetDevice(device);
  cudaError_t e = ensure_pool(device);
  if (e != cudaSuccess) {
    set_err(nullptr, cudaGetErrorString(e));
    return HB_ECUDA;
  }
  const int64_t n = in->nz * in->ny * in->nx;
  const size_t es = (size_t)dtype_size(in->dtype), nn = (size_t)std::max<int64_t>(n, 1);
  const size_t oes = out->dtype == HB_F32 ? 4 : 8;
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  PoolAlloc pa{g_dev[device].pool, s};
  double* d2a = (double*)pa.get(nn * 8);
  double* d2b = (double*)pa.get(nn * 8);
  void* work = pa.get(edt_workspace_bytes(in->nz, in->ny, in->nx));
  const void* d_in = in->data;
  if (in->location != HB_DEVICE && work) {
    void* b = pa.get(nn * es);
    if (b) e = h2d_any(device, b, in->data, (size_t)n * es, s);
    d_in = b;
  }
  void* d_out = out->location == HB_DEVICE ? out->data : (work ? pa.get(nn * oes) : nullptr);
  if (!d2a || !d2b || !work || !d_in || !d_out || pa.err != cudaSuccess)
    e = pa.err != cudaSuccess ? pa.err : cudaErrorMemoryAllocation;
  if (e == cudaSuccess)
    e = edt(d_in, in->dtype, in->nz, in->ny, in->nx, spacing, out->dtype != HB_F32, d_out, d2a, d2b,
            work, s);
  if (e == cudaSuccess && out->location != HB_DEVICE)
    e = d2h_any(device, out->data, d_out, (size_t)n * oes, s);
  cudaError_t se = cudaStreamSynchronize(s);
  if (e == cudaSuccess) e = se;
  pa.release();
  cudaStreamSynchronize(s);
  cudaStreamDestroy(s);
  if (g_dev[device].session.load() == 0) cudaMemPoolTrimTo(g_dev[device].pool, 0);
  if (e != cudaSuccess) {
    set_err(nullptr, std::string("edt: ") + cudaGetErrorString(e));
    cudaGetLastError();
    return e == cudaErrorMemoryAllocation ? HB_EBUDGET_UNAVAILABLE : HB_ECUDA;
  }
  return HB_OK;
}

int32_t hb_histogram(const hb_volume* in, int32_t device, int32_t bins, double lo, double hi,
                     const double* edges, int32_t edges_f32, int64_t* counts) {
  if (!in || bins < 1 || !edges || !counts || !(hi > lo) || !std::isfinite(lo) || !std::isfinite(hi)) {
    set_err(nullptr, "hb_histogram: bins >= 1, finite lo < hi and edges/counts required");
    return HB_EPARAM;
  }
  double* d_edges = nullptr;
  unsigned long long* d_counts = nullptr;
  int32_t rc = for_each_slab(in, device, [&](const void* p, int64_t n, cudaStream_t s) {
    if (!d_counts) {
      cudaError_t e = cudaMallocAsync(&d_counts, sizeof(unsigned long long) * bins, s);
      if (e == cudaSuccess) e = cudaMallocAsync(&d_edges, sizeof(double) * (bins + 1), s);
      if (e != cudaSuccess) return e;
      cudaMemsetAsync(d_counts, 0, sizeof(unsigned long long) * bins, s);
      cudaMemcpyAsync(d_edges, edges, sizeof(double) * (bins + 1), cudaMemcpyHostToDevice, s);
    }
    return histogram(p, in->dtype, n, bins, lo, hi, d_edges, edges_f32 != 0, d_counts, s);
  });
  if (rc == HB_OK && d_counts) {
    cudaError_t e = cudaMemcpy(counts, d_counts, sizeof(unsigned long long) * bins, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) {
      set_err(nullptr, cudaGetErrorString(e));
      rc = HB_ECUDA;
    }
  } else if (rc == HB_OK) {
    std::memset(counts, 0, sizeof(int64_t) * bins);
  }
  if (d_counts) cudaFree(d_counts);
  if (d_edges) cudaFree(d_edges);
  return rc;
}

int64_t hb_device_pool_bytes(int32_t dev) {
  if (dev < 0 || dev >= 64 || !g_dev[dev].init) return 0;
  return pool_attr(dev, cudaMemPoolAttrReservedMemCurrent);
}

int32_t hb_apply_device(const hb_volume* in, hb_volume* out, const hb_stage* stages,
                        int32_t nstages, int64_t z_begin, void* stream, int32_t synchronize,
                        hb_report* rep) {
  NvtxRange nv_range("hb_apply_device");
  if (rep) {
    std::memset(rep, 0, sizeof(*rep));
    rep->failed_chunk = -1;
    rep->chunk_count = 1;
  }
  if (!in || !out || !in->data || !out->data || in->location != HB_DEVICE ||
      out->location != HB_DEVICE) {
    set_err(rep, "hb_apply_device needs device volumes");
    return HB_EPARAM;
  }
  if (in->nz < 1 || in->ny < 1 || in->nx < 1 || out->ny != in->ny || out->nx != in->nx ||
      z_begin < 0 || out->nz < 0 || z_begin + out->nz > in->nz) {
    set_err(rep, "shape mismatch between device blocks");
    return HB_EPARAM;
  }
  std::vector<StageDesc> st;
  std::string msg;
  hb_status rc = normalise(stages, nstages, in->dtype, st, msg);
  if (rc != HB_OK) {
    set_err(rep, msg);
    return rc;
  }
  if (st.back().out_dt != out->dtype) {
    set_err(rep, "output dtype does not match the chain's output dtype");
    return HB_EPARAM;
  }
  int dev = 0;
  cudaPointerAttributes pa_attr;
  if (cudaPointerGetAttributes(&pa_attr, in->data) == cudaSuccess && pa_attr.device >= 0)
    dev = pa_attr.device;
  cudaGetLastError();
  cudaSetDevice(dev);
  std::lock_guard<std::mutex> lk(g_dev[dev].mu);
  cudaError_t e = ensure_pool(dev);
  if (e != cudaSuccess) {
    set_err(rep, std::string("device pool: ") + cudaGetErrorString(e));
    return HB_ECUDA;
  }
  cudaStream_t s = (cudaStream_t)stream;
  if (synchronize) pool_reset_peak(dev);
  PoolAlloc pa{g_dev[dev].pool, s};
  DevIn din{in->data, in->dtype, in->nz, in->ny, in->nx};
  int64_t launches = 0;
  double t0 = now_ms();
  e = run_chain(st, din, z_begin, out->nz, out->data, pa, s, &launches);
  pa.release();
  if (rep) rep->kernel_launches = launches;
  if (e != cudaSuccess) {
    cudaStreamSynchronize(s);
    cudaGetLastError();
    cudaMemPoolTrimTo(g_dev[dev].pool, 0);
    set_err(rep, std::string("CUDA: ") + cudaGetErrorString(e));
    if (rep) rep->failed_chunk = 0;
    return HB_ECUDA;
  }
  if (synchronize) {
    e = cudaStreamSynchronize(s);
    if (rep) {
      rep->device_peak_bytes = pool_attr(dev, cudaMemPoolAttrUsedMemHigh);
      rep->wall_ms = now_ms() - t0;
    }
    cudaMemPoolTrimTo(g_dev[dev].pool, 0);
    if (rep) rep->device_residual_bytes = pool_attr(dev, cudaMemPoolAttrReservedMemCurrent);
    if (e != cudaSuccess) {
      set_err(rep, std::string("CUDA: ") + cudaGetErrorString(e));
      cudaGetLastError();
      if (rep) rep->failed_chunk = 0;
      return HB_ECUDA;
    }
  }
  return HB_OK;
}

// Argument / plan validation shared by hb_run and hb_run_multi: the chunk
// interiors must partition [0, Z) with halos inside the volume.
static int32_t check_run(const hb_volume* in, hb_volume* out, const hb_stage* stages,
                         int32_t nstages, const hb_chunk* chunks, int64_t nchunks,
                         const hb_exec* ex, hb_report* rep, std::vector<StageDesc>& st) {
  if (!in || !out || !in->data || !out->data || !ex || !chunks) {
    set_err(rep, "null argument");
    return HB_EPARAM;
  }
  if (in->location != HB_HOST || out->location != HB_HOST) {
    set_err(rep, "hb_run streams host volumes; use hb_apply_device for device blocks");
    return HB_EPARAM;
  }
  if (in->nz < 1 || in->ny < 1 || in->nx < 1 || out->nz != in->nz || out->ny != in->ny ||
      out->nx != in->nx) {
    set_err(rep, "input/output shapes differ");
    return HB_EPARAM;
  }
  std::string msg;
  hb_status rc = normalise(stages, nstages, in->dtype, st, msg);
  if (rc != HB_OK) {
    set_err(rep, msg);
    return rc;
  }
  if (st.back().out_dt != out->dtype) {
    set_err(rep, "output dtype does not match the chain's output dtype");
    return HB_EPARAM;
  }
  // validate the plan: interiors must partition [0, Z), halos within the volume
  int64_t expect = 0;
  int64_t max_int = 0;
  for (int64_t k = 0; k < nchunks; k++) {
    const hb_chunk& c = chunks[k];
    if (c.z_start != expect || c.z_stop <= c.z_start || c.halo_lo < 0 || c.halo_hi < 0 ||
        c.z_start - c.halo_lo < 0 || c.z_stop + c.halo_hi > in->nz) {
      set_err(rep, "invalid chunk plan at chunk " + std::to_string(k));
      return HB_EPARAM;
    }
    expect = c.z_stop;
    max_int = std::max(max_int, c.z_stop - c.z_start);
  }
  if (expect != in->nz) {
    set_err(rep, "chunk interiors do not cover the volume");
    return HB_EPARAM;
  }
  (void)max_int;
  return HB_OK;
}

// The streaming loop over a run of plan chunks on ONE device (ex->device).
static int32_t run_host_range(const hb_volume* in, hb_volume* out,
                              const std::vector<StageDesc>& st, const hb_chunk* chunks,
                              int64_t nchunks, const hb_exec* ex, hb_report* rep,
                              double t_start) {
  int64_t max_int = 0;
  for (int64_t k = 0; k < nchunks; k++)
    max_int = std::max(max_int, chunks[k].z_stop - chunks[k].z_start);
  const int dev = ex->device;
  if (dev < 0 || dev >= hb_device_count()) {
    set_err(rep, "no CUDA device " + std::to_string(dev));
    return HB_EBUDGET_UNAVAILABLE;
  }
  cudaSetDevice(dev);
  std::lock_guard<std::mutex> lk(g_dev[dev].mu);
  cudaError_t e = ensure_pool(dev);
  if (e != cudaSuccess) {
    set_err(rep, std::string("device pool: ") + cudaGetErrorString(e));
    return HB_ECUDA;
  }
  const size_t plane = (size_t)in->ny * in->nx;
  const size_t in_es = dtype_size(in->dtype), out_es = dtype_size(out->dtype);
  int64_t H = 0;
  for (auto& d : st) H += d.halo;

  // ---- pieces: every plan chunk is streamed as z-pieces of <= S interior
  // slices.  A piece's padded block is clamped to its chunk's padded block, so
  // each piece reproduces the chunk-level (reference) result exactly; pieces
  // bound the device working set and deepen the copy/compute overlap.
  auto slot_bytes_for = [&](int64_t S) -> size_t {
    const int64_t pad = S + 2 * H;
    return (size_t)pad * plane * in_es + (size_t)S * plane * out_es +
           chain_scratch(st, pad, in->ny, in->nx, H, S);
  };
  size_t free_b = 0, total_b = 0;
  cudaMemGetInfo(&free_b, &total_b);
  // Hard limit: physically free device memory.  Soft target: the job budget
  // (the planner's scratch factors are the reference's host estimates; a plan
  // the reference accepts must not fail here just because the device layout
  // differs, so pieces shrink and the pipeline gets shallower first).
  const size_t cap = free_b > (256u << 20) ? free_b - (256u << 20) : 0;
  size_t soft = cap;
  if (ex->device_budget > 0) soft = std::min(cap, (size_t)ex->device_budget);
  // ~160 MiB per pipeline slot (HB_SLOT_MB overrides: smaller slots shorten
  // the pipeline fill / drain of a job, larger ones cut per-piece overhead)
  static const size_t target = [] {
    const char* v = std::getenv("HB_SLOT_MB");
    return (size_t)(v ? std::max(8, std::atoi(v)) : 160) << 20;
  }();
  int64_t S = max_int;
  while (S > 1 && slot_bytes_for(S) > target && S > 2 * H) S = std::max<int64_t>(1, S * 3 / 4);
  int depth = ex->pipeline_depth > 0 ? ex->pipeline_depth : 3;
  while (depth > 1 && (size_t)depth * slot_bytes_for(S) > soft) depth--;
  while (S > 1 && slot_bytes_for(S) > soft) S = std::max<int64_t>(1, S / 2);
  if (slot_bytes_for(S) > cap) {
    rep->minimum_bytes = (int64_t)slot_bytes_for(S);
    set_err(rep, "device budget of " + std::to_string(cap) + " bytes cannot hold one chunk (" +
                     std::to_string(slot_bytes_for(S)) + " bytes needed)");
    return HB_EBUDGET_SMALL;
  }
  struct Piece {
    int64_t chunk, a, b, p0, p1;
  };
  std::vector<Piece> pieces;
  std::vector<int64_t> last_piece(nchunks, -1);
  int64_t max_pad = 0;
  for (int64_t k = 0; k < nchunks; k++) {
    const hb_chunk& c = chunks[k];
    const int64_t cs = c.z_start - c.halo_lo, ce = c.z_stop + c.halo_hi;
    for (int64_t a0 = c.z_start; a0 < c.z_stop; a0 += S) {
      const int64_t b0 = std::min(a0 + S, c.z_stop);
      Piece pc{k, a0, b0, std::max(cs, a0 - H), std::min(ce, b0 + H)};
      max_pad = std::max(max_pad, pc.p1 - pc.p0);
      last_piece[k] = (int64_t)pieces.size();
      pieces.push_back(pc);
    }
  }
  const int64_t npieces = (int64_t)pieces.size();
  depth = (int)std::min<int64_t>(depth, std::max<int64_t>(1, npieces));
  const int threads = auto_threads(ex->host_threads);
  const bool in_pinned = is_pinned(in->data), out_pinned = is_pinned(out->data);
  PinnedRing& ring = g_ring[dev];
  if (!in_pinned || !out_pinned) {
    e = ring.init();
    if (e != cudaSuccess) {
      set_err(rep, std::string("pinned staging: ") + cudaGetErrorString(e));
      return HB_ECUDA;
    }
  }

  cudaStream_t s_in, s_comp, s_out;
  cudaStreamCreateWithFlags(&s_in, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s_comp, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s_out, cudaStreamNonBlocking);
  std::vector<cudaEvent_t> ev_h2d(depth), ev_comp(depth), ev_k0(depth);
  for (int i = 0; i < depth; i++) {
    cudaEventCreate(&ev_h2d[i]);
    cudaEventCreate(&ev_comp[i]);
    cudaEventCreate(&ev_k0[i]);
  }
  std::vector<cudaEvent_t> ev_done(npieces);
  for (auto& v : ev_done) cudaEventCreate(&v);
  cudaEvent_t ev_start;
  cudaEventCreate(&ev_start);

  const double t_alloc0 = now_ms();
  pool_reset_peak(dev);
  std::vector<PoolAlloc> slots;
  std::vector<void*> dbuf_in(depth), dbuf_out(depth);
  for (int i = 0; i < depth; i++) slots.push_back(PoolAlloc{g_dev[dev].pool, s_comp});
  PoolAlloc io{g_dev[dev].pool, s_comp};
  for (int i = 0; i < depth && e == cudaSuccess; i++) {
    dbuf_in[i] = io.get((size_t)max_pad * plane * in_es);
    dbuf_out[i] = io.get((size_t)S * plane * out_es);
    if (!dbuf_in[i] || !dbuf_out[i]) e = io.err;
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(s_comp);
  if (e != cudaSuccess) {
    io.release();
    cudaStreamSynchronize(s_comp);
    cudaGetLastError();
    cudaMemPoolTrimTo(g_dev[dev].pool, 0);
    rep->minimum_bytes = (int64_t)slot_bytes_for(S);
    set_err(rep, std::string("device allocation failed: ") + cudaGetErrorString(e));
    return HB_EBUDGET_SMALL;
  }

  const double t_setup = now_ms();
  hb_status status = HB_OK;
  int64_t launches = 0;
  double kernel_ms = 0;
  std::vector<int64_t> slot_piece(depth, -1);
  cudaEventRecord(ev_start, s_in);

  // finish piece j: its D2H into pageable memory (if needed) and bookkeeping
  auto finish = [&](int64_t j) -> cudaError_t {
    const int slot = (int)(j % depth);
    const Piece& pc = pieces[j];
    NvtxRange fin_range("hb piece finish (D2H)");
    const size_t bytes = (size_t)(pc.b - pc.a) * plane * out_es;
    char* host_dst = (char*)out->data + (size_t)pc.a * plane * out_es;
    cudaError_t err = cudaSuccess;
    if (!out_pinned) {
      cudaStreamWaitEvent(s_out, ev_comp[slot], 0);
      err = d2h_staged(ring, host_dst, dbuf_out[slot], bytes, s_out, threads);
      cudaEventRecord(ev_done[j], s_out);
    }
    cudaEventSynchronize(ev_done[j]);
    float ms = 0;
    if (cudaEventElapsedTime(&ms, ev_k0[slot], ev_comp[slot]) == cudaSuccess) kernel_ms += ms;
    rep->d2h_bytes += (int64_t)bytes;
    slot_piece[slot] = -1;
    return err == cudaSuccess ? cudaGetLastError() : err;
  };

  int64_t j = 0;
  int64_t chunk_now = -1;
  int64_t prev_p0 = 0, prev_p1 = 0;
  int prev_slot = -1;
  for (; j < npieces; j++) {
    const Piece& pc = pieces[j];
    const int slot = (int)(j % depth);
    char nv[48];
    std::snprintf(nv, sizeof(nv), "hb chunk %lld piece %lld", (long long)pc.chunk, (long long)j);
    NvtxRange piece_range(nv);  // host-side enqueue of H2D -> chain -> D2H
    if (pc.chunk != chunk_now) {  // chunk boundary: cancel poll + fault hook
      chunk_now = pc.chunk;
      if (ex->cancel && ex->cancel(ex->cancel_ctx)) {
        status = HB_ECANCELLED;
        set_err(rep, "cancelled before chunk " + std::to_string(chunk_now));
        break;
      }
      if (ex->fault_chunk >= 0 && chunk_now == ex->fault_chunk) {
        status = HB_ECHUNK;
        set_err(rep, "injected fault on chunk " + std::to_string(chunk_now));
        break;
      }
    }
    if (slot_piece[slot] >= 0) {
      e = finish(slot_piece[slot]);
      if (e != cudaSuccess) break;
    }
    // input: reuse the overlap with the previous piece's slab on the device
    // (halo slices cross PCIe once), upload the rest
    int64_t up0 = pc.p0;
    if (prev_slot >= 0 && prev_slot != slot && pc.p0 >= prev_p0 && pc.p0 < prev_p1) {
      const int64_t keep = std::min(prev_p1, pc.p1) - pc.p0;
      e = cudaMemcpyAsync(dbuf_in[slot], (char*)dbuf_in[prev_slot] + (size_t)(pc.p0 - prev_p0) * plane * in_es,
                          (size_t)keep * plane * in_es, cudaMemcpyDeviceToDevice, s_in);
      if (e != cudaSuccess) break;
      up0 = pc.p0 + keep;
    }
    if (up0 < pc.p1) {
      const size_t bytes = (size_t)(pc.p1 - up0) * plane * in_es;
      char* dst = (char*)dbuf_in[slot] + (size_t)(up0 - pc.p0) * plane * in_es;
      const char* src = (const char*)in->data + (size_t)up0 * plane * in_es;
      e = in_pinned ? cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s_in)
                    : h2d_staged(ring, dst, src, bytes, s_in, threads);
      if (e != cudaSuccess) break;
      rep->h2d_bytes += (int64_t)bytes;
    }
    cudaEventRecord(ev_h2d[slot], s_in);
    prev_p0 = pc.p0;
    prev_p1 = pc.p1;
    prev_slot = slot;
    // compute
    cudaStreamWaitEvent(s_comp, ev_h2d[slot], 0);
    cudaEventRecord(ev_k0[slot], s_comp);
    DevIn din{dbuf_in[slot], in->dtype, pc.p1 - pc.p0, in->ny, in->nx};
    e = run_chain(st, din, pc.a - pc.p0, pc.b - pc.a, dbuf_out[slot], slots[slot], s_comp, &launches);
    slots[slot].release();
    if (e != cudaSuccess) break;
    cudaEventRecord(ev_comp[slot], s_comp);
    if (out_pinned) {
      cudaStreamWaitEvent(s_out, ev_comp[slot], 0);
      char* host_dst = (char*)out->data + (size_t)pc.a * plane * out_es;
      e = cudaMemcpyAsync(host_dst, dbuf_out[slot], (size_t)(pc.b - pc.a) * plane * out_es,
                          cudaMemcpyDeviceToHost, s_out);
      if (e != cudaSuccess) break;
      cudaEventRecord(ev_done[j], s_out);
    }
    slot_piece[slot] = j;
  }
  // drain outstanding pieces in order
  if (status == HB_OK && e == cudaSuccess) {
    for (int64_t q = std::max<int64_t>(0, j - depth); q < j; q++) {
      const int slot = (int)(q % depth);
      if (slot_piece[slot] == q) {
        e = finish(q);
        if (e != cudaSuccess) break;
      }
    }
  }
  cudaError_t sync_e = cudaDeviceSynchronize();
  const double t_loop = now_ms();
  if (e == cudaSuccess && status == HB_OK && sync_e != cudaSuccess) e = sync_e;
  const int64_t at_chunk = j < npieces ? pieces[j].chunk : nchunks - 1;
  if (e != cudaSuccess && status == HB_OK) {
    status = HB_ECUDA;
    rep->failed_chunk = at_chunk;
    set_err(rep, std::string("CUDA error on chunk ") + std::to_string(at_chunk) + ": " +
                     cudaGetErrorString(e));
    cudaGetLastError();
  } else if (status != HB_OK) {
    rep->failed_chunk = at_chunk;
  }
  if (status == HB_OK && ex->chunk_seconds) {
    for (int64_t k = 0; k < nchunks; k++) {
      float ms = 0;
      cudaEventElapsedTime(&ms, k == 0 ? ev_start : ev_done[last_piece[k - 1]], ev_done[last_piece[k]]);
      ex->chunk_seconds[k] = ms * 1e-3;
    }
  }
  for (auto& sl : slots) sl.release();
  io.release();
  cudaStreamSynchronize(s_comp);
  const double t_free = now_ms();
  rep->device_peak_bytes = pool_attr(dev, cudaMemPoolAttrUsedMemHigh);
  if (g_dev[dev].session.load() == 0) cudaMemPoolTrimTo(g_dev[dev].pool, 0);
  // job-owned bytes still allocated (0: every buffer went back to the pool);
  // outside a session the pool itself is trimmed to zero as well
  rep->device_residual_bytes = pool_attr(dev, cudaMemPoolAttrUsedMemCurrent);
  if (g_dev[dev].session.load() == 0)
    rep->device_residual_bytes = pool_attr(dev, cudaMemPoolAttrReservedMemCurrent);
  const double t_trim = now_ms();
  for (int i = 0; i < depth; i++) {
    cudaEventDestroy(ev_h2d[i]);
    cudaEventDestroy(ev_comp[i]);
    cudaEventDestroy(ev_k0[i]);
  }
  for (auto& v : ev_done) cudaEventDestroy(v);
  cudaEventDestroy(ev_start);
  cudaStreamDestroy(s_in);
  cudaStreamDestroy(s_comp);
  cudaStreamDestroy(s_out);
  cudaGetLastError();
  rep->chunk_count = nchunks;
  rep->kernel_launches = launches;
  rep->kernel_ms = kernel_ms;
  rep->wall_ms = now_ms() - t_start;
  if (std::getenv("HB_TRACE"))
    std::fprintf(stderr,
                 "[hb_run] pieces=%lld S=%lld depth=%d setup=%.2fms (alloc %.2fms) loop=%.2fms "
                 "teardown=%.2fms (free %.2f trim %.2f destroy %.2f)\n",
                 (long long)npieces, (long long)S, depth, t_setup - t_start, t_setup - t_alloc0,
                 t_loop - t_setup, now_ms() - t_loop, t_free - t_loop, t_trim - t_free,
                 now_ms() - t_trim);
  return status;
}


int32_t hb_run(const hb_volume* in, hb_volume* out, const hb_stage* stages, int32_t nstages,
               const hb_chunk* chunks, int64_t nchunks, const hb_exec* ex, hb_report* rep) {
  hb_report dummy;
  if (!rep) rep = &dummy;
  std::memset(rep, 0, sizeof(*rep));
  rep->failed_chunk = -1;
  const double t_start = now_ms();
  std::vector<StageDesc> st;
  int32_t rc = check_run(in, out, stages, nstages, chunks, nchunks, ex, rep, st);
  if (rc != HB_OK) return rc;
  NvtxRange job("hb_run");
  return run_host_range(in, out, st, chunks, nchunks, ex, rep, t_start);
}

int32_t hb_run_multi(const hb_volume* in, hb_volume* out, const hb_stage* stages,
                     int32_t nstages, const hb_chunk* chunks, int64_t nchunks,
                     const hb_exec* ex, int32_t ndev, const int32_t* devices, hb_report* rep,
                     hb_report* per_device) {
  hb_report dummy;
  if (!rep) rep = &dummy;
  std::memset(rep, 0, sizeof(*rep));
  rep->failed_chunk = -1;
  const double t_start = now_ms();
  if (ndev < 1 || !devices) {
    set_err(rep, "hb_run_multi: ndev >= 1 devices required");
    return HB_EPARAM;
  }
  std::vector<StageDesc> st;
  int32_t rc = check_run(in, out, stages, nstages, chunks, nchunks, ex, rep, st);
  if (rc != HB_OK) return rc;
  for (int i = 0; i < ndev; i++)
    if (devices[i] < 0 || devices[i] >= hb_device_count()) {
      set_err(rep, "no CUDA device " + std::to_string(devices[i]));
      return HB_EBUDGET_UNAVAILABLE;
    }
  // contiguous chunk groups with balanced interior slices: device i owns the
  // chunks whose interior starts in [i*Z/ndev, (i+1)*Z/ndev) — a z-slab per
  // device, each streamed through its own PCIe link; halos at group faces are
  // read from host memory (the out-of-core rule)
  std::vector<int64_t> first(ndev + 1, nchunks);
  {
    int g = 0;
    first[0] = 0;
    for (int64_t k = 0; k < nchunks; k++) {
      while (g + 1 < ndev && chunks[k].z_start >= (in->nz * (g + 1)) / ndev) first[++g] = k;
    }
    for (int i = g + 1; i <= ndev; i++) first[i] = nchunks;
  }
  std::vector<hb_report> reps(ndev);
  std::vector<hb_exec> exs(ndev);
  std::vector<int32_t> codes(ndev, HB_OK);
  std::vector<std::thread> th;
  for (int i = 0; i < ndev; i++) {
    const int64_t k0 = first[i], n = first[i + 1] - first[i];
    std::memset(&reps[i], 0, sizeof(hb_report));
    reps[i].failed_chunk = -1;
    if (n <= 0) continue;
    exs[i] = *ex;
    exs[i].device = devices[i];
    exs[i].chunk_seconds = ex->chunk_seconds ? ex->chunk_seconds + k0 : nullptr;
    exs[i].fault_chunk = ex->fault_chunk >= k0 && ex->fault_chunk < k0 + n ? (int32_t)(ex->fault_chunk - k0) : -1;
    th.emplace_back([&, i, k0, n] {
      codes[i] = run_host_range(in, out, st, chunks + k0, n, &exs[i], &reps[i], now_ms());
      if (codes[i] != HB_OK && reps[i].failed_chunk >= 0) reps[i].failed_chunk += k0;
    });
  }
  for (auto& t : th) t.join();
  int32_t status = HB_OK;
  for (int i = 0; i < ndev; i++) {
    const hb_report& r = reps[i];
    rep->chunk_count += r.chunk_count;
    rep->device_peak_bytes = std::max(rep->device_peak_bytes, r.device_peak_bytes);
    rep->device_residual_bytes += r.device_residual_bytes;
    rep->h2d_bytes += r.h2d_bytes;
    rep->d2h_bytes += r.d2h_bytes;
    rep->kernel_ms = std::max(rep->kernel_ms, r.kernel_ms);
    rep->kernel_launches += r.kernel_launches;
    if (codes[i] != HB_OK && status == HB_OK) {  // the lowest failing group reports
      status = codes[i];
      rep->failed_chunk = r.failed_chunk;
      rep->minimum_bytes = r.minimum_bytes;
      std::memcpy(rep->message, r.message, sizeof(rep->message));
    }
    if (per_device) per_device[i] = r;
  }
  rep->wall_ms = now_ms() - t_start;
  if (status != HB_OK) set_err(nullptr, rep->message);
  return status;
}

int32_t hb_device_alloc(int32_t dev, int64_t bytes, void* stream, void** ptr) {
  if (!ptr || bytes < 0 || dev < 0 || dev >= hb_device_count()) {
    set_err(nullptr, "hb_device_alloc: bad arguments");
    return HB_EPARAM;
  }
  *ptr = nullptr;
  cudaSetDevice(dev);
  {
    std::lock_guard<std::mutex> lk(g_dev[dev].mu);
    cudaError_t e = ensure_pool(dev);
    if (e == cudaSuccess)
      e = cudaMallocFromPoolAsync(ptr, (size_t)std::max<int64_t>(bytes, 256), g_dev[dev].pool,
                                  (cudaStream_t)stream);
    if (e != cudaSuccess) {
      cudaGetLastError();
      *ptr = nullptr;
      set_err(nullptr, std::string("hb_device_alloc: ") + cudaGetErrorString(e));
      return e == cudaErrorMemoryAllocation ? HB_EBUDGET_SMALL : HB_ECUDA;
    }
  }
  return HB_OK;
}

int32_t hb_device_free(int32_t dev, void* ptr, void* stream) {
  if (!ptr) return HB_OK;
  if (dev < 0 || dev >= hb_device_count()) return HB_EPARAM;
  cudaSetDevice(dev);
  cudaError_t e = cudaFreeAsync(ptr, (cudaStream_t)stream);
  if (e != cudaSuccess) {
    cudaGetLastError();
    set_err(nullptr, std::string("hb_device_free: ") + cudaGetErrorString(e));
    return HB_ECUDA;
  }
  return HB_OK;
}

}  // extern "C"
