// gauss_fused.cu — fused single-pass 3D separable Gaussian (fast fp32 mode).
// Placeholder until the tiled kernel lands: reports "not supported" so the
// executor takes the generic three-pass path.
#include "ops.cuh"

namespace hb {
cudaError_t gaussian_fused(const DevIn&, int64_t, int64_t, float*, const Taps&, const EpiArgs&,
                           cudaStream_t, int64_t*) {
  return cudaErrorNotSupported;
}
}  // namespace hb
