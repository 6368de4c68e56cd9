// Does q' = fma(fma(-q, d, a), inv, q), q = a*inv, inv = RN(1/d) reproduce
// __fdiv_rn(a, d) for the mean's divisors and dividends?
#include <cstdio>
#include <cstdint>
__global__ void k(float d, uint32_t n0, uint32_t n, int mode, unsigned long long* bad, float* ex) {
  const float inv = __frcp_rn(d);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    float a;
    if (mode == 0) a = (float)(n0 + i);                       // integer sums
    else a = __uint_as_float(0x3f000000u + (i * 2654435761u) % 0x03000000u);  // floats in [0.5, 32)
    const float q = a * inv;
    const float r = fmaf(-q, d, a);
    const float q2 = fmaf(r, inv, q);
    const float ref = __fdiv_rn(a, d);
    if (q2 != ref) { unsigned long long k = atomicAdd(bad, 1ull); if (k == 0) { ex[0] = a; ex[1] = q2; ex[2] = ref; } }
  }
}
int main() {
  unsigned long long* bad; float* ex; cudaMallocManaged(&bad, 8); cudaMallocManaged(&ex, 12);
  for (float d : {27.f, 125.f, 343.f, 8.f*8*8+0.f, 9.f}) {
    for (int mode = 0; mode < 2; ++mode) {
      *bad = 0;
      uint32_t n = mode == 0 ? (uint32_t)(d * 65536) : (1u << 30);
      k<<<4096, 256>>>(d, 0, n, mode, bad, ex); cudaDeviceSynchronize();
      printf("d=%g mode=%d mismatches=%llu", d, mode, *bad);
      if (*bad) printf("  e.g. a=%.9g q2=%.9g ref=%.9g", ex[0], ex[1], ex[2]);
      printf("\n");
    }
  }
}
