// Throughput microbenchmarks for the instruction mixes the stencil/median/morphology
// kernels rely on (FFMA 3-reg vs const-operand vs FFMA2, DFMA, FMNMX, VIMNMX.U16x2),
// plus HBM copy and pinned PCIe bandwidth. Run once on the B200 box; results feed DESIGN.md.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e){printf("err %s line %d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)

constexpr int ITERS = 4096;
__constant__ float cw[32];

__global__ void k_ffma3(float* out, float a, float b) {
  float x0=threadIdx.x, x1=x0+1, x2=x0+2, x3=x0+3, x4=x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  float y = a, z = b;
  #pragma unroll 16
  for (int i=0;i<ITERS;i++){ x0=fmaf(x0,y,z); x1=fmaf(x1,y,z); x2=fmaf(x2,y,z); x3=fmaf(x3,y,z);
    x4=fmaf(x4,y,z); x5=fmaf(x5,y,z); x6=fmaf(x6,y,z); x7=fmaf(x7,y,z);
    y += 1e-30f; }
  out[blockIdx.x*blockDim.x+threadIdx.x]=x0+x1+x2+x3+x4+x5+x6+x7;
}
__global__ void k_ffma_const(float* out) {
  float x0=threadIdx.x, x1=x0+1, x2=x0+2, x3=x0+3, x4=x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  #pragma unroll 16
  for (int i=0;i<ITERS;i++){ float w=cw[i&15]; x0=fmaf(x0,w,x1); x1=fmaf(x1,w,x2); x2=fmaf(x2,w,x3); x3=fmaf(x3,w,x4);
    x4=fmaf(x4,w,x5); x5=fmaf(x5,w,x6); x6=fmaf(x6,w,x7); x7=fmaf(x7,w,x0);}
  out[blockIdx.x*blockDim.x+threadIdx.x]=x0+x1+x2+x3+x4+x5+x6+x7;
}
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b, unsigned long long c){
  unsigned long long d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
__global__ void k_ffma2(float* out, float a, float b) {
  unsigned long long x[8]; for(int j=0;j<8;j++){ float2 f=make_float2(threadIdx.x+j, j); x[j]=*reinterpret_cast<unsigned long long*>(&f);} 
  float2 yy=make_float2(a,a), zz=make_float2(b,b);
  unsigned long long y=*reinterpret_cast<unsigned long long*>(&yy), z=*reinterpret_cast<unsigned long long*>(&zz);
  #pragma unroll 16
  for (int i=0;i<ITERS;i++){
    #pragma unroll
    for(int j=0;j<8;j++) x[j]=ffma2(x[j],y,z);
  }
  float s=0; for(int j=0;j<8;j++){ float2 f=*reinterpret_cast<float2*>(&x[j]); s+=f.x+f.y;} out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
__global__ void k_fadd(float* out, float a) {
  float x0=threadIdx.x, x1=x0+1, x2=x0+2, x3=x0+3, x4=x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  #pragma unroll 16
  for (int i=0;i<ITERS;i++){ x0=x0+x1; x1=x1+x2; x2=x2+x3; x3=x3+x4; x4=x4+x5; x5=x5+x6; x6=x6+x7; x7=x7+a;}
  out[blockIdx.x*blockDim.x+threadIdx.x]=x0+x1+x2+x3+x4+x5+x6+x7;
}
__global__ void k_dfma(double* out, double a, double b) {
  double x0=threadIdx.x, x1=x0+1, x2=x0+2, x3=x0+3, x4=x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  #pragma unroll 16
  for (int i=0;i<ITERS;i++){ x0=fma(x0,a,b); x1=fma(x1,a,b); x2=fma(x2,a,b); x3=fma(x3,a,b);
    x4=fma(x4,a,b); x5=fma(x5,a,b); x6=fma(x6,a,b); x7=fma(x7,a,b);}
  out[blockIdx.x*blockDim.x+threadIdx.x]=x0+x1+x2+x3+x4+x5+x6+x7;
}
__global__ void k_dadd(double* out, double a) {
  double x0=threadIdx.x, x1=x0+1, x2=x0+2, x3=x0+3, x4=x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  #pragma unroll 16
  for (int i=0;i<ITERS;i++){ x0=__dadd_rn(x0,x1); x1=__dadd_rn(x1,x2); x2=__dadd_rn(x2,x3); x3=__dadd_rn(x3,x4); x4=__dadd_rn(x4,x5); x5=__dadd_rn(x5,x6); x6=__dadd_rn(x6,x7); x7=__dadd_rn(x7,a);}
  out[blockIdx.x*blockDim.x+threadIdx.x]=x0+x1+x2+x3+x4+x5+x6+x7;
}
__global__ void k_fmnmx(float* out, float a) {
  float x0=threadIdx.x, x1=x0+1, x2=x0+2, x3=x0+3, x4=x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  #pragma unroll 16
  for (int i=0;i<ITERS;i++){ x0=fminf(x0,x1); x1=fmaxf(x1,x2); x2=fminf(x2,x3); x3=fmaxf(x3,x4); x4=fminf(x4,x5); x5=fmaxf(x5,x6); x6=fminf(x6,x7); x7=fmaxf(x7,a); a+=1.f;}
  out[blockIdx.x*blockDim.x+threadIdx.x]=x0+x1+x2+x3+x4+x5+x6+x7;
}
__global__ void k_fmnmx3(float* out, float a) {
  float x0=threadIdx.x, x1=x0+1, x2=x0+2, x3=x0+3, x4=x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  #pragma unroll 16
  for (int i=0;i<ITERS;i++){ x0=fminf(x0,fminf(x1,x2)); x1=fmaxf(x1,fmaxf(x2,x3)); x2=fminf(x2,fminf(x3,x4)); x3=fmaxf(x3,fmaxf(x4,x5)); x4=fminf(x4,fminf(x5,x6)); x5=fmaxf(x5,fmaxf(x6,x7)); x6=fminf(x6,fminf(x7,x0)); x7=fmaxf(x7,fmaxf(x0,a)); a+=1.f;}
  out[blockIdx.x*blockDim.x+threadIdx.x]=x0+x1+x2+x3+x4+x5+x6+x7;
}
__device__ __forceinline__ unsigned vmin2(unsigned a, unsigned b){ unsigned d; asm("min.u16x2 %0,%1,%2;":"=r"(d):"r"(a),"r"(b)); return d;}
__device__ __forceinline__ unsigned vmax2(unsigned a, unsigned b){ unsigned d; asm("max.u16x2 %0,%1,%2;":"=r"(d):"r"(a),"r"(b)); return d;}
__global__ void k_vmnmx(unsigned* out, unsigned a) {
  unsigned x0=threadIdx.x, x1=x0+1, x2=x0+2, x3=x0+3, x4=x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  #pragma unroll 16
  for (int i=0;i<ITERS;i++){ x0=vmin2(x0,x1); x1=vmax2(x1,x2); x2=vmin2(x2,x3); x3=vmax2(x3,x4); x4=vmin2(x4,x5); x5=vmax2(x5,x6); x6=vmin2(x6,x7); x7=vmax2(x7,a); a+=0x10001u;}
  out[blockIdx.x*blockDim.x+threadIdx.x]=x0+x1+x2+x3+x4+x5+x6+x7;
}
__global__ void k_imnmx(unsigned* out, unsigned a) {
  unsigned x0=threadIdx.x, x1=x0+1, x2=x0+2, x3=x0+3, x4=x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  #pragma unroll 16
  for (int i=0;i<ITERS;i++){ x0=min(x0,x1); x1=max(x1,x2); x2=min(x2,x3); x3=max(x3,x4); x4=min(x4,x5); x5=max(x5,x6); x6=min(x6,x7); x7=max(x7,a); a+=1u;}
  out[blockIdx.x*blockDim.x+threadIdx.x]=x0+x1+x2+x3+x4+x5+x6+x7;
}
__global__ void k_copy(const float4* __restrict__ a, float4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x*(size_t)blockDim.x+threadIdx.x; i<n; i+= (size_t)gridDim.x*blockDim.x) b[i]=a[i];
}

template<class F> float timeit(F f, int reps=5){
  cudaEvent_t s,e; cudaEventCreate(&s); cudaEventCreate(&e);
  f(); cudaDeviceSynchronize();
  float best=1e30f;
  for(int r=0;r<reps;r++){ cudaEventRecord(s); f(); cudaEventRecord(e); cudaEventSynchronize(e); float ms; cudaEventElapsedTime(&ms,s,e); if(ms<best)best=ms;}
  return best;
}

int main(){
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p,0));
  printf("device %s SMs %d cc %d.%d smemPerBlockOptin %zu L2 %d\n", p.name, p.multiProcessorCount, p.major,p.minor, p.sharedMemPerBlockOptin, p.l2CacheSize);
  int nsm=p.multiProcessorCount; int blocks=nsm*8, threads=256; size_t nth=(size_t)blocks*threads;
  float* fo; double* dout; unsigned* uo; CK(cudaMalloc(&fo,nth*8)); dout=(double*)fo; uo=(unsigned*)fo;
  float hw[32]; for(int i=0;i<32;i++) hw[i]=0.5f+i*1e-3f; cudaMemcpyToSymbol(cw,hw,sizeof(hw));
  double ops = (double)nth*ITERS*8;
  float ms;
  ms=timeit([&]{k_ffma3<<<blocks,threads>>>(fo,1.0001f,0.5f);}); printf("FFMA(3reg)  %.1f Ginstr-lanes/s  (%.2f lanes/clk/SM @%dMHz)\n", ops/ms/1e6, ops/ms/1e3/ (p.clockRate/1e3) / nsm *1e-3*1e3/1e3, p.clockRate/1000);
  ms=timeit([&]{k_ffma_const<<<blocks,threads>>>(fo);}); printf("FFMA(cbank) %.1f G/s\n", ops/ms/1e6);
  ms=timeit([&]{k_ffma2<<<blocks,threads>>>(fo,1.0001f,0.5f);}); printf("FFMA2       %.1f G fma/s (x2 lanes counted)\n", 2*ops/ms/1e6);
  ms=timeit([&]{k_fadd<<<blocks,threads>>>(fo,1.0f);}); printf("FADD        %.1f G/s\n", ops/ms/1e6);
  ms=timeit([&]{k_dfma<<<blocks,threads>>>(dout,1.0001,0.5);}); printf("DFMA        %.1f G/s\n", ops/ms/1e6);
  ms=timeit([&]{k_dadd<<<blocks,threads>>>(dout,1.0);}); printf("DADD        %.1f G/s\n", ops/ms/1e6);
  ms=timeit([&]{k_fmnmx<<<blocks,threads>>>(fo,1.0f);}); printf("FMNMX       %.1f G/s\n", ops/ms/1e6);
  ms=timeit([&]{k_fmnmx3<<<blocks,threads>>>(fo,1.0f);}); printf("FMNMX3(2op) %.1f G minmax-ops/s\n", 2*ops/ms/1e6);
  ms=timeit([&]{k_vmnmx<<<blocks,threads>>>(uo,1u);}); printf("VIMNMX.U16x2 %.1f G/s (x2 values)\n", ops/ms/1e6);
  ms=timeit([&]{k_imnmx<<<blocks,threads>>>(uo,1u);}); printf("IMNMX       %.1f G/s\n", ops/ms/1e6);
  size_t bytes=(size_t)4<<30; float4 *a,*b; CK(cudaMalloc(&a,bytes)); CK(cudaMalloc(&b,bytes)); cudaMemset(a,0,bytes);
  size_t n=bytes/16;
  for (int bpsm : {2,4,8}) { ms=timeit([&]{k_copy<<<nsm*bpsm,1024>>>(a,b,n);}); printf("copy kernel grid %dx1024: %.1f GB/s (r+w)\n", nsm*bpsm, 2.0*bytes/ms/1e6); }
  ms=timeit([&]{cudaMemcpyAsync(b,a,bytes,cudaMemcpyDeviceToDevice);}); printf("cudaMemcpy D2D %.1f GB/s (r+w)\n", 2.0*bytes/ms/1e6);
  size_t hb=(size_t)1<<30; void* h; CK(cudaMallocHost(&h,hb));
  ms=timeit([&]{cudaMemcpyAsync(a,h,hb,cudaMemcpyHostToDevice);}); printf("H2D pinned %.1f GB/s\n", hb/ms/1e6);
  ms=timeit([&]{cudaMemcpyAsync(h,a,hb,cudaMemcpyDeviceToHost);}); printf("D2H pinned %.1f GB/s\n", hb/ms/1e6);
  cudaStream_t s1,s2; cudaStreamCreate(&s1); cudaStreamCreate(&s2); void* h2; CK(cudaMallocHost(&h2,hb));
  ms=timeit([&]{cudaMemcpyAsync(a,h,hb,cudaMemcpyHostToDevice,s1); cudaMemcpyAsync(h2,b,hb,cudaMemcpyDeviceToHost,s2); cudaStreamSynchronize(s1); cudaStreamSynchronize(s2);}); printf("H2D||D2H pinned %.1f GB/s each\n", hb/ms/1e6);
  void* pg = malloc(hb); memset(pg,1,hb);
  ms=timeit([&]{cudaMemcpy(a,pg,hb,cudaMemcpyHostToDevice);},3); printf("H2D pageable %.1f GB/s\n", hb/ms/1e6);
  return 0;
}
