// Issue-rate probe: scalar FFMA/FADD/FMUL vs packed FFMA2/FADD2/FMUL2 (sm_100a).
// 8 independent chains per thread, 16 warps/SM x 148 SMs; prints G-op/s per
// instruction kind (an x2 op counts 2 lanes of work per lane).
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c){u64 r; asm volatile("fma.rn.f32x2 %0,%1,%2,%3;":"=l"(r):"l"(a),"l"(b),"l"(c)); return r;}
__device__ __forceinline__ u64 add2(u64 a, u64 b){u64 r; asm volatile("add.rn.f32x2 %0,%1,%2;":"=l"(r):"l"(a),"l"(b)); return r;}
__device__ __forceinline__ u64 mul2(u64 a, u64 b){u64 r; asm volatile("mul.rn.f32x2 %0,%1,%2;":"=l"(r):"l"(a),"l"(b)); return r;}
template<int K> __global__ void kscalar(float* out, float b, float c, int iters){
  float x[8]; for(int i=0;i<8;i++) x[i]=threadIdx.x*1e-3f+i;
  for(int it=0; it<iters; it++){
    #pragma unroll
    for(int i=0;i<8;i++){
      if(K==0) asm volatile("fma.rn.f32 %0,%0,%1,%2;":"+f"(x[i]):"f"(b),"f"(c));
      if(K==1) asm volatile("add.rn.f32 %0,%0,%1;":"+f"(x[i]):"f"(c));
      if(K==2) asm volatile("mul.rn.f32 %0,%0,%1;":"+f"(x[i]):"f"(b));
    }
  }
  float s=0; for(int i=0;i<8;i++) s+=x[i]; out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
template<int K> __global__ void kpacked(float* out, float b, float c, int iters){
  u64 x[8]; for(int i=0;i<8;i++){float2 f=make_float2(threadIdx.x*1e-3f+i, i); x[i]=*(u64*)&f;}
  float2 bf=make_float2(b,b), cf=make_float2(c,c); u64 bb=*(u64*)&bf, cc=*(u64*)&cf;
  for(int it=0; it<iters; it++){
    #pragma unroll
    for(int i=0;i<8;i++){
      if(K==0) x[i]=fma2(x[i],bb,cc);
      if(K==1) x[i]=add2(x[i],cc);
      if(K==2) x[i]=mul2(x[i],bb);
    }
  }
  float s=0; for(int i=0;i<8;i++){float2 f=*(float2*)&x[i]; s+=f.x+f.y;} out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
template<class F> void run(const char* name, F f, int lanes_per_op){
  float* out; cudaMalloc(&out, 148*512*4);
  int iters=20000; cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(out,iters); cudaDeviceSynchronize();
  cudaEventRecord(a); f(out,iters); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms,a,b);
  double inst = 148.0*512/32*8*iters;   // warp instructions
  printf("%-8s %8.3f ms  %7.2f warp-inst/clk/SM  %8.1f G lane-ops/s\n", name, ms,
         inst/(ms*1e-3)/148/1.965e9, inst*32*lanes_per_op/(ms*1e-3)/1e9);
  cudaFree(out);
}
int main(){
  run("FFMA",  [](float*o,int n){kscalar<0><<<148,512>>>(o,1.0001f,1e-7f,n);},1);
  run("FFMA2", [](float*o,int n){kpacked<0><<<148,512>>>(o,1.0001f,1e-7f,n);},2);
  run("FADD",  [](float*o,int n){kscalar<1><<<148,512>>>(o,1.0001f,1e-7f,n);},1);
  run("FADD2", [](float*o,int n){kpacked<1><<<148,512>>>(o,1.0001f,1e-7f,n);},2);
  run("FMUL",  [](float*o,int n){kscalar<2><<<148,512>>>(o,1.0001f,1e-7f,n);},1);
  run("FMUL2", [](float*o,int n){kpacked<2><<<148,512>>>(o,1.0001f,1e-7f,n);},2);
  return 0;
}
