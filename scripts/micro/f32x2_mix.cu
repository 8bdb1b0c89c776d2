// Does a packed FADD2 (2 fma-pipe cycles) leave its second issue slot free
// for an ALU instruction? Loop bodies per iteration and thread:
//   S: 16 FADD + 8 SHF      P: 8 FADD2 + 8 SHF     (same FP work)
// Issue-bound S needs 24 slots/iteration; P needs 16 if the slot is free.
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 add2(u64 a, u64 b){u64 r; asm volatile("add.rn.f32x2 %0,%1,%2;":"=l"(r):"l"(a),"l"(b)); return r;}
template<int P> __global__ void k(float* out, float c, int iters, unsigned m){
  u64 x[8]; float y[16]; unsigned z[8];
  for(int i=0;i<8;i++){float2 f=make_float2(threadIdx.x*1e-3f+i, i); x[i]=*(u64*)&f; z[i]=threadIdx.x+i;}
  for(int i=0;i<16;i++) y[i]=threadIdx.x*1e-3f+i;
  float2 cf=make_float2(c,c); u64 cc=*(u64*)&cf;
  for(int it=0; it<iters; it++){
    #pragma unroll
    for(int i=0;i<8;i++){
      if(P){ x[i]=add2(x[i],cc); }
      else { asm volatile("add.rn.f32 %0,%0,%1;":"+f"(y[2*i]):"f"(c)); asm volatile("add.rn.f32 %0,%0,%1;":"+f"(y[2*i+1]):"f"(c)); }
      asm volatile("shf.l.wrap.b32 %0,%0,%0,%1;":"+r"(z[i]):"r"(m));
    }
  }
  float s=0; for(int i=0;i<8;i++){float2 f=*(float2*)&x[i]; s+=f.x+f.y+z[i];} for(int i=0;i<16;i++) s+=y[i];
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
template<class F> void run(const char* name, F f){
  float* out; cudaMalloc(&out, 148*512*4);
  int iters=20000; cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(out,iters); cudaDeviceSynchronize();
  cudaEventRecord(a); f(out,iters); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms,a,b);
  double iter_per_smsp = 148.0*512/32/4/148*iters;   // warp-iterations per SMSP
  printf("%-4s %8.3f ms  %6.2f cycles per warp-iteration per SMSP\n", name, ms, ms*1e-3*1.965e9/ (iter_per_smsp));
  cudaFree(out);
}
int main(){
  run("S", [](float*o,int n){k<0><<<148,512>>>(o,1e-7f,n,3u);});
  run("P", [](float*o,int n){k<1><<<148,512>>>(o,1e-7f,n,3u);});
  return 0;
}
