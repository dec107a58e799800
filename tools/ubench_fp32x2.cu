// Microbenchmark: scalar exact (FADD,FMUL,FADD) vs packed exact (FADD2,FFMA2(+rt zero),FADD2) issue rate on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void scalar_k(float* out, float a0, float b0, int iters){
  float a[8], s[8];
  for (int i=0;i<8;i++){ a[i]=a0+threadIdx.x*1e-3f+i; s[i]=0.f; }
  for (int it=0; it<iters; ++it){
#pragma unroll
    for (int i=0;i<8;i++){ float d=__fsub_rn(a[i],b0); s[i]=__fadd_rn(s[i],__fmul_rn(d,d)); a[i]=__fadd_rn(a[i],1e-7f);}
  }
  float t=0; for(int i=0;i<8;i++) t+=s[i]; if (t==1234.5f) out[threadIdx.x]=t;
}
__global__ void packed_k(float* out, float a0, float b0, int iters, unsigned long long zero){
  unsigned long long a[8], s[8], b; float2 bb=make_float2(b0,b0); b=*(unsigned long long*)&bb;
  float2 inc=make_float2(1e-7f,1e-7f); unsigned long long incu=*(unsigned long long*)&inc;
  for (int i=0;i<8;i++){ float2 t=make_float2(a0+threadIdx.x*1e-3f+i, a0+i+0.5f); a[i]=*(unsigned long long*)&t; s[i]=0ull; }
  for (int it=0; it<iters; ++it){
#pragma unroll
    for (int i=0;i<8;i++){ unsigned long long d,p;
      asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a[i]), "l"(b));
      asm("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(p) : "l"(d), "l"(zero));
      asm("add.rn.f32x2 %0, %1, %2;" : "=l"(s[i]) : "l"(s[i]), "l"(p));
      asm("add.rn.f32x2 %0, %1, %2;" : "=l"(a[i]) : "l"(a[i]), "l"(incu));
    }
  }
  float t=0; for(int i=0;i<8;i++){ float2 f=*(float2*)&s[i]; t+=f.x+f.y;} if (t==1234.5f) out[threadIdx.x]=t;
}
int main(){
  float* out; cudaMalloc(&out, 1<<20);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int iters=20000; cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep=0; rep<2; ++rep){
  for (int blocks_per_sm=2; blocks_per_sm<=8; blocks_per_sm*=2){
    dim3 g(sms*blocks_per_sm), b(256);
    scalar_k<<<g,b>>>(out,1.f,0.5f,10);
    cudaEventRecord(e0); scalar_k<<<g,b>>>(out,1.f,0.5f,iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms,e0,e1);
    double pairdims = (double)g.x*b.x*iters*8; // each = 1 pair-dim (3 exact ops) + 1 extra add
    printf("scalar  bps=%d: %.3f ms, %.2f T pair-dim/s (4 instr each)\n", blocks_per_sm, ms, pairdims/ms/1e9);
    packed_k<<<g,b>>>(out,1.f,0.5f,10,0ull);
    cudaEventRecord(e0); packed_k<<<g,b>>>(out,1.f,0.5f,iters,0ull); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms,e0,e1);
    pairdims = (double)g.x*b.x*iters*8*2;
    printf("packed  bps=%d: %.3f ms, %.2f T pair-dim/s (4 x2-instr per 2)\n", blocks_per_sm, ms, pairdims/ms/1e9);
  }}
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0); printf("sms=%d clk=%d kHz\n", sms, clk);
  return 0;
}
