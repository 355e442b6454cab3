// Step-0 hardware probe: FP64 pipe ceilings on sm_100a.
// Measures DFMA (SIMT) and DMMA (mma.sync .f64) issue-limited throughput with
// register-resident operands. Not part of the product path.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e){printf("err %s line %d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)

__global__ void dfma_peak(double* out, int iters, double s){
  double a[8];
  for(int i=0;i<8;i++) a[i]=threadIdx.x*1e-3+i;
  double b=s, c=1e-9;
  for(int it=0;it<iters;it++){
#pragma unroll
    for(int i=0;i<8;i++) a[i]=fma(a[i],b,c);
  }
  double r=0; for(int i=0;i<8;i++) r+=a[i];
  if(r==12345.0) out[0]=r;
}

__global__ void dmma884_peak(double* out, int iters){
  double acc[8][2];
  for(int i=0;i<8;i++){acc[i][0]=0;acc[i][1]=0;}
  double a=threadIdx.x*1e-3, b=1e-3;
  for(int it=0;it<iters;it++){
#pragma unroll
    for(int i=0;i<8;i++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
        : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
  }
  double r=0; for(int i=0;i<8;i++) r+=acc[i][0]+acc[i][1];
  if(r==12345.0) out[0]=r;
}

__global__ void dmma16816_peak(double* out, int iters){
  double acc[4][4];
  for(int i=0;i<4;i++) for(int j=0;j<4;j++) acc[i][j]=0;
  double a[8], b[4];
  for(int i=0;i<8;i++) a[i]=threadIdx.x*1e-3+i; for(int i=0;i<4;i++) b[i]=1e-3*i;
  for(int it=0;it<iters;it++){
#pragma unroll
    for(int i=0;i<4;i++)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
        : "+d"(acc[i][0]), "+d"(acc[i][1]), "+d"(acc[i][2]), "+d"(acc[i][3])
        : "d"(a[0]),"d"(a[1]),"d"(a[2]),"d"(a[3]),"d"(a[4]),"d"(a[5]),"d"(a[6]),"d"(a[7]),
          "d"(b[0]),"d"(b[1]),"d"(b[2]),"d"(b[3]));
  }
  double r=0; for(int i=0;i<4;i++) for(int j=0;j<4;j++) r+=acc[i][j];
  if(r==12345.0) out[0]=r;
}

int main(){
  double* d; CK(cudaMalloc(&d,8));
  int dev; cudaGetDevice(&dev); cudaDeviceProp p; cudaGetDeviceProperties(&p,dev);
  int sms=p.multiProcessorCount; int clk; cudaDeviceGetAttribute(&clk,cudaDevAttrClockRate,dev);
  printf("{\"gpu\":\"%s\",\"sms\":%d,\"clock_khz\":%d", p.name, sms, clk);
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for(int threads: {128,256,512}){
    int blocks=sms*(1024/threads)*2; int iters=4096;
    dfma_peak<<<blocks,threads>>>(d,16,1.0); CK(cudaDeviceSynchronize());
    float best=1e9;
    for(int r=0;r<5;r++){cudaEventRecord(e0); dfma_peak<<<blocks,threads>>>(d,iters,1.0000001); cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms,e0,e1); if(ms<best)best=ms;}
    double fl=2.0*8*iters*(double)blocks*threads; printf(",\"dfma_tflops_t%d\":%.3f",threads,fl/best/1e9);
  }
  for(int threads: {128,256,512}){
    int blocks=sms*(1024/threads)*2; int iters=2048;
    dmma884_peak<<<blocks,threads>>>(d,16); CK(cudaDeviceSynchronize());
    float best=1e9;
    for(int r=0;r<5;r++){cudaEventRecord(e0); dmma884_peak<<<blocks,threads>>>(d,iters); cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms,e0,e1); if(ms<best)best=ms;}
    double fl=2.0*256*8*iters*(double)blocks*(threads/32); printf(",\"dmma884_tflops_t%d\":%.3f",threads,fl/best/1e9);
  }
  for(int threads: {128,256,512}){
    int blocks=sms*(1024/threads)*2; int iters=512;
    dmma16816_peak<<<blocks,threads>>>(d,16); CK(cudaDeviceSynchronize());
    float best=1e9;
    for(int r=0;r<5;r++){cudaEventRecord(e0); dmma16816_peak<<<blocks,threads>>>(d,iters); cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms,e0,e1); if(ms<best)best=ms;}
    double fl=2.0*2048*4*iters*(double)blocks*(threads/32); printf(",\"dmma16816_tflops_t%d\":%.3f",threads,fl/best/1e9);
  }
  printf("}\n");
  return 0;
}
