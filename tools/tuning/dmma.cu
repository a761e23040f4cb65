#include <cstdio>
#include <cuda_runtime.h>
extern "C" __global__ void k_m8n8k4(double* out, int iters){
  double a = threadIdx.x*1e-3, b = 1.0001;
  double c[8][2];
  #pragma unroll
  for(int i=0;i<8;i++){c[i][0]=0;c[i][1]=0;}
  for(int it=0; it<iters; ++it){
    #pragma unroll
    for(int i=0;i<8;i++){
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s=0; for(int i=0;i<8;i++) s+=c[i][0]+c[i][1];
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
extern "C" __global__ void k_m16n8k4(double* out, int iters){
  double a0 = threadIdx.x*1e-3, a1=a0+1, b = 1.0001;
  double c[8][4];
  #pragma unroll
  for(int i=0;i<8;i++){c[i][0]=0;c[i][1]=0;c[i][2]=0;c[i][3]=0;}
  for(int it=0; it<iters; ++it){
    #pragma unroll
    for(int i=0;i<8;i++){
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};" : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a0), "d"(a1), "d"(b));
    }
  }
  double s=0; for(int i=0;i<8;i++) s+=c[i][0]+c[i][1]+c[i][2]+c[i][3];
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
extern "C" __global__ void k_m16n8k16(double* out, int iters){
  double a[8], b[4];
  for(int i=0;i<8;i++) a[i]=threadIdx.x*1e-3+i; for(int i=0;i<4;i++) b[i]=1.0+i*1e-4;
  double c[4][4];
  #pragma unroll
  for(int i=0;i<4;i++){c[i][0]=0;c[i][1]=0;c[i][2]=0;c[i][3]=0;}
  for(int it=0; it<iters; ++it){
    #pragma unroll
    for(int i=0;i<4;i++){
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};" : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a[0]),"d"(a[1]),"d"(a[2]),"d"(a[3]),"d"(a[4]),"d"(a[5]),"d"(a[6]),"d"(a[7]), "d"(b[0]),"d"(b[1]),"d"(b[2]),"d"(b[3]));
    }
  }
  double s=0; for(int i=0;i<4;i++) s+=c[i][0]+c[i][1]+c[i][2]+c[i][3];
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
extern "C" __global__ void k_dfma(double* out, int iters){
  double a = threadIdx.x*1e-3, b = 1.0001;
  double c[16];
  #pragma unroll
  for(int i=0;i<16;i++) c[i]=i;
  for(int it=0; it<iters; ++it){
    #pragma unroll
    for(int i=0;i<16;i++) c[i]=fma(c[i],b,a);
  }
  double s=0; for(int i=0;i<16;i++) s+=c[i];
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
int main(){
  double* out; cudaMalloc(&out, 148*8*1024*8);
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters=20000;
  struct K{const char* n; void(*f)(double*,int); double flop_per_warp_iter;} ks[]={
    {"m8n8k4",k_m8n8k4, 8*2.0*8*8*4},{"m16n8k4",k_m16n8k4,8*2.0*16*8*4},{"m16n8k16",k_m16n8k16,4*2.0*16*8*16},{"dfma",k_dfma,16*2.0*32}};
  for (auto& k: ks){
   for(int warps=4; warps<=32; warps*=2){
    int bs=warps*32; int grid=148*2;
    k.f<<<grid,bs>>>(out,100); cudaDeviceSynchronize();
    cudaEventRecord(e0); k.f<<<grid,bs>>>(out,iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms,e0,e1);
    double flops = (double)grid*warps*iters*k.flop_per_warp_iter;
    printf("%s warps/blk=%d grid=%d: %.3f ms  %.2f TFLOP/s  err=%s\n", k.n, warps, grid, ms, flops/ms/1e9, cudaGetErrorString(cudaGetLastError()));
   }
  }
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0); printf("clock kHz %d\n", clk);
}
