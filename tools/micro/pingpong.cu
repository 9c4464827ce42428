// Cross-SM flag ping-pong latency (relaxed gpu-scope store/load through L2),
// and intra-CTA __syncthreads step latency; dev microbenchmark.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ long long ldr(const long long* p){long long v;asm volatile("ld.relaxed.gpu.global.b64 %0,[%1];":"=l"(v):"l"(p):"memory");return v;}
__device__ __forceinline__ void str(long long* p,long long v){asm volatile("st.relaxed.gpu.global.b64 [%0],%1;"::"l"(p),"l"(v):"memory");}
__device__ __forceinline__ unsigned long long gt(){unsigned long long t;asm volatile("mov.u64 %0,%globaltimer;":"=l"(t));return t;}
__global__ void pingpong(long long* a, long long* b, int iters, unsigned long long* out){
  if(threadIdx.x) return;
  unsigned long long t0=gt();
  if(blockIdx.x==0){ for(int i=1;i<=iters;i++){ str(a,i); while(ldr(b)!=i); } out[0]=gt()-t0; }
  else if(blockIdx.x==gridDim.x-1){ for(int i=1;i<=iters;i++){ while(ldr(a)!=i); str(b,i);} }
}
__global__ void barsteps(int iters, unsigned long long* out, double* sink){
  __shared__ double xs[1024];
  double acc=threadIdx.x;
  unsigned long long t0=gt();
  for(int i=0;i<iters;i++){ xs[threadIdx.x]=acc; __syncthreads(); acc+=xs[(threadIdx.x+37)&1023]*1.0000001; __syncthreads(); }
  if(threadIdx.x==0) out[1]=gt()-t0;
  sink[threadIdx.x]=acc;
}
int main(){
  long long *a,*b; unsigned long long* out; double* sink;
  cudaMalloc(&a,4096); cudaMalloc(&b,4096); cudaMalloc(&out,64); cudaMalloc(&sink,8192);
  for(int g : {2, 148}){
    cudaMemset(a,0,8); cudaMemset(b,0,8);
    int iters=20000;
    pingpong<<<g,32>>>(a,b,iters,out); cudaDeviceSynchronize();
    unsigned long long h[2]; cudaMemcpy(h,out,16,cudaMemcpyDeviceToHost);
    printf("pingpong grid=%d: %.3f us per round trip\n", g, h[0]/1e3/iters);
  }
  int iters=20000;
  barsteps<<<1,1024>>>(iters,out,sink); cudaDeviceSynchronize();
  unsigned long long h[2]; cudaMemcpy(h,out,16,cudaMemcpyDeviceToHost);
  printf("1024-thread step (2 syncthreads + smem): %.3f us\n", h[1]/1e3/iters);
  barsteps<<<148,1024>>>(iters,out,sink); cudaDeviceSynchronize();
  cudaMemcpy(h,out,16,cudaMemcpyDeviceToHost);
  printf("1024-thread step, 148 CTAs: %.3f us\n", h[1]/1e3/iters);
  return 0;
}
