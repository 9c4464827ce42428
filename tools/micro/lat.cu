// Primitive latencies on sm_100a (dev microbenchmark): dependent LDS chain,
// DFMA chain, DDIV chain, st.relaxed.gpu + dependent work.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* g, long long* out, int n) {
  __shared__ int idx[1024];
  __shared__ double xs[1024];
  int t = threadIdx.x;
  idx[t] = (t * 7 + 1) & 1023; xs[t] = 1.0 + t * 1e-9;
  __syncthreads();
  if (t) return;
  long long c0 = clock64();
  int j = 0;
  for (int i = 0; i < n; i++) j = idx[j];
  long long c1 = clock64();
  double a = xs[j & 1023], b = 1.0000001;
  for (int i = 0; i < n; i++) a = fma(a, b, 1e-9);
  long long c2 = clock64();
  double d = a;
  for (int i = 0; i < n; i++) d = __ddiv_rn(1.0, d + 1.0);
  long long c3 = clock64();
  for (int i = 0; i < n; i++) { asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" :: "l"(g + (i & 7)), "d"(d) : "memory"); d = d * 1.0000001; }
  long long c4 = clock64();
  double e = d;
  for (int i = 0; i < n; i++) e = xs[(int)(e * 0.0) + (i & 1023)] + e * 0.5;
  long long c5 = clock64();
  out[0] = (c1 - c0) / n; out[1] = (c2 - c1) / n; out[2] = (c3 - c2) / n; out[3] = (c4 - c3) / n; out[4] = (c5 - c4) / n;
  g[100] = a + d + e + j;
}
int main() {
  double* g; long long* o; cudaMalloc(&g, 4096); cudaMalloc(&o, 64);
  k<<<1, 1024>>>(g, o, 1000); cudaDeviceSynchronize();
  k<<<1, 1024>>>(g, o, 10000); cudaDeviceSynchronize();
  long long h[5]; cudaMemcpy(h, o, 40, cudaMemcpyDeviceToHost);
  printf("cycles: dep LDS %lld, DFMA %lld, DDIV %lld, STG.strong+DMUL %lld, LDS+DFMA chain %lld\n", h[0], h[1], h[2], h[3], h[4]);
}
