// Latency microbenchmarks on the B200 (diagnostics for the slice phase).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void chain(double* out, long long* t, int n, double x0, double y) {
  __shared__ double sm[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) sm[i] = y * i;
  __syncthreads();
  if (threadIdx.x != 0) return;
  double a = x0;
  long long c0 = clock64();
  for (int i = 0; i < n; ++i) { a = a + y; a = a + y; a = a + y; a = a + y; }
  long long c1 = clock64();
  double b = x0;
  for (int i = 0; i < n; ++i) { b = fma(b, y, y); b = fma(b, y, y); b = fma(b, y, y); b = fma(b, y, y); }
  long long c2 = clock64();
  float f = (float)x0;
  for (int i = 0; i < n; ++i) { f = f + (float)y; f = f + (float)y; f = f + (float)y; f = f + (float)y; }
  long long c3 = clock64();
  // cumsum-like: add chain with smem operand + store
  double acc = 0;
  for (int i = 0; i < 1024; ++i) { acc = acc + sm[i]; sm[1024 + (i & 1023)] = acc; }
  long long c4 = clock64();
  // volatile smem pointer chase
  volatile int* vi = (volatile int*)sm;
  int idx = 0;
  for (int i = 0; i < n; ++i) idx = vi[idx & 7];
  long long c5 = clock64();
  out[0] = a + b + f + acc + idx;
  t[0] = (c1 - c0) / (4 * n);
  t[1] = (c2 - c1) / (4 * n);
  t[2] = (c3 - c2) / (4 * n);
  t[3] = (c4 - c3) / 1024;
  t[4] = (c5 - c4) / n;
}

__global__ void syncs(long long* t, int n) {
  long long c0 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  long long c1 = clock64();
  if (threadIdx.x == 0) t[5] = (c1 - c0) / n;
}

int main() {
  double* d; long long* t;
  cudaMalloc(&d, 8); cudaMalloc(&t, 64);
  chain<<<1, 256>>>(d, t, 1000, 1.0, 1e-3);
  syncs<<<1, 256>>>(t, 1000);
  long long h[8];
  cudaMemcpy(h, t, 48, cudaMemcpyDeviceToHost);
  printf("cycles: dependent DADD %lld, DFMA %lld, FADD %lld, cumsum elem (LDS+DADD+STS) %lld, LDS chase %lld, syncthreads(256) %lld\n",
         h[0], h[1], h[2], h[3], h[4], h[5]);
  return 0;
}
