// FP64 issue rate on one SM: W warps, each with 8 independent DADD chains
// (throughput) or 1 chain (latency), cycles per warp-instruction.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -o tools/fp64_bench tools/fp64_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int NCH>
__global__ void k(double* out, long long* t, int n, double y) {
  double a[NCH];
#pragma unroll
  for (int c = 0; c < NCH; ++c) a[c] = y * (threadIdx.x + c);
  __syncthreads();
  long long c0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int c = 0; c < NCH; ++c) a[c] = a[c] + y;
  }
  __syncthreads();
  long long c1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < NCH; ++c) s += a[c];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) t[0] = c1 - c0;
}

int main() {
  double* out;
  long long* t;
  cudaMalloc(&out, 1024 * 8);
  cudaMallocManaged(&t, 8);
  const int n = 4096;
  for (int w : {1, 4, 8, 16, 32}) {
    k<1><<<1, 32 * w>>>(out, t, n, 1.0000001);
    cudaDeviceSynchronize();
    k<1><<<1, 32 * w>>>(out, t, n, 1.0000001);
    cudaDeviceSynchronize();
    const double lat = (double)t[0] / n;
    k<8><<<1, 32 * w>>>(out, t, n, 1.0000001);
    cudaDeviceSynchronize();
    k<8><<<1, 32 * w>>>(out, t, n, 1.0000001);
    cudaDeviceSynchronize();
    const double thr = (double)t[0] / (8.0 * n);
    printf("warps/SM %2d: 1 chain: %.2f cycles per DADD per warp; 8 chains: %.2f cycles per DADD "
           "per warp -> %.2f warp-DADDs per cycle per SM\n", w, lat, thr, w / thr);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
