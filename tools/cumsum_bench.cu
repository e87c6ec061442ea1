// Cycle counts of the field solve's sequential scan variants on one CTA
// (diagnostic for the slice phase of the fine kernel).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -o tools/cumsum_bench tools/cumsum_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2511_13386_b200/csrc/pk_device.cuh"

using namespace pk;

__global__ void bench(double* out, long long* t, int n, double y) {
  extern __shared__ double sm[];
  for (int i = threadIdx.x; i < 2 * n; i += blockDim.x) sm[i] = y * (i % 17);
  __syncthreads();
  long long c0 = clock64();
  smem_cumsum(sm, sm + n, n);
  __syncthreads();
  long long c1 = clock64();
  smem_cumsum(sm, sm, n);  // in place
  __syncthreads();
  long long c2 = clock64();
  if (threadIdx.x == 0) {  // a subtrahend on every operand (the slow form)
    double a = -0.0;
    for (int i = 0; i < n; ++i) {
      a = a + (sm[i] - y);
      sm[n + i] = a;
    }
  }
  __syncthreads();
  long long c3 = clock64();
  warp_cumsum([&](int i) { return sm[i]; }, [&](int i, double v) { sm[n + i] = v; }, n);
  __syncthreads();
  long long c4 = clock64();
  if (threadIdx.x == 0) {
    // register-only dependent chain
    double a = y, b = sm[1];
    for (int i = 0; i < n; i += 4) {
      a = a + b;
      a = a + b;
      a = a + b;
      a = a + b;
    }
    sm[2] = a;
  }
  __syncthreads();
  long long c5 = clock64();
  if (threadIdx.x == 0) {
    out[0] = sm[n - 1] + sm[2 * n - 1] + sm[0] + sm[2];
    t[0] = c1 - c0;
    t[1] = c2 - c1;
    t[2] = c3 - c2;
    t[3] = c4 - c3;
    t[4] = c5 - c4;
  }
}

int main() {
  double* out;
  long long* t;
  cudaMalloc(&out, 8);
  cudaMallocManaged(&t, 8 * 8);
  for (int n : {256, 1024, 8192}) {
    const int smem = 2 * n * 8;
    cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int rep = 0; rep < 2; ++rep) {
      bench<<<1, 128, smem>>>(out, t, n, 1.0000001);
      cudaDeviceSynchronize();
    }
    printf("n=%d cycles/elt: smem_cumsum %.2f, in place %.2f, operand-subtrahend loop %.2f, "
           "generic warp_cumsum %.2f, register chain %.2f\n",
           n, (double)t[0] / n, (double)t[1] / n, (double)t[2] / n, (double)t[3] / n,
           (double)t[4] / n);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
