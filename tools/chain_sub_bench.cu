// Does a subtrahend folded into the np.cumsum chain cost extra?  Thread 0
// chains x[i] - corr with the subtractions of the next block interleaved
// between the current block's dependent adds (one asm block per 8).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -o tools/chain_sub_bench tools/chain_sub_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2511_13386_b200/csrc/pk_device.cuh"

using namespace pk;

// acc += c_k (c = already corrected), store; load next 8 raw into nn; after
// the fourth add, subtract corr from the next 8 (in place in nn)
#define PK_CS8S(acc, c, nn, lda, sta, corr)                                               \
  asm volatile(                                                                            \
      "{\n\t"                                                                              \
      "ld.shared.f64 %1, [%17];\n\t"                                                       \
      "ld.shared.f64 %2, [%17+8];\n\t"                                                     \
      "ld.shared.f64 %3, [%17+16];\n\t"                                                    \
      "ld.shared.f64 %4, [%17+24];\n\t"                                                    \
      "ld.shared.f64 %5, [%17+32];\n\t"                                                    \
      "ld.shared.f64 %6, [%17+40];\n\t"                                                    \
      "ld.shared.f64 %7, [%17+48];\n\t"                                                    \
      "ld.shared.f64 %8, [%17+56];\n\t"                                                    \
      "add.rn.f64 %0, %0, %9;\n\tst.shared.f64 [%18], %0;\n\t"                             \
      "add.rn.f64 %0, %0, %10;\n\tst.shared.f64 [%18+8], %0;\n\t"                          \
      "add.rn.f64 %0, %0, %11;\n\tst.shared.f64 [%18+16], %0;\n\t"                         \
      "add.rn.f64 %0, %0, %12;\n\tst.shared.f64 [%18+24], %0;\n\t"                         \
      "sub.rn.f64 %1, %1, %19;\n\t"                                                        \
      "sub.rn.f64 %2, %2, %19;\n\t"                                                        \
      "add.rn.f64 %0, %0, %13;\n\tst.shared.f64 [%18+32], %0;\n\t"                         \
      "sub.rn.f64 %3, %3, %19;\n\t"                                                        \
      "sub.rn.f64 %4, %4, %19;\n\t"                                                        \
      "add.rn.f64 %0, %0, %14;\n\tst.shared.f64 [%18+40], %0;\n\t"                         \
      "sub.rn.f64 %5, %5, %19;\n\t"                                                        \
      "sub.rn.f64 %6, %6, %19;\n\t"                                                        \
      "add.rn.f64 %0, %0, %15;\n\tst.shared.f64 [%18+48], %0;\n\t"                         \
      "sub.rn.f64 %7, %7, %19;\n\t"                                                        \
      "sub.rn.f64 %8, %8, %19;\n\t"                                                        \
      "add.rn.f64 %0, %0, %16;\n\tst.shared.f64 [%18+56], %0;\n\t"                         \
      "}"                                                                                   \
      : "+d"(acc), "=&d"(nn[0]), "=&d"(nn[1]), "=&d"(nn[2]), "=&d"(nn[3]), "=&d"(nn[4]),   \
        "=&d"(nn[5]), "=&d"(nn[6]), "=&d"(nn[7])                                           \
      : "d"(c[0]), "d"(c[1]), "d"(c[2]), "d"(c[3]), "d"(c[4]), "d"(c[5]), "d"(c[6]),       \
        "d"(c[7]), "r"(lda), "r"(sta), "d"(corr)                                           \
      : "memory")

__device__ void cumsum_sub(double* x, int n, double corr) {
  if (threadIdx.x != 0) return;
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(x);
  double acc = -0.0;
  const int n2 = n - n % 16;
  double A[8], Bv[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) A[k] = lds64(s + 8 * k) - corr;
  for (int i = 0; i < n2; i += 16) {
    PK_CS8S(acc, A, Bv, s + 8 * (i + 8), s + 8 * i, corr);
    const uint32_t nxt = i + 16 < n2 ? s + 8 * (i + 16) : s;
    PK_CS8S(acc, Bv, A, nxt, s + 8 * (i + 8), corr);
  }
  for (int i = n2; i < n; ++i) {
    acc = acc + (lds64(s + 8 * i) - corr);
    sts64(s + 8 * i, acc);
  }
}

__global__ void bench(double* out, long long* t, int n, double corr) {
  extern __shared__ double sm[];
  double* a = sm;
  double* b = sm + n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) a[i] = b[i] = 1e-3 * (i % 17) - 0.008;
  __syncthreads();
  long long c0 = clock64();
  for (int i = threadIdx.x; i < n; i += blockDim.x) a[i] = a[i] - corr;
  __syncthreads();
  smem_cumsum(a, a, n);
  __syncthreads();
  long long c1 = clock64();
  cumsum_sub(b, n, corr);
  __syncthreads();
  long long c2 = clock64();
  bool same = true;
  for (int i = threadIdx.x; i < n; i += blockDim.x) same &= __double_as_longlong(a[i]) == __double_as_longlong(b[i]);
  same = __syncthreads_and(same);
  if (threadIdx.x == 0) {
    t[0] = c1 - c0;
    t[1] = c2 - c1;
    t[2] = same;
    out[0] = a[n - 1];
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
      bench<<<1, 128, smem>>>(out, t, n, 1.2345e-4);
      cudaDeviceSynchronize();
    }
    printf("n=%d: corr pass + chain %.2f cycles/elt, folded %.2f cycles/elt, bitwise equal %lld\n", n,
           (double)t[0] / n, (double)t[1] / n, t[2]);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
