// Sequential-scan variants for the exact field (np.cumsum order): cycles per
// element of the chain thread with the rest of the CTA parked at a barrier.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -o tools/cumsum_bench2 tools/cumsum_bench2.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2511_13386_b200/csrc/pk_device.cuh"

using namespace pk;

// B: 16-byte loads and stores (half the shared-memory instructions)
#define CS8V(acc, c, nn, lda, sta)                                                        \
  asm volatile(                                                                            \
      "{\n\t"                                                                              \
      "ld.shared.v2.f64 {%1, %2}, [%17];\n\t"                                              \
      "ld.shared.v2.f64 {%3, %4}, [%17+16];\n\t"                                           \
      "ld.shared.v2.f64 {%5, %6}, [%17+32];\n\t"                                           \
      "ld.shared.v2.f64 {%7, %8}, [%17+48];\n\t"                                           \
      ".reg .f64 t0, t1, t2, t3, t4, t5, t6;\n\t"                                          \
      "add.rn.f64 t0, %0, %9;\n\t"                                                         \
      "add.rn.f64 t1, t0, %10;\n\tst.shared.v2.f64 [%18], {t0, t1};\n\t"                   \
      "add.rn.f64 t2, t1, %11;\n\t"                                                        \
      "add.rn.f64 t3, t2, %12;\n\tst.shared.v2.f64 [%18+16], {t2, t3};\n\t"                \
      "add.rn.f64 t4, t3, %13;\n\t"                                                        \
      "add.rn.f64 t5, t4, %14;\n\tst.shared.v2.f64 [%18+32], {t4, t5};\n\t"                \
      "add.rn.f64 t6, t5, %15;\n\t"                                                        \
      "add.rn.f64 %0, t6, %16;\n\tst.shared.v2.f64 [%18+48], {t6, %0};\n\t"                \
      "}"                                                                                   \
      : "+d"(acc), "=&d"(nn[0]), "=&d"(nn[1]), "=&d"(nn[2]), "=&d"(nn[3]), "=&d"(nn[4]),   \
        "=&d"(nn[5]), "=&d"(nn[6]), "=&d"(nn[7])                                           \
      : "d"(c[0]), "d"(c[1]), "d"(c[2]), "d"(c[3]), "d"(c[4]), "d"(c[5]), "d"(c[6]),       \
        "d"(c[7]), "r"(lda), "r"(sta)                                                      \
      : "memory")

__device__ __forceinline__ void cumsum_v2(const double* src, double* dst, int n) {
  if (threadIdx.x != 0) return;
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(src);
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
  double acc = -0.0;
  const int n2 = n - n % 16;
  double A[8], Bv[8];
  for (int k = 0; k < 8; ++k) A[k] = lds64(s + 8 * k);
  for (int i = 0; i < n2; i += 16) {
    CS8V(acc, A, Bv, s + 8 * (i + 8), d + 8 * i);
    const uint32_t nxt = i + 16 < n2 ? s + 8 * (i + 16) : s;
    CS8V(acc, Bv, A, nxt, d + 8 * (i + 8));
  }
  for (int i = n2; i < n; ++i) {
    acc = acc + lds64(s + 8 * i);
    sts64(d + 8 * i, acc);
  }
}

// C: the whole warp runs the chain on broadcast operands (one coalesced load
// per 32 elements, operand k by shuffle), lane k keeps the k-th running sum,
// one coalesced store per 32 elements
__device__ __forceinline__ void cumsum_warp(const double* src, double* dst, int n) {
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  double acc = -0.0;
  double x = src[lane];
  for (int i = 0; i < n; i += 32) {
    const double xn = i + 32 < n ? src[i + 32 + lane] : 0.0;
    double keep = 0.0;
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      const double c = __shfl_sync(0xffffffffu, x, k);
      acc = acc + c;
      if (lane == k) keep = acc;
    }
    dst[i + lane] = keep;
    x = xn;
  }
}

// D: broadcast loads (every lane reads the same 16 bytes), lane k keeps
__device__ __forceinline__ void cumsum_bcast(const double* src, double* dst, int n) {
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(src);
  double acc = -0.0;
  double A[32], Bn[32];
#pragma unroll
  for (int k = 0; k < 32; k += 2)
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(A[k]), "=d"(A[k + 1]) : "r"(s + 8 * k));
  for (int i = 0; i < n; i += 32) {
    const uint32_t nx_ = i + 32 < n ? s + 8 * (i + 32) : s;
#pragma unroll
    for (int k = 0; k < 32; k += 2)
      asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(Bn[k]), "=d"(Bn[k + 1]) : "r"(nx_ + 8 * k));
    double keep = 0.0;
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      acc = acc + A[k];
      if (lane == k) keep = acc;
    }
    dst[i + lane] = keep;
#pragma unroll
    for (int k = 0; k < 32; ++k) A[k] = Bn[k];
  }
}

// E: D with ping-pong blocks of 16 (no register copies), not inlined
static __device__ __noinline__ void cumsum_bcast2(uint32_t s, uint32_t d, int n, double init) {
  const int lane = threadIdx.x & 31;
  double acc = init;
  const int n2 = n - n % 32;
  double A[16], Bn[16];
  if (n2 > 0) {
#pragma unroll
    for (int k = 0; k < 16; k += 2)
      asm volatile("ld.volatile.shared.v2.f64 {%0, %1}, [%2];" : "=d"(A[k]), "=d"(A[k + 1]) : "r"(s + 8 * k));
  }
#pragma unroll 1
  for (int i = 0; i < n2; i += 32) {
#pragma unroll
    for (int k = 0; k < 16; k += 2)
      asm volatile("ld.volatile.shared.v2.f64 {%0, %1}, [%2];" : "=d"(Bn[k]), "=d"(Bn[k + 1]) : "r"(s + 8 * (i + 16 + k)));
    double keep = 0.0;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      acc = acc + A[k];
      keep = lane == k ? acc : keep;
    }
    const uint32_t nxt = i + 32 < n2 ? s + 8 * (i + 32) : s;
#pragma unroll
    for (int k = 0; k < 16; k += 2)
      asm volatile("ld.volatile.shared.v2.f64 {%0, %1}, [%2];" : "=d"(A[k]), "=d"(A[k + 1]) : "r"(nxt + 8 * k));
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      acc = acc + Bn[k];
      keep = lane == 16 + k ? acc : keep;
    }
    asm volatile("st.volatile.shared.f64 [%0], %1;" ::"r"(d + 8 * (i + lane)), "d"(keep) : "memory");
  }
  __syncwarp();
  if (lane == 0)
    for (int i = n2; i < n; ++i) {
      acc = acc + lds64(s + 8 * i);
      sts64(d + 8 * i, acc);
    }
}
#define CS8NV(acc, c, nn, lda, sta)                                                      \
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
      "add.rn.f64 %0, %0, %13;\n\tst.shared.f64 [%18+32], %0;\n\t"                         \
      "add.rn.f64 %0, %0, %14;\n\tst.shared.f64 [%18+40], %0;\n\t"                         \
      "add.rn.f64 %0, %0, %15;\n\tst.shared.f64 [%18+48], %0;\n\t"                         \
      "add.rn.f64 %0, %0, %16;\n\tst.shared.f64 [%18+56], %0;\n\t"                         \
      "}"                                                                                   \
      : "+d"(acc), "=&d"(nn[0]), "=&d"(nn[1]), "=&d"(nn[2]), "=&d"(nn[3]), "=&d"(nn[4]),   \
        "=&d"(nn[5]), "=&d"(nn[6]), "=&d"(nn[7])                                           \
      : "d"(c[0]), "d"(c[1]), "d"(c[2]), "d"(c[3]), "d"(c[4]), "d"(c[5]), "d"(c[6]),       \
        "d"(c[7]), "r"(lda), "r"(sta)                                                      \
      : "memory")


static __device__ __noinline__ void chain_nv(uint32_t s, uint32_t d, int n, double init) {
  double acc = init;
  const int n2 = n - n % 16;
  double A[8], Bv[8];
  for (int k = 0; k < 8; ++k) A[k] = lds64(s + 8 * k);
  for (int i = 0; i < n2; i += 16) {
    CS8NV(acc, A, Bv, s + 8 * (i + 8), d + 8 * i);
    const uint32_t nxt = i + 16 < n2 ? s + 8 * (i + 16) : s;
    CS8NV(acc, Bv, A, nxt, d + 8 * (i + 8));
  }
}
static __device__ __noinline__ void chain_v2(uint32_t s, uint32_t d, int n, double init) {
  double acc = init;
  const int n2 = n - n % 16;
  double A[8], Bv[8];
  for (int k = 0; k < 8; ++k) A[k] = lds64(s + 8 * k);
  for (int i = 0; i < n2; i += 16) {
    CS8V(acc, A, Bv, s + 8 * (i + 8), d + 8 * i);
    const uint32_t nxt = i + 16 < n2 ? s + 8 * (i + 16) : s;
    CS8V(acc, Bv, A, nxt, d + 8 * (i + 8));
  }
}

template <int V>
__global__ void __launch_bounds__(256, 2) bench(double* out, long long* t, int n, double y) {
  extern __shared__ __align__(16) double sm[];
  for (int i = threadIdx.x; i < n; i += blockDim.x) sm[i] = y * ((i * 7) % 17 - 8) * 1e-5;
  __syncthreads();
  long long c0 = clock64();
  if (V == 0) smem_cumsum(sm, sm, n);
  if (V == 1) cumsum_v2(sm, sm, n);
  if (V == 2) cumsum_warp(sm, sm, n);
  if (V == 3) cumsum_bcast(sm, sm, n);
  if (V == 5 && threadIdx.x == 0) chain_nv((uint32_t)__cvta_generic_to_shared(sm), (uint32_t)__cvta_generic_to_shared(sm), n, -0.0);
  if (V == 6 && threadIdx.x == 0) chain_v2((uint32_t)__cvta_generic_to_shared(sm), (uint32_t)__cvta_generic_to_shared(sm), n, -0.0);
  if (V == 4 && threadIdx.x < 32) cumsum_bcast2((uint32_t)__cvta_generic_to_shared(sm), (uint32_t)__cvta_generic_to_shared(sm), n, -0.0);
  __syncthreads();
  long long c1 = clock64();
  if (threadIdx.x == 0) {
    t[0] = c1 - c0;
    double chk = 0.0;
    for (int i = 0; i < n; i += 97) chk += sm[i];
    out[0] = chk + sm[n - 1];
  }
}

int main() {
  double* out;
  long long* t;
  cudaMallocManaged(&out, 8);
  cudaMallocManaged(&t, 8 * 8);
  for (int n : {256, 1024, 8192}) {
    const int smem = n * 8;
    double ref = 0;
    for (int v = 0; v < 7; ++v) {
      for (int rep = 0; rep < 2; ++rep) {
        if (v == 0) { cudaFuncSetAttribute(bench<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); bench<0><<<1, 256, smem>>>(out, t, n, 1.0000001); }
        if (v == 1) { cudaFuncSetAttribute(bench<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); bench<1><<<1, 256, smem>>>(out, t, n, 1.0000001); }
        if (v == 2) { cudaFuncSetAttribute(bench<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); bench<2><<<1, 256, smem>>>(out, t, n, 1.0000001); }
        if (v == 3) { cudaFuncSetAttribute(bench<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); bench<3><<<1, 256, smem>>>(out, t, n, 1.0000001); }
        if (v == 4) { cudaFuncSetAttribute(bench<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); bench<4><<<1, 256, smem>>>(out, t, n, 1.0000001); }
        if (v == 5) { cudaFuncSetAttribute(bench<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); bench<5><<<1, 256, smem>>>(out, t, n, 1.0000001); }
        if (v == 6) { cudaFuncSetAttribute(bench<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); bench<6><<<1, 256, smem>>>(out, t, n, 1.0000001); }
        cudaDeviceSynchronize();
      }
      if (v == 0) ref = out[0];
      printf("n=%d variant %d: %.2f cycles/elt, checksum %s (%.17g)\n", n, v, (double)t[0] / n,
             out[0] == ref ? "equal" : "DIFFERENT", out[0]);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
