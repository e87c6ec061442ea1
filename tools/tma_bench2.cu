// Multi-lane cp.async.bulk issue: L lanes of one warp each issue one 1 KiB
// row copy per iteration into its own padded slot (one mbarrier per group of
// L rows, expect_tx = L KiB).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k(const double* g, int nrow, int L, long long* out) {
  extern __shared__ __align__(16) unsigned char sm[];
  constexpr int S = 8;           // groups in flight
  uint64_t* mb = (uint64_t*)sm;
  double* ring = (double*)(sm + 1024);
  const int rowd = 128, RS = 136;
  for (int i = threadIdx.x; i < S; i += blockDim.x) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(mb + i)));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  const int lane = threadIdx.x;
  long long c0 = clock64();
  const int ng = nrow / L;
  for (int q = 0; q < ng; ++q) {
    const int slot = q % S;
    const uint32_t m = su32(mb + slot);
    if (q >= S) {
      uint32_t par = ((q - S) / S) & 1, ok;
      do { asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }" : "=r"(ok) : "r"(m), "r"(par) : "memory"); } while (!ok);
    }
    if (lane == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(m), "r"(L * rowd * 8) : "memory");
    __syncwarp();
    if (lane < L) {
      const double* src = g + ((size_t)blockIdx.x * nrow + q * L + lane) * rowd;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
                   "r"(su32(ring + ((size_t)slot * 8 + lane) * RS)), "l"(src), "r"(rowd * 8), "r"(m) : "memory");
    }
  }
  for (int q = ng - S; q < ng; ++q) {
    if (q < 0) continue;
    const int slot = q % S; uint32_t m = su32(mb + slot), par = (q / S) & 1, ok;
    do { asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }" : "=r"(ok) : "r"(m), "r"(par) : "memory"); } while (!ok);
  }
  long long c1 = clock64();
  if (blockIdx.x == 0 && lane == 0) out[0] = (c1 - c0) / ng;
}

int main() {
  const int nrow = 4096;
  double* g; long long* o; long long h = 0;
  if (cudaMalloc(&g, (size_t)296 * nrow * 1024 + (1 << 20)) != cudaSuccess) return 1;
  cudaMalloc(&o, 8);
  const int smem = 1024 + 8 * 8 * 136 * 8;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int Ls[4] = {1, 2, 4, 8}, nbs[3] = {1, 148, 296};
  for (int li = 0; li < 4; ++li)
    for (int bi = 0; bi < 3; ++bi) {
      const int L = Ls[li], nb = nbs[bi];
      k<<<nb, 32, smem>>>(g, nrow, L, o);
      if (cudaDeviceSynchronize() != cudaSuccess) { printf("fault\n"); return 1; }
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0);
      k<<<nb, 32, smem>>>(g, nrow, L, o);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      cudaMemcpy(&h, o, 8, cudaMemcpyDeviceToHost);
      printf("lanes %d blocks %3d: %lld cycles per group of %d rows, %.1f GB/s\n", L, nb, h, L,
             (double)nb * nrow * 1024 / (ms * 1e-3) / 1e9);
    }
  return 0;
}
