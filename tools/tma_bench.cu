// cp.async.bulk issue-rate microbenchmark: one thread issues N row copies
// (row bytes B) into a ring of S slots, waiting on each slot's mbarrier
// before reuse.  Reports cycles per issued copy.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int S>
__global__ void k(const double* g, int nrow, int rowd, long long* out, int per_copy_rows) {
  extern __shared__ __align__(16) unsigned char sm[];
  uint64_t* mb = (uint64_t*)sm;
  double* ring = (double*)(sm + 1024);
  for (int i = threadIdx.x; i < S; i += blockDim.x) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(mb + i)));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  if (threadIdx.x != 0) return;
  const uint32_t bytes = rowd * 8 * per_copy_rows;
  long long c0 = clock64();
  int nq = nrow / per_copy_rows;
  for (int q = 0; q < nq; ++q) {
    int slot = q % S;
    uint32_t m = su32(mb + slot);
    if (q >= S) {
      uint32_t par = ((q - S) / S) & 1, ok;
      do { asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }" : "=r"(ok) : "r"(m), "r"(par) : "memory"); } while (!ok);
    }
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(m), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
                 "r"(su32(ring + (size_t)slot * rowd * per_copy_rows)), "l"(g + (size_t)((q * per_copy_rows) % 100000) * rowd * 0 + (size_t)(blockIdx.x * 4096 + q * per_copy_rows) * rowd), "r"(bytes), "r"(m) : "memory");
  }
  for (int q = nq - S; q < nq; ++q) {
    if (q < 0) continue;
    int slot = q % S; uint32_t m = su32(mb + slot), par = (q / S) & 1, ok;
    do { asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }" : "=r"(ok) : "r"(m), "r"(par) : "memory"); } while (!ok);
  }
  long long c1 = clock64();
  if (blockIdx.x == 0) out[0] = (c1 - c0) / nq;
}

int main() {
  const int rowd = 128, nrow = 4096, blocks = 296;
  double* g; long long* o; long long h = 0;
  if (cudaMalloc(&g, (size_t)blocks * nrow * rowd * 8 + (1 << 20)) != cudaSuccess) return 1;
  cudaMalloc(&o, 8);
  const int smem = 1024 + 40 * rowd * 8;  // 40 rows of ring in every case
  cudaFuncSetAttribute(k<40>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<20>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<10>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int pcrs[4] = {1, 2, 4, 8};
  for (int pi = 0; pi < 4; ++pi) {
    const int pcr = pcrs[pi];
    int nbs[3] = {1, 148, 296};
    for (int bi = 0; bi < 3; ++bi) {
      const int nb = nbs[bi];
      auto launch = [&]() {
        if (pcr == 1) k<40><<<nb, 32, smem>>>(g, nrow, rowd, o, pcr);
        else if (pcr == 2) k<20><<<nb, 32, smem>>>(g, nrow, rowd, o, pcr);
        else if (pcr == 4) k<10><<<nb, 32, smem>>>(g, nrow, rowd, o, pcr);
        else k<5><<<nb, 32, smem>>>(g, nrow, rowd, o, pcr);
      };
      launch();
      if (cudaDeviceSynchronize() != cudaSuccess) { printf("fault\n"); return 1; }
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      cudaMemcpy(&h, o, 8, cudaMemcpyDeviceToHost);
      double gbs = (double)nb * nrow * rowd * 8 / (ms * 1e-3) / 1e9;
      printf("rows/copy %d blocks %3d: %lld cycles per copy, %.1f GB/s  (err %s)\n", pcr, nb, h, gbs, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
