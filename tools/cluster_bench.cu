// Cluster barrier vs mbarrier signalling latency (8-CTA clusters).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/cluster_bench tools/cluster_bench.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void __cluster_dims__(8, 1, 1) bench(long long* t, int reps) {
  __shared__ __align__(8) unsigned long long mb;
  cg::cluster_group cl = cg::this_cluster();
  const unsigned rank = cl.block_rank();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(&mb)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cl.sync();
  long long c0 = clock64();
  for (int r = 0; r < reps; ++r) cl.sync();
  long long c1 = clock64();
  // ping: rank 0 arrives remotely on every other CTA's mbarrier, they wait (phase r)
  for (int r = 0; r < reps; ++r) {
    if (rank == 0) {
      __syncthreads();
      if (threadIdx.x == 0)
        for (unsigned c = 1; c < 8; ++c) {
          const unsigned la = (unsigned)__cvta_generic_to_shared(&mb);
          unsigned ra;
          asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(c));
          asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(ra) : "memory");
        }
    } else {
      if (threadIdx.x == 0) {
        const unsigned la = (unsigned)__cvta_generic_to_shared(&mb);
        unsigned done = 0;
        while (!done)
          asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                       : "=r"(done) : "r"(la), "r"((unsigned)(r & 1)) : "memory");
      }
      __syncthreads();
    }
  }
  long long c2 = clock64();
  cl.sync();
  if (threadIdx.x == 0 && rank == 1) {
    t[0] = (c1 - c0) / reps;
    t[1] = (c2 - c1) / reps;
  }
}

int main() {
  long long* t;
  cudaMallocManaged(&t, 16);
  for (int nt : {128, 256}) {
    bench<<<8, nt>>>(t, 1000);
    cudaDeviceSynchronize();
    bench<<<8, nt>>>(t, 1000);
    cudaDeviceSynchronize();
    printf("threads %d: cluster.sync %lld cycles; rank-0 -> mbarrier release/acquire round %lld cycles\n", nt, t[0], t[1]);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
