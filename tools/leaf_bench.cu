// Cycle counts of one numpy pairwise leaf (128 terms, 8 accumulators) on the
// device: group_leaf through a generic pointer vs shared-window loads.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -o tools/leaf_bench tools/leaf_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2511_13386_b200/csrc/pk_device.cuh"

using namespace pk;

__global__ void bench(double* out, long long* t, int reps) {
  __shared__ double x[1024];  // (x[512..] holds the plan below)
  for (int i = threadIdx.x; i < 512; i += blockDim.x) x[i] = 1e-3 * (i % 13) - 0.004;
  __syncthreads();
  double acc = 0.0;
  double* volatile gp = x;  // opaque generic pointer
  const double* xp = gp;
  long long c0 = clock64();
  for (int r = 0; r < reps; ++r) {
    const double v = group_leaf([&](int i) { return xp[i]; }, 0, 128, true);
    acc += v;
    __syncwarp();
  }
  long long c1 = clock64();
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(x);
  for (int r = 0; r < reps; ++r) {
    const double v = group_leaf([&](int i) { return lds64(s + 8 * i); }, 0, 128, true);
    acc += v;
    __syncwarp();
  }
  long long c2 = clock64();
  for (int r = 0; r < reps; ++r) {  // 2 sums interleaved (defect + |rho|)
    const double v = group_leaf([&](int i) { return xp[i]; }, 0, 128, true);
    const double w = group_leaf([&](int i) { return fabs(xp[i + 128]); }, 0, 128, true);
    acc += v + w;
    __syncwarp();
  }
  long long c3 = clock64();
  // the field's pw_perfect (nx = 256: two leaves) and the chain before it
  PwPlan& P = *reinterpret_cast<PwPlan*>(x + 512);  // (plan in shared memory)
  if (threadIdx.x == 0) {
    P.n = 256; P.nleaf = 2; P.nnode = 1; P.nlevel = 1; P.perfect = 1;
    P.leaf_off[0] = 0; P.leaf_len[0] = 128; P.leaf_off[1] = 128; P.leaf_len[1] = 128;
    P.node_a[0] = 0; P.node_b[0] = 1; P.level_end[0] = 1;
  }
  __syncthreads();
  double red[8];
  long long c4 = clock64();
  for (int r = 0; r < reps; ++r) {
    double mm[1];
    pw_perfect<1>([&](int, int i) { return xp[i]; }, P, red, mm);
    acc += mm[0];
  }
  long long c5 = clock64();
  for (int r = 0; r < reps; ++r) {
    double mm[2];
    pw_perfect<2>([&](int s2, int i) { return s2 ? fabs(xp[i + 256]) : xp[i]; }, P, red, mm);
    acc += mm[0] + mm[1];
  }
  long long c6 = clock64();
  for (int r = 0; r < reps; ++r) {
    smem_cumsum(gp, gp, 256);
    __syncthreads();
    double mm[1];
    pw_perfect<1>([&](int, int i) { return xp[i]; }, P, red, mm);
    acc += mm[0];
  }
  long long c7 = clock64();
  for (int r = 0; r < reps; ++r) {
    smem_cumsum(gp, gp, 256);
    __syncthreads();
  }
  long long c8 = clock64();
  if (threadIdx.x == 0) {
    t[3] = (c5 - c4) / reps;
    t[4] = (c6 - c5) / reps;
    t[5] = (c7 - c6) / reps;
    t[6] = (c8 - c7) / reps;
    t[0] = (c1 - c0) / reps;
    t[1] = (c2 - c1) / reps;
    t[2] = (c3 - c2) / reps;
  }
  out[threadIdx.x] = acc;
}

int main() {
  double* out;
  long long* t;
  cudaMalloc(&out, 1024 * 8);
  cudaMallocManaged(&t, 8 * 8);
  for (int nt : {32, 128}) {
    bench<<<1, nt>>>(out, t, 100);
    cudaDeviceSynchronize();
    bench<<<1, nt>>>(out, t, 100);
    cudaDeviceSynchronize();
    printf("threads %d: group_leaf generic %lld, shared-window %lld, two leaves %lld cycles; "
           "pw_perfect<1> %lld, <2> %lld; chain+bar+mean %lld, chain+bar %lld\n", nt,
           t[0], t[1], t[2], t[3], t[4], t[5], t[6]);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
