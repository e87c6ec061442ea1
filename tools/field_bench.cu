// Cycle counts of the exact field solve's variants on one CTA with the slice
// vectors in shared memory (diagnostic for the slice phase and the chain
// kernel): the pass-by-pass sequence, field_exact_onchip (shuffle trees).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -o tools/field_bench tools/field_bench.cu
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <cuda_runtime.h>
#include <vector>

#include "../paper_2511_13386_b200/csrc/pk_device.cuh"

using namespace pk;

// pass-by-pass (slice_field's generic exact path)
__device__ bool field_passes(const double* rho, double* x, int nx, double dx, const PwPlan& P,
                             double* red, double& mean) {
  double defect, abssum;
  block_pairwise2([&](int i) { return x[i]; }, [&](int i) { return fabs(rho[i]); }, P, red, defect,
                  abssum);
  if (fabs(defect) > 1e300 * fmax(abssum * dx, 1e-300)) return false;
  const double corr = defect / (double)nx;
  for (int i = threadIdx.x; i < nx; i += blockDim.x) x[i] = x[i] - corr;
  __syncthreads();
  smem_cumsum(x, x, nx);
  __syncthreads();
  mean = block_pairwise([&](int i) { return x[i]; }, P, red) / (double)nx;
  return true;
}

__device__ long long g_st[4];

__global__ void bench(const PwPlan* gP, double* out, long long* t, int nx, int reps) {
  extern __shared__ double sm[];
  __shared__ PwPlan P;
  double* rho = sm;
  double* x = sm + nx;
  double* red = sm + 2 * nx;
  if (threadIdx.x == 0) P = *gP;
  for (int i = threadIdx.x; i < nx; i += blockDim.x) rho[i] = 1.0 + 0.3 * sin(0.01 * i);
  __syncthreads();
  const double dx = 0.0245;
  double acc = 0.0;
  for (int v = 0; v < 2; ++v) {
    long long tot = 0;
    for (int r = 0; r < reps; ++r) {
      for (int i = threadIdx.x; i < nx; i += blockDim.x) x[i] = (rho[i] - 1.0) * dx;
      __syncthreads();
      const long long c0 = clock64();
      double mean = 0.0;
      bool ok;
      if (v == 0) ok = field_passes(rho, x, nx, dx, P, red, mean);
      else ok = field_exact_onchip([&](int i) { return fabs(rho[i]); }, x, nx, dx, 1e300, P, red, mean, g_st);
      __syncthreads();
      tot += clock64() - c0;
      acc += ok ? mean + x[nx - 1] : 0.0;
    }
    if (threadIdx.x == 0) t[v] = tot / reps;
  }
  if (threadIdx.x == 0) out[0] = acc;
}

// numpy pairwise plan (same construction as pk_api.cu build_plan)
struct PB {
  std::vector<int> lo, ll;
  struct N { int a, b, lev; };
  std::vector<N> nd;
  std::pair<int, int> rec(int off, int n) {
    if (n <= 128) { lo.push_back(off); ll.push_back(n); return {(int)lo.size() - 1, 0}; }
    int n2 = n / 2; n2 -= n2 % 8;
    auto l = rec(off, n2); auto r = rec(off + n2, n - n2);
    int lev = std::max(l.second, r.second) + 1;
    nd.push_back({l.first, r.first, lev});
    return {~((int)nd.size() - 1), lev};
  }
};

static void plan(int n, PwPlan* P) {
  PB pb; pb.rec(0, n);
  const int nl = (int)pb.lo.size(), nn = (int)pb.nd.size();
  memset(P, 0, sizeof(*P));
  P->n = n; P->nleaf = nl; P->nnode = nn;
  for (int i = 0; i < nl; ++i) { P->leaf_off[i] = pb.lo[i]; P->leaf_len[i] = pb.ll[i]; }
  int ml = 0; for (auto& x : pb.nd) ml = std::max(ml, x.lev);
  std::vector<int> ord(nn), slot(nn);
  for (int i = 0; i < nn; ++i) ord[i] = i;
  std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return pb.nd[a].lev < pb.nd[b].lev; });
  for (int i = 0; i < nn; ++i) slot[ord[i]] = i;
  auto op = [&](int id) { return id >= 0 ? id : nl + slot[~id]; };
  for (int i = 0; i < nn; ++i) { P->node_a[i] = op(pb.nd[ord[i]].a); P->node_b[i] = op(pb.nd[ord[i]].b); }
  P->nlevel = ml;
  for (int l = 1; l <= ml; ++l) { int e = 0; for (int i = 0; i < nn; ++i) if (pb.nd[ord[i]].lev <= l) e = i + 1; P->level_end[l - 1] = e; }
  P->perfect = (nl & (nl - 1)) == 0 && (1 << ml) == nl;  // (power-of-two nx only here)
}

int main() {
  double* out; long long* t; PwPlan* dP;
  cudaMalloc(&out, 8); cudaMalloc(&t, 64); cudaMalloc(&dP, sizeof(PwPlan));
  for (int nx : {256, 512, 1024, 8192})
    for (int nt : {128, 256, 512}) {
      PwPlan P; plan(nx, &P);
      cudaMemcpy(dP, &P, sizeof(P), cudaMemcpyHostToDevice);
      const int smem = (2 * nx + 2 * (MAX_LEAF + MAX_NODE)) * 8;
      cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      bench<<<1, nt, smem>>>(dP, out, t, nx, 20);
      long long h[2];
      cudaError_t e = cudaMemcpy(h, t, sizeof(h), cudaMemcpyDeviceToHost);
      long long st[4], z[4] = {0, 0, 0, 0};
      cudaMemcpyFromSymbol(st, g_st, sizeof(st));
      cudaMemcpyToSymbol(g_st, z, sizeof(z));
      printf("   onchip stages per call: sums %lld corr %lld chain %lld mean %lld\n", st[0] / 20, st[1] / 20, st[2] / 20, st[3] / 20);
      printf("nx %5d NT %3d: passes %7lld  onchip %7lld cycles (%s)\n", nx, nt, h[0], h[1],
             cudaGetErrorString(e));
    }
  return 0;
}
