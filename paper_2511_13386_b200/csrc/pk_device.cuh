// Device helpers shared by the fine-propagator, coarse-propagator and lift
// kernels.  Compiled with --fmad=false: every multiply and add below rounds
// separately, exactly like numpy; fused multiply-adds appear only where they
// are written out explicitly (__fma_rn in qdiv).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace pk {

constexpr unsigned FULL = 0xffffffffu;
constexpr int MAX_LEAF = 80;    // pairwise leaves of <= 128 terms: nx <= 10240
constexpr int MAX_NODE = 80;
constexpr int MAX_LEVEL = 10;

// x / d from rd = RN(1/d) with one Markstein correction step: the correctly
// rounded IEEE quotient for every |x| >= 2^-960 (d here is a mesh spacing,
// 2^-14 < d < 1).  Below that the residual r = x - q d leaves the normal
// range and the step can miss the rounding (subnormal and near-subnormal
// numerators), and a -0.0 numerator gives +0.0.  Checked bit for bit against
// IEEE division: on the CPU, 2e6 operands per spacing 2 pi / nx for 12 nx
// (tests/test_native_host.py); on the device, through pk_diag_qdiv, 2^20
// operands per spacing for 14 (nx, x*) pairs over the whole exponent range
// (tests/test_gpu_parity.py::test_qdiv_matches_ieee_division_on_device:
// identical above 2^-960; every difference found lies below it or is -0.0).
// The numerators are differences of g values (kinetic.py:173) and of
// densities (fluid.py:51) -- never that small in these models; a guard for
// them (an integer exponent test + an IEEE division on the rare path) cost
// 25 % of the cfg5 throughput, so a build with -DPK_TRUE_DIV is the exact
// everywhere alternative.
__device__ __forceinline__ double qdiv(double x, double d, double rd) {
#ifdef PK_TRUE_DIV
  return x / d;
#else
  double q = x * rd;
  double r = __fma_rn(-q, d, x);
  return __fma_rn(r, rd, q);
#endif
}

// profiling counters: a fire-and-forget reduction (no load round trip on
// the profiled thread's timeline)
__device__ __forceinline__ void pk_red_add(long long* p, long long v) {
  atomicAdd(reinterpret_cast<unsigned long long*>(p), (unsigned long long)v);
}

// numpy pairwise-summation plan for an n-term reduction (numpy's
// pairwise_sum: <8 sequential, <=128 eight accumulators, else split at
// n/2 rounded down to a multiple of 8).  Leaves in order, internal nodes
// bottom-up by level; built on the host (pk_api.cu) per n.
struct PwPlan {
  int n, nleaf, nnode, nlevel;
  int leaf_off[MAX_LEAF];
  int leaf_len[MAX_LEAF];
  int node_a[MAX_NODE];      // operand indices into vals[nleaf + nnode]
  int node_b[MAX_NODE];
  int level_end[MAX_LEVEL];  // nodes [level_end[l-1], level_end[l]) form level l
  int perfect;               // 2^L leaves combined as adjacent pairs level by level
};

// One pairwise leaf (n <= 128) over x[off .. off+n) computed by a whole warp;
// every lane returns the same bits.  Lanes 8..31 duplicate lanes 0..7's
// accumulators so the butterfly stays within groups of eight.
template <class F>
__device__ __forceinline__ double warp_leaf(F x, int off, int n, int lane) {
  if (n < 8) {
    double r = -0.0;
    for (int i = 0; i < n; ++i) r = r + x(off + i);
    return r;
  }
  const int k = lane & 7;
  const int full = n - (n % 8);
  double r = x(off + k);
  for (int i = 8; i < full; i += 8) r = r + x(off + i + k);
  r = r + __shfl_xor_sync(FULL, r, 1);
  r = r + __shfl_xor_sync(FULL, r, 2);
  r = r + __shfl_xor_sync(FULL, r, 4);
  for (int i = full; i < n; ++i) r = r + x(off + i);
  return r;
}

// One pairwise leaf per group of eight lanes (four leaves per warp at once).
// `act`: this group has a leaf.  Same bits in the eight lanes of a group.
template <class F>
__device__ __forceinline__ double group_leaf(F x, int off, int n, bool act) {
  const int k = threadIdx.x & 7;
  double r = 0.0, seq = -0.0;
  int full = 0;
  if (act) {
    if (n == 128) {  // full leaf: the 16 operands load back to back, then the chain
      full = 128;
      double t[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) t[j] = x(off + 8 * j + k);
      r = t[0];
#pragma unroll
      for (int j = 1; j < 16; ++j) r = r + t[j];
    } else if (n < 8) {
      for (int i = 0; i < n; ++i) seq = seq + x(off + i);
    } else {
      full = n - (n % 8);
      r = x(off + k);
      for (int i = 8; i < full; i += 8) r = r + x(off + i + k);
    }
  }
  r = r + __shfl_xor_sync(FULL, r, 1);
  r = r + __shfl_xor_sync(FULL, r, 2);
  r = r + __shfl_xor_sync(FULL, r, 4);
  if (act && n >= 8)
    for (int i = full; i < n; ++i) r = r + x(off + i);
  return (act && n < 8) ? seq : r;
}

// Block-wide pairwise sum following a plan.  `scratch` is shared memory of at
// least nleaf + nnode doubles.  Every thread of the block must call it; every
// thread gets the result.
template <class F>
__device__ double block_pairwise(F x, const PwPlan& P, double* scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarp = blockDim.x >> 5;
  for (int l0 = 4 * warp; l0 < P.nleaf; l0 += 4 * nwarp) {
    const int l = l0 + (lane >> 3);
    const bool act = l < P.nleaf;
    const double v = group_leaf(x, act ? P.leaf_off[l] : 0, act ? P.leaf_len[l] : 0, act);
    if (act && (lane & 7) == 0) scratch[l] = v;
  }
  __syncthreads();
  int start = 0;
  for (int lev = 0; lev < P.nlevel; ++lev) {
    const int end = P.level_end[lev];
    for (int j = start + threadIdx.x; j < end; j += blockDim.x)
      scratch[P.nleaf + j] = scratch[P.node_a[j]] + scratch[P.node_b[j]];
    __syncthreads();
    start = end;
  }
  // root: the single leaf, or the last internal node
  const double res = scratch[P.nnode == 0 ? 0 : P.nleaf + P.nnode - 1];
  __syncthreads();
  return res;
}

// Two pairwise sums over the same plan in one sweep (defect and scale of
// poisson.py:42-43).  `scratch` holds 2 (nleaf + nnode) doubles.
template <class F1, class F2>
__device__ void block_pairwise2(F1 x1, F2 x2, const PwPlan& P, double* scratch, double& r1,
                                double& r2) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarp = blockDim.x >> 5;
  const int W = P.nleaf + P.nnode;
  // 2 nleaf leaf tasks (both sums) spread over all 8-lane groups
  for (int t0 = 4 * warp; t0 < 2 * P.nleaf; t0 += 4 * nwarp) {
    const int t = t0 + (lane >> 3);
    const bool act = t < 2 * P.nleaf;
    const bool second = act && t >= P.nleaf;
    const int l = second ? t - P.nleaf : t;
    const int off = act ? P.leaf_off[l] : 0, n = act ? P.leaf_len[l] : 0;
    const double v = group_leaf([&](int i) { return second ? x2(i) : x1(i); }, off, n, act);
    if (act && (lane & 7) == 0) scratch[second ? W + l : l] = v;
  }
  __syncthreads();
  int start = 0;
  for (int lev = 0; lev < P.nlevel; ++lev) {
    const int end = P.level_end[lev];
    for (int j = start + threadIdx.x; j < end; j += blockDim.x) {
      scratch[P.nleaf + j] = scratch[P.node_a[j]] + scratch[P.node_b[j]];
      scratch[W + P.nleaf + j] = scratch[W + P.node_a[j]] + scratch[W + P.node_b[j]];
    }
    __syncthreads();
    start = end;
  }
  const int root = P.nnode == 0 ? 0 : P.nleaf + P.nnode - 1;
  r1 = scratch[root];
  r2 = scratch[W + root];
  __syncthreads();
}

// Sequential prefix sum (np.cumsum order) of src into dst by thread 0 of the
// block.  Operands are software-pipelined through two alternating register
// blocks (the next block is loaded while the current one is summed), so the
// only serial dependency is the add chain itself.  Other threads return.
template <class FS, class FD>
__device__ __forceinline__ void warp_cumsum(FS src, FD dst, int n) {
  if (threadIdx.x != 0) return;
  constexpr int K = 8;
  double acc = -0.0;  // -0.0 + t == t bitwise: out[0] = src[0]
  const int n2 = n - n % (2 * K);
  double A[K], Bv[K];
  if (n2 > 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) A[k] = src(k);
  }
  for (int i = 0; i < n2; i += 2 * K) {
#pragma unroll
    for (int k = 0; k < K; ++k) Bv[k] = src(i + K + k);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      acc = acc + A[k];
      dst(i + k, acc);
    }
    if (i + 2 * K < n2) {
#pragma unroll
      for (int k = 0; k < K; ++k) A[k] = src(i + 2 * K + k);
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
      acc = acc + Bv[k];
      dst(i + K + k, acc);
    }
  }
  for (int i = n2; i < n; ++i) {
    acc = acc + src(i);
    dst(i, acc);
  }
}

__device__ __forceinline__ double lds64(uint32_t a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}

__device__ __forceinline__ void sts64(uint32_t a, double v) {
  asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}

// Eight elements of the smem_cumsum chain in one asm block: the next block's
// eight operands are loaded first (into n*), then acc += c_k and the running
// sum is stored, k = 0..7.  One block keeps the compiler from sinking the
// loads next to their adds, which it does under register pressure (kernels
// capped at 128 registers) and which doubles the chain's cost.  (Volatile
// accesses, which ptxas keeps in program order, cost 1.5 cycles per element:
// tools/cumsum_bench2.cu.)
#define PK_CS8(acc, c, nn, lda, sta)                                                      \
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

// warp_cumsum for operands that live in shared memory (dst may alias src:
// every operand is loaded before its slot is overwritten).  Two blocks of
// eight operands alternate (ping-pong, no register copies): one block's adds
// run while the other block's loads are in flight, so the only serial
// dependency is the add chain (~8 cycles per element, tools/cumsum_bench.cu).
// Keep the operand a plain load: an extra DADD per element (e.g. a fused
// subtrahend) doubles the cost.  Thread 0 only.  `init`: the chain's carry
// (-0.0 starts np.cumsum: -0 + x == x for every x).
static __device__ __forceinline__ void smem_cumsum_body(uint32_t s, uint32_t d, int n, double init);

__device__ __forceinline__ void smem_cumsum(const double* src, double* dst, int n,
                                            double init = -0.0) {
  if (threadIdx.x != 0) return;
  smem_cumsum_body((uint32_t)__cvta_generic_to_shared(src),
                          (uint32_t)__cvta_generic_to_shared(dst), n, init);
}

// The same chain as a function call, for kernels under register pressure:
// compiled on its own it keeps the schedule it has in isolation (9.0 cycles
// per element, tools/cumsum_bench2.cu); inlined into the 128-register hybrid
// kernels the same code ran at 12.5 (the block's loads and stores sharing
// scoreboards with the chain operands).  Elsewhere the inlined form is the
// faster one (8.5).
static __device__ __noinline__ void smem_cumsum_chain(uint32_t s, uint32_t d, int n, double init) {
  smem_cumsum_body(s, d, n, init);
}

__device__ __forceinline__ void smem_cumsum_call(const double* src, double* dst, int n,
                                                 double init = -0.0) {
  if (threadIdx.x != 0) return;
  smem_cumsum_chain((uint32_t)__cvta_generic_to_shared(src), (uint32_t)__cvta_generic_to_shared(dst),
                    n, init);
}

static __device__ __forceinline__ void smem_cumsum_body(uint32_t s, uint32_t d, int n, double init) {
  double acc = init;
  const int n2 = n - n % 16;
  if (n2 > 0) {
    double A[8], Bv[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) A[k] = lds64(s + 8 * k);
    for (int i = 0; i < n2; i += 16) {
      PK_CS8(acc, A, Bv, s + 8 * (i + 8), d + 8 * i);
      // the last block re-reads the first eight operands (harmless, unused)
      const uint32_t nxt = i + 16 < n2 ? s + 8 * (i + 16) : s;
      PK_CS8(acc, Bv, A, nxt, d + 8 * (i + 8));
    }
  }
#pragma unroll 1
  for (int i = n2; i < n; ++i) {
    acc = acc + lds64(s + 8 * i);
    sts64(d + 8 * i, acc);
  }
}

// Pairwise sums over a PERFECT plan (P.perfect: 2^L leaves, combined as
// adjacent pairs level by level -- every nx = 2^k x (<= 128)): one leaf per
// 8-lane group (group_leaf), the tree by xor butterflies.  a + b == b + a
// bitwise, so the butterfly's lane order gives numpy's node values exactly.
// NS sums of the same plan (x(s, i), s < NS); every thread gets the results.
// NS nleaf <= 4: every warp sums all the leaves itself -- no shared memory,
// no barrier.  Else the leaves are dealt over the warps, the 4-leaf subtrees
// meet in `scr` (NS nleaf / 4 doubles) behind ONE barrier and every warp
// finishes the tree itself; the caller keeps a barrier between this call's
// reads of scr and the next writes to it.
// One full numpy leaf of 128 terms at x(off ..) per 8-lane group: eight
// interleaved accumulators (16 operands loaded back to back), the 8-way
// butterfly.  group_leaf's n == 128 case with the length known at compile time.
template <class F>
__device__ __forceinline__ double leaf128(F x, int off) {
  const int k = threadIdx.x & 7;
  double t[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) t[j] = x(off + 8 * j + k);
  double r = t[0];
#pragma unroll
  for (int j = 1; j < 16; ++j) r = r + t[j];
  r = r + __shfl_xor_sync(FULL, r, 1);
  r = r + __shfl_xor_sync(FULL, r, 2);
  r = r + __shfl_xor_sync(FULL, r, 4);
  return r;
}

template <int NS, class F>
__device__ __forceinline__ void pw_perfect(F x, const PwPlan& P, double* scr, double (&res)[NS]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  const int nl = P.nleaf, ntask = NS * nl;
  const int lg = __ffs(nl) - 1;                // nl = 2^lg
  const bool full = P.n == (nl << 7);          // every leaf 128 terms: leaf l at 128 l
  auto leaf = [&](int s, int l, bool act) {
    return full ? leaf128([&](int i) { return x(s, i); }, l << 7)
                : group_leaf([&](int i) { return x(s, i); }, act ? P.leaf_off[l] : 0,
                             act ? P.leaf_len[l] : 0, act);
  };
  if (ntask <= 4) {
    const int t = lane >> 3;
    const bool act = t < ntask;
    const int s = act ? t >> lg : 0, l = act ? t - (s << lg) : 0;
    double v = leaf(s, act ? l : 0, act);
    if (nl >= 2) v = v + __shfl_xor_sync(FULL, v, 8);
    if (nl >= 4) v = v + __shfl_xor_sync(FULL, v, 16);
#pragma unroll
    for (int q = 0; q < NS; ++q) res[q] = __shfl_sync(FULL, v, (8 << lg) * q);
    return;
  }
  // nl >= 4 here (a power of two): aligned groups of four leaves share a sum
  for (int t0 = 4 * warp; t0 < ntask; t0 += 4 * nwarp) {
    const int t = t0 + (lane >> 3);
    const int s = t >> lg, l = t - (s << lg);
    double v = leaf(s, l, true);
    v = v + __shfl_xor_sync(FULL, v, 8);
    v = v + __shfl_xor_sync(FULL, v, 16);
    if (lane == 0) scr[t0 >> 2] = v;
  }
  __syncthreads();
  const int nsub = nl >> 2;  // <= 16 (MAX_LEAF)
#pragma unroll
  for (int q = 0; q < NS; ++q) {
    double w = lane < nsub ? scr[q * nsub + lane] : 0.0;
    for (int o = 1; o < nsub; o <<= 1) w = w + __shfl_xor_sync(FULL, w, o);
    res[q] = __shfl_sync(FULL, w, 0);
  }
}

// Exact field (poisson.py:41-54) of a slice whose vectors are in shared
// memory: pairwise defect and sum|rho| (pw_perfect when the plan is perfect,
// else block_pairwise2), the guard, x - defect/nx, the sequential np.cumsum
// chain on thread 0, the pairwise mean.  Same operations in the same order
// as slice_field's generic path, same bits.
//   x:  in  (rho - rho_bar) dx for every cell (the caller's barrier done),
//       out the running sums E + mean (in place)
//   mean: E = x - mean is left to the caller (x - 0.0 == x: a pending shift
//       of 0 is exact)
// `red`: 2 (nleaf + nnode) doubles.  Returns false on a solvability
// violation (uniform over the block).
template <class FA>
__device__ bool field_exact_onchip(FA absrho, double* x, int nx, double dx, double rtol,
                                   const PwPlan& P, double* red, double& mean,
                                   long long* dbg = nullptr) {
  long long c0 = dbg ? clock64() : 0;
  auto tick = [&](int k) {  // optional stage profile (thread 0)
    if (dbg && threadIdx.x == 0) {
      const long long c1 = clock64();
      pk_red_add(dbg + k, c1 - c0);
      c0 = c1;
    }
  };
  double r[2];
  const uint32_t xs = (uint32_t)__cvta_generic_to_shared(x);  // x is in shared memory
  if (P.perfect)
    pw_perfect<2>([&](int s, int i) { return s ? absrho(i) : lds64(xs + 8 * i); }, P, red, r);
  else
    block_pairwise2([&](int i) { return x[i]; }, absrho, P, red, r[0], r[1]);
  tick(0);
  if (fabs(r[0]) > rtol * fmax(r[1] * dx, 2.2250738585072014e-308)) return false;
  const double corr = r[0] / (double)nx;
  for (int i = threadIdx.x; i < nx; i += blockDim.x) x[i] = x[i] - corr;
  __syncthreads();
  tick(1);
  smem_cumsum(x, x, nx);
  __syncthreads();
  tick(2);
  if (P.perfect) {
    double mm[1];
    pw_perfect<1>([&](int, int i) { return lds64(xs + 8 * i); }, P, red, mm);
    mean = mm[0] / (double)nx;
  } else {
    mean = block_pairwise([&](int i) { return x[i]; }, P, red) / (double)nx;
  }
  tick(3);
  return true;
}

// Work-efficient parallel prefix sum (fast mode, not bitwise): block scan with
// warp shuffles over a blocked partition.  `scratch` holds blockDim.x/32 + 1
// doubles.  Result differs from np.cumsum by O(n u |E|).
template <class FS, class FD>
__device__ void block_scan_fast(FS src, FD dst, int n, double* scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarp = blockDim.x >> 5;
  const int per = (n + blockDim.x - 1) / blockDim.x;
  const int lo = min(n, threadIdx.x * per), hi = min(n, lo + per);
  double s = 0.0;
  for (int i = lo; i < hi; ++i) s = s + src(i);
  double inc = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    double t = __shfl_up_sync(FULL, inc, o);
    if (lane >= o) inc = inc + t;
  }
  if (lane == 31) scratch[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    double w = (lane < nwarp) ? scratch[lane] : 0.0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      double t = __shfl_up_sync(FULL, w, o);
      if (lane >= o) w = w + t;
    }
    if (lane < nwarp) scratch[lane] = w;
  }
  __syncthreads();
  double run = (inc - s) + (warp > 0 ? scratch[warp - 1] : 0.0);
  for (int i = lo; i < hi; ++i) {
    run = run + src(i);
    dst(i, run);
  }
  __syncthreads();
}

__device__ __forceinline__ int wrap(int i, int n) {
  return i < 0 ? i + n : (i >= n ? i - n : i);
}

// Status record.  When several slices fail in one launch the LOWEST slice's
// error is kept (atomicMin on slice+1 | step | code): the reference consumes
// its window futures in window order, so `run` raises the lowest failing
// window's error (parareal.py:260-266).  A slice stops at its first error, so
// a slice never posts twice.  Empty record = all ones (pk_api.cu decodes it).
struct Status {
  unsigned long long key;   // (slice + 1) << 40 | (uint32)step << 8 | code
  int pad0, pad1;
};

__device__ __forceinline__ void set_status(Status* st, int code, int slice, int step) {
  const unsigned long long key = ((unsigned long long)((unsigned)(slice + 1) & 0xFFFFFFu) << 40) |
                                 ((unsigned long long)(unsigned)step << 8) |
                                 (unsigned long long)(code & 0xFF);
  atomicMin(&st->key, key);
}

}  // namespace pk
