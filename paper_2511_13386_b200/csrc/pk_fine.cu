// Fine propagator F on B200: one thread-block cluster per slice runs the
// whole window (all steps) in a single persistent launch.
//
// Per step (hybrid.py:123-188, kinetic.py:255-273):
//   micro phase   every warp of the cluster streams its share of the kinetic
//                 interface rows: TMA bulk copies (cp.async.bulk + mbarrier)
//                 feed a per-warp shared-memory ring, the warp computes
//                 g' = k1 g - k2 (upwind transport - M d_x<xi g> + xi M J)
//                 (kinetic.py:148-224) from rows i-1, i, i+1 and writes g' and
//                 the row moments <xi g'>, <g'^2>.  Only kinetic rows are
//                 visited (compacted row list).
//   cluster barrier
//   slice phase   the leader CTA, on shared-memory copies of the slice
//                 vectors: masked rho update (hybrid.py:117-119, kinetic.py:
//                 232-240, fluid.py:55-57), field solve (poisson.py:21-54), J,
//                 remainder/perturbation indicators and labels for the next
//                 step (adaptation.py:120-181), Chapman-Enskog re-initialisation
//                 of flipped rows (lifting.py:38-105), projection
//                 coefficients and the next kinetic-row list.
//   cluster barrier
// g is double-buffered in HBM/L2 (the mixed update reads stale neighbours,
// SURVEY F9).  Arithmetic follows numpy's operation order
// so results are bitwise equal to the reference.
#include <cooperative_groups.h>
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "../../include/pk.h"
#include "pk_rows.cuh"
#include "pk_big.cuh"

namespace cg = cooperative_groups;

// The file compiles either as one translation unit or, for a parallel build
// (build.py), once per PK_FINE_PART: part 0 holds the standalone operators and
// the dispatcher, parts 1.. one fine_kernel layout each.
#ifndef PK_FINE_PART
#define PK_FINE_PART -1
#endif
#define PK_IN_PART(n) (PK_FINE_PART < 0 || PK_FINE_PART == (n))

namespace pk {

// ---------------------------------------------------------------------------
// TMA bulk copy + mbarrier primitives.

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* m, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(m)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* m, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(m)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* m) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(m))
      : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* m, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_u32(m)), "r"(parity)
        : "memory");
  } while (!done);
}

__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---------------------------------------------------------------------------
// Per-slice view.  "Local" vectors belong to the leader CTA's slice phase and
// live in shared memory when they fit (else in the global workspace);
// "shared" vectors are exchanged between the CTAs of the cluster through L2.
struct SliceView {
  int b, nx, nv;
  // leader-local
  double *rho, *E, *Eprev, *J, *tA, *tB, *tC, *tD, *tE, *bm, *blift;
  uint8_t *kc, *ki, *flip, *nza, *nzb, *kcn, *kin;
  // cluster-shared (global)
  double *gJ, *dco, *vco;
  // row moments <xi g>, <g^2>: written by every warp of the cluster (fl_w /
  // sq_w: the leader's shared memory through DSMEM, or global), read by the
  // leader (fl / sq)
  double *fl, *sq, *fl_w, *sq_w;
  int8_t* vsg;
  int* klist;
  int* kpos;
  int* kstream;
  int* nk;
  int* zlist;
  int* nzl;
  int* abort_;
  double* ga;
  double* gb;
  double rb;
  // exact on-chip field: E = E[i] - Emean is still to be applied (Epend)
  double Emean;
  bool Epend;
};

// number of leader-local double / byte vectors (all-kinetic mode needs the
// first NLOC_DK / NLOC_BK only)
constexpr int NLOC_D = 13;
constexpr int NLOC_B = 7;
constexpr int NLOC_DK = 5;
constexpr int NLOC_BK = 2;

__device__ __forceinline__ void bind_shared(SliceView& v, const FineArgs& a, int b) {
  const int nx = a.m.nx;
  const size_t o = (size_t)b * nx;
  v.b = b;
  v.nx = nx;
  v.nv = a.m.nv;
  v.gJ = a.J + o;
  v.dco = a.dco + o;
  v.vco = a.vco + o;
  v.vsg = a.vsg + o;
  v.klist = a.klist + o;
  v.kpos = a.kpos + o;
  v.kstream = a.kstream + 3 * o;
  v.nk = a.nk + b;
  v.zlist = a.zlist + o;
  v.nzl = a.nzl + b;
  v.abort_ = a.abort_ + b;
  v.ga = a.ga + o * a.m.nv;
  v.gb = a.gb + o * a.m.nv;
  v.rb = a.rho_bar[b];
  v.Emean = 0.0;
  v.Epend = false;
}

// Leader-local vectors either in shared memory (loc != null: the same smem
// offset in every CTA of the cluster) or global.  In the shared-memory
// layout the micro phase writes the row moments straight into the leader's
// shared memory through DSMEM.
__device__ __forceinline__ void bind_local(SliceView& v, const FineArgs& a, int b, double* loc,
                                           bool leader, int owner) {
  const int nx = a.m.nx;
  const size_t o = (size_t)b * nx;
  if (loc) {
    const int nd = a.adaptation ? NLOC_D : NLOC_DK;
    const int nb = a.adaptation ? NLOC_B : NLOC_BK;
    double* p = loc;
    double* fl = nullptr;
    double* sq = nullptr;
    double** d[NLOC_D] = {&v.rho, &v.E, &v.Eprev, &v.J, &fl, &v.tA, &v.tB,
                          &sq, &v.tC, &v.tD, &v.tE, &v.bm, &v.blift};
    // all-kinetic mode keeps only rho, E, E_prev, J and the moments on chip
    for (int k = 0; k < NLOC_D; ++k) *d[k] = k < nd ? p + (size_t)k * nx : nullptr;
    uint8_t* q = reinterpret_cast<uint8_t*>(p + (size_t)nd * nx);
    uint8_t** e[NLOC_B] = {&v.kc, &v.ki, &v.flip, &v.nza, &v.nzb, &v.kcn, &v.kin};
    for (int k = 0; k < NLOC_B; ++k) *e[k] = k < nb ? q + (size_t)k * nx : nullptr;
    if (!a.adaptation) {  // unused in all-kinetic mode: sq and nz flags in global
      v.nza = a.nza + o;
      v.nzb = a.nzb + o;
      sq = a.sq + o;
    }
    cg::cluster_group cl = cg::this_cluster();
    v.fl = fl;
    v.sq = sq;
    v.fl_w = cl.map_shared_rank(fl, owner);
    v.sq_w = a.adaptation ? cl.map_shared_rank(sq, owner) : sq;
    if (!leader) {
      v.rho = v.E = v.Eprev = v.J = v.tA = v.tB = v.tC = v.tD = v.tE = v.bm = v.blift = nullptr;
    }
  } else {
    v.fl = v.fl_w = a.fl + o;
    v.sq = v.sq_w = a.sq + o;
    v.rho = a.rho + o;
    v.E = a.E + o;
    v.Eprev = a.Eprev + o;
    v.J = a.lJ + o;
    v.tA = a.tA + o;
    v.tB = a.tB + o;
    v.tC = a.tC + o;
    v.tD = a.tD + o;
    v.tE = a.tE + o;
    v.bm = a.bm + o;
    v.blift = a.blift + o;
    v.kc = a.kc + o;
    v.ki = a.ki + o;
    v.flip = a.flip + o;
    v.nza = a.nza + o;
    v.nzb = a.nzb + o;
    v.kcn = a.kcn + o;
    v.kin = a.kin + o;
  }
}

// ---------------------------------------------------------------------------
// Slice-level operations, executed by ONE CTA (all threads).

// 7-point stencil of order p at i (adaptation.py:65-73).
__device__ __forceinline__ double stencil_at(const double* v, int i, int nx, const MeshDev& m,
                                             int p) {
  double acc = 0.0;
#pragma unroll
  for (int o = 0; o < 7; ++o) {
    const double c = m.stc[p - 1][o];
    if (c != 0.0) acc = acc + c * v[wrap(i + o - 3, nx)];
  }
  return acc * m.sts[p - 1];
}

// stencil_at on a register window w[o] = v[i + o - 3] (same terms, same order).
// With the reference's table (m.stc_std) the zero terms it skips are known:
// the offset-0 term of orders 1 and 3 -- no per-term test.
// sqrt with +0 answered inline: the device sqrt takes a slow subroutine for
// zero operands, and fluid interfaces have <g^2> = 0 (sqrt(+0) = +0: same bits)
__device__ __forceinline__ double sqrt0(double x) { return x == 0.0 ? x : sqrt(x); }

__device__ __forceinline__ double stencil_reg(const double (&w)[7], const MeshDev& m, int p) {
  double acc = 0.0;
  if (m.stc_std) {
#pragma unroll
    for (int o = 0; o < 7; ++o)
      if (!((p == 1 || p == 3) && o == 3)) acc = acc + m.stc[p - 1][o] * w[o];
    return acc * m.sts[p - 1];
  }
#pragma unroll
  for (int o = 0; o < 7; ++o) {
    const double c = m.stc[p - 1][o];
    if (c != 0.0) acc = acc + c * w[o];
  }
  return acc * m.sts[p - 1];
}

// E_out = solve_field(rho); false on a solvability violation.
// poisson.py:41-54: src=(rho-rb)dx; defect=sum(src); guard; src-=defect/nx;
// E=cumsum(src); E-=mean(E).
// Fast mode (exact_scan == 0) field of rho into E_out: plain-tree sums and a
// parallel prefix, two block barriers (poisson.py:41-54 up to reassociation:
// not bitwise, O(nx u |E|) from np.cumsum).  Warp w owns a contiguous chunk of
// cells, read in coalesced rounds of 32; within a round a warp scan, the
// running carry across rounds; the warp offsets and -- folded into the same
// barrier -- sum(E) for the zero-mean gauge come from per-warp partials
// (sum_w C_w off_w + A_w).  Works on shared or global vectors alike.
static __device__ bool slice_field_fast(const MeshDev& m, const double* __restrict__ rho, double rb,
                                 double* __restrict__ E_out, double rtol, double* red) {
  const int nx = m.nx;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int cw = ((nx + nw - 1) / nw + 31) & ~31;
  const int lo = min(nx, warp * cw), hi = min(nx, lo + cw);
  const double dx = m.dx;
  auto wsum = [&](double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = v + __shfl_xor_sync(FULL, v, o);
    return v;
  };
  constexpr int U = 4;
  double ls = 0.0, la = 0.0;
  for (int b = lo; b < hi; b += 32 * U) {
    double r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = b + 32 * u + lane;
      r[u] = i < hi ? rho[i] : rb;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = b + 32 * u + lane;
      ls = ls + (r[u] - rb) * dx;
      la = la + (i < hi ? fabs(r[u]) : 0.0);
    }
  }
  ls = wsum(ls);
  la = wsum(la);
  if (lane == 0) {
    red[warp] = ls;
    red[32 + warp] = la;
  }
  __syncthreads();
  const double defect = wsum(lane < nw ? red[lane] : 0.0);
  const double abssum = wsum(lane < nw ? red[32 + lane] : 0.0);
  if (fabs(defect) > rtol * fmax(abssum * dx, 2.2250738585072014e-308)) return false;
  const double corr = defect / (double)nx;
  double carry = 0.0, part = 0.0;
  for (int b = lo; b < hi; b += 32 * U) {
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = b + 32 * u + lane;
      v[u] = i < hi ? (rho[i] - rb) * dx - corr : 0.0;
    }
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const double y = __shfl_up_sync(FULL, v[u], o);
        if (lane >= o) v[u] = v[u] + y;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = b + 32 * u + lane;
      const double e = carry + v[u];
      if (i < hi) {
        E_out[i] = e;
        part = part + e;
      }
      carry = carry + __shfl_sync(FULL, v[u], 31);
    }
  }
  const double aw = wsum(part);
  if (lane == 0) {
    red[64 + warp] = carry;                    // warp total
    red[96 + warp] = aw;                       // sum of the warp-local prefixes
    red[128 + warp] = (double)(hi - lo);       // cells in the warp
  }
  __syncthreads();
  double wi = lane < nw ? red[64 + lane] : 0.0;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_up_sync(FULL, wi, o);
    if (lane >= o) wi = wi + y;
  }
  double we = __shfl_up_sync(FULL, wi, 1);
  if (lane == 0) we = 0.0;
  const double tot = wsum(lane < nw ? red[128 + lane] * we + red[96 + lane] : 0.0);
  const double mean = tot / (double)nx;
  const double off = __shfl_sync(FULL, we, warp);
  for (int b = lo; b < hi; b += 32 * U) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = b + 32 * u + lane;
      if (i < hi) E_out[i] = (off + E_out[i]) - mean;
    }
  }
  __syncthreads();
  return true;
}

// Fast-mode field over EVERY CTA of the cluster (global-memory slice vectors,
// the hybrid dist slice phase): CTA r takes the r-th contiguous chunk of the
// cells, its warps contiguous sub-chunks read in coalesced rounds; the CTA
// partials meet in the leader's shared memory through DSMEM (two cluster
// barriers), so each pass is nx / (C x warps) cells per warp instead of one
// CTA walking all of them.  Same arithmetic shape as slice_field_fast.
static __device__ bool cluster_field_fast(const MeshDev& m, const double* __restrict__ rho, double rb,
                                   double* __restrict__ E_out, double rtol, double* red,
                                   int rank, int C) {
  const int nx = m.nx;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int cc = ((nx + C - 1) / C + 31) & ~31;
  const int clo = min(nx, rank * cc), chi = min(nx, clo + cc);
  const int cw = ((chi - clo + nw - 1) / nw + 31) & ~31;
  const int lo = min(chi, clo + warp * cw), hi = min(chi, lo + cw);
  const double dx = m.dx;
  double* lred = cg::this_cluster().map_shared_rank(red, 0);   // the leader's scratch
  auto wsum = [&](double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = v + __shfl_xor_sync(FULL, v, o);
    return v;
  };
  constexpr int U = 4;
  double ls = 0.0, la = 0.0;
  for (int b = lo; b < hi; b += 32 * U) {
    double r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = b + 32 * u + lane;
      r[u] = i < hi ? rho[i] : rb;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = b + 32 * u + lane;
      ls = ls + (r[u] - rb) * dx;
      la = la + (i < hi ? fabs(r[u]) : 0.0);
    }
  }
  ls = wsum(ls);
  la = wsum(la);
  if (lane == 0) {
    red[warp] = ls;
    red[32 + warp] = la;
  }
  __syncthreads();
  if (warp == 0) {
    const double cs_ = wsum(lane < nw ? red[lane] : 0.0);
    const double ca = wsum(lane < nw ? red[32 + lane] : 0.0);
    if (lane == 0) {
      lred[192 + rank] = cs_;
      lred[208 + rank] = ca;
    }
  }
  cg::this_cluster().sync();
  const double defect = wsum(lane < C ? lred[192 + lane] : 0.0);
  const double abssum = wsum(lane < C ? lred[208 + lane] : 0.0);
  if (fabs(defect) > rtol * fmax(abssum * dx, 2.2250738585072014e-308)) return false;
  const double corr = defect / (double)nx;
  double carry = 0.0, part = 0.0;
  for (int b = lo; b < hi; b += 32 * U) {
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = b + 32 * u + lane;
      v[u] = i < hi ? (rho[i] - rb) * dx - corr : 0.0;
    }
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const double y = __shfl_up_sync(FULL, v[u], o);
        if (lane >= o) v[u] = v[u] + y;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = b + 32 * u + lane;
      const double e = carry + v[u];
      if (i < hi) {
        E_out[i] = e;
        part = part + e;
      }
      carry = carry + __shfl_sync(FULL, v[u], 31);
    }
  }
  const double aw = wsum(part);
  if (lane == 0) {
    red[64 + warp] = carry;
    red[96 + warp] = aw;
    red[128 + warp] = (double)(hi - lo);
  }
  __syncthreads();
  // this CTA's warp offsets, and its partials for the cluster
  double wi = lane < nw ? red[64 + lane] : 0.0;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_up_sync(FULL, wi, o);
    if (lane >= o) wi = wi + y;
  }
  double we = __shfl_up_sync(FULL, wi, 1);
  if (lane == 0) we = 0.0;
  const double woff = __shfl_sync(FULL, we, warp);
  if (warp == 0) {
    const double at = wsum(lane < nw ? red[128 + lane] * we + red[96 + lane] : 0.0);
    if (lane == 31) lred[224 + rank] = wi;            // CTA total
    if (lane == 0) {
      lred[240 + rank] = at;                          // sum of the CTA-local prefixes
      lred[256 + rank] = (double)(chi - clo);         // cells in the CTA
    }
  }
  cg::this_cluster().sync();
  double ti = lane < C ? lred[224 + lane] : 0.0;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_up_sync(FULL, ti, o);
    if (lane >= o) ti = ti + y;
  }
  double te = __shfl_up_sync(FULL, ti, 1);
  if (lane == 0) te = 0.0;
  const double tot = wsum(lane < C ? lred[256 + lane] * te + lred[240 + lane] : 0.0);
  const double mean = tot / (double)nx;
  const double off = __shfl_sync(FULL, te, rank) + woff;
  for (int b = lo; b < hi; b += 32 * U) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = b + 32 * u + lane;
      if (i < hi) E_out[i] = (off + E_out[i]) - mean;
    }
  }
  cg::this_cluster().sync();   // E complete (and the leader's scratch free) everywhere
  return true;
}

static __device__ bool slice_field(const MeshDev& m, const double* rho, double rb, double* src,
                            double* E_out, double rtol, int exact_scan, bool on_chip,
                            const Smem& sm, long long* dbg = nullptr, bool src_ready = false,
                            double* mean_out = nullptr) {
  const int nx = m.nx;
  long long c0 = dbg ? clock64() : 0;
#define PK_TICK(k)                         \
  if (dbg && threadIdx.x == 0) {           \
    const long long c1 = clock64();        \
    pk_red_add(dbg + k, c1 - c0);          \
    c0 = c1;                               \
  }
  if (!exact_scan) {
    PK_TICK(0)
    const bool ok = slice_field_fast(m, rho, rb, E_out, rtol, sm.red);
    PK_TICK(3)
    return ok;
  }
  if (sm.scan && exact_scan && !on_chip) {
    // global-memory slice vectors with a buffer of scan_cap doubles on chip:
    // src is formed where it is read (same bits), the scan runs on the buffer
    // (chunk by chunk, the carry continuing the chain, when nx > scan_cap)
    double defect, abssum;
    PK_TICK(0)
    if (sm.plan->perfect) {  // (butterfly tree, 16 operands in flight per lane: pw_perfect)
      double r2[2];
      pw_perfect<2>([&](int s, int i) { return s ? fabs(rho[i]) : (rho[i] - rb) * m.dx; }, *sm.plan,
                    sm.red, r2);
      defect = r2[0];
      abssum = r2[1];
    } else {
      block_pairwise2([&](int i) { return (rho[i] - rb) * m.dx; },
                      [&](int i) { return fabs(rho[i]); }, *sm.plan, sm.red, defect, abssum);
    }
    PK_TICK(1)
    if (fabs(defect) > rtol * fmax(abssum * m.dx, 2.2250738585072014e-308)) return false;
    const double corr = defect / (double)nx;
    double* sc = sm.scan;
    if (sm.scan_cap >= nx) {  // whole: the mean and E - mean from the buffer too
      for (int i = threadIdx.x; i < nx; i += blockDim.x) sc[i] = (rho[i] - rb) * m.dx - corr;
      __syncthreads();
      PK_TICK(2)
      smem_cumsum_call(sc, sc, nx, -0.0);
      __syncthreads();
      PK_TICK(3)
      double mean;
      if (sm.plan->perfect) {
        const uint32_t scs = (uint32_t)__cvta_generic_to_shared(sc);
        double mm[1];
        pw_perfect<1>([&](int, int i) { return lds64(scs + 8 * i); }, *sm.plan, sm.red, mm);
        mean = mm[0] / (double)nx;
      } else {
        mean = block_pairwise([&](int i) { return sc[i]; }, *sm.plan, sm.red) / (double)nx;
      }
      PK_TICK(4)
      for (int i = threadIdx.x; i < nx; i += blockDim.x) E_out[i] = sc[i] - mean;
      __syncthreads();
      PK_TICK(5)
      return true;
    }
    double carry = -0.0;  // np.cumsum's chain starts from the first operand
    for (int q0 = 0; q0 < nx; q0 += sm.scan_cap) {
      const int len = min(sm.scan_cap, nx - q0);
      for (int i = threadIdx.x; i < len; i += blockDim.x)
        sc[i] = (rho[q0 + i] - rb) * m.dx - corr;
      __syncthreads();
      smem_cumsum_call(sc, sc, len, carry);
      __syncthreads();
      carry = sc[len - 1];
      for (int i = threadIdx.x; i < len; i += blockDim.x) E_out[q0 + i] = sc[i];
      __syncthreads();
    }
    PK_TICK(3)
    const double mean =
        block_pairwise([&](int i) { return E_out[i]; }, *sm.plan, sm.red) / (double)nx;
    PK_TICK(4)
    for (int i = threadIdx.x; i < nx; i += blockDim.x) E_out[i] = E_out[i] - mean;
    __syncthreads();
    PK_TICK(5)
    return true;
  }
  if (!src_ready) {  // (finish_step forms src in its rho-update pass)
    for (int i = threadIdx.x; i < nx; i += blockDim.x) src[i] = (rho[i] - rb) * m.dx;
    __syncthreads();
  }
  if (on_chip) {
    // vectors on chip: field_exact_onchip, in place on E_out
    if (src != E_out) {
      for (int i = threadIdx.x; i < nx; i += blockDim.x) E_out[i] = src[i];
      __syncthreads();
    }
    PK_TICK(0)
    double mean;
    const uint32_t rs = (uint32_t)__cvta_generic_to_shared(rho);  // on chip: shared memory
    if (!field_exact_onchip([&](int i) { return fabs(lds64(rs + 8 * i)); }, E_out, nx, m.dx, rtol,
                            *sm.plan, sm.red, mean, dbg ? dbg + 1 : nullptr))
      return false;
    if (dbg) c0 = clock64();  // (field_exact_onchip ticked pairwise2 / corr / cumsum / mean)
    if (mean_out) {  // the caller applies E - mean where it next reads E
      *mean_out = mean;
    } else {
      for (int i = threadIdx.x; i < nx; i += blockDim.x) E_out[i] = E_out[i] - mean;
      __syncthreads();
    }
    PK_TICK(5)
    return true;
  }
  PK_TICK(0)
  double defect, abssum;
  block_pairwise2([&](int i) { return src[i]; }, [&](int i) { return fabs(rho[i]); }, *sm.plan,
                  sm.red, defect, abssum);
  PK_TICK(1)
  const double scale = abssum * m.dx;
  // `abs(defect) > rtol * max(scale, tiny)`: a NaN defect compares False in
  // Python too, so only a genuine violation raises.
  if (fabs(defect) > rtol * fmax(scale, 2.2250738585072014e-308)) return false;
  const double corr = defect / (double)nx;
  for (int i = threadIdx.x; i < nx; i += blockDim.x) src[i] = src[i] - corr;
  __syncthreads();
  PK_TICK(2)
  if (exact_scan) {
    if (on_chip)  // src and E_out in this CTA's shared memory
      smem_cumsum(src, E_out, nx);
    else
      warp_cumsum([&](int i) { return src[i]; }, [&](int i, double v) { E_out[i] = v; }, nx);
  } else {
    block_scan_fast([&](int i) { return src[i]; }, [&](int i, double v) { E_out[i] = v; }, nx,
                    sm.red);
  }
  __syncthreads();
  PK_TICK(3)
  const double mean = block_pairwise([&](int i) { return E_out[i]; }, *sm.plan, sm.red) / (double)nx;
  PK_TICK(4)
  for (int i = threadIdx.x; i < nx; i += blockDim.x) E_out[i] = E_out[i] - mean;
  __syncthreads();
  PK_TICK(5)
#undef PK_TICK
  return true;
}

// J_{i+1/2} = (rho_{i+1}-rho_i)/dx - E*0.5*(rho_i+rho_{i+1})   (fluid.py:48-52)
// ((.)/dx as the correctly rounded Markstein quotient, qdiv in pk_device.cuh)
__device__ __forceinline__ double flux_J(double r, double rn, double e, double dx, double rdx) {
  return qdiv(rn - r, dx, rdx) - e * 0.5 * (r + rn);
}

// Block-wide exclusive scan of per-thread counts; returns the total.
static __device__ int block_excl_scan(int v, int* out_prefix, int* sbuf) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  int inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int t = __shfl_up_sync(FULL, inc, o);
    if (lane >= o) inc += t;
  }
  if (lane == 31) sbuf[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    int w = lane < nwarp ? sbuf[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int t = __shfl_up_sync(FULL, w, o);
      if (lane >= o) w += t;
    }
    if (lane < nwarp) sbuf[lane] = w;
  }
  __syncthreads();
  *out_prefix = inc - v + (warp > 0 ? sbuf[warp - 1] : 0);
  const int total = sbuf[nwarp - 1];
  __syncthreads();
  return total;
}

// Unordered compaction: every lane of the warp calls it (same trip count);
// lanes with f append i to list through one warp-aggregated shared atomic.
__device__ __forceinline__ void list_append(bool f, int i, int* list, int* count) {
  const unsigned bal = __ballot_sync(FULL, f);
  if (!bal) return;
  const int lane = threadIdx.x & 31, lead = __ffs(bal) - 1;
  int base = 0;
  if (lane == lead) base = atomicAdd(count, __popc(bal));
  base = __shfl_sync(FULL, base, lead);
  if (f) list[base + __popc(bal & ((1u << lane) - 1u))] = i;
}

// Who runs a slice phase: the leader CTA alone, or (hybrid slices whose
// vectors live in global memory) every CTA of the cluster, elements and rows
// dealt over all of their threads / warps, with cluster barriers between
// dependent loops and the list counters in the leader's shared memory.
struct Par {
  int r0, rs;    // this thread's first element, element stride
  int w0, ws;    // this warp's first row, row stride
  int rank, C;   // CTA rank among the participants, participants
  bool dist;
  int* flags;    // the leader's misc ints: [0] any flip, [40]/[41] list sizes,
                 // [42] field ok, [48 + r] scan totals of rank r
  __device__ void sync() const {
    if (dist) cg::this_cluster().sync();
    else __syncthreads();
  }
  // exclusive prefix of v over the participants' threads in (rank, thread)
  // order; returns the total.  `sbuf`: this CTA's block_excl_scan scratch.
  __device__ int scan(int v, int* pre, int* sbuf) const {
    int p;
    const int tot = block_excl_scan(v, &p, sbuf);
    if (!dist) {
      *pre = p;
      return tot;
    }
    if (threadIdx.x == 0) flags[48 + rank] = tot;
    sync();
    int base = 0, all = 0;
    for (int r = 0; r < C; ++r) {
      const int t = flags[48 + r];
      base += r < rank ? t : 0;
      all += t;
    }
    *pre = p + base;
    return all;
  }
};

__device__ __forceinline__ Par leader_par(const Smem& sm) {
  Par P;
  P.r0 = threadIdx.x;
  P.rs = blockDim.x;
  P.w0 = threadIdx.x >> 5;
  P.ws = blockDim.x >> 5;
  P.rank = 0;
  P.C = 1;
  P.dist = false;
  P.flags = sm.misc;
  return P;
}

// Kinetic-row list segment (contiguous cells) for the one-scan klist/kstream:
// cnt kinetic cells, the first/last of them, and the stream rows its entries
// after the first add (each entry q adds min(3, i_q - i_{q-1}) rows, the
// first entry of the whole list 3).  Associative (segment A then B).
struct KSeg {
  int cnt, first, last, inner;
};

__device__ __forceinline__ KSeg kseg_comb(const KSeg& a, const KSeg& b) {
  KSeg r;
  r.cnt = a.cnt + b.cnt;
  r.first = a.cnt ? a.first : b.first;
  r.last = b.cnt ? b.last : a.last;
  r.inner = a.inner + b.inner + ((a.cnt && b.cnt) ? min(3, b.first - a.last) : 0);
  return r;
}

__device__ __forceinline__ KSeg kseg_shfl_up(const KSeg& x, int o) {
  KSeg r;
  r.cnt = __shfl_up_sync(FULL, x.cnt, o);
  r.first = __shfl_up_sync(FULL, x.first, o);
  r.last = __shfl_up_sync(FULL, x.last, o);
  r.inner = __shfl_up_sync(FULL, x.inner, o);
  return r;
}

// Block-wide exclusive scan of KSeg (thread order); returns the total.
// `wt`: 4 * nwarp ints of shared memory.  One barrier.
static __device__ KSeg kseg_block_scan(const KSeg& mine, KSeg& excl, int* wt) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  const KSeg id = {0, 0, 0, 0};
  KSeg inc = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const KSeg y = kseg_shfl_up(inc, o);
    if (lane >= o) inc = kseg_comb(y, inc);
  }
  if (lane == 31) {
    wt[4 * warp] = inc.cnt;
    wt[4 * warp + 1] = inc.first;
    wt[4 * warp + 2] = inc.last;
    wt[4 * warp + 3] = inc.inner;
  }
  KSeg e = kseg_shfl_up(inc, 1);
  if (lane == 0) e = id;
  __syncthreads();
  KSeg wp = id, tot = id;
  for (int w = 0; w < nwarp; ++w) {
    const KSeg t = {wt[4 * w], wt[4 * w + 1], wt[4 * w + 2], wt[4 * w + 3]};
    if (w < warp) wp = kseg_comb(wp, t);
    tot = kseg_comb(tot, t);
  }
  excl = kseg_comb(wp, e);
  return tot;
}

// prepare_step's hybrid slice phase in five passes (the leader CTA alone, or
// -- Par::dist -- every CTA of the cluster on global-memory vectors with
// cluster barriers): the same values as the pass-by-pass form below with
// fewer passes and barriers -- J, (E - E_prev)/dt and J_c in one pass
// (J_{i-1} recomputed: same operands, same bits), the masked moment b_m folded
// into the dco pass (b_m(i +- 1) recomputed from the OLD kinetic-interface
// flags, so the new labels are stored only after the scan's barrier), and the
// kinetic-row list with its stream positions from ONE block scan of KSeg
// segments.  The field's pending zero-mean shift (v.Emean) is applied where E
// is read and stored in the dco pass, where no other thread reads E.
template <int T>
__device__ bool prepare_step_fused(const FineArgs& a, const SliceView& v, const Smem& sm,
                                   double dt, int moment_all, double* gin, uint8_t* nzin,
                                   uint8_t* nzout, int step, const Par& P, long long* dbg) {
  long long c0 = dbg ? clock64() : 0;
  auto tick = [&](int k) {
    if (dbg && threadIdx.x == 0) {
      const long long c1 = clock64();
      pk_red_add(dbg + k, c1 - c0);
      c0 = c1;
    }
  };
  const MeshDev& m = a.m;
  const int nx = m.nx, nv = m.nv;
  const int tid = P.r0, nt = P.rs;  // this thread's first element, element stride
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int* sflags = P.flags;  // the leader's: [0] any flip, [40]/[41] list sizes
  const double Em = v.Emean;
  const double* __restrict__ rho_ = v.rho;
  double* __restrict__ E_ = v.E;
  const double* __restrict__ Ep_ = v.Eprev;
  auto Ef = [&](int i) { return E_[i] - Em; };  // x - 0.0 == x when nothing is pending
  if (P.rank == 0 && threadIdx.x == 0) {
    sflags[0] = 0;
    sflags[40] = 0;
    sflags[41] = 0;
  }
  // P1: J (fluid.py:48-52), (E - E_prev)/dt, J_c = (J_{i-1} + J_i)/2
  {
    const double rdt = 1.0 / dt;
    double* __restrict__ J_ = v.J;
    double* __restrict__ gJ_ = v.gJ;
    double* __restrict__ tA_ = v.tA;
    double* __restrict__ tB_ = v.tB;
    constexpr int U = 2;
    for (int i0 = tid; i0 < nx; i0 += U * nt) {
      double rm[U], r0[U], r1[U], em[U], e0[U], ep[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = min(i0 + u * nt, nx - 1);
        const int ip = wrap(i - 1, nx);
        rm[u] = rho_[ip];
        r0[u] = rho_[i];
        r1[u] = rho_[wrap(i + 1, nx)];
        em[u] = Ef(ip);
        e0[u] = Ef(i);
        ep[u] = Ep_[i];
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = i0 + u * nt;
        if (i < nx) {
          const double J = flux_J(r0[u], r1[u], e0[u], m.dx, m.rdx);
          const double Jm = flux_J(rm[u], r0[u], em[u], m.dx, m.rdx);
          J_[i] = J;
          gJ_[i] = J;
          tA_[i] = qdiv(e0[u] - ep[u], dt, rdt);
          tB_[i] = 0.5 * (Jm + J);
        }
      }
    }
  }
  P.sync();
  tick(0);
  // P2: remainder indicator (adaptation.py:120-152), perturbation norm
  // (155-159), labels (161-181)
  {
    const double three_rb = 3.0 * v.rb;
    const double* __restrict__ tA_ = v.tA;
    const double* __restrict__ tB_ = v.tB;
    const double* __restrict__ sq_ = v.sq;
    const uint8_t* __restrict__ ki_ = v.ki;
    double* __restrict__ tC_ = v.tC;
    double* __restrict__ tD_ = v.tD;
    uint8_t* __restrict__ kcn_ = v.kcn;
    const double* __restrict__ rsc = a.rscale ? a.rscale + (size_t)v.b * nx : nullptr;
    constexpr int U = 2;
    for (int i0 = tid; i0 < nx; i0 += U * nt) {
      double wB[U][7], wR[U][7], a0[U], a1[U], e0[U], e1[U], s0[U], s1[U], rs[U];
      int k0[U], k1[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = min(i0 + u * nt, nx - 1);
        const int ip = wrap(i - 1, nx);
#pragma unroll
        for (int o = 0; o < 7; ++o) {
          const int j = wrap(i + o - 3, nx);
          wB[u][o] = tB_[j];
          wR[u][o] = rho_[j];
        }
        a0[u] = tA_[ip];
        a1[u] = tA_[i];
        e0[u] = Ef(ip);
        e1[u] = Ef(i);
        s0[u] = sq_[ip];
        s1[u] = sq_[i];
        k0[u] = ki_[ip];
        k1[u] = ki_[i];
        rs[u] = rsc ? rsc[i] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = i0 + u * nt;
        if (i < nx) {
          const double dtEc = 0.5 * (a0[u] + a1[u]);
          const double Ec = 0.5 * (e0[u] + e1[u]);
          const double d1J = stencil_reg(wB[u], m, 1);
          const double d2J = stencil_reg(wB[u], m, 2);
          const double d3J = stencil_reg(wB[u], m, 3);
          const double d1r = stencil_reg(wR[u], m, 1);
          const double rho = wR[u][3];
          const double Jc = wB[u][3];
          const double R =
              -d3J + Ec * d2J + (2.0 * rho - three_rb) * d1J + 2.0 * Jc * d1r - d1r * dtEc;
          tC_[i] = R;    // unscaled R (lift, higher_order)
          tD_[i] = d1J;  // D1(J_c) (lift drift)
          const double Rs = rsc ? rs[u] * R : R;
          const double sqp = (moment_all || k0[u]) ? s0[u] : 0.0;
          const double sqi = (moment_all || k1[u]) ? s1[u] : 0.0;
          const double gn = sqrt0(0.5 * (sqp + sqi));
          const bool fR = fabs(Rs) < a.delta0;
          const bool fg = gn < a.eta0;
          const bool fluid = a.combine_and ? (fR && fg) : (fR || fg);
          kcn_[i] = fluid ? 0 : 1;
        }
      }
    }
  }
  P.sync();
  tick(1);
  // P3: kinetic interfaces and F -> K flips, listed (klist is free until the
  // row list below)
  int anyflip = 0;
  {
    const uint8_t* __restrict__ kcn_ = v.kcn;
    const uint8_t* __restrict__ ki_ = v.ki;
    uint8_t* __restrict__ kin_ = v.kin;
    uint8_t* __restrict__ flip_ = v.flip;
    constexpr int U = 4;
    for (int i00 = 0; i00 < nx; i00 += U * nt) {  // uniform trip count (ballots inside)
      int c0v[U], c1v[U], k[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = min(i00 + u * nt + tid, nx - 1);
        c0v[u] = kcn_[i];
        c1v[u] = kcn_[wrap(i + 1, nx)];
        k[u] = ki_[i];
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = i00 + u * nt + tid;
        uint8_t f = 0;
        if (i < nx) {
          const uint8_t kin = (uint8_t)(c0v[u] | c1v[u]);
          kin_[i] = kin;
          f = (kin && !k[u]) ? 1 : 0;
          flip_[i] = f;
        }
        anyflip |= f;
        list_append(f != 0, i, v.klist, &sflags[40]);
      }
    }
  }
  if (anyflip) atomicOr(&sflags[0], 1);
  P.sync();
  tick(2);
  const int nflip = sflags[40];
  if (dbg && threadIdx.x == 0) pk_red_add(dbg + 10, nflip);
  if (sflags[0]) {
    if (a.reinit == 0) {
      if (a.lift_order != 1 && a.lift_order != 2) {
        if (P.rank == 0 && threadIdx.x == 0) set_status(a.status, PK_ERR_BAD_LIFT, v.b, step);
        return false;
      }
      if (a.lift_order >= 2 && a.time_elim != 0 && a.time_elim != 1) {
        if (P.rank == 0 && threadIdx.x == 0) set_status(a.status, PK_ERR_BAD_LIFT, v.b, step);
        return false;
      }
      // lift scalars at the flipped interfaces (lifting.py:63-88); dE_dt = (E - E_prev)/dt
      for (int q = tid; q < nflip; q += nt) {
        const int i = v.klist[q];
        const int in_ = wrap(i + 1, nx);
        const double dJ = 0.5 * (v.tD[i] + v.tD[in_]);
        v.tE[i] = dJ - Ef(i) * v.J[i];           // drift
        v.tA[i] = 0.5 * (v.tC[i] + v.tC[in_]);   // R_if
      }
      P.sync();
      for (int q = P.w0; q < nflip; q += P.ws) {
        const int i = v.klist[q];
        LiftRow L;
        const size_t o = (size_t)v.b * nx + i;
        L.negJ = a.neg_eps[o] * v.J[i];
        L.e2 = a.eps2[o];
        L.drift = v.tE[i];
        L.Rif = v.tA[i];
        double bx, bsq;
        if constexpr (T < 0) {
          double* row = gin + (size_t)i * nv;
          double* scr = sm.wrow + warp * BIG_SCR;
          big_row_lift(row, L, a.lift_order, a.time_elim == 1, 1, m, scr, lane);
          big_row_moments(row, m, scr, false, bx, bsq);
        } else {
          double g[Layout<T>::S];
          row_lift<T>(g, L, a.lift_order, a.time_elim == 1, 1, sm, m, sm.wrow + warp * nv, lane);
          row_store<T>(g, gin + (size_t)i * nv, lane, nv);
          row_moments<T>(g, sm, m, sm.wrow + warp * nv, lane, bx, bsq);
        }
        if (lane == 0) v.blift[i] = bx;
      }
    } else if (a.reinit == 1) {
      for (int q = P.w0; q < nflip; q += P.ws) {
        const int i = v.klist[q];
        row_zero_store<T>(gin + (size_t)i * nv, lane, nv);
        if (lane == 0) v.blift[i] = 0.0;
      }
    } else {
      if (P.rank == 0 && threadIdx.x == 0) set_status(a.status, PK_ERR_BAD_REINIT, v.b, step);
      return false;
    }
    P.sync();
  }
  tick(3);
  // P4: masked projection moment b_m (hybrid.py:103-105) at i-1, i+1 from the
  // post-flip rows and the OLD interface flags, dco (kinetic.py:190-191),
  // E-upwind factors (177-178), the zero list (hybrid.py:166), E stored
  {
    const uint8_t* __restrict__ ki_ = v.ki;
    const uint8_t* __restrict__ kin_ = v.kin;
    const uint8_t* __restrict__ flip_ = v.flip;
    const double* __restrict__ blift_ = v.blift;
    const double* __restrict__ fl_ = v.fl;
    double* __restrict__ dco_ = v.dco;
    double* __restrict__ vco_ = v.vco;
    int8_t* __restrict__ vsg_ = v.vsg;
    uint8_t* __restrict__ nzo = nzout;
    auto bm = [&](int j) {
      const bool valid = moment_all || ki_[j];
      return kin_[j] ? (flip_[j] ? blift_[j] : (valid ? fl_[j] : 0.0)) : 0.0;
    };
    const bool pend = v.Epend;
    constexpr int U = 2;
    for (int i00 = 0; i00 < nx; i00 += U * nt) {  // uniform trip count (ballots inside)
      double b1[U], b0[U], e[U];
      int kn[U], nz[U], fp[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = min(i00 + u * nt + tid, nx - 1);
        b1[u] = bm(wrap(i + 1, nx));
        b0[u] = bm(wrap(i - 1, nx));
        e[u] = Ef(i);
        kn[u] = kin_[i];
        nz[u] = nzo[i];
        fp[u] = flip_[i];
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = i00 + u * nt + tid;
        bool z = false;
        if (i < nx) {
          dco_[i] = qdiv(b1[u] - b0[u], m.two_dx, m.rtwo_dx);
          vsg_[i] = e[u] > 0.0 ? 1 : (e[u] < 0.0 ? -1 : 0);
          vco_[i] = qdiv(e[u], m.dvx, m.rdvx);
          if (pend) E_[i] = e[u];
          if (!moment_all && fp[u]) nzin[i] = 1;
          z = !kn[u] && nz[u];
          if (z) nzo[i] = 0;
        }
        list_append(z, i, v.zlist, &sflags[41]);
      }
    }
  }
  tick(5);
  // P5: the order-preserving kinetic-row list and its row-stream positions
  // (one KSeg scan over contiguous chunks); the new labels stored
  {
    const uint8_t* __restrict__ kin_ = v.kin;
    const int per = (nx + nt - 1) / nt;
    const int lo = min(nx, tid * per), hi = min(nx, lo + per);
    KSeg mine = {0, 0, 0, 0};
    for (int i = lo; i < hi; ++i)
      if (kin_[i]) {
        if (mine.cnt) mine.inner += min(3, i - mine.last);
        else mine.first = i;
        mine.last = i;
        ++mine.cnt;
      }
    KSeg ex;
    KSeg tot = kseg_block_scan(mine, ex, sm.misc + 64);  // (barrier: P4 is done here)
    if (P.dist) {  // CTA totals meet in the leader's reduction scratch (free here)
      int* ct = reinterpret_cast<int*>(cg::this_cluster().map_shared_rank(sm.red, 0)) + 576;
      if (threadIdx.x == 0) {
        ct[4 * P.rank] = tot.cnt;
        ct[4 * P.rank + 1] = tot.first;
        ct[4 * P.rank + 2] = tot.last;
        ct[4 * P.rank + 3] = tot.inner;
      }
      P.sync();  // (also: every CTA's P4 is done)
      KSeg pre = {0, 0, 0, 0}, all = {0, 0, 0, 0};
      for (int r = 0; r < P.C; ++r) {
        const KSeg t = {ct[4 * r], ct[4 * r + 1], ct[4 * r + 2], ct[4 * r + 3]};
        if (r < P.rank) pre = kseg_comb(pre, t);
        all = kseg_comb(all, t);
      }
      ex = kseg_comb(pre, ex);
      tot = all;
    }
    int q = ex.cnt, prev = ex.last;
    int pos = ex.cnt ? 3 + ex.inner : 0;  // stream rows of the entries before this chunk
    for (int i = lo; i < hi; ++i) {
      v.kc[i] = v.kcn[i];
      const uint8_t kn = kin_[i];
      v.ki[i] = kn;
      if (kn) {
        const int nn = q == 0 ? 3 : min(3, i - prev);
        pos += nn;
        v.klist[q] = i;
        v.kpos[q] = pos;
        for (int t = 0; t < nn; ++t) v.kstream[pos - nn + t] = i + 2 - nn + t;
        prev = i;
        ++q;
      }
    }
    if (P.rank == 0 && threadIdx.x == 0) {
      *v.nk = tot.cnt;
      *v.nzl = sflags[41];
      if (dbg) {
        pk_red_add(dbg + 11, sflags[41]);
        pk_red_add(dbg + 12, tot.cnt);
      }
    }
  }
  P.sync();
  tick(7);
  return true;
}

// ---------------------------------------------------------------------------
// Slice phase: prepare step `s` (labels, flips, projection coefficients, row
// list) from rho, E (start of step s), Eprev and the moments fl/sq of the
// rows stored in gin.  `moment_all`: moments are valid on every row
// (prologue: user g) rather than only on the previous step's kinetic rows.
template <int T, bool AD>
__device__ bool prepare_step(const FineArgs& a, const SliceView& v, const Smem& sm, double dt,
                             int moment_all, double* gin, uint8_t* nzin, uint8_t* nzout,
                             int step, const Par& P, long long* dbg = nullptr) {
  long long c0 = dbg ? clock64() : 0;
#define PK_PTICK(k)                        \
  if (dbg && threadIdx.x == 0) {           \
    const long long c1 = clock64();        \
    pk_red_add(dbg + k, c1 - c0);          \
    c0 = c1;                               \
  }
  const MeshDev& m = a.m;
  const int nx = m.nx, nv = m.nv;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5;
  int* sflags = P.flags;  // leader's: [0] any flip, [40]/[41] list sizes

  if constexpr (!AD) {
    // all-kinetic: J, and the projection/E-upwind coefficients from the
    // unmasked moments (kinetic.py:177-178,190-191,221)
    const double Em = v.Emean;  // pending zero-mean shift of E (0.0: none)
    for (int i = tid; i < nx; i += nt) {
      const int in_ = wrap(i + 1, nx), ip = wrap(i - 1, nx);
      v.kc[i] = 1;  // adaptation off: all kinetic (hybrid.py:167-168)
      v.ki[i] = 1;
      const double e = v.E[i] - Em;
      if (v.Epend) v.E[i] = e;
      const double J = flux_J(v.rho[i], v.rho[in_], e, m.dx, m.rdx);
      v.J[i] = J;
      v.gJ[i] = J;
      v.dco[i] = qdiv(v.fl[in_] - v.fl[ip], m.two_dx, m.rtwo_dx);
      v.vsg[i] = e > 0.0 ? 1 : (e < 0.0 ? -1 : 0);
      v.vco[i] = qdiv(e, m.dvx, m.rdvx);
    }
    if (tid == 0) *v.nk = nx;
    __syncthreads();
    return true;
  }

  if (!a.pass_prepare)
    return prepare_step_fused<T>(a, v, sm, dt, moment_all, gin, nzin, nzout, step, P, dbg);
  // The element loops below run over global memory when the slice vectors do
  // not fit on chip (large nx): every operand of U iterations is loaded
  // unconditionally first (restrict views, no load behind a branch), so the
  // L2 round trips of consecutive iterations overlap.
  const double* __restrict__ rho_ = v.rho;
  double* __restrict__ E_ = v.E;
  const double* __restrict__ Ep_ = v.Eprev;
  double* __restrict__ J_ = v.J;
  double* __restrict__ gJ_ = v.gJ;
  double* __restrict__ tA_ = v.tA;
  double* __restrict__ tB_ = v.tB;
  {
    constexpr int U = 4;
    for (int i0 = P.r0; i0 < nx; i0 += U * P.rs) {
      double r0[U], r1[U], e[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = min(i0 + u * P.rs, nx - 1);
        r0[u] = rho_[i];
        r1[u] = rho_[wrap(i + 1, nx)];
        e[u] = E_[i] - v.Emean;  // the pending zero-mean shift (0.0: none)
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = i0 + u * P.rs;
        if (i < nx) {
          if (v.Epend) E_[i] = e[u];
          const double J = flux_J(r0[u], r1[u], e[u], m.dx, m.rdx);
          J_[i] = J;
          gJ_[i] = J;
        }
      }
    }
  }
  if (P.rank == 0 && tid == 0) {
    sflags[0] = 0;
    sflags[40] = 0;
    sflags[41] = 0;
  }
  P.sync();
  PK_PTICK(0)
  // remainder indicator (adaptation.py:120-152) at cells
  {
    const double rdt = 1.0 / dt;   // qdiv's reciprocal for (E - E_prev) / dt
    constexpr int U = 4;
    for (int i0 = P.r0; i0 < nx; i0 += U * P.rs) {
      double e[U], ep[U], j0[U], j1[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = min(i0 + u * P.rs, nx - 1);
        e[u] = E_[i];
        ep[u] = Ep_[i];
        j0[u] = J_[wrap(i - 1, nx)];
        j1[u] = J_[i];
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = i0 + u * P.rs;
        if (i < nx) {
          tA_[i] = qdiv(e[u] - ep[u], dt, rdt);  // (E - E_prev)/dt
          tB_[i] = 0.5 * (j0[u] + j1[u]);  // J_c
        }
      }
    }
  }
  P.sync();
  {
    const double three_rb = 3.0 * v.rb;
    const double* __restrict__ sq_ = v.sq;
    const uint8_t* __restrict__ ki_ = v.ki;
    double* __restrict__ tC_ = v.tC;
    double* __restrict__ tD_ = v.tD;
    uint8_t* __restrict__ kcn_ = v.kcn;
    const double* __restrict__ rsc = a.rscale ? a.rscale + (size_t)v.b * nx : nullptr;
    constexpr int U = 2;
    for (int i0 = P.r0; i0 < nx; i0 += U * P.rs) {
      double wB[U][7], wR[U][7], a0[U], a1[U], e0[U], e1[U], s0[U], s1[U], rs[U];
      int k0[U], k1[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = min(i0 + u * P.rs, nx - 1);
        const int ip = wrap(i - 1, nx);
#pragma unroll
        for (int o = 0; o < 7; ++o) {
          const int j = wrap(i + o - 3, nx);
          wB[u][o] = tB_[j];
          wR[u][o] = rho_[j];
        }
        a0[u] = tA_[ip];
        a1[u] = tA_[i];
        e0[u] = E_[ip];
        e1[u] = E_[i];
        s0[u] = sq_[ip];
        s1[u] = sq_[i];
        k0[u] = ki_[ip];
        k1[u] = ki_[i];
        rs[u] = rsc ? rsc[i] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = i0 + u * P.rs;
        if (i < nx) {
          const double dtEc = 0.5 * (a0[u] + a1[u]);
          const double Ec = 0.5 * (e0[u] + e1[u]);
          const double d1J = stencil_reg(wB[u], m, 1);
          const double d2J = stencil_reg(wB[u], m, 2);
          const double d3J = stencil_reg(wB[u], m, 3);
          const double d1r = stencil_reg(wR[u], m, 1);
          const double rho = wR[u][3];
          const double Jc = wB[u][3];
          const double R =
              -d3J + Ec * d2J + (2.0 * rho - three_rb) * d1J + 2.0 * Jc * d1r - d1r * dtEc;
          tC_[i] = R;    // unscaled R (lift, higher_order)
          tD_[i] = d1J;  // D1(J_c) (lift drift)
          const double Rs = rsc ? rs[u] * R : R;
          // perturbation indicator (adaptation.py:155-159) on the incoming g
          const double sqp = (moment_all || k0[u]) ? s0[u] : 0.0;
          const double sqi = (moment_all || k1[u]) ? s1[u] : 0.0;
          const double gn = sqrt0(0.5 * (sqp + sqi));
          const bool fR = fabs(Rs) < a.delta0;
          const bool fg = gn < a.eta0;
          const bool fluid = a.combine_and ? (fR && fg) : (fR || fg);
          kcn_[i] = fluid ? 0 : 1;
        }
      }
    }
  }
  P.sync();
  PK_PTICK(1)
  // flipped interfaces (F -> K) are listed (klist is free until the row list
  // below), so the row work touches only them
  int anyflip = 0;
  {
    const uint8_t* __restrict__ kcn_ = v.kcn;
    const uint8_t* __restrict__ ki_ = v.ki;
    uint8_t* __restrict__ kin_ = v.kin;
    uint8_t* __restrict__ flip_ = v.flip;
    constexpr int U = 4;
    for (int i00 = 0; i00 < nx; i00 += U * P.rs) {  // uniform trip count (ballots inside)
      int c0[U], c1[U], k[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = min(i00 + u * P.rs + P.r0, nx - 1);
        c0[u] = kcn_[i];
        c1[u] = kcn_[wrap(i + 1, nx)];
        k[u] = ki_[i];
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = i00 + u * P.rs + P.r0;
        uint8_t f = 0;
        if (i < nx) {
          const uint8_t kin = (uint8_t)(c0[u] | c1[u]);
          kin_[i] = kin;
          f = (kin && !k[u]) ? 1 : 0;
          flip_[i] = f;
        }
        anyflip |= f;
        list_append(f != 0, i, v.klist, &sflags[40]);
      }
    }
  }
  if (anyflip) atomicOr(&sflags[0], 1);
  P.sync();
  PK_PTICK(2)
  const int nflip = sflags[40];
  if (dbg && tid == 0) pk_red_add(dbg + 10, nflip);
  if (sflags[0]) {
    if (a.reinit == 0) {
      if (a.lift_order != 1 && a.lift_order != 2) {
        if (tid == 0) set_status(a.status, PK_ERR_BAD_LIFT, v.b, step);
        return false;
      }
      if (a.lift_order >= 2 && a.time_elim != 0 && a.time_elim != 1) {
        if (tid == 0) set_status(a.status, PK_ERR_BAD_LIFT, v.b, step);
        return false;
      }
      // lift scalars at the flipped interfaces (lifting.py:63-88); dE_dt = (E - E_prev)/dt
      for (int q = P.r0; q < nflip; q += P.rs) {
        const int i = v.klist[q];
        const int in_ = wrap(i + 1, nx);
        const double dJ = 0.5 * (v.tD[i] + v.tD[in_]);
        v.tE[i] = dJ - E_[i] * v.J[i];           // drift
        v.tA[i] = 0.5 * (v.tC[i] + v.tC[in_]);   // R_if
      }
      P.sync();
      for (int q = P.w0; q < nflip; q += P.ws) {
        const int i = v.klist[q];
        LiftRow L;
        const size_t o = (size_t)v.b * nx + i;
        L.negJ = a.neg_eps[o] * v.J[i];
        L.e2 = a.eps2[o];
        L.drift = v.tE[i];
        L.Rif = v.tA[i];
        double bx, bsq;
        if constexpr (T < 0) {
          double* row = gin + (size_t)i * nv;
          double* scr = sm.wrow + warp * BIG_SCR;
          big_row_lift(row, L, a.lift_order, a.time_elim == 1, 1, m, scr, lane);
          big_row_moments(row, m, scr, false, bx, bsq);
        } else {
          double g[Layout<T>::S];
          row_lift<T>(g, L, a.lift_order, a.time_elim == 1, 1, sm, m, sm.wrow + warp * nv, lane);
          row_store<T>(g, gin + (size_t)i * nv, lane, nv);
          row_moments<T>(g, sm, m, sm.wrow + warp * nv, lane, bx, bsq);
        }
        if (lane == 0) v.blift[i] = bx;
      }
    } else if (a.reinit == 1) {
      for (int q = P.w0; q < nflip; q += P.ws) {
        const int i = v.klist[q];
        row_zero_store<T>(gin + (size_t)i * nv, lane, nv);
        if (lane == 0) v.blift[i] = 0.0;
      }
    } else {
      if (tid == 0) set_status(a.status, PK_ERR_BAD_REINIT, v.b, step);
      return false;
    }
  }
  P.sync();
  // masked projection moment (hybrid.py:103-105) on the post-flip rows
  PK_PTICK(3)
  {
    uint8_t* __restrict__ ki_ = v.ki;
    uint8_t* __restrict__ kc_ = v.kc;
    const uint8_t* __restrict__ kin_ = v.kin;
    const uint8_t* __restrict__ kcn_ = v.kcn;
    const uint8_t* __restrict__ flip_ = v.flip;
    const double* __restrict__ blift_ = v.blift;
    const double* __restrict__ fl_ = v.fl;
    double* __restrict__ bm_ = v.bm;
    constexpr int U = 4;
    for (int i0 = P.r0; i0 < nx; i0 += U * P.rs) {
      int k[U], kn[U], kcv[U], f[U];
      double bl[U], fv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = min(i0 + u * P.rs, nx - 1);
        k[u] = ki_[i];
        kn[u] = kin_[i];
        kcv[u] = kcn_[i];
        f[u] = flip_[i];
        bl[u] = blift_[i];
        fv[u] = fl_[i];
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = i0 + u * P.rs;
        if (i < nx) {
          const bool valid = moment_all || k[u];
          bm_[i] = kn[u] ? (f[u] ? bl[u] : (valid ? fv[u] : 0.0)) : 0.0;
          if (!moment_all && f[u]) nzin[i] = 1;
          kc_[i] = (uint8_t)kcv[u];
          ki_[i] = (uint8_t)kn[u];
        }
      }
    }
  }
  P.sync();
  PK_PTICK(4)
  // projection coefficient dc (kinetic.py:190-191) and E-upwind factor
  // max(E,0)/dvx or min(E,0)/dvx (kinetic.py:177-178); zero the output rows of
  // interfaces that are not kinetic this step but may hold data in the output
  // buffer (kinetic->fluid transitions, hybrid.py:166)
  {
    const double* __restrict__ bm_ = v.bm;
    const uint8_t* __restrict__ ki_ = v.ki;
    double* __restrict__ dco_ = v.dco;
    double* __restrict__ vco_ = v.vco;
    int8_t* __restrict__ vsg_ = v.vsg;
    uint8_t* __restrict__ nzo = nzout;
    constexpr int U = 4;
    for (int i00 = 0; i00 < nx; i00 += U * P.rs) {  // uniform trip count (ballots inside)
      double b1[U], b0[U], e[U];
      int k[U], nz[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = min(i00 + u * P.rs + P.r0, nx - 1);
        b1[u] = bm_[wrap(i + 1, nx)];
        b0[u] = bm_[wrap(i - 1, nx)];
        e[u] = E_[i];
        k[u] = ki_[i];
        nz[u] = nzo[i];
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = i00 + u * P.rs + P.r0;
        bool z = false;
        if (i < nx) {
          dco_[i] = qdiv(b1[u] - b0[u], m.two_dx, m.rtwo_dx);
          vsg_[i] = e[u] > 0.0 ? 1 : (e[u] < 0.0 ? -1 : 0);
          vco_[i] = qdiv(e[u], m.dvx, m.rdvx);
          z = !k[u] && nz[u];
          if (z) nzo[i] = 0;
        }
        // rows to zero are listed; the next micro phase zeroes them, spread
        // over every warp of the cluster
        list_append(z, i, v.zlist, &sflags[41]);
      }
    }
  }
  P.sync();
  PK_PTICK(5)
  if (P.rank == 0 && tid == 0) {
    *v.nzl = sflags[41];
    if (dbg) pk_red_add(dbg + 11, sflags[41]);
  }
  PK_PTICK(6)
  // compacted kinetic-row list (order preserving: contiguous chunks per
  // participating thread, in (rank, thread) order)
  const int per = (nx + P.rs - 1) / P.rs;
  const int lo = min(nx, P.r0 * per), hi = min(nx, lo + per);
  int cnt = 0;
  for (int i = lo; i < hi; ++i) cnt += v.ki[i] ? 1 : 0;
  int pre;
  const int total = P.scan(cnt, &pre, sm.misc + 1);
  for (int i = lo; i < hi; ++i)
    if (v.ki[i]) v.klist[pre++] = i;
  if (P.rank == 0 && tid == 0) *v.nk = total;
  if (dbg && tid == 0) pk_red_add(dbg + 12, total);
  P.sync();
  PK_PTICK(7)
  // row-stream positions for the producer/consumer micro phase: entry p needs
  // rows i-1, i, i+1; the rows not already needed by entry p-1 are
  // min(3, i_p - i_{p-1}); kpos[p] = inclusive scan (stream end after p)
  {
    const int pe = (total + P.rs - 1) / P.rs;
    const int a0 = min(total, P.r0 * pe), a1 = min(total, a0 + pe);
    int c = 0;
    for (int q = a0; q < a1; ++q) c += q == 0 ? 3 : min(3, v.klist[q] - v.klist[q - 1]);
    int pre2;
    P.scan(c, &pre2, sm.misc + 1);
    for (int q = a0; q < a1; ++q) {
      const int i = v.klist[q];
      const int nn = q == 0 ? 3 : min(3, i - v.klist[q - 1]);
      pre2 += nn;
      v.kpos[q] = pre2;
      // the stream's row ids: entry q adds rows i+2-nn .. i+1 (unwrapped)
      for (int t = 0; t < nn; ++t) v.kstream[pre2 - nn + t] = i + 2 - nn + t;
    }
  }
  P.sync();
  PK_PTICK(8)
#undef PK_PTICK
  return true;
}

// Slice phase after step s: masked rho update and field.  Returns false on a
// solvability violation.  kc/ki are the labels the step ran with.
static __device__ bool finish_step(const FineArgs& a, SliceView& v, const Smem& sm, int ph, int step,
                            const Par& Q) {
  const MeshDev& m = a.m;
  const int nx = m.nx;
  const int tid = threadIdx.x;
  const PhaseDev& P = a.ph[ph];
  const size_t o = (size_t)v.b * nx;
  const double cflu = P.cflu[v.b];
  const double cs = P.cmacs ? P.cmacs[v.b] : __longlong_as_double(0x7ff8000000000000LL);
  // the exact field's source (rho' - rho_bar) dx is formed here, into the
  // buffer the field is solved in (the outgoing E_prev, rotated below), when
  // the leader solves on that buffer (slice_field's generic path)
  const bool pre_src = a.exact_scan && !Q.dist && !(sm.scan && a.local_smem == 0);
  double* const src = v.Eprev;
  const double rb = v.rb, dx = m.dx;
  for (int i = Q.r0; i < nx; i += Q.rs) {
    const int ip = wrap(i - 1, nx);
    const double rho = v.rho[i];
    double r;
    if (v.kc[i]) {
      const double fi = v.ki[i] ? v.fl[i] : 0.0;
      const double fp = v.ki[ip] ? v.fl[ip] : 0.0;
      // constant eps: one scalar, no per-row loads (bitwise the same value)
      const double ci = cs == cs ? cs : P.cmac[o + i], cp = cs == cs ? cs : P.cmac[o + ip];
      r = (ci == cp) ? rho - ci * (fi - fp) : rho - (ci * fi - cp * fp);
    } else {
      r = rho + cflu * (v.J[i] - v.J[ip]);
    }
    v.rho[i] = r;  // in place: each rho_i update reads only its own rho_i
    if (pre_src) src[i] = (r - rb) * dx;
  }
  Q.sync();
  // the new field is solved in place in the E_prev buffer; the old E becomes
  // E_prev (pointer rotation)
  double* t = v.Eprev;
  v.Eprev = v.E;
  v.E = t;
  bool ok = true;
  if (Q.dist && !a.exact_scan) {  // fast mode: every CTA of the cluster
    const long long t0 = (a.prof && v.b == 0 && Q.rank == 0 && tid == 0) ? clock64() : 0;
    ok = cluster_field_fast(m, v.rho, v.rb, v.E, a.rtol, sm.red, Q.rank, Q.C);
    if (t0) pk_red_add(a.prof + 11, clock64() - t0);
  } else if (Q.rank == 0) {  // the leader CTA solves the field
    // on chip, exact: the zero-mean shift stays pending (v.Emean) until the
    // next prepare_step's first pass (or the end of the window) applies it
    const bool pend = a.exact_scan && a.local_smem != 0 && !Q.dist;
    ok = slice_field(m, v.rho, v.rb, v.E, v.E, a.rtol, a.exact_scan, a.local_smem != 0, sm,
                     (a.prof && v.b == 0) ? a.prof + 8 : nullptr, pre_src,
                     pend ? &v.Emean : nullptr);
    v.Epend = pend && ok;
    if (!v.Epend) v.Emean = 0.0;
  }
  if (Q.dist && a.exact_scan) {
    if (Q.rank == 0 && tid == 0) Q.flags[42] = ok;
    Q.sync();
    ok = Q.flags[42] != 0;
  }
  if (!ok) {
    if (Q.rank == 0 && tid == 0) set_status(a.status, PK_ERR_SOLVABILITY, v.b, step);
    return false;
  }
  return true;
}

// ---------------------------------------------------------------------------
// Micro phase, TMA path (fast layouts): this warp's share of the kinetic
// rows.  The rows it needs (i-1, i, i+1 for each listed i, deduplicated;
// the list is sorted so the unwrapped row sequence is increasing) form a
// stream; stream position q lives in ring slot (qb+q) % S and completes phase
// ((qb+q) / S) & 1 of that slot's mbarrier.  One lane issues the bulk
// copies up to S-1 rows ahead of the consumer.
struct RowStream {
  int p_prod, e_next, e_end, hi_p, q_prod;  // producer
  int hi_c, qhi_c;                          // consumer
};

template <int T, int S>
__device__ void micro_phase_tma(const FineArgs& a, const SliceView& v, const Smem& sm, int ph,
                                const double* gin, double* gout, int wg, int nwg, double* ring,
                                uint64_t* mbar, uint32_t& qbase) {
  const MeshDev& m = a.m;
  const int nx = m.nx;
  constexpr int NV = 32 * T;
  const int lane = threadIdx.x & 31;
  const int nk = __ldcg(v.nk);
  const bool dense = nk == nx;
  const int p0 = (int)(((long long)wg * nk) / nwg);
  const int p1 = (int)(((long long)(wg + 1) * nk) / nwg);
  if (p0 >= p1) return;
  const PhaseDev& P = a.ph[ph];
  const size_t o = (size_t)v.b * nx;
  FastConsts<T> C;
  C.load(sm.vx, sm.M, sm.xiM, lane);
  auto rowid = [&](int p) { return dense ? p : __ldcg(v.klist + p); };

  // the rows written by the previous step / slice phase are read below by TMA
  // (async proxy)
  if (lane == 0) fence_proxy_async_global();
  __syncwarp();

  RowStream st;
  st.p_prod = p0;
  st.e_next = 1;
  st.e_end = 0;  // empty: fetch the first entry's range
  st.hi_p = -3;
  st.q_prod = 0;
  st.hi_c = -3;
  st.qhi_c = -1;
  const uint32_t bytes = NV * 8;

  auto pump = [&](int q_limit) {
    while (st.q_prod < q_limit) {
      if (st.e_next > st.e_end) {
        if (st.p_prod >= p1) break;
        const int i = rowid(st.p_prod++);
        st.e_next = max(i - 1, st.hi_p + 1);
        st.e_end = i + 1;
        continue;
      }
      if (lane == 0) {
        const uint32_t Q = qbase + (uint32_t)st.q_prod;
        const int slot = (int)(Q % S);
        uint64_t* mb = mbar + slot;
        // slot reuse: its previous contents were read into registers and
        // consumed by this warp's arithmetic before this point (program
        // order), so no proxy fence is needed here
        mbar_expect_tx(mb, bytes);
        bulk_g2s(ring + slot * NV, gin + (size_t)wrap(st.e_next, nx) * NV, bytes, mb);
      }
      st.hi_p = st.e_next;
      ++st.e_next;
      ++st.q_prod;
    }
  };
  auto fetch = [&](double (&r)[T], int q) {
    const uint32_t Q = qbase + (uint32_t)q;
    const int slot = (int)(Q % S);
    mbar_wait(mbar + slot, (Q / S) & 1);
    const double* src = ring + slot * NV;
#pragma unroll
    for (int s = 0; s < T; ++s) r[s] = src[Fast<T>::col(lane, s)];
  };

  pump(S);
  // per-row coefficients, 32 list entries at a time (one coalesced load per
  // array, broadcast by shuffle)
  double c_vco = 0, c_dco = 0, c_J = 0, c_k1 = 0, c_k2 = 0;
  int c_vsg = 0, c_row = 0;
  int cbase = p0 - 64;
  double gp[T], gc[T], gn[T];
  int prev_i = -5;
  for (int p = p0; p < p1; ++p) {
    if (p - cbase >= 32) {
      cbase = p;
      const int pl = p + lane;
      if (pl < p1) {
        const int r = rowid(pl);
        c_row = r;
        c_vco = __ldcg(v.vco + r);
        c_dco = __ldcg(v.dco + r);
        c_J = __ldcg(v.gJ + r);
        c_vsg = __ldcg(v.vsg + r);
        c_k1 = __ldg(P.k1 + o + r);
        c_k2 = __ldg(P.k2 + o + r);
      }
    }
    const int src = p - cbase;
    const int i = __shfl_sync(FULL, c_row, src);
    // stream positions of rows i-1, i, i+1
    int q_im1;
    if (i - 1 > st.hi_c) {
      q_im1 = st.qhi_c + 1;
      st.qhi_c += 3;
    } else {
      st.qhi_c += (i + 1) - st.hi_c;
      q_im1 = st.qhi_c - 2;
    }
    st.hi_c = i + 1;
    if (i == prev_i + 1) {
#pragma unroll
      for (int s = 0; s < T; ++s) {
        gp[s] = gc[s];
        gc[s] = gn[s];
      }
      fetch(gn, q_im1 + 2);
    } else {
      fetch(gp, q_im1);
      fetch(gc, q_im1 + 1);
      fetch(gn, q_im1 + 2);
    }
    RowCoef rc;
    rc.vsg = __shfl_sync(FULL, c_vsg, src);
    rc.vco = __shfl_sync(FULL, c_vco, src);
    rc.dc = __shfl_sync(FULL, c_dco, src);
    rc.J = __shfl_sync(FULL, c_J, src);
    rc.k1 = __shfl_sync(FULL, c_k1, src);
    rc.k2 = __shfl_sync(FULL, c_k2, src);
    double out[T];
    fast_micro<T>(gp, gc, gn, out, C, rc, m.dx, m.rdx, lane);
    __syncwarp();
    pump(q_im1 + 1 + S);  // positions < pos(i) are free (already consumed)
    fast_store<T>(out, gout + (size_t)i * NV, lane);
    double bx, bsq;
    fast_moments<T>(out, sm, m.dv3, lane, bx, bsq);
    if (lane == 0) {
      v.fl_w[i] = bx;
      v.sq_w[i] = bsq;
    }
    prev_i = i;
  }
  qbase += (uint32_t)st.q_prod;
}

// Micro phase, G8 layout (nv = 16 CH: 64, 128): eight lanes own one row and
// lane k owns the whole pairwise chain k of the velocity fold (columns
// k + 8m and their mirrors nv-1-k-8m), so the bracket needs no cross-lane
// traffic until the final 8-way tree; a warp advances four rows at a time.
// Every operand (row i, its x-neighbours, the velocity neighbours) is read
// from the TMA ring in shared memory; ring rows are padded by 64 B so the
// four groups of a warp hit distinct bank halves.
template <int CH, int S, bool DENSE, bool SQ>
__device__ void micro_phase_g8(const FineArgs& a, const SliceView& v, const Smem& sm, int ph,
                               const double* gin, double* gout, int p0, int p1, double* ring,
                               uint64_t* mbar, uint32_t& qbase) {
  constexpr int NV = 16 * CH;
  constexpr int RS = NV + 8;  // ring row stride in doubles (64 B pad)
  // an operation holds rows p-1 .. p+4 of the stream at once: a shallower
  // ring would wait forever for a slot it has not released
  static_assert(S >= 6, "G8 ring needs >= 6 slots per warp");
  const MeshDev& m = a.m;
  const int nx = m.nx;
  const int lane = threadIdx.x & 31;
  const int k = lane & 7, gr = lane >> 3;
  const PhaseDev& P = a.ph[ph];
  const size_t o = (size_t)v.b * nx;
  const uint32_t s_vx = smem_u32(sm.vx), s_M = smem_u32(sm.M);
  const uint32_t s_ring = smem_u32(ring), s_mbar = smem_u32(mbar);
  const double dx = m.dx, rdx = m.rdx, dv3 = m.dv3;
  const double NaN_ = __longlong_as_double(0x7ff8000000000000LL);
  const double k1u = P.k1s ? P.k1s[v.b] : NaN_, k2u = P.k2s ? P.k2s[v.b] : NaN_;
  const bool kuni = k1u == k1u && k2u == k2u;
  auto rowid = [&](int p) { return DENSE ? p : __ldcg(v.klist + p); };
  // listed rows: this warp's next 32 row ids ride in the lanes (one L2 round
  // trip for the producer logic and the first coefficient batch together; a
  // load per listed row made the start of a sparse phase a chain of them)
  int rw_base = p0;
  int rw = (!DENSE && p0 + lane < p1) ? __ldcg(v.klist + p0 + lane) : 0;
  auto rowid_u = [&](int p) {  // p uniform over the warp
    if (DENSE) return p;
    if (p - rw_base >= 32) {
      rw_base = p;
      rw = p + lane < p1 ? __ldcg(v.klist + p + lane) : 0;
    }
    return __shfl_sync(FULL, rw, p - rw_base);
  };

  if (lane == 0) fence_proxy_async_global();  // rows written by the generic proxy, read by TMA
  __syncwarp();

  // ---- row stream: producer (lane 0 issues) and consumer position logic ----
  // DENSE: the stream is rows p0-1 .. p1, position q <-> row p0-1+q.
  RowStream st;
  st.p_prod = p0;
  st.e_next = 1;
  st.e_end = 0;
  st.hi_p = -3;
  st.q_prod = 0;
  st.hi_c = -3;
  st.qhi_c = -1;
  const int q_end = DENSE ? (p1 - p0 + 2) : 0x7fffffff;
  constexpr uint32_t bytes = NV * 8;
  auto issue = [&](int q, int row) {
    if (lane == 0) {
      const uint32_t Q = qbase + (uint32_t)q;
      const uint32_t slot = Q % S;
      const uint32_t mb = s_mbar + 8 * slot;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes)
                   : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
              "r"(s_ring + slot * (RS * 8)),
          "l"(gin + (size_t)wrap(row, nx) * NV), "r"(bytes), "r"(mb)
          : "memory");
    }
  };
  auto pump = [&](int q_limit) {
    if (DENSE) {
      // all pending rows in ONE instruction, one lane per row: a bulk copy
      // costs ~185 cycles of issue per thread, lanes overlap (~52 per extra)
      const int lim = min(q_limit, q_end);
      const int n = lim - st.q_prod;
      if (n > 0 && lane < n) {
        const int q = st.q_prod + lane;
        const uint32_t Q = qbase + (uint32_t)q;
        const uint32_t slot = Q % S;
        const uint32_t mb = s_mbar + 8 * slot;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes)
                     : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
                "r"(s_ring + slot * (RS * 8)),
            "l"(gin + (size_t)wrap(p0 - 1 + q, nx) * NV), "r"(bytes), "r"(mb)
            : "memory");
      }
      if (n > 0) st.q_prod = lim;
      return;
    }
    while (st.q_prod < q_limit) {
      if (st.e_next > st.e_end) {
        if (st.p_prod >= p1) break;
        const int i = rowid_u(st.p_prod++);
        st.e_next = max(i - 1, st.hi_p + 1);
        st.e_end = i + 1;
        continue;
      }
      issue(st.q_prod, st.e_next);
      st.hi_p = st.e_next;
      ++st.e_next;
      ++st.q_prod;
    }
  };
  auto slot_addr = [&](int q) {
    const uint32_t Q = qbase + (uint32_t)q;
    const uint32_t slot = Q % S;
    const uint32_t mb = s_mbar + 8 * slot, par = (Q / S) & 1;
    uint32_t done;
    do {
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
          : "=r"(done)
          : "r"(mb), "r"(par)
          : "memory");
    } while (!done);
    return s_ring + slot * (RS * 8);
  };

  // this lane's column constants (columns k + 8 mm and their mirrors) stay in
  // registers for the whole phase
  double vxr[CH], Mr[CH];
#pragma unroll
  for (int mm = 0; mm < CH; ++mm) {
    vxr[mm] = lds64(s_vx + 8 * (k + 8 * mm));
    Mr[mm] = lds64(s_M + 8 * (k + 8 * mm));
  }
  pump(S);
  // per-row coefficients, one row per lane, 32 rows per batch
  struct Coef {
    double vco = 0, dco = 0, J = 0, k1 = 0, k2 = 0;
    int row = 0;
  };
  auto load_batch = [&](int base, Coef& c) {
    const int pl = base + lane;
    if (pl < p1) {
      const int r = (!DENSE && base == rw_base) ? rw : rowid(pl);
      // signed E-upwind factor: (g - g_nb) * (+-vco) reproduces both of the
      // reference's forms bitwise (kinetic.py:176-187); 0 when E == 0
      const int sg = __ldcg(v.vsg + r);
      const double vco = __ldcg(v.vco + r);
      c.vco = sg > 0 ? vco : (sg < 0 ? -vco : 0.0);
      c.dco = __ldcg(v.dco + r);
      c.J = __ldcg(v.gJ + r);
      if (!kuni) {  // constant eps: kappa1/2 are per-slice scalars
        c.k1 = __ldg(P.k1 + o + r);
        c.k2 = __ldg(P.k2 + o + r);
      }
      // neighbour direction rides in the sign bit of the row id
      c.row = sg > 0 ? r : -1 - r;
    }
  };
  Coef cur, nxt;
  int cbase = p0 - 64;
  if (DENSE) {  // rows advance four per operation: batches at p0 + 32 n, the next one in flight
    cbase = p0;
    load_batch(p0, cur);
    load_batch(p0 + 32, nxt);
  }
  for (int p = p0; p < p1;) {
    if (DENSE) {
      if (p - cbase >= 32) {
        cur = nxt;
        cbase += 32;
        load_batch(cbase + 32, nxt);
      }
    } else if (p + 4 - cbase > 32) {
      cbase = p;
      load_batch(p, cur);
    }
    const double c_vco = cur.vco, c_dco = cur.dco, c_J = cur.J, c_k1 = cur.k1, c_k2 = cur.k2;
    const int c_row = cur.row;
    // entries of this operation (up to four, within the ring window)
    int nent, my_q, last_q;
    if (DENSE) {
      nent = min(4, p1 - p);
      my_q = p + gr - p0;            // position of row (p+gr)-1
      last_q = p + nent - 1 - p0;
    } else {
      nent = 0;
      my_q = 0;
      last_q = 0;
      int q0 = 0;
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        if (p + g < p1 && nent == g) {
          int i = __shfl_sync(FULL, c_row, p + g - cbase);
          i = i < 0 ? -1 - i : i;
          int q_im1, hi = st.hi_c, qhi = st.qhi_c;
          if (i - 1 > hi) {
            q_im1 = qhi + 1;
            qhi += 3;
          } else {
            qhi += (i + 1) - hi;
            q_im1 = qhi - 2;
          }
          if (g == 0) q0 = q_im1;
          if (g == 0 || q_im1 + 2 - q0 + 1 <= S) {
            st.hi_c = i + 1;
            st.qhi_c = qhi;
            nent = g + 1;
            last_q = q_im1;
            if (g == gr) my_q = q_im1;
          }
        }
      }
    }
    const bool active = gr < nent;
    const int src = min(p + gr - cbase, 31);
    const int rsg = __shfl_sync(FULL, c_row, src);
    const double svco = __shfl_sync(FULL, c_vco, src);
    const double dc = __shfl_sync(FULL, c_dco, src);
    const double J = __shfl_sync(FULL, c_J, src);
    const double k1 = kuni ? k1u : __shfl_sync(FULL, c_k1, src);
    const double k2 = kuni ? k2u : __shfl_sync(FULL, c_k2, src);
    const bool up = rsg >= 0;          // E > 0 (or 0): velocity neighbour j-1
    const int i = up ? rsg : -1 - rsg;
    double bx = 0.0, bsq = 0.0;
    if (active) {
      const uint32_t rp = slot_addr(my_q), rcu = slot_addr(my_q + 1), rn = slot_addr(my_q + 2);
      double* row = gout + (size_t)i * NV;
#pragma unroll
      for (int mm = 0; mm < CH; ++mm) {
        const int c = k + 8 * mm, u = NV - 1 - c;
        // mirrored grid (m.mirror): vx[u] = -vx[c], M[u] = M[c], and xiM is
        // vx * M as the host formed it, so one column's constants serve both
        // halves and xiM costs a multiply instead of a shared-memory load
        const double vxc = vxr[mm], vxu = -vxc;
        const double Mc = Mr[mm];
        const double xMc = vxc * Mc, xMu = -xMc;
        double lo, hi;
        {  // lower half, xi < 0: x-upwind from row i+1; zero inflow at -v*
          const double g = lds64(rcu + 8 * c);
          double oo = vxc * (lds64(rn + 8 * c) - g);
          oo = qdiv(oo, dx, rdx);
          const int cn = up ? c - 1 : c + 1;
          const double nb = cn >= 0 ? lds64(rcu + 8 * cn) : 0.0;
          oo = oo + (g - nb) * svco;
          oo = oo - Mc * dc;
          const double forcing = oo + xMc * J;
          lo = k1 * g - k2 * forcing;
        }
        {  // upper half, xi > 0: x-upwind from row i-1; zero inflow at +v*
          const double g = lds64(rcu + 8 * u);
          double oo = vxu * (g - lds64(rp + 8 * u));
          oo = qdiv(oo, dx, rdx);
          const int un = up ? u - 1 : u + 1;
          const double nb = un < NV ? lds64(rcu + 8 * un) : 0.0;
          oo = oo + (g - nb) * svco;
          oo = oo - Mc * dc;
          const double forcing = oo + xMu * J;
          hi = k1 * g - k2 * forcing;
        }
        __stcg(row + c, lo);
        __stcg(row + u, hi);
        // row moments: fold (lo + mirror), in-lane pairwise chain k
        const double f = vxc * lo + vxu * hi;
        bx = mm == 0 ? f : bx + f;
        if (SQ) {
          const double h = lo * lo + hi * hi;
          bsq = mm == 0 ? h : bsq + h;
        }
      }
    }
    __syncwarp();
    pump(last_q + 1 + S);  // positions < pos(last row) are consumed
    bx = bx + __shfl_xor_sync(FULL, bx, 1);
    bx = bx + __shfl_xor_sync(FULL, bx, 2);
    bx = bx + __shfl_xor_sync(FULL, bx, 4);
    if (SQ) {
      bsq = bsq + __shfl_xor_sync(FULL, bsq, 1);
      bsq = bsq + __shfl_xor_sync(FULL, bsq, 2);
      bsq = bsq + __shfl_xor_sync(FULL, bsq, 4);
    }
    if (active && k == 0) {
      v.fl_w[i] = bx * dv3;
      if (SQ) v.sq_w[i] = bsq * dv3;
    }
    p += nent;
  }
  qbase += (uint32_t)st.q_prod;
}

// ---------------------------------------------------------------------------
// Micro phase, producer/consumer pipeline with the GS layout (nv = 64 SEG:
// 64, 128, 256).
//
// One producer warp per CTA streams the rows this CTA needs (each fetched
// once; i-1, i, i+1 of every listed row, deduplicated) into a CTA-wide TMA
// ring: `full[slot]` completes when a row has landed, `done[op]` when a
// consumer warp has finished an operation, which is what allows a slot to be
// refilled.  Consumer warps take operations round-robin; an operation is
// 4/SEG listed rows, each served by 8 SEG lanes.  Lane (k, seg) owns terms
// m = 4 seg .. 4 seg + 3 of pairwise chain k of the velocity fold (columns
// k + 8m and their mirrors nv-1-k-8m): 8 values, velocity constants in
// registers, 3 shared-memory reads per value, and the chain passes between
// segments in numpy's order with one shuffle hop per segment.
template <int SEG>
struct GS {
  static constexpr int NV = 64 * SEG;   // velocities
  static constexpr int LPR = 8 * SEG;   // lanes per row
  static constexpr int RPO = 4 / SEG;   // rows per operation
  static constexpr int RS = NV + 8;     // ring row stride (doubles): 64 B pad
};

// velocity constants of a lane's 8 columns; xi M is recomputed as
// fl(vx * M), which is exactly how the host formed it (mesh.py:167)
template <int SEG>
struct GSConsts {
  uint32_t s_vx, s_M, s_xiM;  // shared-memory addresses of the constant rows
  __device__ void load(const Smem& sm, int) {
    s_vx = smem_u32(sm.vx);
    s_M = smem_u32(sm.M);
    s_xiM = smem_u32(sm.xiM);
  }
};

__device__ __forceinline__ void mbar_wait_u32(uint32_t mb, uint32_t par) {
  uint32_t ok;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(mb), "r"(par)
        : "memory");
  } while (!ok);
}

template <int SEG, int R>
__device__ void micro_phase_pc(const FineArgs& a, const SliceView& v, int ph, const double* gin,
                               double* gout, int e0, int e1, bool dense, int nc, double* ring,
                               uint64_t* full, uint64_t* done, uint32_t& qbase, uint32_t& obase,
                               const GSConsts<SEG>& C) {
  using L = GS<SEG>;
  constexpr int NV = L::NV, RPO = L::RPO, RS = L::RS, Q = R;
  const MeshDev& m = a.m;
  const int nx = m.nx;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nent = e1 - e0;
  const int nops = (nent + RPO - 1) / RPO;
  const int kp0 = dense ? 0 : __ldcg(v.kpos + e0);
  const int nstream = nent <= 0 ? 0 : (dense ? nent + 2 : __ldcg(v.kpos + e1 - 1) - kp0 + 3);
  const int ngrp = (nstream + 7) >> 3;  // rows travel in groups of 8 (one barrier per group)
  constexpr int NG = R / 8;
  const uint32_t s_ring = smem_u32(ring), s_full = smem_u32(full), s_done = smem_u32(done);
  constexpr uint32_t bytes = NV * 8;

  if (nent > 0 && warp == nc) {
    // ---------------- producer warp ----------------
    // eight lanes issue one padded row each per group: a bulk copy costs
    // ~185 cycles of issue per thread, so rows are issued eight at a time
    if (lane == 0) fence_proxy_async_global();  // rows written by the generic proxy
    __syncwarp();
    const int i0 = dense ? e0 : __ldcg(v.klist + e0);
    int pw = e0;
    int jw = 0;  // next operation whose completion has not been observed
    // stream positions of the entries after pw, 32 at a time in the lanes
    // (kpos is increasing): one L2 round trip per 32 entries -- walking kpos
    // entry by entry cost a dependent L2 load per entry, ~700 cycles a row,
    // and bounded the whole sparse micro phase
    auto kwin = [&](int base) {
      const int q = base + 1 + lane;
      return !dense && q < e1 ? __ldcg(v.kpos + q) - kp0 : 0x7fffffff;
    };
    int wb = e0, kq = kwin(e0);
    for (int g = 0; g < ngrp; ++g) {
      const uint32_t G = (qbase >> 3) + (uint32_t)g;
      if (g >= NG) {
        // the group's previous occupant (positions up to x) is free once every
        // operation up to its last reader is done; operations run on
        // different warps and finish out of order, so wait for all of them
        const int x = (g - NG) * 8 + 7;
        int plast;
        if (dense) {
          plast = min(e0 + x, e1 - 1);
        } else {
          // position of row i-1 of entry p is kpos[p] - kpos[e0]: the last
          // entry whose rows start at or before x
          for (;;) {
            const int off = pw - wb;  // lane off + t holds entry pw + 1 + t
            const unsigned bal = __ballot_sync(FULL, lane >= off && kq <= x) >> off;
            pw += bal == FULL ? 32 : __ffs(~bal) - 1;
            if (pw - wb < 32) break;
            wb = pw;  // window used up: the next 32 entries
            kq = kwin(wb);
          }
          plast = pw;
        }
        const int jl = (plast - e0) / RPO;
        for (; jw <= jl; ++jw) {
          const uint32_t J = obase + (uint32_t)jw;
          mbar_wait_u32(s_done + 8 * (J % Q), (J / Q) & 1);
        }
      }
      const int nrows = min(8, nstream - 8 * g);
      const uint32_t mb = s_full + 8 * (G % NG);
      if (lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb),
                     "r"(bytes * nrows)
                     : "memory");
      __syncwarp();
      if (lane < nrows) {
        const int q = 8 * g + lane;
        const int row = dense ? e0 - 1 + q : (q < 3 ? i0 - 1 + q : __ldcg(v.kstream + kp0 + q - 3));
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
                "r"(s_ring + ((G % NG) * 8 + lane) * (RS * 8)),
            "l"(gin + (size_t)wrap(row, nx) * NV), "r"(bytes), "r"(mb)
            : "memory");
      }
    }
  } else if (nent > 0 && warp < nc) {
    // ---------------- consumers ----------------
    const int k = lane & 7, seg = (lane >> 3) % SEG, grp = lane / L::LPR;
    const double dx = m.dx, rdx = m.rdx, dv3 = m.dv3;
    const PhaseDev& P = a.ph[ph];
    const size_t o = (size_t)v.b * nx;
    // coefficients of the next 32/RPO operations of this warp, one entry per lane
    double c_vco = 0, c_dco = 0, c_J = 0, c_k1 = 0, c_k2 = 0;
    int c_row = 0, c_pos = 0;
    int jb = -1 << 30;  // first operation of the loaded batch
    constexpr int OPB = 32 / RPO;
    // optional profile (slice 0's leader CTA, consumer warp 0): cycles spent
    // on coefficients, waiting for rows, and in the row operation
    const bool cprof = a.prof && v.b == 0 && warp == 0 && blockIdx.x == 0;
    long long tq0 = cprof ? clock64() : 0, tq_coef = 0, tq_wait = 0, tq_op = 0;
    for (int j = warp; j < nops; j += nc) {
      const int jj = (j - warp) / nc;  // this warp's operation ordinal
      if (jj - jb >= OPB) {
        jb = jj;
        const int pl = e0 + (warp + (jb + lane / RPO) * nc) * RPO + lane % RPO;
        if (pl < e1) {
          const int r = dense ? pl : __ldcg(v.klist + pl);
          const int sg = __ldcg(v.vsg + r);
          const double vco = __ldcg(v.vco + r);
          // signed E-upwind factor: (g - g_nb) * (+-vco) reproduces both of
          // the reference's forms bitwise (kinetic.py:176-187); 0 when E == 0
          c_vco = sg > 0 ? vco : (sg < 0 ? -vco : 0.0);
          c_dco = __ldcg(v.dco + r);
          c_J = __ldcg(v.gJ + r);
          c_k1 = __ldg(P.k1 + o + r);
          c_k2 = __ldg(P.k2 + o + r);
          c_row = sg > 0 ? r : -1 - r;  // velocity-neighbour side in the sign
          c_pos = dense ? pl - e0 : __ldcg(v.kpos + pl) - kp0;
        }
      }
      const int src = (jj - jb) * RPO + grp;
      const int p = e0 + j * RPO + grp;
      const bool active = p < e1;
      const int rsg = __shfl_sync(FULL, c_row, src);
      const int pos = __shfl_sync(FULL, c_pos, src);
      const double svco = __shfl_sync(FULL, c_vco, src);
      const double dc = __shfl_sync(FULL, c_dco, src);
      const double Jv = __shfl_sync(FULL, c_J, src);
      const double k1 = __shfl_sync(FULL, c_k1, src);
      const double k2 = __shfl_sync(FULL, c_k2, src);
      const bool up = rsg >= 0;
      const int i = up ? rsg : -1 - rsg;
      double f[4], h[4];
      if (cprof) { const long long t = clock64(); tq_coef += t - tq0; tq0 = t; }
      if (active) {
        uint32_t ra[3];
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          const uint32_t Qp = qbase + (uint32_t)(pos + d), G = Qp >> 3;
          mbar_wait_u32(s_full + 8 * (G % NG), (G / NG) & 1);
          ra[d] = s_ring + ((G % NG) * 8 + (Qp & 7)) * (RS * 8);
        }
        if (cprof) { const long long t = clock64(); tq_wait += t - tq0; tq0 = t; }
        const uint32_t rp = ra[0], rc = ra[1], rn = ra[2];
        double* row = gout + (size_t)i * NV;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int c = k + 8 * (4 * seg + t), u = NV - 1 - c;
          double lo, hi, xl, xh;
          {  // lower half, xi < 0: x-upwind from row i+1; zero inflow at -v*
            const double g = lds64(rc + 8 * c);
            xl = lds64(C.s_vx + 8 * c);
            double oo = xl * (lds64(rn + 8 * c) - g);
            oo = qdiv(oo, dx, rdx);
            const int cn = up ? c - 1 : c + 1;
            const double nb = cn >= 0 ? lds64(rc + 8 * cn) : 0.0;
            oo = oo + (g - nb) * svco;
            oo = oo - lds64(C.s_M + 8 * c) * dc;
            const double forcing = oo + lds64(C.s_xiM + 8 * c) * Jv;
            lo = k1 * g - k2 * forcing;
          }
          {  // upper half, xi > 0: x-upwind from row i-1; zero inflow at +v*
            const double g = lds64(rc + 8 * u);
            xh = lds64(C.s_vx + 8 * u);
            double oo = xh * (g - lds64(rp + 8 * u));
            oo = qdiv(oo, dx, rdx);
            const int un = up ? u - 1 : u + 1;
            const double nb = un < NV ? lds64(rc + 8 * un) : 0.0;
            oo = oo + (g - nb) * svco;
            oo = oo - lds64(C.s_M + 8 * u) * dc;
            const double forcing = oo + lds64(C.s_xiM + 8 * u) * Jv;
            hi = k1 * g - k2 * forcing;
          }
          __stcg(row + c, lo);
          __stcg(row + u, hi);
          f[t] = xl * lo + xh * hi;  // fold of xi g' (mesh.py:95-109)
          h[t] = lo * lo + hi * hi;              // fold of g'^2
        }
      } else {
#pragma unroll
        for (int t = 0; t < 4; ++t) f[t] = h[t] = 0.0;
      }
      __syncwarp();
      if (lane == 0) {  // this operation's ring rows are consumed
        const uint32_t J = obase + (uint32_t)j;
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s_done + 8 * (J % Q))
                     : "memory");
      }
      // pairwise chain k in numpy's order, passed segment to segment
      double bx = ((f[0] + f[1]) + f[2]) + f[3];
      double bq = ((h[0] + h[1]) + h[2]) + h[3];
#pragma unroll
      for (int s2 = 1; s2 < SEG; ++s2) {
        const double ix = __shfl_up_sync(FULL, bx, 8);
        const double iq = __shfl_up_sync(FULL, bq, 8);
        if (seg == s2) {
          bx = (((ix + f[0]) + f[1]) + f[2]) + f[3];
          bq = (((iq + h[0]) + h[1]) + h[2]) + h[3];
        }
      }
      bx = bx + __shfl_xor_sync(FULL, bx, 1);
      bx = bx + __shfl_xor_sync(FULL, bx, 2);
      bx = bx + __shfl_xor_sync(FULL, bx, 4);
      bq = bq + __shfl_xor_sync(FULL, bq, 1);
      bq = bq + __shfl_xor_sync(FULL, bq, 2);
      bq = bq + __shfl_xor_sync(FULL, bq, 4);
      if (active && k == 0 && seg == SEG - 1) {
        v.fl_w[i] = bx * dv3;
        v.sq_w[i] = bq * dv3;
      }
      if (cprof) { const long long t = clock64(); tq_op += t - tq0; tq0 = t; }
    }
    if (cprof && lane == 0) {
      a.prof[29] += tq_coef;
      a.prof[30] += tq_wait;
      a.prof[31] += tq_op;
    }
  }
  qbase += (uint32_t)(8 * ngrp);
  obase += (uint32_t)nops;
}

// Micro phase, generic layout (any nv <= 256, no TMA): direct row loads.
static __device__ void micro_phase_gen(const FineArgs& a, const SliceView& v, const Smem& sm, int ph,
                                const double* gin, double* gout, int wg, int nwg) {
  const MeshDev& m = a.m;
  const int nx = m.nx, nv = m.nv;
  const int lane = threadIdx.x & 31;
  const int nk = __ldcg(v.nk);
  const bool dense = nk == nx;
  const int p0 = (int)(((long long)wg * nk) / nwg);
  const int p1 = (int)(((long long)(wg + 1) * nk) / nwg);
  const PhaseDev& P = a.ph[ph];
  const size_t o = (size_t)v.b * nx;
  double* wrow = sm.wrow + (threadIdx.x >> 5) * nv;
  for (int p = p0; p < p1; ++p) {
    const int i = dense ? p : __ldcg(v.klist + p);
    double gp[GT], gc[GT], gn[GT];
    gen_load(gp, gin + (size_t)wrap(i - 1, nx) * nv, lane, nv);
    gen_load(gc, gin + (size_t)i * nv, lane, nv);
    gen_load(gn, gin + (size_t)wrap(i + 1, nx) * nv, lane, nv);
    RowCoef rc;
    rc.vsg = __ldcg(v.vsg + i);
    rc.vco = __ldcg(v.vco + i);
    rc.dc = __ldcg(v.dco + i);
    rc.J = __ldcg(v.gJ + i);
    rc.k1 = P.k1[o + i];
    rc.k2 = P.k2[o + i];
    double out[GT];
    gen_micro(gp, gc, gn, out, sm.vx, sm.M, sm.xiM, rc, nv, m.nvyz, wrow, m.dx, m.rdx, lane);
    gen_store(out, gout + (size_t)i * nv, lane, nv);
    double bx, bsq;
    gen_moments(out, sm, nv, m.nvyz, m.dv3, wrow, lane, bx, bsq);
    if (lane == 0) {
      v.fl_w[i] = bx;
      v.sq_w[i] = bsq;
    }
  }
}

// Micro phase, big rows (pk_big.cuh): one warp per listed row.
static __device__ void micro_phase_big(const FineArgs& a, const SliceView& v, const Smem& sm, int ph,
                                const double* gin, double* gout, int wg, int nwg) {
  const MeshDev& m = a.m;
  const int nx = m.nx, nv = m.nv;
  const int lane = threadIdx.x & 31;
  const int nk = __ldcg(v.nk);
  const bool dense = nk == nx;
  const int p0 = (int)(((long long)wg * nk) / nwg);
  const int p1 = (int)(((long long)(wg + 1) * nk) / nwg);
  const PhaseDev& P = a.ph[ph];
  const size_t o = (size_t)v.b * nx;
  double* scr = sm.wrow + (threadIdx.x >> 5) * BIG_SCR;
  for (int p = p0; p < p1; ++p) {
    const int i = dense ? p : __ldcg(v.klist + p);
    RowCoef rc;
    rc.vsg = __ldcg(v.vsg + i);
    rc.vco = __ldcg(v.vco + i);
    rc.dc = __ldcg(v.dco + i);
    rc.J = __ldcg(v.gJ + i);
    rc.k1 = P.k1[o + i];
    rc.k2 = P.k2[o + i];
    double* row = gout + (size_t)i * nv;
    big_micro_row(gin + (size_t)wrap(i - 1, nx) * nv, gin + (size_t)i * nv,
                  gin + (size_t)wrap(i + 1, nx) * nv, row, m, rc, lane);
    double bx, bsq;
    big_row_moments(row, m, scr, a.adaptation != 0, bx, bsq);
    if (lane == 0) {
      v.fl_w[i] = bx;
      v.sq_w[i] = bsq;
    }
  }
}

// Big rows, one CTA per row (FineArgs::bigc): the reference's default 1D-3V
// grid, 32 xi planes of nvy nvz = 256 (vy, vz) columns, mirrored, xi constant
// on each plane.
//
// The thread layout follows the row moments.  <q> folds plane jx with plane
// 31-jx and sums the 4096 folded terms pairwise (mesh.py:95-133): 32 leaves
// of 128 (fold plane jx = l / 2, column block l % 2), each leaf eight
// interleaved accumulators (columns k + 8 m, m = 0..15, in order) combined by
// a butterfly, then a perfectly balanced tree over the leaves.  Thread (l, k)
// -- warp l / 4, lanes 8 (l % 4) + k -- updates exactly the nodes of its
// accumulator: columns 128 (l % 2) + k + 8 m of planes jx and 31 - jx (xi < 0
// and its mirror xi > 0), 32 nodes (their M in registers), and accumulates
// its fold terms in registers in leaf order; the leaf butterfly is
// group_leaf's (shuffles in the 8-lane group), the tree a 32-lane butterfly
// of warp 0 over the leaves in order.  One barrier per row.  Node updates:
// the operations of big_micro_row (kinetic.py:148-224) in its order, the
// zero upwind term skipped as in the fast layouts (equal up to the sign of
// zero).
//
// Staging.  Dense phases (every row kinetic, rows p0..p1-1 in order): the
// lower halves (planes 0-15) of rows p0..p1 and the upper halves (planes
// 16-31) of rows p0-1..p1-1 stream through three 32 KB shared-memory slots
// each, one TMA bulk copy per half, issued two rows ahead; row i then reads
// its own halves, the lower half of row i+1 (x neighbour for xi < 0) and the
// upper half of row i-1 (for xi > 0) from shared memory -- no global loads in
// the node loop.  Sparse phases (listed rows, hybrid): two full-row slots,
// the next listed row landing while the current one is worked on, the x
// neighbour from L2.
constexpr int BIGC_NXI = 32;   // xi planes
constexpr int BIGC_S = 256;    // (vy, vz) columns per plane

// running fill counters of the staging mbarriers: [0] full-row slots
// (mbar 0-1), [1] lower-half slots (mbar 2-4), [2] upper-half slots (mbar 5-7)
struct BigcCnt {
  uint32_t q[3];
};

// SQ: the <g^2> row moment (adaptation on) is formed too
template <bool SQ>
static __device__ void micro_phase_bigc(const FineArgs& a, const SliceView& v, const Smem& sm, int ph,
                                 const double* gin, double* gout, int crank, int C, double* rbuf,
                                 const double* sxi, uint64_t* mbar, BigcCnt& cnt) {
  constexpr int S = BIGC_S, X = BIGC_NXI, NM = 16, HX = X / 2;
  const MeshDev& m = a.m;
  const int nx = m.nx, nv = m.nv, hv = nv / 2;
  const int nk = __ldcg(v.nk);
  const bool dense = nk == nx;
  const int p0 = (int)(((long long)crank * nk) / C), p1 = (int)(((long long)(crank + 1) * nk) / C);
  if (p0 >= p1) return;
  const PhaseDev& P = a.ph[ph];
  const size_t o = (size_t)v.b * nx;
  const int tid = threadIdx.x, lane = tid & 31;
  const int l = tid >> 3, k = lane & 7;  // leaf, accumulator
  const int jx = l >> 1, jm = X - 1 - jx;
  const int col0 = (l & 1) * 128 + k;
  constexpr bool sq = SQ;
  const double xl = sxi[jx], xh = sxi[jm];
  const double dx = m.dx, rdx = m.rdx;
  double Ml[NM], Mh[NM];
#pragma unroll
  for (int u = 0; u < NM; ++u) {
    Ml[u] = __ldg(m.M + jx * S + col0 + 8 * (u ^ (l & 1)));  // (node order of the bank swizzle)
    Mh[u] = __ldg(m.M + jm * S + col0 + 8 * (u ^ (l & 1)));
  }
  auto rowid = [&](int p) { return dense ? p : __ldcg(v.klist + p); };
  auto coef = [&](int i) {
    RowCoef rc;
    rc.vsg = __ldcg(v.vsg + i);
    rc.vco = __ldcg(v.vco + i);
    rc.dc = __ldcg(v.dco + i);
    rc.J = __ldcg(v.gJ + i);
    rc.k1 = P.k1[o + i];
    rc.k2 = P.k2[o + i];
    return rc;
  };
  // one bulk copy of `bytes` from src into slot `dst`, completing mbarrier mb
  auto copy = [&](double* dst, const double* src, uint32_t bytes, uint64_t* mb) {
    mbar_expect_tx(mb, bytes);
    bulk_g2s(dst, src, bytes, mb);
  };
  // Bank swizzle.  The two leaves of a half warp (column blocks 0 and 1 of
  // one plane) sit 1 KB apart: the same 16 banks, a 2-way conflict on every
  // load.  Lanes of block 1 therefore visit their 16 columns in the order
  // 1, 0, 3, 2, ... (node u ^ odd at loop index u: the other 16 banks), and
  // the fold terms of a pair are added in node order afterwards -- the same
  // chain.  Staged data is read through the shared window (ld.shared, 32-bit
  // addresses; [0] for even u, [1] for odd u, + 64 u bytes).
  const int odd = l & 1;
  auto node = [&](int u) { return u ^ odd; };
  struct Addr {
    uint32_t e, o;
  };
  auto addr = [&](const double* base) {  // base: the thread's column k of a staged plane
    const uint32_t b = (uint32_t)__cvta_generic_to_shared(base);
    return Addr{b + (odd ? 64u : 0u), b - (odd ? 64u : 0u)};
  };
  auto lds = [&](const Addr& a_, int u) {
    double x;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(x) : "r"(((u & 1) ? a_.o : a_.e) + 64u * (uint32_t)u));
    return x;
  };
  // The node update of plane jx (lower, xi < 0) and jm (upper, xi > 0) for
  // u = 0..15: g/gb/gf the node and its xi neighbours, xn the x neighbour
  // (staged, or xa/xb when XS is false).  Stores the outputs of row i and
  // leaves the fold-term accumulators in a1/a2.
  auto row_update = [&](const RowCoef& rc, auto XS, const Addr& gl, const Addr& bl, const Addr& fl,
                        const Addr& xl_, const Addr& gh, const Addr& bh, const Addr& fh,
                        const Addr& xh_, const double (&xa)[NM], const double (&xb)[NM], int i,
                        double& a1, double& a2) {
    // (outputs stored as they are formed: no output registers held over the row)
    double* const ol = gout + (size_t)i * nv + jx * S + col0;
    double* const oh = gout + (size_t)i * nv + jm * S + col0;
    const double Ep = rc.vsg > 0 ? rc.vco : 0.0;
    const double Em = rc.vsg < 0 ? rc.vco : 0.0;
    double f1[2], f2[2];
#pragma unroll
    for (int u = 0; u < NM; ++u) {
      double lo, hi;
      {  // plane jx, xi < 0: x-upwind from row i+1; zero xi-inflow below plane 0
        const double g = lds(gl, u);
        const double gb = jx > 0 ? lds(bl, u) : 0.0;
        const double gf = lds(fl, u);
        const double xn = decltype(XS)::value ? lds(xl_, u) : xa[u];
        double w = xl * (xn - g);
        w = qdiv(w, dx, rdx);
        const double dm = g - gb;  // (gb = 0.0 below plane 0: g - 0.0 == g bitwise)
        w = w + dm * Ep;
        const double dp = gf - g;  // (jx + 1 <= 16 < X)
        w = w + dp * Em;
        const double Mc = Ml[u];
        w = w - Mc * rc.dc;
        const double forcing = w + (xl * Mc) * rc.J;
        lo = rc.k1 * g - rc.k2 * forcing;
      }
      {  // plane 31 - jx, xi > 0: x-upwind from row i-1; zero inflow above plane 31
        const double g = lds(gh, u);
        const double gb = lds(bh, u);
        const double gf = jm + 1 < X ? lds(fh, u) : 0.0;
        const double xn = decltype(XS)::value ? lds(xh_, u) : xb[u];
        double w = xh * (g - xn);
        w = qdiv(w, dx, rdx);
        const double dm = g - gb;  // (jm - 1 >= 15 >= 0)
        w = w + dm * Ep;
        const double dp = jm + 1 == X ? -g : gf - g;
        w = w + dp * Em;
        const double Mc = Mh[u];
        w = w - Mc * rc.dc;
        const double forcing = w + (xh * Mc) * rc.J;
        hi = rc.k1 * g - rc.k2 * forcing;
      }
      __stcg(ol + 8 * node(u), lo);
      __stcg(oh + 8 * node(u), hi);
      // fold terms (q(j) + q(mirror j)), accumulated in leaf (node) order
      f1[u & 1] = xl * lo + xh * hi;
      if (sq) f2[u & 1] = lo * lo + hi * hi;
      if (u & 1) {
        const double s0 = odd ? f1[1] : f1[0], s1 = odd ? f1[0] : f1[1];
        a1 = u == 1 ? s0 : a1 + s0;
        a1 = a1 + s1;
        if (sq) {
          const double t0 = odd ? f2[1] : f2[0], t1 = odd ? f2[0] : f2[1];
          a2 = u == 1 ? t0 : a2 + t0;
          a2 = a2 + t1;
        }
      }
    }
  };
  // leaf butterflies, the tree over the leaves and the moments of row i
  auto row_finish = [&](int i, double a1, double a2) {
    a1 = a1 + __shfl_xor_sync(FULL, a1, 1);
    a1 = a1 + __shfl_xor_sync(FULL, a1, 2);
    a1 = a1 + __shfl_xor_sync(FULL, a1, 4);
    if (sq) {
      a2 = a2 + __shfl_xor_sync(FULL, a2, 1);
      a2 = a2 + __shfl_xor_sync(FULL, a2, 2);
      a2 = a2 + __shfl_xor_sync(FULL, a2, 4);
    }
    if (k == 0) {
      sm.red[l] = a1;
      sm.red[32 + l] = a2;
    }
    __syncthreads();  // leaves ready; every thread is done with the staged data
    if (tid < 32) {   // balanced tree over the 32 leaves in order
      double r1 = sm.red[lane], r2 = sm.red[32 + lane];
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        r1 = r1 + __shfl_xor_sync(FULL, r1, d);
        if (sq) r2 = r2 + __shfl_xor_sync(FULL, r2, d);
      }
      if (tid == 0) {
        v.fl_w[i] = r1 * m.dv3;
        if (sq) v.sq_w[i] = r2 * m.dv3;
      }
      __syncwarp();
    }
  };
  if (tid == 0) fence_proxy_async_global();  // rows written by the generic proxy, read by TMA

  if (dense) {
    // lower halves L_t = row p0 + t (t = 0..n), upper halves U_t = row p0 - 1 + t
    const int n = p1 - p0;
    const uint32_t lb = cnt.q[1], ub = cnt.q[2];
    double* const lslot = rbuf;           // 3 lower-half slots
    double* const uslot = rbuf + 3 * hv;  // 3 upper-half slots
    auto issue_l = [&](int t) {
      const uint32_t T = lb + (uint32_t)t;
      copy(lslot + (T % 3) * hv, gin + (size_t)wrap(p0 + t, nx) * nv, hv * 8, mbar + 2 + T % 3);
    };
    auto issue_u = [&](int t) {
      const uint32_t T = ub + (uint32_t)t;
      copy(uslot + (T % 3) * hv, gin + (size_t)wrap(p0 - 1 + t, nx) * nv + hv, hv * 8,
           mbar + 5 + T % 3);
    };
    auto wait_l = [&](int t) {
      const uint32_t T = lb + (uint32_t)t;
      mbar_wait(mbar + 2 + T % 3, (T / 3) & 1);
      return lslot + (T % 3) * hv;
    };
    auto wait_u = [&](int t) {
      const uint32_t T = ub + (uint32_t)t;
      mbar_wait(mbar + 5 + T % 3, (T / 3) & 1);
      return uslot + (T % 3) * hv;
    };
    if (tid == 0)
      for (int t = 0; t < 3 && t <= n; ++t) {
        issue_l(t);
        issue_u(t);
      }
    RowCoef rc = coef(p0);
    for (int q = 0; q < n; ++q) {
      const int i = p0 + q;
      RowCoef rn = rc;
      if (q + 1 < n) rn = coef(i + 1);
      const double* Lc = wait_l(q);      // own lower half
      const double* Ln = wait_l(q + 1);  // row i+1, lower half
      const double* Up = wait_u(q);      // row i-1, upper half
      const double* Uc = wait_u(q + 1);  // own upper half
      const double* rl = Lc + jx * S + col0;
      const double* rh = Uc + (jm - HX) * S + col0;
      const Addr gl = addr(rl), bl = addr(rl - S);
      const Addr fl = addr(jx + 1 < HX ? rl + S : Uc + col0);  // plane jx + 1
      const Addr xl_ = addr(Ln + jx * S + col0);
      const Addr gh = addr(rh), fh = addr(rh + S);
      const Addr bh = addr(jm > HX ? rh - S : Lc + (HX - 1) * S + col0);  // plane jm - 1
      const Addr xh_ = addr(Up + (jm - HX) * S + col0);
      double a1 = 0.0, a2 = 0.0;
      row_update(rc, std::true_type{}, gl, bl, fl, xl_, gh, bh, fh, xh_, Ml, Mh, i, a1, a2);
      row_finish(i, a1, a2);
      // (after row_finish's barrier) slots of L_q and U_q are free: L_{q+3}, U_{q+3}
      if (tid == 0) {
        if (q + 3 <= n) issue_l(q + 3);
        if (q + 3 <= n) issue_u(q + 3);
      }
      rc = rn;
    }
    cnt.q[1] += (uint32_t)(n + 1);
    cnt.q[2] += (uint32_t)(n + 1);
    return;
  }

  // sparse: two full-row slots, the x neighbours from L2
  uint32_t& qbase = cnt.q[0];
  const uint32_t bytes = (uint32_t)nv * 8;
  // row q of this phase goes to slot (qbase + q) & 1 at parity ((qbase + q) >> 1) & 1
  auto issue = [&](int q, int i) {
    if (tid == 0) {
      const uint32_t Q = qbase + (uint32_t)q;
      copy(rbuf + (size_t)(Q & 1) * nv, gin + (size_t)i * nv, bytes, mbar + (Q & 1));
    }
  };
  int i_cur = rowid(p0);
  issue(0, i_cur);
  int i_nxt = p0 + 1 < p1 ? rowid(p0 + 1) : 0;
  if (p0 + 1 < p1) issue(1, i_nxt);
  RowCoef rc = coef(i_cur);
  for (int p = p0; p < p1; ++p) {
    const int q = p - p0;
    const uint32_t Q = qbase + (uint32_t)q;
    const double* rb = rbuf + (size_t)(Q & 1) * nv;
    const int i = i_cur;
    // next row's id and coefficients ride ahead of the current row's work
    const int i_n2 = p + 2 < p1 ? rowid(p + 2) : 0;
    RowCoef rn = rc;
    if (p + 1 < p1) rn = coef(i_nxt);
    // x neighbours from L2 first (row i+1 on the lower plane, i-1 on the upper)
    const double* gnl = gin + (size_t)wrap(i + 1, nx) * nv + jx * S + col0;
    const double* gph = gin + (size_t)wrap(i - 1, nx) * nv + jm * S + col0;
    double xa[NM], xb[NM];
#pragma unroll
    for (int u = 0; u < NM; ++u) {
      xa[u] = __ldcg(gnl + 8 * node(u));
      xb[u] = __ldcg(gph + 8 * node(u));
    }
    mbar_wait(mbar + (Q & 1), (Q >> 1) & 1);
    const double* rl = rb + jx * S + col0;
    const double* rh = rb + jm * S + col0;
    const Addr gl = addr(rl), bl = addr(rl - S), fl = addr(rl + S);
    const Addr gh = addr(rh), bh = addr(rh - S), fh = addr(rh + S);
    double a1 = 0.0, a2 = 0.0;
    row_update(rc, std::false_type{}, gl, bl, fl, gl, gh, bh, fh, gh, xa, xb, i, a1, a2);
    row_finish(i, a1, a2);
    if (p + 2 < p1) issue(q + 2, i_n2);  // (the staged row was only read: no proxy fence)
    i_cur = i_nxt;
    i_nxt = i_n2;
    rc = rn;
  }
  qbase += (uint32_t)(p1 - p0);
}

// Prologue row pass of the one-CTA-per-row big-row layout without a lift:
// copy the input rows into the step-0 input buffer and form their moments in
// micro_phase_bigc's thread layout (same leaves, butterflies and tree), every
// CTA of the cluster / group its share of the rows.
static __device__ void prologue_rows_bigc(const FineArgs& a, const SliceView& v, const Smem& sm,
                                          double* gin0, const double* sxi, int crank, int C) {
  constexpr int S = BIGC_S, X = BIGC_NXI, NM = 16;
  const MeshDev& m = a.m;
  const int nx = m.nx, nv = m.nv;
  const int tid = threadIdx.x, lane = tid & 31;
  const int l = tid >> 3, k = lane & 7;
  const int jx = l >> 1, jm = X - 1 - jx;
  const int col0 = (l & 1) * 128 + k;
  const double xl = sxi[jx], xh = sxi[jm];
  const int p0 = (int)(((long long)crank * nx) / C), p1 = (int)(((long long)(crank + 1) * nx) / C);
  const bool cp = gin0 != v.ga;
  for (int i = p0; i < p1; ++i) {
    const double* rl = v.ga + (size_t)i * nv + jx * S + col0;
    const double* rh = v.ga + (size_t)i * nv + jm * S + col0;
    double lo[NM], hi[NM];
#pragma unroll
    for (int u = 0; u < NM; ++u) {
      lo[u] = __ldcg(rl + 8 * u);
      hi[u] = __ldcg(rh + 8 * u);
    }
    double a1 = 0.0, a2 = 0.0;
#pragma unroll
    for (int u = 0; u < NM; ++u) {
      if (cp) {
        __stcg(gin0 + (size_t)i * nv + jx * S + col0 + 8 * u, lo[u]);
        __stcg(gin0 + (size_t)i * nv + jm * S + col0 + 8 * u, hi[u]);
      }
      const double f1 = xl * lo[u] + xh * hi[u];
      const double f2 = lo[u] * lo[u] + hi[u] * hi[u];
      a1 = u == 0 ? f1 : a1 + f1;
      a2 = u == 0 ? f2 : a2 + f2;
    }
#pragma unroll
    for (int d = 1; d < 8; d <<= 1) {
      a1 = a1 + __shfl_xor_sync(FULL, a1, d);
      a2 = a2 + __shfl_xor_sync(FULL, a2, d);
    }
    if (k == 0) {
      sm.red[l] = a1;
      sm.red[32 + l] = a2;
    }
    __syncthreads();
    if (tid < 32) {
      double r1 = sm.red[lane], r2 = sm.red[32 + lane];
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        r1 = r1 + __shfl_xor_sync(FULL, r1, d);
        r2 = r2 + __shfl_xor_sync(FULL, r2, d);
      }
      if (tid == 0) {
        v.fl_w[i] = r1 * m.dv3;
        v.sq_w[i] = r2 * m.dv3;
      }
    }
    __syncthreads();  // sm.red is rewritten by the next row
  }
}

// Prologue row pass: (optionally lift and) copy the input rows into the
// step-0 input buffer and compute their moments.
template <int T>
__device__ void prologue_rows(const FineArgs& a, const SliceView& v, const Smem& sm, double* gin0,
                              bool lift, const double* lJ, const double* ldrift,
                              const double* lRif, int wg, int nwg) {
  const MeshDev& m = a.m;
  const int nx = m.nx, nv = m.nv;
  const int lane = threadIdx.x & 31;
  constexpr int S = Layout<T>::S;
  double* wrow = sm.wrow + (threadIdx.x >> 5) * nv;
  const int p0 = (int)(((long long)wg * nx) / nwg);
  const int p1 = (int)(((long long)(wg + 1) * nx) / nwg);
  if constexpr (T < 0) {  // big rows: work on the rows in global memory
    double* scr = sm.wrow + (threadIdx.x >> 5) * BIG_SCR;
    for (int i = p0; i < p1; ++i) {
      double* row = gin0 + (size_t)i * nv;
      if (lift) {
        LiftRow L;
        const size_t o = (size_t)v.b * nx + i;
        L.negJ = a.neg_eps[o] * __ldcg(lJ + i);
        L.e2 = a.eps2[o];
        L.drift = __ldcg(ldrift + i);
        L.Rif = __ldcg(lRif + i);
        big_row_lift(row, L, a.lift_order, a.time_elim == 1, 1, m, scr, lane);
      } else if (gin0 != v.ga) {
        big_row_copy(v.ga + (size_t)i * nv, row, nv, lane);
      }
      double bx, bsq;
      big_row_moments(row, m, scr, true, bx, bsq);
      if (lane == 0) {
        v.fl_w[i] = bx;
        v.sq_w[i] = bsq;
      }
    }
    return;
  }
  for (int i = p0; i < p1; ++i) {
    double g[S];
    if (lift) {
      LiftRow L;
      const size_t o = (size_t)v.b * nx + i;
      L.negJ = a.neg_eps[o] * __ldcg(lJ + i);
      L.e2 = a.eps2[o];
      L.drift = __ldcg(ldrift + i);
      L.Rif = __ldcg(lRif + i);
      row_lift<T>(g, L, a.lift_order, a.time_elim == 1, 1, sm, m, wrow, lane);
      row_store<T>(g, gin0 + (size_t)i * nv, lane, nv);
    } else {
      row_load<T>(g, v.ga + (size_t)i * nv, lane, nv);
      if (gin0 != v.ga) row_store<T>(g, gin0 + (size_t)i * nv, lane, nv);
    }
    double bx, bsq;
    row_moments<T>(g, sm, m, wrow, lane, bx, bsq);
    if (lane == 0) {
      v.fl_w[i] = bx;
      v.sq_w[i] = bsq;
    }
  }
}

// Window-start lift scalars (parareal.py:171-178: lift(rho_in, E) with
// dE_dt = None, i.e. dtE_c = 0), written to cluster-shared arrays (global)
// for every CTA's prologue row pass.
static __device__ bool lift_scalars(const FineArgs& a, const SliceView& v, const Smem& sm, double* out_J,
                             double* out_drift, double* out_Rif) {
  const MeshDev& m = a.m;
  const int nx = m.nx, tid = threadIdx.x, nt = blockDim.x;
  if (a.lift_order != 1 && a.lift_order != 2) return false;
  if (a.lift_order == 2 && a.time_elim != 0 && a.time_elim != 1) return false;
  const bool higher = a.lift_order == 2 && a.time_elim == 1;
  // temporaries: J_c in tA, D1(J_c) in tB (leader-local in every layout),
  // R in the global scratch tC (once per window)
  double* Jc = a.tA + (size_t)v.b * nx;   // global scratch: once per window
  double* d1 = a.tB + (size_t)v.b * nx;
  double* R = a.tC + (size_t)v.b * nx;
  for (int i = tid; i < nx; i += nt) {
    const int ip = wrap(i - 1, nx);
    Jc[i] = 0.5 * (v.J[ip] + v.J[i]);
  }
  __syncthreads();
  const double three_rb = 3.0 * v.rb;
  for (int i = tid; i < nx; i += nt) {
    const double d1J = stencil_at(Jc, i, nx, m, 1);
    d1[i] = d1J;
    if (higher) {
      const int ip = wrap(i - 1, nx);
      const double Ec = 0.5 * (v.E[ip] + v.E[i]);
      const double d2J = stencil_at(Jc, i, nx, m, 2);
      const double d3J = stencil_at(Jc, i, nx, m, 3);
      const double d1r = stencil_at(v.rho, i, nx, m, 1);
      const double dtEc = 0.0;
      R[i] = -d3J + Ec * d2J + (2.0 * v.rho[i] - three_rb) * d1J + 2.0 * Jc[i] * d1r - d1r * dtEc;
    }
  }
  __syncthreads();
  for (int i = tid; i < nx; i += nt) {
    const int in_ = wrap(i + 1, nx);
    const double dJ = 0.5 * (d1[i] + d1[in_]);
    out_J[i] = v.J[i];
    out_drift[i] = dJ - v.E[i] * v.J[i];
    out_Rif[i] = higher ? 0.5 * (R[i] + R[in_]) : 0.0;
  }
  __syncthreads();
  return true;
}

// Micro phase of a cluster that runs several all-kinetic slices: the
// cluster's rows, slice after slice, split evenly over its warps; a warp whose
// share crosses a slice boundary streams each slice's part on its own (row
// moments go to the owning CTA's shared memory through DSMEM).
template <int CH, int S>
__device__ __forceinline__ void micro_slices(const FineArgs& a, const SliceView& v, const Smem& sm,
                                             int s, int b0, int Kq, int wg, int nwg, double* ring,
                                             uint64_t* mbar, uint32_t& qbase) {
  const int nx = a.m.nx, R = Kq * nx;
  const int r1 = (int)(((long long)(wg + 1) * R) / nwg);
  for (int r = (int)(((long long)wg * R) / nwg); r < r1;) {
    const int k = r / nx, bb = b0 + k;
    const int e = min(r1, (k + 1) * nx);
    const int n0 = a.ph[0].nsteps[bb], nb = n0 + a.ph[1].nsteps[bb];
    if (s < nb && !__ldcg(a.abort_ + bb)) {
      const size_t o = (size_t)bb * nx;
      SliceView u = v;
      u.b = bb;
      u.gJ = a.J + o;
      u.dco = a.dco + o;
      u.vco = a.vco + o;
      u.vsg = a.vsg + o;
      u.fl_w = a.sg > 1 ? a.fl + o : cg::this_cluster().map_shared_rank(v.fl, k);
      double* ga = a.ga + o * a.m.nv;
      double* gb = a.gb + o * a.m.nv;
      const bool odd = ((s + (nb & 1)) & 1) != 0;  // step s reads buf(s), as in fine_kernel
      micro_phase_g8<CH, S, true, false>(a, u, sm, s < n0 ? 0 : 1, odd ? gb : ga, odd ? ga : gb,
                                         r - k * nx, e - k * nx, ring, mbar, qbase);
    }
    r = e;
  }
}

__device__ __forceinline__ void cluster_barrier(int C) {
  if (C > 1) {
    cg::this_cluster().sync();
  } else {
    // one CTA per slice: the next micro phase's bulk copies (async proxy, from
    // L2) read rows that OTHER warps of this CTA stored in this phase.
    // __syncthreads() orders them for the CTA's threads only; the stores
    // must also be performed at L2 before the copies are issued (the cluster
    // and group barriers release at cluster / gpu scope and imply it).
    // Without the fence a slice now and then read a stale halo row
    // (tools/flake_probe.py: 3 of 24 fresh processes, last-bit differences).
    __threadfence();
    __syncthreads();
  }
}

// Barrier of a software group (FineArgs::sg): C co-resident CTAs (cooperative
// launch) count arrivals on one global counter; the n-th barrier of the
// kernel waits for C * n arrivals.  Release/acquire at gpu scope, as a grid
// sync: every write before the barrier is visible to every CTA after it.
constexpr unsigned long long kMomentSentinel = 0x7FF4C0DE5E47C0DEull;  // signalling NaN

__device__ __forceinline__ void st_relaxed_u64(double* p, unsigned long long x) {
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(x) : "memory");
}

__device__ __forceinline__ unsigned long long ld_relaxed_u64(const double* p) {
  unsigned long long x;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(x) : "l"(p) : "memory");
  return x;
}

__device__ __forceinline__ void group_barrier(unsigned* cnt, int C, unsigned& n) {
  __syncthreads();
  ++n;
  if (threadIdx.x == 0) {
    const unsigned target = (unsigned)C * n;
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
    unsigned v;
    for (;;) {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(cnt) : "memory");
      if (v >= target) break;
      __nanosleep(32);
    }
  }
  __syncthreads();
}

// AD: adaptation on (hybrid) or off (all-kinetic, compiled without the
// labels / lifts / row lists of the hybrid slice phase)
template <int T, int S, int G, int NT, bool AD>
// (the G8 layouts with 8 warps and the GS layout with 16 run one CTA per SM)
__global__ void __launch_bounds__(NT, (T < 0 || (G > 0 && NT > 128) || (G < 0 && NT > 256)) ? 1 : 2)
    fine_kernel(const FineArgs a) {
  // ring row stride (doubles); G > 0: per-warp G8 rings, G < 0: CTA-wide
  // producer/consumer ring of the GS layout with SEG = -G
  constexpr int RSN = G > 0 ? 16 * G + 8 : (G < 0 ? 64 * (-G) + 8 : 32 * (T > 0 ? T : 1));
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const long long t_kstart = a.prof ? clock64() : 0;
  const MeshDev& m = a.m;
  const int nx = m.nx, nv = m.nv;
  int C = 1;
  int crank = 0;
  if (a.sg > 1) {  // software group of sg consecutive CTAs (hardware cluster of 1)
    C = a.sg;
    crank = (int)(blockIdx.x % (unsigned)C);
  } else {
    cg::cluster_group cl = cg::this_cluster();
    C = (int)cl.num_blocks();
    crank = (int)cl.block_rank();
  }
  unsigned* const sgc = a.sg > 1 ? a.sg_cnt + blockIdx.x / (unsigned)C : nullptr;
  unsigned sgn = 0;
  auto barrier = [&]() {
    if (sgc) group_barrier(sgc, C, sgn);
    else cluster_barrier(C);
  };
  // a cluster runs K consecutive slices (K = 1 unless the launcher packs
  // several all-kinetic slices per cluster): CTA k < K owns slice b0 + k (its
  // slice phase and on-chip vectors), every CTA streams an equal share of the
  // cluster's rows
  const int K = a.kps > 1 ? a.kps : 1;
  const int b0 = (blockIdx.x / C) * K;
  const int Kq = min(K, a.B - b0);
  const bool leader = crank < Kq;
  const int b = leader ? b0 + crank : b0;
  const int nwpc = blockDim.x >> 5;
  const int warp = threadIdx.x >> 5;
  // shared memory carve-up
  Smem sm;
  double* ring = nullptr;
  uint64_t* mbar = nullptr;
  double* sm_loc = nullptr;
  {
    unsigned char* p = smem_raw;
    mbar = reinterpret_cast<uint64_t*>(p);
    p += 128 * 8;
    sm.plan = reinterpret_cast<PwPlan*>(p);
    p += (sizeof(PwPlan) + 15) / 16 * 16;
    if (T >= 0) {  // velocity constants on chip (big rows read them from global)
      sm.vx = reinterpret_cast<double*>(p); p += nv * 8;
      sm.M = reinterpret_cast<double*>(p); p += nv * 8;
      sm.xiM = reinterpret_cast<double*>(p); p += nv * 8;
      sm.w2 = reinterpret_cast<double*>(p); p += nv * 8;
    } else {
      sm.vx = const_cast<double*>(m.vx);
      sm.M = const_cast<double*>(m.M);
      sm.xiM = const_cast<double*>(m.xiM);
      sm.w2 = const_cast<double*>(m.w2);
    }
    sm.red = reinterpret_cast<double*>(p); p += 2 * (MAX_LEAF + MAX_NODE) * 8;
    sm.misc = reinterpret_cast<int*>(p); p += 160 * 4;
    sm.wrow = reinterpret_cast<double*>(p);
    if (T == 0) p += (size_t)nwpc * nv * 8;       // generic-layout row scratch
    if (T < 0 && !a.bigc) p += (size_t)nwpc * BIG_SCR * 8;   // big rows: plan scratch
    if (T < 0 && a.bigc) {
      // big rows, one CTA per row: row staging (six half-row or two full-row
      // slots), xi per plane; the plan scratch of the per-warp row operations
      // (prologue, lifts: never during a micro phase) lives in the staging
      p = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(p) + 15) & ~uintptr_t(15));
      ring = reinterpret_cast<double*>(p);
      sm.wrow = ring;
      p += ((size_t)3 * nv + nv / m.nvyz + 1) / 2 * 16;
    }
    if (T > 0) {
      ring = reinterpret_cast<double*>(p);
      p += (size_t)(G < 0 ? 1 : nwpc) * S * RSN * 8;
    }
    if (a.local_smem) sm_loc = reinterpret_cast<double*>(p);  // same offset in every CTA
    sm.scan = !a.local_smem && a.scan_smem ? reinterpret_cast<double*>(p) : nullptr;
    sm.scan_cap = a.scan_smem;
  }
  {
    const int* src = reinterpret_cast<const int*>(m.plan_x);
    int* dst = reinterpret_cast<int*>(sm.plan);
    for (int i = threadIdx.x; i < (int)(sizeof(PwPlan) / 4); i += blockDim.x) dst[i] = src[i];
    if (T >= 0)
      for (int j = threadIdx.x; j < nv; j += blockDim.x) {
        sm.vx[j] = m.vx[j];
        sm.M[j] = m.M[j];
        sm.xiM[j] = m.xiM[j];
        sm.w2[j] = m.w2[j];
      }
    if (T > 0 && threadIdx.x < (G < 0 ? 2 * S : nwpc * S)) mbar_init(mbar + threadIdx.x, 1);
    if (T < 0 && a.bigc) {
      if (threadIdx.x < 8) mbar_init(mbar + threadIdx.x, 1);
      for (int j = threadIdx.x; j < nv / m.nvyz; j += blockDim.x)
        ring[3 * (size_t)nv + j] = m.vx[(size_t)j * m.nvyz];
    }
    if (T > 0 || (T < 0 && a.bigc)) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  SliceView v;
  bind_shared(v, a, b);
  bind_local(v, a, b, sm_loc, leader, leader ? crank : 0);
  // Software group: the row moments arrive in global memory (a.fl), the value
  // being its own flag -- the owner re-arms every entry with a signalling-NaN
  // sentinel (arithmetic only makes quiet NaNs) before the barrier that opens
  // the next micro phase, and after that phase polls its entries until none
  // is the sentinel, pulling them on chip.  No barrier (and no release fence
  // behind the phase's row stores) between the micro and the slice phase.
  const bool sgo = a.sg > 1 && leader && sm_loc;  // an owner in a software group
  if (a.sg > 1) v.fl_w = a.fl + (size_t)b * nx;
  auto arm_moments = [&]() {
    for (int i = threadIdx.x; i < nx; i += blockDim.x) st_relaxed_u64(v.fl_w + i, kMomentSentinel);
  };
  auto pull_moments = [&]() {  // moments written by this CTA (prologue)
    for (int i = threadIdx.x; i < nx; i += blockDim.x) v.fl[i] = __ldcg(v.fl_w + i);
    __syncthreads();
    arm_moments();
  };
  auto poll_moments = [&]() {  // moments written by the whole group (micro phase)
    constexpr int U = 8;
    for (int i0 = threadIdx.x; i0 < nx; i0 += U * blockDim.x) {
      unsigned long long x[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = i0 + u * blockDim.x;
        x[u] = i < nx ? ld_relaxed_u64(v.fl_w + i) : 0ull;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = i0 + u * blockDim.x;
        if (i < nx) {
          while (x[u] == kMomentSentinel) {
            __nanosleep(64);
            x[u] = ld_relaxed_u64(v.fl_w + i);
          }
          v.fl[i] = __longlong_as_double((long long)x[u]);
        }
      }
    }
    __syncthreads();
    arm_moments();
  };
  const int n0 = a.ph[0].nsteps[b], n1 = a.ph[1].nsteps[b];
  const int nst = n0 + n1;
  int nst_all = nst;  // steps of the longest slice of the cluster
  for (int k = 0; k < Kq && K > 1; ++k)
    nst_all = max(nst_all, a.ph[0].nsteps[b0 + k] + a.ph[1].nsteps[b0 + k]);
  const int wg = crank * nwpc + warp;
  const int nwg = C * nwpc;
  const int initf = a.init_flags ? a.init_flags[b] : 0;
  const bool lift0 = (initf & 1) != 0;   // g := lift(rho, E)   (parareal.py:171-178)
  const bool eprev0 = (initf & 2) != 0;  // E_prev := E         (hybrid.py:68-72)
  // step s reads buf(s) and writes buf(s+1); the last output lands in ga.
  auto buf = [&](int s) { return ((s + (nst & 1)) & 1) ? v.gb : v.ga; };
  auto nzf = [&](int s) { return ((s + (nst & 1)) & 1) ? v.nzb : v.nza; };
  int* abort_flag = v.abort_;
  const size_t o = (size_t)b * nx;
  uint32_t qbase = 0, obase = 0;
  BigcCnt bcnt = {{0u, 0u, 0u}};
  GSConsts<G < 0 ? -G : 1> gsc;
  if constexpr (G < 0) gsc.load(sm, threadIdx.x & 31);
  double* ring_w = ring ? ring + (size_t)(G < 0 ? 0 : warp) * S * RSN : nullptr;
  uint64_t* mbar_w = mbar + warp * S;

  // ---- prologue ----
  if (leader) {
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int i = tid; i < nx; i += nt) {
      v.nza[i] = 1;
      v.nzb[i] = 1;
      if (sm_loc) {
        v.rho[i] = a.rho[o + i];
        v.Eprev[i] = a.Eprev[o + i];
        v.kc[i] = a.kc[o + i];
        v.ki[i] = a.ki[o + i];
      }
    }
    if (tid == 0) *abort_flag = 0;
    __syncthreads();
    bool ok = slice_field(m, v.rho, v.rb, v.E, v.E, a.rtol, a.exact_scan, a.local_smem != 0, sm);
    if (!ok) {
      if (tid == 0) {
        set_status(a.status, PK_ERR_SOLVABILITY, b, 0);
        *abort_flag = 1;
      }
    } else {
      for (int i = tid; i < nx; i += nt) {
        v.J[i] = flux_J(v.rho[i], v.rho[wrap(i + 1, nx)], v.E[i], m.dx, m.rdx);
        if (eprev0) v.Eprev[i] = v.E[i];
      }
      __syncthreads();
      // window-start lift scalars go to cluster-shared scratch (dco/vco/gJ
      // are not in use before the first prepare_step)
      if (lift0 && !lift_scalars(a, v, sm, v.gJ, v.dco, v.vco)) {
        if (tid == 0) {
          set_status(a.status, PK_ERR_BAD_LIFT, b, 0);
          *abort_flag = 1;
        }
      }
    }
    __syncthreads();
  }
  barrier();
  if (K == 1 && __ldcg(abort_flag)) return;
  if (T < 0 && a.bigc && !lift0 && K == 1)
    prologue_rows_bigc(a, v, sm, buf(0), ring + 3 * (size_t)nv, crank, C);
  else if (K == 1)
    prologue_rows<T>(a, v, sm, buf(0), lift0, v.gJ, v.dco, v.vco, wg, nwg);
  else if (leader && !__ldcg(abort_flag))  // several slices: each owner's warps
    prologue_rows<T>(a, v, sm, buf(0), lift0, v.gJ, v.dco, v.vco, warp, nwpc);
  barrier();
  if (sgo) pull_moments();
  // hybrid slices with global-memory vectors run their slice phases on every
  // CTA of the cluster; otherwise the leader runs them alone
  Par par = leader_par(sm);
  const bool dist = AD && C > 1 && K == 1 && !sm_loc;
  if (dist) {
    par.rank = crank;
    par.C = C;
    par.dist = true;
    par.r0 = crank * blockDim.x + threadIdx.x;
    par.rs = C * blockDim.x;
    par.w0 = crank * nwpc + warp;
    par.ws = C * nwpc;
    par.flags = cg::this_cluster().map_shared_rank(sm.misc, 0);
  }
  if ((dist || leader) && !__ldcg(abort_flag)) {
    const double dt0 = (n0 > 0 ? a.ph[0].dt : a.ph[1].dt)[b];
    if (!prepare_step<T, AD>(a, v, sm, dt0, 1, buf(0), nzf(0), nzf(1), 0, par)) {
      if (threadIdx.x == 0) *abort_flag = 1;
    }
  }
  barrier();
  if (K == 1 && __ldcg(abort_flag)) return;

  // ---- steps ----
  // optional phase profile (slice 0, leader thread 0): clock64 deltas of
  // [micro, barrier, finish, prepare, barrier]
  const bool prof = a.prof && b == 0 && leader && threadIdx.x == 0;
  // per-CTA [micro, first barrier] cycles and SM id at prof[32 + 3 * blockIdx.x]
  const bool profc = a.prof && threadIdx.x == 0 && blockIdx.x < 1024;
  long long pc_m = 0, pc_b = 0, pc_t = 0;
  long long tp[6] = {0, 0, 0, 0, 0, 0};
  long long c0 = prof ? clock64() : 0, c1;
  if (prof) a.prof[6] += c0 - t_kstart;  // prologue
  // optional row counters (pk_count_rows): the slice owner's thread 0
  const bool rcnt = a.rowcnt && leader && threadIdx.x == 0;
  long long rc_rows = 0, rc_zero = 0;
  for (int s = 0; s < nst_all; ++s) {
    const int ph = s < n0 ? 0 : 1;
    if constexpr (AD) {  // rows the slice phase listed for zeroing in this step's output
      const int nzr = __ldcg(v.nzl);
      for (int q = wg; q < nzr; q += nwg)
        row_zero_store<T>(buf(s + 1) + (size_t)__ldcg(v.zlist + q) * nv, threadIdx.x & 31, nv);
      if (rcnt && s < nst) rc_zero += nzr;
    }
    if (rcnt && s < nst) rc_rows += AD ? __ldcg(v.nk) : nx;
    if (profc) pc_t = clock64();
    if constexpr (G < 0) {
      const int nkk = __ldcg(v.nk);
      const int e0 = (int)(((long long)crank * nkk) / C), e1 = (int)(((long long)(crank + 1) * nkk) / C);
      micro_phase_pc<-G, S>(a, v, ph, buf(s), buf(s + 1), e0, e1, nkk == nx, nwpc - 1, ring, mbar,
                            mbar + S, qbase, obase, gsc);
    } else if constexpr (G > 0) {
      const int nkk = __ldcg(v.nk);
      const int q0 = (int)(((long long)wg * nkk) / nwg), q1 = (int)(((long long)(wg + 1) * nkk) / nwg);
      if (!AD && K > 1) {
        if constexpr (!AD) micro_slices<G, S>(a, v, sm, s, b0, Kq, wg, nwg, ring_w, mbar_w, qbase);
      } else if (q0 < q1) {
        // the |g|^2 row moment feeds only the adaptation labels
        if constexpr (!AD)
          micro_phase_g8<G, S, true, false>(a, v, sm, ph, buf(s), buf(s + 1), q0, q1, ring_w, mbar_w,
                                            qbase);
        else if (nkk == nx)
          micro_phase_g8<G, S, true, true>(a, v, sm, ph, buf(s), buf(s + 1), q0, q1, ring_w, mbar_w,
                                           qbase);
        else
          micro_phase_g8<G, S, false, true>(a, v, sm, ph, buf(s), buf(s + 1), q0, q1, ring_w, mbar_w,
                                            qbase);
      }
    }
    else if constexpr (T > 0)
      micro_phase_tma<T, S>(a, v, sm, ph, buf(s), buf(s + 1), wg, nwg, ring_w, mbar_w, qbase);
    else if constexpr (T == 0)
      micro_phase_gen(a, v, sm, ph, buf(s), buf(s + 1), wg, nwg);
    else if (a.bigc)
      micro_phase_bigc<AD>(a, v, sm, ph, buf(s), buf(s + 1), crank, C, ring, ring + 3 * (size_t)nv,
                       mbar, bcnt);
    else
      micro_phase_big(a, v, sm, ph, buf(s), buf(s + 1), wg, nwg);
    if (prof) { c1 = clock64(); tp[0] += c1 - c0; c0 = c1; }
    if (profc) { const long long t = clock64(); pc_m += t - pc_t; pc_t = t; }
    if (a.sg > 1) {  // (owner of a live slice: every row of it was streamed this step)
      if (sgo && s < nst && !__ldcg(abort_flag)) poll_moments();
    } else {
      barrier();
    }
    if (prof) { c1 = clock64(); tp[1] += c1 - c0; c0 = c1; }
    if (profc) pc_b += clock64() - pc_t;
    // host cancel request (speculative parareal windows that are not needed
    // any more): sampled by the slice's leader thread only, here, so that the
    // load's L2 round trip hides behind the slice phase
    int cancel_req = 0;
    if (K == 1 && a.sg <= 1 && leader && threadIdx.x == 0 && a.cancel)
      asm volatile("ld.global.cg.s32 %0, [%1];" : "=r"(cancel_req) : "l"(a.cancel));
    // (K == 1: s < nst always, and an aborted slice has returned)
    if ((dist || leader) && s < nst && !(K > 1 && __ldcg(abort_flag))) {
      bool ok = finish_step(a, v, sm, ph, s, par);
      if (prof) { c1 = clock64(); tp[2] += c1 - c0; c0 = c1; }
      if (ok && s + 1 < nst) {
        // step s+1 reads buf(s+1) and writes buf(s+2) == buf(s); after step
        // s the rows of buf(s+1) hold data exactly on step s's kinetic rows.
        if (AD) {
          uint8_t* nzn = nzf(s + 1);
          for (int i = par.r0; i < nx; i += par.rs) nzn[i] = v.ki[i];
          par.sync();
        }
        const int phn = (s + 1) < n0 ? 0 : 1;
        ok = prepare_step<T, AD>(a, v, sm, a.ph[phn].dt[b], 0, buf(s + 1), nzf(s + 1), nzf(s),
                                 s + 1, par, (a.prof && b == 0 && leader) ? a.prof + 16 : nullptr);
      } else if (ok && v.Epend) {  // last step: the field's pending zero-mean shift
        for (int i = threadIdx.x; i < nx; i += blockDim.x) v.E[i] = v.E[i] - v.Emean;
        __syncthreads();
      }
      v.Epend = false;
      v.Emean = 0.0;
      if (!ok && threadIdx.x == 0) *abort_flag = 1;
      if (prof) { c1 = clock64(); tp[3] += c1 - c0; c0 = c1; }
    }
    // (the cancel request sampled above, passed on as an abort before the
    // barrier, so every CTA of the cluster sees the same value)
    if (cancel_req) *abort_flag = 1;
    barrier();
    if (prof) { c1 = clock64(); tp[4] += c1 - c0; c0 = c1; }
    if (K == 1 && __ldcg(abort_flag)) return;
  }
  if (profc) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    a.prof[32 + 3 * blockIdx.x] += pc_m;
    a.prof[33 + 3 * blockIdx.x] += pc_b;
    a.prof[34 + 3 * blockIdx.x] = smid;
  }
  if (prof) {
    for (int k = 0; k < 5; ++k) a.prof[k] += tp[k];
    a.prof[5] += nst;
    a.prof[15] = a.local_smem;
  }
  if (rcnt) {
    a.rowcnt[2 * (size_t)b] += rc_rows;
    a.rowcnt[2 * (size_t)b + 1] += rc_zero;
  }
  // ---- epilogue: leader-local state back to the caller's arrays ----
  if (K > 1 && __ldcg(abort_flag)) return;  // as a single-slice cluster would have
  if (leader && sm_loc) {
    for (int i = threadIdx.x; i < nx; i += blockDim.x) {
      a.rho[o + i] = v.rho[i];
      a.E[o + i] = v.E[i];
      a.Eprev[o + i] = v.Eprev[i];
      a.kc[o + i] = v.kc[i];
      a.ki[o + i] = v.ki[i];
    }
  } else if (leader) {
    // global mode: rho/E/Eprev rotate through rho/E/Eprev/tA/tB pointers
    for (int i = threadIdx.x; i < nx; i += blockDim.x) {
      const double r = v.rho[i], e = v.E[i], ep = v.Eprev[i];
      a.rho[o + i] = r;
      a.E[o + i] = e;
      a.Eprev[o + i] = ep;
    }
  }
}

// ---------------------------------------------------------------------------
// Standalone operators: lift (lifting.py:38-105) and solve_field
// (poisson.py:21-54) over B slices, one CTA per slice.

#if PK_IN_PART(0)
template <int T>
__global__ void __launch_bounds__(256) lift_kernel(const LiftArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const MeshDev& m = a.m;
  const int nx = m.nx, nv = m.nv, b = blockIdx.x;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
  Smem sm;
  {
    unsigned char* p = smem_raw;
    sm.plan = nullptr;
    sm.red = nullptr;
    sm.misc = nullptr;
    if (T >= 0) {
      sm.vx = reinterpret_cast<double*>(p); p += nv * 8;
      sm.M = reinterpret_cast<double*>(p); p += nv * 8;
      sm.xiM = reinterpret_cast<double*>(p); p += nv * 8;
      sm.w2 = reinterpret_cast<double*>(p); p += nv * 8;
      sm.wrow = reinterpret_cast<double*>(p); p += (blockDim.x >> 5) * nv * 8;
    } else {  // big rows: constants from global, per-warp plan scratch only
      sm.wrow = reinterpret_cast<double*>(p);
    }
  }
  if (T >= 0)
    for (int j = tid; j < nv; j += nt) {
      sm.vx[j] = m.vx[j];
      sm.M[j] = m.M[j];
      sm.xiM[j] = m.xiM[j];
      sm.w2[j] = m.w2[j];
    }
  const size_t o = (size_t)b * nx;
  const double* rho = a.rho + o;
  const double* E = a.E + o;
  double *J = a.J + o, *Jc = a.tA + o, *d1 = a.tB + o, *drift = a.tC + o, *R = a.tD + o,
         *Rif = a.tE + o;
  for (int i = tid; i < nx; i += nt) J[i] = flux_J(rho[i], rho[wrap(i + 1, nx)], E[i], m.dx, m.rdx);
  __syncthreads();
  const bool higher = a.order >= 2 && a.time_elim == 1;
  if (a.order >= 2) {
    for (int i = tid; i < nx; i += nt) Jc[i] = 0.5 * (J[wrap(i - 1, nx)] + J[i]);
    __syncthreads();
    const double three_rb = 3.0 * a.rho_bar[b];
    for (int i = tid; i < nx; i += nt) {
      const double d1J = stencil_at(Jc, i, nx, m, 1);
      d1[i] = d1J;
      if (higher) {
        const int ip = wrap(i - 1, nx);
        const double Ec = 0.5 * (E[ip] + E[i]);
        const double dtEc = a.dE_dt ? 0.5 * (a.dE_dt[o + ip] + a.dE_dt[o + i]) : 0.0;
        const double d2J = stencil_at(Jc, i, nx, m, 2);
        const double d3J = stencil_at(Jc, i, nx, m, 3);
        const double d1r = stencil_at(rho, i, nx, m, 1);
        R[i] = -d3J + Ec * d2J + (2.0 * rho[i] - three_rb) * d1J + 2.0 * Jc[i] * d1r - d1r * dtEc;
      }
    }
    __syncthreads();
    for (int i = tid; i < nx; i += nt) {
      const int in_ = wrap(i + 1, nx);
      const double dJ = 0.5 * (d1[i] + d1[in_]);
      drift[i] = dJ - E[i] * J[i];
      Rif[i] = higher ? 0.5 * (R[i] + R[in_]) : 0.0;
    }
  }
  __syncthreads();
  const int nwarp = nt >> 5;
  double* wrow = sm.wrow + warp * nv;
  for (int i = warp; i < nx; i += nwarp) {
    LiftRow L;
    L.negJ = a.neg_eps[o + i] * J[i];
    L.e2 = a.eps2[o + i];
    L.drift = a.order >= 2 ? drift[i] : 0.0;
    L.Rif = a.order >= 2 ? Rif[i] : 0.0;
    if constexpr (T < 0) {
      big_row_lift(a.g_out + (o + i) * nv, L, a.order, higher, a.project, m,
                   sm.wrow + warp * BIG_SCR, lane);
    } else {
      double g[Layout<T>::S];
      row_lift<T>(g, L, a.order, higher, a.project, sm, m, wrow, lane);
      row_store<T>(g, a.g_out + (o + i) * nv, lane, nv);
    }
  }
}

__global__ void __launch_bounds__(256) field_kernel(const FieldArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem sm;
  sm.plan = reinterpret_cast<PwPlan*>(smem_raw);
  sm.red = reinterpret_cast<double*>(smem_raw + (sizeof(PwPlan) + 15) / 16 * 16);
  {
    const int* src = reinterpret_cast<const int*>(a.m.plan_x);
    int* dst = reinterpret_cast<int*>(sm.plan);
    for (int i = threadIdx.x; i < (int)(sizeof(PwPlan) / 4); i += blockDim.x) dst[i] = src[i];
  }
  __syncthreads();
  const size_t o = (size_t)blockIdx.x * a.m.nx;
  if (!slice_field(a.m, a.rho + o, a.rho_bar[blockIdx.x], a.src + o, a.E + o, a.rtol,
                   a.exact_scan, false, sm)) {
    if (threadIdx.x == 0) set_status(a.status, PK_ERR_SOLVABILITY, blockIdx.x, 0);
  }
}

#endif  // PK_IN_PART(0)

// ---------------------------------------------------------------------------
// Host-side launch.

constexpr int kThreads = 256;

static size_t base_smem(int nv, int T, int S, int G, int NT) {
  size_t s = 128 * 8 + (sizeof(PwPlan) + 15) / 16 * 16 + (T >= 0 ? 4 * (size_t)nv * 8 : 0) +
             2 * (MAX_LEAF + MAX_NODE) * 8 + 160 * 4;
  if (T < 0) s += (NT / 32) * (size_t)BIG_SCR * 8;
  else if (T == 0) s += (NT / 32) * (size_t)nv * 8;
  else if (G < 0) s += (size_t)S * (nv + 8) * 8;
  else s += (size_t)(NT / 32) * S * (G != 0 ? nv + 8 : nv) * 8;
  return s;
}

// the one-CTA-per-row big-row layout (micro_phase_bigc): 32 xi planes of
// nvy nvz = 256 columns, mirrored grid with xi constant on each plane
static bool bigc_layout(const MeshDev& m) {
  return m.nvyz == BIGC_S && m.nv == BIGC_S * BIGC_NXI && m.mirror && m.xplane;
}

static size_t local_smem(int nx, int adaptation) {
  return adaptation ? (size_t)nx * (NLOC_D * 8 + NLOC_B) + 16
                    : (size_t)nx * (NLOC_DK * 8 + NLOC_BK) + 16;
}

// layout of the calling thread's last fine launch (pk_fine_last_launch)
extern thread_local int last_launch[4];
#if PK_IN_PART(0)
thread_local int last_launch[4] = {0, 0, 0, 0};

void fine_last_launch(int out[4]) {
  for (int i = 0; i < 4; ++i) out[i] = last_launch[i];
}
#endif

template <int T, int S, int G, int NT, bool AD>
static cudaError_t launch_TA(FineArgs a, int C, cudaStream_t st) {
  // big rows: one CTA per row through shared-memory row buffers when two rows
  // fit (one CTA per SM); else the warp-per-row layout on global rows
  static const bool no_bigc = getenv("PK_NO_BIGC") != nullptr;
  const size_t rowbufs = ((size_t)3 * a.m.nv + a.m.nv / a.m.nvyz + 1) / 2 * 16 + 16;
  const size_t scr = (NT / 32) * (size_t)BIG_SCR * 8;  // (T < 0) plan scratch, aliased under bigc
  a.bigc = T < 0 && NT == 256 && !no_bigc && bigc_layout(a.m) &&
           base_smem(a.m.nv, T, S, G, NT) - scr + rowbufs + 16 * 8 <= 226 * 1024 &&
           (size_t)(NT / 32) * BIG_SCR <= 2 * (size_t)a.m.nv;
  const size_t base = base_smem(a.m.nv, T, S, G, NT) + (a.bigc ? rowbufs - scr : 0);
  // slice vectors on chip when they fit: two CTAs per SM when the grid needs
  // them, the whole SM's shared memory when the grid has one CTA per SM
  static int num_sms = 0;
  if (!num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const size_t need = base + local_smem(a.m.nx, a.adaptation);
  // half the cluster if that puts the slice vectors on chip (one CTA per SM)
  if (!a.bigc && need > 112 * 1024 && need <= 226 * 1024 && C >= 2 &&
      (size_t)a.B * (C / 2) <= (size_t)num_sms)
    C /= 2;
  const size_t limit = a.bigc || (size_t)a.B * C <= (size_t)num_sms ? 226 * 1024 : 112 * 1024;
  // test hook: PK_FORCE_GLOBAL_SLICE=1 keeps the slice vectors in global
  // memory (whole scan buffer on chip), =2 also cuts the scan buffer to 48
  // doubles (chunked scan), so small golden cases exercise the large-nx paths
  static const int force_global =
      getenv("PK_FORCE_GLOBAL_SLICE") ? atoi(getenv("PK_FORCE_GLOBAL_SLICE")) : 0;
  size_t smem;
  a.local_smem = 0;
  a.scan_smem = 0;
  if (!force_global && base + local_smem(a.m.nx, a.adaptation) <= limit) {
    a.local_smem = 1;
    smem = base + local_smem(a.m.nx, a.adaptation);
  } else {  // global slice vectors, the field scan through an on-chip buffer
    const size_t room = limit > base ? (limit - base) / 8 : 0;
    int cap = (int)std::min<size_t>((size_t)a.m.nx, room);
    if (force_global == 2) cap = std::min(cap, 48);
    if (cap < std::min(16, a.m.nx)) return cudaErrorInvalidValue;  // (never: tens of KB left)
    a.scan_smem = cap;
    smem = base + (size_t)cap * 8;
  }
  auto kern = fine_kernel<T, S, G, NT, AD>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if constexpr ((G > 0 && NT > 128) || (G < 0 && NT > 256)) {
    // the wide layouts (8-warp G8, 16-warp GS) only when every cluster of the
    // grid is resident at one CTA per SM; else the caller falls back
    if ((size_t)a.B * C > (size_t)num_sms) return cudaErrorNotSupported;
    if (C > 1) {
      if (C > 8 && cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) !=
                       cudaSuccess)
        return cudaErrorNotSupported;
      cudaLaunchConfig_t qc = {};
      qc.gridDim = dim3(C);
      qc.blockDim = dim3(NT);
      qc.dynamicSmemBytes = smem;
      cudaLaunchAttribute qa[1];
      qa[0].id = cudaLaunchAttributeClusterDimension;
      qa[0].val.clusterDim.x = C;
      qa[0].val.clusterDim.y = 1;
      qa[0].val.clusterDim.z = 1;
      qc.attrs = qa;
      qc.numAttrs = 1;
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, kern, &qc) != cudaSuccess) {
        cudaGetLastError();
        return cudaErrorNotSupported;
      }
      if (n < a.B) return cudaErrorNotSupported;
    }
  }
  static const bool dbg_packing = getenv("PK_DEBUG_PACKING") != nullptr;
  const bool autok = a.kps == 0;
  // Few large slices (e.g. cfg4's 8 windows per GPU of 8192 cells: 64 CTAs on
  // 148 SMs): grow the 8-CTA clusters up to 16 CTAs while every cluster of
  // the grid stays resident (GPC packing: 12 x 8 does not fit, 10 x 8 does)
  // and every warp keeps >= 8 rows -- the micro phase shrinks with the share.
  static const bool no_grow = getenv("PK_NO_GROW") != nullptr;
  if (!no_grow && autok && C == 8 && !a.bigc && T != 0 &&
      (long long)a.m.nx >= 9LL * (NT / 32) * 8 && (size_t)a.B * 9 <= 2 * (size_t)num_sms) {
    static size_t g_smem = 0;
    static int g_max[17];
    if (g_smem != smem) {
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      if (e != cudaSuccess) return e;
      for (int cc = 9; cc <= 16; ++cc) {
        cudaLaunchConfig_t qc = {};
        qc.gridDim = dim3(cc);
        qc.blockDim = dim3(NT);
        qc.dynamicSmemBytes = smem;
        cudaLaunchAttribute qa[1];
        qa[0].id = cudaLaunchAttributeClusterDimension;
        qa[0].val.clusterDim.x = cc;
        qa[0].val.clusterDim.y = 1;
        qa[0].val.clusterDim.z = 1;
        qc.attrs = qa;
        qc.numAttrs = 1;
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, kern, &qc) != cudaSuccess) {
          cudaGetLastError();
          n = 0;
        }
        g_max[cc] = n;
      }
      g_smem = smem;
    }
    for (int cc = 16; cc > 8; --cc)
      if (g_max[cc] >= a.B && (long long)a.m.nx >= (long long)cc * (NT / 32) * 8) {
        C = cc;
        break;
      }
  }
  a.kps = 1;
  a.sg = 0;
  if constexpr (T < 0) {
    // Big rows, one CTA per row and one CTA per SM: the cluster size that
    // keeps every cluster resident.  GPC packing admits fewer clusters than
    // num_sms / C (37 slices x 4 CTAs = 148 CTAs run as two waves, 32 + 5);
    // a second wave doubles the launch.  Cost of a size: waves x rows per CTA.
    // All-kinetic slices with on-chip vectors may run as software groups
    // instead (cooperative launch, moments through global memory as for the
    // G8 layouts): no GPC limit, every SM busy.
    if (a.bigc && autok) {
      static size_t b_smem = 0;
      static int b_max[17];
      if (b_smem != smem) {
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
        for (int cc = 1; cc <= 16; ++cc) {
          cudaLaunchConfig_t qc = {};
          qc.gridDim = dim3(cc);
          qc.blockDim = dim3(NT);
          qc.dynamicSmemBytes = smem;
          cudaLaunchAttribute qa[1];
          qa[0].id = cudaLaunchAttributeClusterDimension;
          qa[0].val.clusterDim.x = cc;
          qa[0].val.clusterDim.y = 1;
          qa[0].val.clusterDim.z = 1;
          qc.attrs = qa;
          qc.numAttrs = 1;
          int n = 0;
          if (cudaOccupancyMaxActiveClusters(&n, kern, &qc) != cudaSuccess) {
            cudaGetLastError();
            n = 0;
          }
          b_max[cc] = n;
        }
        b_smem = smem;
        if (dbg_packing) {
          fprintf(stderr, "pk big rows: smem %zu, max active clusters:", smem);
          for (int cc = 1; cc <= 16; ++cc) fprintf(stderr, " %d:%d", cc, b_max[cc]);
          fprintf(stderr, "\n");
        }
      }
      auto rows = [&](int cc) { return (long long)((a.m.nx + cc - 1) / cc); };
      long long best = -1;
      for (int cc = 1; cc <= 16; ++cc) {
        if (b_max[cc] <= 0 || a.m.nx < 2 * cc) continue;
        const long long cost = (long long)((a.B + b_max[cc] - 1) / b_max[cc]) * rows(cc);
        if (best < 0 || cost < best) {
          best = cost;
          C = cc;
        }
      }
      static const bool no_sg = getenv("PK_NO_SG") != nullptr;
      if (!AD && !no_sg && a.local_smem && best >= 0)
        for (int cc = 2; cc <= 16; ++cc) {
          if ((long long)a.B * cc > num_sms || a.m.nx < 2 * cc) continue;
          // (the group barrier costs more than a cluster barrier: strictly fewer rows)
          if (rows(cc) < best) {
            best = rows(cc);
            C = cc;
            a.sg = cc;
          }
        }
    }
  }
  if constexpr (!AD && G > 0) {
    // More slices than SMs (one CTA per slice, some SMs with one CTA and some
    // with two): pack K slices into clusters of C > K CTAs so that every CTA
    // streams K/C of a slice, e.g. 200 slices as 67 clusters of 4 CTAs x 3
    // slices.  Only packings whose clusters are all co-resident (one wave,
    // cudaOccupancyMaxActiveClusters: GPC packing caps 8-CTA clusters at 33
    // on a B200, so 256 slices keep one CTA each) qualify.
    if (autok && C == 1 && a.B > num_sms && a.local_smem && smem <= 112 * 1024) {
      static size_t q_smem = 0;
      static int q_max[17];
      if (q_smem != smem) {
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
        for (int cc = 2; cc <= 16; ++cc) {
          cudaLaunchConfig_t qc = {};
          qc.gridDim = dim3(cc);
          qc.blockDim = dim3(NT);
          qc.dynamicSmemBytes = smem;
          cudaLaunchAttribute qa[1];
          qa[0].id = cudaLaunchAttributeClusterDimension;
          qa[0].val.clusterDim.x = cc;
          qa[0].val.clusterDim.y = 1;
          qa[0].val.clusterDim.z = 1;
          qc.attrs = qa;
          qc.numAttrs = 1;
          int n = 0;
          if (cudaOccupancyMaxActiveClusters(&n, kern, &qc) != cudaSuccess) {
            cudaGetLastError();
            n = 0;
          }
          q_max[cc] = n;
        }
        q_smem = smem;
        if (dbg_packing) {
          fprintf(stderr, "pk packing: smem %zu, max active clusters:", smem);
          for (int cc = 2; cc <= 16; ++cc) fprintf(stderr, " %d:%d", cc, q_max[cc]);
          fprintf(stderr, "\n");
        }
      }
      double best = 1.0;
      for (int cc = 2; cc <= 16; ++cc)
        for (int kk = 1; kk < cc; ++kk) {
          const double load = (double)kk / cc;
          if (load >= best || (a.B + kk - 1) / kk > q_max[cc]) continue;
          if ((long long)kk * a.m.nx < 32LL * cc * (NT / 32)) continue;  // >= 32 rows per warp
          best = load;
          C = cc;
          a.kps = kk;
        }
      // Software groups (cooperative launch, no hardware cluster): the GPC
      // packing limit does not apply, only the CTA slots of the whole chip,
      // e.g. 256 slices as 37 groups of 8 CTAs x 7 slices on 296 slots.  The
      // group barrier costs more than a cluster barrier: only a strictly
      // lighter load than the best hardware packing qualifies.
      static const bool no_sg = getenv("PK_NO_SG") != nullptr;
      int occ = 0;
      if (!no_sg && cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT, smem) != cudaSuccess) {
        cudaGetLastError();
        occ = 0;
      }
      const long long slots = (long long)occ * num_sms;
      for (int cc = 2; cc <= 16 && !no_sg; ++cc)
        for (int kk = 1; kk < cc; ++kk) {
          const double load = (double)kk / cc;
          if (load >= best - 1e-9 || (long long)(a.B + kk - 1) / kk * cc > slots) continue;
          if ((long long)kk * a.m.nx < 32LL * cc * (NT / 32)) continue;
          best = load;
          C = cc;
          a.kps = kk;
          a.sg = cc;
        }
    }
  }
  // Hardware clusters of a persistent kernel that are not all resident run in
  // waves, each a whole launch long (GPC packing admits fewer clusters than
  // CTA slots / C: e.g. 33 clusters of 4 at one CTA per SM).  When this grid
  // would need more than one wave, take the size <= C with the least
  // waves x rows per CTA from the measured residency (big rows chose above).
  if (a.sg <= 1 && a.kps == 1 && autok && C > 1 && !a.bigc) {
    static size_t w_smem = 0;
    static int w_max[17];
    if (w_smem != smem) {
      for (int cc = 0; cc <= 16; ++cc) w_max[cc] = -1;
      w_smem = smem;
    }
    auto max_active = [&](int cc) {
      if (w_max[cc] < 0) {
        if (cc > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaLaunchConfig_t qc = {};
        qc.gridDim = dim3(cc);
        qc.blockDim = dim3(NT);
        qc.dynamicSmemBytes = smem;
        cudaLaunchAttribute qa[1];
        qa[0].id = cudaLaunchAttributeClusterDimension;
        qa[0].val.clusterDim.x = cc;
        qa[0].val.clusterDim.y = 1;
        qa[0].val.clusterDim.z = 1;
        qc.attrs = qa;
        qc.numAttrs = 1;
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, kern, &qc) != cudaSuccess) {
          cudaGetLastError();
          n = 0;
        }
        w_max[cc] = n;
      }
      return w_max[cc];
    };
    const int n0 = max_active(C);
    if (n0 > 0 && a.B > n0) {
      long long best = (long long)((a.B + n0 - 1) / n0) * ((a.m.nx + C - 1) / C);
      for (int cc = C - 1; cc >= 1; --cc) {
        const int n = max_active(cc);
        if (n <= 0) continue;
        const long long cost = (long long)((a.B + n - 1) / n) * ((a.m.nx + cc - 1) / cc);
        if (cost < best) {
          best = cost;
          C = cc;
        }
      }
      if (dbg_packing) fprintf(stderr, "pk packing: B %d does not fit in one wave, clusters of %d\n", a.B, C);
    }
  }
  const bool sg = a.sg > 1;
  static const bool pass_prepare = getenv("PK_PASS_PREPARE") != nullptr;
  a.pass_prepare = pass_prepare ? 1 : 0;
  if (dbg_packing)
    fprintf(stderr, "pk packing: B %d, %s of %d CTAs x %d slices\n", a.B,
            a.sg > 1 ? "software group" : "cluster", C, a.kps);
  last_launch[0] = C;
  last_launch[1] = a.kps;
  last_launch[2] = a.local_smem;
  last_launch[3] = a.bigc ? (sg ? 3 : 2) : (sg ? 1 : 0);
  if (sg) {
    e = cudaMemsetAsync(a.sg_cnt, 0, (size_t)((a.B + a.kps - 1) / a.kps) * sizeof(unsigned), st);
    if (e != cudaSuccess) return e;
  }
  if (C > 8 && !sg) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((a.B + a.kps - 1) / a.kps * C);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  if (sg) {  // every group's CTAs must be co-resident: the launch fails otherwise
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
  } else {
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
  }
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, a);
}

template <int T, int S, int G, int NT>
static cudaError_t launch_T(const FineArgs& a, int C, cudaStream_t st) {
  return a.adaptation ? launch_TA<T, S, G, NT, true>(a, C, st)
                      : launch_TA<T, S, G, NT, false>(a, C, st);
}

// one fine_kernel layout (both adaptation modes) per part
#define PK_LAYOUT(n, name, ...)                                           \
  cudaError_t name(const FineArgs& a, int C, cudaStream_t st);            \
  PK_LAYOUT_BODY_##n(name, __VA_ARGS__)
#define PK_LAYOUT_DEF(name, ...) \
  cudaError_t name(const FineArgs& a, int C, cudaStream_t st) { return launch_T<__VA_ARGS__>(a, C, st); }
#if PK_IN_PART(0)
#define PK_LAYOUT_BODY_0(name, ...) PK_LAYOUT_DEF(name, __VA_ARGS__)
#else
#define PK_LAYOUT_BODY_0(name, ...)
#endif
#if PK_IN_PART(1)
#define PK_LAYOUT_BODY_1(name, ...) PK_LAYOUT_DEF(name, __VA_ARGS__)
#else
#define PK_LAYOUT_BODY_1(name, ...)
#endif
#if PK_IN_PART(2)
#define PK_LAYOUT_BODY_2(name, ...) PK_LAYOUT_DEF(name, __VA_ARGS__)
#else
#define PK_LAYOUT_BODY_2(name, ...)
#endif
#if PK_IN_PART(3)
#define PK_LAYOUT_BODY_3(name, ...) PK_LAYOUT_DEF(name, __VA_ARGS__)
#else
#define PK_LAYOUT_BODY_3(name, ...)
#endif
#if PK_IN_PART(4)
#define PK_LAYOUT_BODY_4(name, ...) PK_LAYOUT_DEF(name, __VA_ARGS__)
#else
#define PK_LAYOUT_BODY_4(name, ...)
#endif
#if PK_IN_PART(5)
#define PK_LAYOUT_BODY_5(name, ...) PK_LAYOUT_DEF(name, __VA_ARGS__)
#else
#define PK_LAYOUT_BODY_5(name, ...)
#endif
#if PK_IN_PART(6)
#define PK_LAYOUT_BODY_6(name, ...) PK_LAYOUT_DEF(name, __VA_ARGS__)
#else
#define PK_LAYOUT_BODY_6(name, ...)
#endif
#if PK_IN_PART(7)
#define PK_LAYOUT_BODY_7(name, ...) PK_LAYOUT_DEF(name, __VA_ARGS__)
#else
#define PK_LAYOUT_BODY_7(name, ...)
#endif
#if PK_IN_PART(8)
#define PK_LAYOUT_BODY_8(name, ...) PK_LAYOUT_DEF(name, __VA_ARGS__)
#else
#define PK_LAYOUT_BODY_8(name, ...)
#endif
PK_LAYOUT(0, fine_generic, 0, 1, 0, 256)      // generic rows (<= 256 nodes)
PK_LAYOUT(1, fine_big, -1, 1, 0, 256)         // big 1D-3V rows
PK_LAYOUT(2, fine_g8_64w, 2, 16, 4, 256)      // nv = 64, G8, 8 warps
PK_LAYOUT(3, fine_g8_64, 2, 16, 4, 128)       // nv = 64, G8, 4 warps
PK_LAYOUT(4, fine_g8_128w, 4, 14, 8, 256)     // nv = 128, G8, 8 warps
PK_LAYOUT(5, fine_g8_128, 4, 14, 8, 128)      // nv = 128, G8, 4 warps
PK_LAYOUT(6, fine_gs_256, 8, 20, -4, 256)     // nv = 256, producer/consumer
PK_LAYOUT(7, fine_tma_512, 16, 3, 0, 256)     // nv = 512
PK_LAYOUT(8, fine_gs_256w, 8, 40, -4, 512)    // nv = 256, 15 consumer warps, 40-row ring

#if PK_IN_PART(0)
template <int T>
static cudaError_t launch_lift_T(const LiftArgs& a, cudaStream_t st) {
  const size_t smem = T < 0 ? (kThreads / 32) * (size_t)BIG_SCR * 8
                            : 4 * a.m.nv * 8 + (kThreads / 32) * a.m.nv * 8;
  cudaError_t e =
      cudaFuncSetAttribute(lift_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  lift_kernel<T><<<a.B, kThreads, smem, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_lift(const LiftArgs& a, cudaStream_t st) {
  if (a.m.nvyz > 1) return a.m.nv <= 32 * GT ? launch_lift_T<0>(a, st) : launch_lift_T<-1>(a, st);
  switch (a.m.nv) {
    case 64: return launch_lift_T<2>(a, st);
    case 128: return launch_lift_T<4>(a, st);
    case 256: return launch_lift_T<8>(a, st);
    case 512: return launch_lift_T<16>(a, st);
    default:
      if (a.m.nv <= 32 * GT) return launch_lift_T<0>(a, st);
      return cudaErrorInvalidValue;
  }
}

// ---------------------------------------------------------------------------
// Standalone adaptation indicators (adaptation.py:120-181): the public K3
// operators on the device, in the arithmetic of prepare_step (the in-kernel
// copy F uses every step).  One CTA per slice.

// R = -D3(J_c) + E_c D2(J_c) + (2 rho - 3 rho_bar) D1(J_c) + 2 J_c D1(rho)
//     - D1(rho) dtE_c   (remainder_from_fields / remainder_indicator,
// adaptation.py:120-152)
__global__ void __launch_bounds__(256) remainder_kernel(const IndArgs a) {
  extern __shared__ __align__(16) double ism[];
  const MeshDev& m = a.m;
  const int nx = m.nx, b = blockIdx.x, tid = threadIdx.x, nt = blockDim.x;
  const size_t o = (size_t)b * nx;
  const double* rho = a.rho + o;
  const double* E = a.E + o;
  double* J = ism;         // fluid_flux at interfaces, then dE/dt at interfaces
  double* Jc = ism + nx;   // J_c at cells
  double* dE = ism;
  for (int i = tid; i < nx; i += nt) J[i] = flux_J(rho[i], rho[wrap(i + 1, nx)], E[i], m.dx, m.rdx);
  __syncthreads();
  for (int i = tid; i < nx; i += nt) Jc[i] = 0.5 * (J[wrap(i - 1, nx)] + J[i]);
  __syncthreads();
  for (int i = tid; i < nx; i += nt)
    dE[i] = a.dtE_c ? a.dtE_c[o + i] : (E[i] - a.E_prev[o + i]) / a.dt;
  __syncthreads();
  const double three_rb = 3.0 * a.rho_bar[b];
  for (int i = tid; i < nx; i += nt) {
    const int ip = wrap(i - 1, nx);
    const double dtEc = a.dtE_c ? dE[i] : 0.5 * (dE[ip] + dE[i]);
    const double Ec = 0.5 * (E[ip] + E[i]);
    const double d1J = stencil_at(Jc, i, nx, m, 1);
    const double d2J = stencil_at(Jc, i, nx, m, 2);
    const double d3J = stencil_at(Jc, i, nx, m, 3);
    const double d1r = stencil_at(rho, i, nx, m, 1);
    a.R[o + i] = -d3J + Ec * d2J + (2.0 * rho[i] - three_rb) * d1J + 2.0 * Jc[i] * d1r -
                 d1r * dtEc;
  }
}

// gnorm_i = sqrt(0.5 (<g^2>_{i-1} + <g^2>_i)) (perturbation_indicator,
// adaptation.py:155-159); <.> the folded pairwise bracket, one warp per row.
__global__ void __launch_bounds__(256) gnorm_kernel(const IndArgs a) {
  extern __shared__ __align__(16) double ism[];
  const MeshDev& m = a.m;
  const int nx = m.nx, nv = m.nv, b = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  double* sq = ism;
  double* scr = ism + nx + warp * BIG_SCR;
  const double* g = a.g + (size_t)b * nx * nv;
  for (int i = warp; i < nx; i += nwarp) {
    const double* row = g + (size_t)i * nv;
    const double v = big_bracket([&](int c) { const double x = row[c]; return x * x; }, m, scr);
    if (lane == 0) sq[i] = v;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nx; i += blockDim.x)
    a.gnorm[(size_t)b * nx + i] = sqrt0(0.5 * (sq[wrap(i - 1, nx)] + sq[i]));
}

// labels (update_labels, DomainLabels.from_cells; adaptation.py:100-105,162-181)
__global__ void labels_kernel(const IndArgs a) {
  const int nx = a.m.nx;
  const int64_t n = (int64_t)a.B * nx;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b0 = k - k % nx;
    auto kin = [&](int64_t q) {
      const bool fR = fabs(a.Rin[q]) < a.delta0;
      const bool fg = a.gin[q] < a.eta0;
      return !(a.combine_and ? (fR && fg) : (fR || fg));
    };
    const bool kc = kin(k);
    const int64_t kn = (k + 1 - b0 == nx) ? b0 : k + 1;
    a.kc[k] = kc ? 1 : 0;
    a.ki[k] = (kc || kin(kn)) ? 1 : 0;
  }
}

cudaError_t launch_indicators(const IndArgs& a, int which, cudaStream_t st) {
  const int nx = a.m.nx;
  if (which == 0) {
    const size_t smem = 2 * (size_t)nx * 8;
    cudaError_t e = cudaFuncSetAttribute(remainder_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    remainder_kernel<<<a.B, 256, smem, st>>>(a);
  } else if (which == 1) {
    const size_t smem = ((size_t)nx + 8 * (size_t)BIG_SCR) * 8;
    cudaError_t e =
        cudaFuncSetAttribute(gnorm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    gnorm_kernel<<<a.B, 256, smem, st>>>(a);
  } else {
    const int64_t n = (int64_t)a.B * nx;
    const int64_t want = (n + 255) / 256;
    labels_kernel<<<(int)(want < 148 * 8 ? (want > 0 ? want : 1) : 148 * 8), 256, 0, st>>>(a);
  }
  return cudaGetLastError();
}

cudaError_t launch_field(const FieldArgs& a, cudaStream_t st) {
  // slice_field's block_pairwise2 keeps two reductions in flight
  const size_t smem = (sizeof(PwPlan) + 15) / 16 * 16 + 2 * (MAX_LEAF + MAX_NODE) * 8;
  cudaError_t e =
      cudaFuncSetAttribute(field_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  field_kernel<<<a.B, kThreads, smem, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_fine(const FineArgs& a, int C, cudaStream_t st) {
  if (a.m.nvyz > 1) {  // 1D-3V rows: generic layout up to 256 nodes, big rows beyond
    if (a.m.nv <= 32 * GT) return fine_generic(a, C, st);
    return fine_big(a, C, st);
  }
  if ((a.m.nv == 64 || a.m.nv == 128) && !a.m.mirror)  // G8 needs the mirrored grid
    return fine_generic(a, C, st);
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  // a grid of at most one CTA per SM (few, latency-bound slices: parareal
  // windows): 8 warps per CTA at the full register file -- half the rows per
  // warp and half the cells per thread in the slice phase
  // (launch_TA may still halve C; it refuses the wide layout with
  // cudaErrorNotSupported unless every cluster is resident)
  static const bool no_wide = getenv("PK_NO_WIDE") != nullptr;
  const bool wide = !no_wide && (long long)a.B * (C > 1 ? C / 2 : 1) <= nsm;
  cudaError_t e = cudaErrorNotSupported;
  switch (a.m.nv) {
    // producer/consumer GS pipeline: 7 consumer warps + 1 producer warp
    case 64:  // G8 per-warp rings, 4 warps (8 at one CTA per SM)
      if (wide) e = fine_g8_64w(a, C, st);
      if (e == cudaErrorNotSupported) e = fine_g8_64(a, C, st);
      return e;
    case 128:
      if (wide) e = fine_g8_128w(a, C, st);
      if (e == cudaErrorNotSupported) e = fine_g8_128(a, C, st);
      return e;
      // (8 warps at two CTAs per SM, <= 128 registers: no spills, but the micro
      // loop loses its ILP and the step takes 1.6x longer)
    case 256:
      // few slices at one CTA per SM (cfg4's 8 windows per GPU: kinetic rows
      // are served one per consumer warp at ~4k cycles each): 15 consumer
      // warps and a 40-row ring instead of 7 and 20
      if (wide) e = fine_gs_256w(a, C, st);
      if (e == cudaErrorNotSupported) e = fine_gs_256(a, C, st);
      return e;
    case 512: return fine_tma_512(a, C, st);
    default:
      if (a.m.nv <= 32 * GT) return fine_generic(a, C, st);
      return cudaErrorInvalidValue;
  }
}
#endif  // PK_IN_PART(0)

}  // namespace pk
