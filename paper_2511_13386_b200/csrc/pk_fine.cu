// Fine propagator F on B200: one thread-block cluster per slice runs the
// whole window (all steps) in a single persistent launch.
//
// Per step (hybrid.py:123-188, kinetic.py:255-273):
//   micro phase   all CTAs of the cluster, one warp per interface row:
//                 g' = k1 g - k2 (upwind transport - M d_x<xi g> + xi M J)
//                 (kinetic.py:148-224) and the row moments <xi g'>, <g'^2>;
//                 only kinetic rows are visited (compacted row list).
//   cluster barrier
//   slice phase   the leader CTA: masked rho update (hybrid.py:117-119,
//                 kinetic.py:232-240, fluid.py:55-57), field solve
//                 (poisson.py:21-54), J, remainder/perturbation indicators and
//                 labels for the next step (adaptation.py:120-181), Chapman-
//                 Enskog re-initialisation of flipped rows (lifting.py:38-105),
//                 projection coefficients and the next kinetic-row list.
//   cluster barrier
// g is double-buffered in HBM/L2 (the mixed update reads stale neighbours,
// SURVEY F9).  Arithmetic follows numpy's operation order (Appendix A of
// SURVEY.md) so results are bitwise equal to the reference.
#include <cooperative_groups.h>

#include "../../include/pk.h"
#include "pk_args.h"

namespace cg = cooperative_groups;

namespace pk {

// ---------------------------------------------------------------------------
// Row layouts.  A warp owns one interface row g[i, 0..nv).

// Fast layout, nv = 64 P: lane l, slot s < P holds column 32 s + l (xi < 0),
// slot T-1-s holds its mirror nv-1-(32 s + l) (xi > 0).  Mirror pairs sit in
// one lane, so the velocity fold is register-local; loads stay coalesced.
template <int T>
struct Fast {
  static constexpr int P = T / 2;
  __device__ static __forceinline__ int col(int lane, int s) {
    return s < P ? 32 * s + lane : 32 * s + 31 - lane;
  }
};

template <int T>
__device__ __forceinline__ void fast_load(double (&v)[T], const double* row, int lane) {
#pragma unroll
  for (int s = 0; s < T; ++s) v[s] = __ldcg(row + Fast<T>::col(lane, s));
}

template <int T>
__device__ __forceinline__ void fast_store(const double (&v)[T], double* row, int lane) {
#pragma unroll
  for (int s = 0; s < T; ++s) __stcg(row + Fast<T>::col(lane, s), v[s]);
}

// Folded velocity integral of q (mesh.py:95-133): mirror-pair fold, then
// numpy's pairwise order (eight interleaved accumulators per block of <= 128
// folded terms, xor-butterfly tree), times dv3.  Same bits on every lane.
template <int T>
__device__ __forceinline__ double fast_bracket(const double (&q)[T], int lane, double dv3) {
  constexpr int P = T / 2;
  double f[P];
#pragma unroll
  for (int t = 0; t < P; ++t) f[t] = q[t] + q[T - 1 - t];
  const int k = lane & 7;
  auto block = [&](int t0, int t1) {
    double r = __shfl_sync(FULL, f[t0], k);
#pragma unroll
    for (int t = t0; t < t1; ++t) {
#pragma unroll
      for (int qq = (t == t0 ? 1 : 0); qq < 4; ++qq) r = r + __shfl_sync(FULL, f[t], k + 8 * qq);
    }
    r = r + __shfl_xor_sync(FULL, r, 1);
    r = r + __shfl_xor_sync(FULL, r, 2);
    r = r + __shfl_xor_sync(FULL, r, 4);
    return r;
  };
  double tot;
  if constexpr (P <= 4) {
    tot = block(0, P);
  } else {  // 256 folded terms: numpy splits at 128
    const double a = block(0, 4);
    const double b = block(4, 8);
    tot = a + b;
  }
  return tot * dv3;
}

// Per-lane velocity constants in slot order.
template <int T>
struct FastConsts {
  double vx[T], M[T], xiM[T];
  __device__ void load(const double* svx, const double* sM, const double* sxiM, int lane) {
#pragma unroll
    for (int s = 0; s < T; ++s) {
      const int c = Fast<T>::col(lane, s);
      vx[s] = svx[c];
      M[s] = sM[c];
      xiM[s] = sxiM[c];
    }
  }
};

struct RowCoef {
  double vco, dc, J, k1, k2;
  int vsg;
};

// One micro update of row i (kinetic.py:164-193,220-224 / hybrid.py:91-110).
// gp, gc, gn: rows i-1, i, i+1 (as stored).  out: g'.
template <int T>
__device__ __forceinline__ void fast_micro(const double (&gp)[T], const double (&gc)[T],
                                           const double (&gn)[T], double (&out)[T],
                                           const FastConsts<T>& C, const RowCoef& rc,
                                           double dx, double rdx, int lane) {
  constexpr int P = T / 2;
  // velocity-upwind neighbours, chosen by sign(E): zero inflow at +-v*
  double nb[T];
  if (rc.vsg > 0) {  // need g_{j-1}
    double up[T], dn[T];
#pragma unroll
    for (int s = 0; s < T; ++s) {
      if (s < P) up[s] = __shfl_sync(FULL, gc[s], (lane + 31) & 31);
      else dn[s] = __shfl_sync(FULL, gc[s], (lane + 1) & 31);
    }
#pragma unroll
    for (int s = 0; s < T; ++s) {
      if (s < P) nb[s] = lane >= 1 ? up[s] : (s >= 1 ? up[s > 0 ? s - 1 : 0] : 0.0);
      else nb[s] = lane <= 30 ? dn[s] : (s > P ? dn[s > P ? s - 1 : P] : gc[P - 1]);
    }
  } else if (rc.vsg < 0) {  // need g_{j+1}
    double up[T], dn[T];
#pragma unroll
    for (int s = 0; s < T; ++s) {
      if (s < P) dn[s] = __shfl_sync(FULL, gc[s], (lane + 1) & 31);
      else up[s] = __shfl_sync(FULL, gc[s], (lane + 31) & 31);
    }
#pragma unroll
    for (int s = 0; s < T; ++s) {
      if (s < P) nb[s] = lane <= 30 ? dn[s] : (s + 1 < P ? dn[s + 1 < P ? s + 1 : 0] : gc[P]);
      else nb[s] = lane >= 1 ? up[s] : (s + 1 < T ? up[s + 1 < T ? s + 1 : T - 1] : 0.0);
    }
  }
#pragma unroll
  for (int s = 0; s < T; ++s) {
    const double g = gc[s];
    // x-upwind by sign(xi): xi<0 uses (g_{i+1}-g_i), xi>0 uses (g_i-g_{i-1})
    double o = (s < P) ? C.vx[s] * (gn[s] - g) : C.vx[s] * (g - gp[s]);
    o = qdiv(o, dx, rdx);
    if (rc.vsg > 0) o = o + (g - nb[s]) * rc.vco;
    else if (rc.vsg < 0) o = o + (nb[s] - g) * rc.vco;
    o = o - C.M[s] * rc.dc;
    const double forcing = o + C.xiM[s] * rc.J;
    out[s] = rc.k1 * g - rc.k2 * forcing;
  }
}

// ---------------------------------------------------------------------------
// Generic layout (any nv <= 256): lane l, slot s holds column 32 s + l.  The
// fold and the pairwise sum go through a per-warp shared-memory row.
constexpr int GT = 8;  // slots: nv <= 256

__device__ __forceinline__ void gen_load(double (&v)[GT], const double* row, int lane, int nv) {
#pragma unroll
  for (int s = 0; s < GT; ++s) {
    const int c = 32 * s + lane;
    v[s] = c < nv ? __ldcg(row + c) : 0.0;
  }
}

__device__ __forceinline__ void gen_store(const double (&v)[GT], double* row, int lane, int nv) {
#pragma unroll
  for (int s = 0; s < GT; ++s) {
    const int c = 32 * s + lane;
    if (c < nv) __stcg(row + c, v[s]);
  }
}

__device__ __forceinline__ double gen_bracket(const double (&q)[GT], double* wrow, int lane,
                                              int nv, double dv3) {
#pragma unroll
  for (int s = 0; s < GT; ++s) {
    const int c = 32 * s + lane;
    if (c < nv) wrow[c] = q[s];
  }
  __syncwarp();
  const int h = nv / 2;
  double mid = (nv & 1) ? wrow[h] : 0.0;
  double f[GT];
#pragma unroll
  for (int s = 0; s < GT; ++s) {
    const int j = 32 * s + lane;
    f[s] = j < h ? wrow[j] + wrow[nv - 1 - j] : 0.0;
  }
  __syncwarp();
#pragma unroll
  for (int s = 0; s < GT; ++s) {
    const int j = 32 * s + lane;
    if (j < h) wrow[j] = f[s];
  }
  __syncwarp();
  double tot = warp_leaf([&](int j) { return wrow[j]; }, 0, h, lane);
  if (nv & 1) tot = tot + mid;
  __syncwarp();
  return tot * dv3;
}

__device__ __forceinline__ void gen_micro(const double (&gp)[GT], const double (&gc)[GT],
                                          const double (&gn)[GT], double (&out)[GT],
                                          const double* svx, const double* sM, const double* sxiM,
                                          const RowCoef& rc, int nv, double dx, double rdx,
                                          int lane) {
  double left[GT], right[GT];
#pragma unroll
  for (int s = 0; s < GT; ++s) {
    const double u = __shfl_sync(FULL, gc[s], (lane + 31) & 31);
    const double d = __shfl_sync(FULL, gc[s], (lane + 1) & 31);
    left[s] = u;
    right[s] = d;
  }
  double lfix[GT], rfix[GT];
#pragma unroll
  for (int s = 0; s < GT; ++s) {
    const int c = 32 * s + lane;
    // column c-1 for lane 0 is lane 31 of slot s-1; column c+1 for lane 31 is lane 0 of slot s+1
    lfix[s] = lane >= 1 ? left[s] : (s >= 1 ? left[s >= 1 ? s - 1 : 0] : 0.0);
    rfix[s] = lane <= 30 ? right[s] : (s + 1 < GT ? right[s + 1 < GT ? s + 1 : 0] : 0.0);
    if (c == 0) lfix[s] = 0.0;
    if (c + 1 >= nv) rfix[s] = 0.0;
  }
  const double Ep = rc.vsg > 0 ? rc.vco : 0.0;
  const double Em = rc.vsg < 0 ? rc.vco : 0.0;
#pragma unroll
  for (int s = 0; s < GT; ++s) {
    const int c = 32 * s + lane;
    if (c >= nv) {
      out[s] = 0.0;
      continue;
    }
    const double xi = svx[c];
    const double xp = xi > 0.0 ? xi : 0.0;
    const double xm = xi < 0.0 ? xi : 0.0;
    const double g = gc[s];
    double o = xp * (g - gp[s]);
    o = o + xm * (gn[s] - g);
    o = qdiv(o, dx, rdx);
    // literal reference terms (both signs) for the generic path
    const double dm = (c == 0) ? g : g - lfix[s];
    o = o + dm * Ep;
    const double dp = (c == nv - 1) ? -g : rfix[s] - g;
    o = o + dp * Em;
    o = o - sM[c] * rc.dc;
    const double forcing = o + sxiM[c] * rc.J;
    out[s] = rc.k1 * g - rc.k2 * forcing;
  }
}

// ---------------------------------------------------------------------------
// Shared memory layout of a CTA.
struct Smem {
  double* vx;
  double* M;
  double* xiM;
  double* w2;
  PwPlan* plan;
  double* red;    // pairwise scratch (MAX_LEAF + MAX_NODE)
  double* wrow;   // generic rows: one nv-row per warp
  int* misc;      // small ints
};

// Per-slice view of the workspace.
struct SliceView {
  int b, nx, nv;
  double *rho, *E, *Eprev, *J, *fl, *sq, *bm, *dco, *vco, *tA, *tB, *tC, *tD, *tE, *blift;
  int8_t* vsg;
  uint8_t *kc, *ki, *flip, *nza, *nzb, *kcn, *kin;
  int* klist;
  int* nk;
  int* abort_;
  double* ga;
  double* gb;
  double rb;
};

__device__ __forceinline__ SliceView make_view(const FineArgs& a, int b) {
  SliceView v;
  const int nx = a.m.nx;
  const size_t o = (size_t)b * nx;
  v.b = b;
  v.nx = nx;
  v.nv = a.m.nv;
  v.rho = a.rho + o; v.E = a.E + o; v.Eprev = a.Eprev + o; v.J = a.J + o; v.fl = a.fl + o;
  v.sq = a.sq + o; v.bm = a.bm + o; v.dco = a.dco + o; v.vco = a.vco + o; v.tA = a.tA + o;
  v.tB = a.tB + o; v.tC = a.tC + o; v.tD = a.tD + o; v.tE = a.tE + o; v.blift = a.blift + o;
  v.vsg = a.vsg + o; v.kc = a.kc + o; v.ki = a.ki + o; v.flip = a.flip + o; v.nza = a.nza + o;
  v.nzb = a.nzb + o; v.kcn = a.kcn + o; v.kin = a.kin + o; v.klist = a.klist + o;
  v.nk = a.nk + b; v.abort_ = a.abort_ + b;
  v.ga = a.ga + o * a.m.nv;
  v.gb = a.gb + o * a.m.nv;
  v.rb = a.rho_bar[b];
  return v;
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
    if (c != 0.0) acc = acc + c * __ldcg(v + wrap(i + o - 3, nx));
  }
  return acc * m.sts[p - 1];
}

// E = solve_field(rho) into E_out; returns false on a solvability violation.
// poisson.py:41-54: src=(rho-rb)dx; defect=sum(src); guard; src-=defect/nx;
// E=cumsum(src); E-=mean(E).
__device__ bool slice_field(const MeshDev& m, const double* rho, double rb, double* src,
                            double* E_out, double rtol, int exact_scan, const Smem& sm) {
  const int nx = m.nx;
  for (int i = threadIdx.x; i < nx; i += blockDim.x) src[i] = (__ldcg(rho + i) - rb) * m.dx;
  __syncthreads();
  const double defect = block_pairwise([&](int i) { return src[i]; }, *sm.plan, sm.red);
  const double scale =
      block_pairwise([&](int i) { return fabs(__ldcg(rho + i)); }, *sm.plan, sm.red) * m.dx;
  // `abs(defect) > rtol * max(scale, tiny)`: a NaN defect compares False
  // in Python too, so only a genuine violation raises.
  const double lim = rtol * fmax(scale, 2.2250738585072014e-308);
  if (fabs(defect) > lim) return false;
  const double corr = defect / (double)nx;
  for (int i = threadIdx.x; i < nx; i += blockDim.x) src[i] = src[i] - corr;
  __syncthreads();
  if (exact_scan) {
    warp_cumsum([&](int i) { return src[i]; }, [&](int i, double v) { E_out[i] = v; }, nx);
  } else {
    block_scan_fast([&](int i) { return src[i]; }, [&](int i, double v) { E_out[i] = v; }, nx,
                    sm.red);
  }
  __syncthreads();
  const double mean =
      block_pairwise([&](int i) { return __ldcg(E_out + i); }, *sm.plan, sm.red) / (double)nx;
  for (int i = threadIdx.x; i < nx; i += blockDim.x) E_out[i] = E_out[i] - mean;
  __syncthreads();
  return true;
}

// J_{i+1/2} = (rho_{i+1}-rho_i)/dx - E*0.5*(rho_i+rho_{i+1})   (fluid.py:48-52)
__device__ __forceinline__ double flux_J(double r, double rn, double e, double dx) {
  return (rn - r) / dx - e * 0.5 * (r + rn);
}

// Block-wide exclusive scan of per-thread counts; returns the total.
__device__ int block_excl_scan(int v, int* out_prefix, int* sbuf) {
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

// ---------------------------------------------------------------------------
// Row-level helpers (warp per row) used by the slice phase and the prologue.

struct LiftRow {
  double negJ;   // (-eps_i) * J_i
  double e2;     // eps_i ** 2
  double drift;  // dJ_i - E_i J_i       (order 2)
  double Rif;    // R at the interface   (higher_order)
};

// lifting.py:63-105 for one row: g = xi M (-eps J) [+ (eps^2 w) drift]
// [+ (eps^2 M) R_if]; two zero-mass projections.  Returns <xi g> and <g^2>
// via bx/bsq.
template <int T>
__device__ void fast_lift_row(double (&g)[T], const LiftRow& L, int order, int higher, int project,
                              const Smem& sm, const MeshDev& m, int lane) {
#pragma unroll
  for (int s = 0; s < T; ++s) {
    const int c = Fast<T>::col(lane, s);
    double v = sm.xiM[c] * L.negJ;
    if (order >= 2) {
      v = v + (L.e2 * sm.w2[c]) * L.drift;
      if (higher) v = v + (L.e2 * sm.M[c]) * L.Rif;
    }
    g[s] = v;
  }
  if (project) {
    for (int pass = 0; pass < 2; ++pass) {
      const double bb = fast_bracket<T>(g, lane, m.dv3) / m.m0;
#pragma unroll
      for (int s = 0; s < T; ++s) g[s] = g[s] - bb * sm.M[Fast<T>::col(lane, s)];
    }
  }
}

__device__ void gen_lift_row(double (&g)[GT], const LiftRow& L, int order, int higher, int project,
                             const Smem& sm, const MeshDev& m, double* wrow, int lane) {
  const int nv = m.nv;
#pragma unroll
  for (int s = 0; s < GT; ++s) {
    const int c = 32 * s + lane;
    if (c >= nv) {
      g[s] = 0.0;
      continue;
    }
    double v = sm.xiM[c] * L.negJ;
    if (order >= 2) {
      v = v + (L.e2 * sm.w2[c]) * L.drift;
      if (higher) v = v + (L.e2 * sm.M[c]) * L.Rif;
    }
    g[s] = v;
  }
  if (project) {
    for (int pass = 0; pass < 2; ++pass) {
      const double bb = gen_bracket(g, wrow, lane, nv, m.dv3) / m.m0;
#pragma unroll
      for (int s = 0; s < GT; ++s) {
        const int c = 32 * s + lane;
        if (c < nv) g[s] = g[s] - bb * sm.M[c];
      }
    }
  }
}

// Row moments <xi g>, <g^2>.
template <int T>
__device__ __forceinline__ void fast_moments(const double (&g)[T], const Smem& sm, double dv3,
                                             int lane, double& bx, double& bsq) {
  double q[T], r[T];
#pragma unroll
  for (int s = 0; s < T; ++s) {
    q[s] = sm.vx[Fast<T>::col(lane, s)] * g[s];
    r[s] = g[s] * g[s];
  }
  bx = fast_bracket<T>(q, lane, dv3);
  bsq = fast_bracket<T>(r, lane, dv3);
}

__device__ __forceinline__ void gen_moments(const double (&g)[GT], const Smem& sm, int nv,
                                            double dv3, double* wrow, int lane, double& bx,
                                            double& bsq) {
  double q[GT], r[GT];
#pragma unroll
  for (int s = 0; s < GT; ++s) {
    const int c = 32 * s + lane;
    q[s] = c < nv ? sm.vx[c] * g[s] : 0.0;
    r[s] = g[s] * g[s];
  }
  bx = gen_bracket(q, wrow, lane, nv, dv3);
  bsq = gen_bracket(r, wrow, lane, nv, dv3);
}

// Layout dispatch: T == 0 selects the generic layout.
template <int T>
struct Layout {
  static constexpr int S = T == 0 ? GT : T;
};

template <int T>
__device__ __forceinline__ void row_load(double (&v)[Layout<T>::S], const double* row, int lane,
                                         int nv) {
  if constexpr (T == 0) gen_load(v, row, lane, nv);
  else fast_load<T>(v, row, lane);
}

template <int T>
__device__ __forceinline__ void row_store(const double (&v)[Layout<T>::S], double* row, int lane,
                                          int nv) {
  if constexpr (T == 0) gen_store(v, row, lane, nv);
  else fast_store<T>(v, row, lane);
}

template <int T>
__device__ __forceinline__ void row_zero_store(double* row, int lane, int nv) {
  double z[Layout<T>::S];
#pragma unroll
  for (int s = 0; s < Layout<T>::S; ++s) z[s] = 0.0;
  row_store<T>(z, row, lane, nv);
}

template <int T>
__device__ __forceinline__ void row_moments(const double (&g)[Layout<T>::S], const Smem& sm,
                                            const MeshDev& m, double* wrow, int lane, double& bx,
                                            double& bsq) {
  if constexpr (T == 0) gen_moments(g, sm, m.nv, m.dv3, wrow, lane, bx, bsq);
  else fast_moments<T>(g, sm, m.dv3, lane, bx, bsq);
}

template <int T>
__device__ __forceinline__ void row_lift(double (&g)[Layout<T>::S], const LiftRow& L, int order,
                                         int higher, int project, const Smem& sm,
                                         const MeshDev& m, double* wrow, int lane) {
  if constexpr (T == 0) gen_lift_row(g, L, order, higher, project, sm, m, wrow, lane);
  else fast_lift_row<T>(g, L, order, higher, project, sm, m, lane);
}

// ---------------------------------------------------------------------------
// Slice phase: prepare step `s` (labels, flips, projection coefficients,
// row list).  `moment_all`: the fl/sq moments are valid on every row
// (prologue: user g) rather than only on the previous step's kinetic rows.
// gin: the input buffer of step s; gout: its output buffer.
template <int T>
__device__ bool prepare_step(const FineArgs& a, const SliceView& v, const Smem& sm, double dt,
                             int moment_all, double* gin, double* gout, uint8_t* nzin,
                             uint8_t* nzout, int step) {
  const MeshDev& m = a.m;
  const int nx = m.nx, nv = m.nv;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nwarp = nt >> 5;
  int* sflags = sm.misc;  // [0]: any flip, [1..32]: scan scratch

  // J from the (new) rho and E   (micro_step's fluid_flux, kinetic.py:221)
  for (int i = tid; i < nx; i += nt) {
    const int in_ = wrap(i + 1, nx);
    v.J[i] = flux_J(__ldcg(v.rho + i), __ldcg(v.rho + in_), __ldcg(v.E + i), m.dx);
  }
  if (tid == 0) sflags[0] = 0;
  __syncthreads();

  if (a.adaptation) {
    // remainder indicator (adaptation.py:120-152) at cells
    for (int i = tid; i < nx; i += nt) {
      const int ip = wrap(i - 1, nx);
      v.tA[i] = (__ldcg(v.E + i) - __ldcg(v.Eprev + i)) / dt;      // (E - E_prev)/dt
      v.tB[i] = 0.5 * (__ldcg(v.J + ip) + __ldcg(v.J + i));        // J_c
    }
    __syncthreads();
    const double three_rb = 3.0 * v.rb;
    for (int i = tid; i < nx; i += nt) {
      const int ip = wrap(i - 1, nx);
      const double dtEc = 0.5 * (__ldcg(v.tA + ip) + __ldcg(v.tA + i));
      const double Ec = 0.5 * (__ldcg(v.E + ip) + __ldcg(v.E + i));
      const double d1J = stencil_at(v.tB, i, nx, m, 1);
      const double d2J = stencil_at(v.tB, i, nx, m, 2);
      const double d3J = stencil_at(v.tB, i, nx, m, 3);
      const double d1r = stencil_at(v.rho, i, nx, m, 1);
      const double rho = __ldcg(v.rho + i);
      const double Jc = __ldcg(v.tB + i);
      const double R = -d3J + Ec * d2J + (2.0 * rho - three_rb) * d1J + 2.0 * Jc * d1r - d1r * dtEc;
      v.tC[i] = R;    // unscaled R (lift, higher_order)
      v.tD[i] = d1J;  // D1(J_c) (lift drift)
      const double Rs = a.rscale ? a.rscale[(size_t)v.b * nx + i] * R : R;
      // perturbation indicator (adaptation.py:155-159) on the incoming g
      const double sqp = (moment_all || v.ki[ip]) ? __ldcg(v.sq + ip) : 0.0;
      const double sqi = (moment_all || v.ki[i]) ? __ldcg(v.sq + i) : 0.0;
      const double gn = sqrt(0.5 * (sqp + sqi));
      const bool fR = fabs(Rs) < a.delta0;
      const bool fg = gn < a.eta0;
      const bool fluid = a.combine_and ? (fR && fg) : (fR || fg);
      v.kcn[i] = fluid ? 0 : 1;
    }
    __syncthreads();
    int anyflip = 0;
    for (int i = tid; i < nx; i += nt) {
      const uint8_t kin = v.kcn[i] | v.kcn[wrap(i + 1, nx)];
      v.kin[i] = kin;
      const uint8_t f = (kin && !v.ki[i]) ? 1 : 0;
      v.flip[i] = f;
      anyflip |= f;
    }
    if (anyflip) atomicOr(&sflags[0], 1);
    __syncthreads();
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
        for (int i = tid; i < nx; i += nt) {
          if (!v.flip[i]) continue;
          const int in_ = wrap(i + 1, nx);
          const double dJ = 0.5 * (__ldcg(v.tD + i) + __ldcg(v.tD + in_));
          v.tE[i] = dJ - __ldcg(v.E + i) * __ldcg(v.J + i);      // drift
          v.tA[i] = 0.5 * (__ldcg(v.tC + i) + __ldcg(v.tC + in_));  // R_if (tA no longer needed)
        }
        __syncthreads();
        for (int i = warp; i < nx; i += nwarp) {
          if (!v.flip[i]) continue;
          LiftRow L;
          const size_t o = (size_t)v.b * nx + i;
          L.negJ = a.neg_eps[o] * __ldcg(v.J + i);
          L.e2 = a.eps2[o];
          L.drift = __ldcg(v.tE + i);
          L.Rif = __ldcg(v.tA + i);
          double g[Layout<T>::S];
          row_lift<T>(g, L, a.lift_order, a.time_elim == 1, 1, sm, m, sm.wrow + warp * nv, lane);
          row_store<T>(g, gin + (size_t)i * nv, lane, nv);
          double bx, bsq;
          row_moments<T>(g, sm, m, sm.wrow + warp * nv, lane, bx, bsq);
          if (lane == 0) v.blift[i] = bx;
        }
      } else if (a.reinit == 1) {
        for (int i = warp; i < nx; i += nwarp) {
          if (!v.flip[i]) continue;
          row_zero_store<T>(gin + (size_t)i * nv, lane, nv);
          if (lane == 0) v.blift[i] = 0.0;
        }
      } else {
        if (tid == 0) set_status(a.status, PK_ERR_BAD_REINIT, v.b, step);
        return false;
      }
    }
    __syncthreads();
    // masked projection moment (hybrid.py:103-105) on the post-flip rows
    for (int i = tid; i < nx; i += nt) {
      const bool valid = moment_all || v.ki[i];
      const double b = v.kin[i] ? (v.flip[i] ? __ldcg(v.blift + i) : (valid ? __ldcg(v.fl + i) : 0.0))
                                : 0.0;
      v.bm[i] = b;
      if (!moment_all && v.flip[i]) nzin[i] = 1;
    }
    __syncthreads();
    for (int i = tid; i < nx; i += nt) {
      v.kc[i] = v.kcn[i];
      v.ki[i] = v.kin[i];
    }
  } else {
    for (int i = tid; i < nx; i += nt) {
      v.bm[i] = __ldcg(v.fl + i);
      v.kc[i] = 1;
      v.ki[i] = 1;
    }
  }
  __syncthreads();
  // projection coefficient dc (kinetic.py:190-191) and the E-upwind factor
  // max(E,0)/dvx or min(E,0)/dvx (kinetic.py:177-178)
  int cnt = 0;
  const int per = (nx + nt - 1) / nt;
  const int lo = min(nx, tid * per), hi = min(nx, lo + per);
  for (int i = tid; i < nx; i += nt) {
    const double bn = __ldcg(v.bm + wrap(i + 1, nx));
    const double bp = __ldcg(v.bm + wrap(i - 1, nx));
    v.dco[i] = (bn - bp) / m.two_dx;
    const double e = __ldcg(v.E + i);
    v.vsg[i] = e > 0.0 ? 1 : (e < 0.0 ? -1 : 0);
    v.vco[i] = e / m.dvx;
  }
  // zero the output rows of interfaces that are not kinetic this step but may
  // hold data in the output buffer (kinetic->fluid transitions, hybrid.py:166)
  for (int i = warp; i < nx; i += nwarp) {
    if (!v.ki[i] && nzout[i]) {
      row_zero_store<T>(gout + (size_t)i * nv, lane, nv);
      if (lane == 0) nzout[i] = 0;
    }
  }
  // compacted kinetic-row list (order preserving)
  for (int i = lo; i < hi; ++i) cnt += v.ki[i] ? 1 : 0;
  int pre;
  const int total = block_excl_scan(cnt, &pre, sm.misc + 1);
  for (int i = lo; i < hi; ++i)
    if (v.ki[i]) v.klist[pre++] = i;
  if (tid == 0) *v.nk = total;
  __syncthreads();
  return true;
}

// Slice phase after step s: masked rho update and field.  Returns false on a
// solvability violation.  kc/ki are the labels the step ran with.
__device__ bool finish_step(const FineArgs& a, const SliceView& v, const Smem& sm, int ph,
                            int step) {
  const MeshDev& m = a.m;
  const int nx = m.nx;
  const int tid = threadIdx.x, nt = blockDim.x;
  const PhaseDev& P = a.ph[ph];
  const size_t o = (size_t)v.b * nx;
  const double cflu = P.cflu[v.b];
  for (int i = tid; i < nx; i += nt) {
    const int ip = wrap(i - 1, nx);
    const double rho = __ldcg(v.rho + i);
    double r;
    if (v.kc[i]) {
      const double fi = v.ki[i] ? __ldcg(v.fl + i) : 0.0;
      const double fp = v.ki[ip] ? __ldcg(v.fl + ip) : 0.0;
      const double ci = P.cmac[o + i], cp = P.cmac[o + ip];
      r = (ci == cp) ? rho - ci * (fi - fp) : rho - (ci * fi - cp * fp);
    } else {
      r = rho + cflu * (__ldcg(v.J + i) - __ldcg(v.J + ip));
    }
    v.tA[i] = r;
  }
  __syncthreads();
  for (int i = tid; i < nx; i += nt) v.rho[i] = v.tA[i];
  __syncthreads();
  if (!slice_field(m, v.rho, v.rb, v.tA, v.tB, a.rtol, a.exact_scan, sm)) {
    if (tid == 0) set_status(a.status, PK_ERR_SOLVABILITY, v.b, step);
    return false;
  }
  for (int i = tid; i < nx; i += nt) {
    v.Eprev[i] = v.E[i];
    v.E[i] = v.tB[i];
  }
  __syncthreads();
  return true;
}

// ---------------------------------------------------------------------------
// Micro phase: this warp's share of the kinetic rows of one step.
template <int T, int D>
__device__ void micro_phase(const FineArgs& a, const SliceView& v, const Smem& sm, int ph,
                            const double* gin, double* gout, int wg, int nwg) {
  const MeshDev& m = a.m;
  const int nx = m.nx, nv = m.nv;
  const int lane = threadIdx.x & 31;
  constexpr int S = Layout<T>::S;
  const int nk = __ldcg(v.nk);
  const bool dense = nk == nx;
  const int p0 = (int)(((long long)wg * nk) / nwg);
  const int p1 = (int)(((long long)(wg + 1) * nk) / nwg);
  if (p0 >= p1) return;
  const PhaseDev& P = a.ph[ph];
  const size_t o = (size_t)v.b * nx;
  double* wrow = sm.wrow + (threadIdx.x >> 5) * nv;
  FastConsts<T == 0 ? 2 : T> C;
  if constexpr (T != 0) C.load(sm.vx, sm.M, sm.xiM, lane);
  auto rowid = [&](int p) { return dense ? p : __ldcg(v.klist + p); };

  double gp[S], gc[S], gn[S];
  double pf[D][S];
  // prime the prefetch ring with rows list(p)+1
#pragma unroll
  for (int d = 0; d < D; ++d)
    if (p0 + d < p1) row_load<T>(pf[d], gin + (size_t)wrap(rowid(p0 + d) + 1, nx) * nv, lane, nv);
  int last = -2;
  for (int base = p0; base < p1; base += D) {
#pragma unroll
    for (int u = 0; u < D; ++u) {
      const int p = base + u;
      if (p < p1) {
        const int i = rowid(p);
        if (i == last + 1) {
#pragma unroll
          for (int s = 0; s < S; ++s) {
            gp[s] = gc[s];
            gc[s] = gn[s];
          }
        } else {
          row_load<T>(gp, gin + (size_t)wrap(i - 1, nx) * nv, lane, nv);
          row_load<T>(gc, gin + (size_t)i * nv, lane, nv);
        }
#pragma unroll
        for (int s = 0; s < S; ++s) gn[s] = pf[u][s];
        if (p + D < p1) row_load<T>(pf[u], gin + (size_t)wrap(rowid(p + D) + 1, nx) * nv, lane, nv);
        RowCoef rc;
        rc.vsg = __ldcg(v.vsg + i);
        rc.vco = __ldcg(v.vco + i);
        rc.dc = __ldcg(v.dco + i);
        rc.J = __ldcg(v.J + i);
        rc.k1 = P.k1[o + i];
        rc.k2 = P.k2[o + i];
        double out[S];
        if constexpr (T == 0)
          gen_micro(gp, gc, gn, out, sm.vx, sm.M, sm.xiM, rc, nv, m.dx, m.rdx, lane);
        else
          fast_micro<T>(gp, gc, gn, out, C, rc, m.dx, m.rdx, lane);
        row_store<T>(out, gout + (size_t)i * nv, lane, nv);
        double bx, bsq;
        row_moments<T>(out, sm, m, wrow, lane, bx, bsq);
        if (lane == 0) {
          v.fl[i] = bx;
          v.sq[i] = bsq;
        }
        last = i;
      }
    }
  }
}

// Prologue row pass: (optionally lift and) copy the input rows into the
// step-0 input buffer and compute their moments.
template <int T>
__device__ void prologue_rows(const FineArgs& a, const SliceView& v, const Smem& sm, double* gin0,
                              bool lift, int wg, int nwg) {
  const MeshDev& m = a.m;
  const int nx = m.nx, nv = m.nv;
  const int lane = threadIdx.x & 31;
  constexpr int S = Layout<T>::S;
  double* wrow = sm.wrow + (threadIdx.x >> 5) * nv;
  const int p0 = (int)(((long long)wg * nx) / nwg);
  const int p1 = (int)(((long long)(wg + 1) * nx) / nwg);
  for (int i = p0; i < p1; ++i) {
    double g[S];
    if (lift) {
      LiftRow L;
      const size_t o = (size_t)v.b * nx + i;
      L.negJ = a.neg_eps[o] * __ldcg(v.J + i);
      L.e2 = a.eps2[o];
      L.drift = __ldcg(v.tE + i);
      L.Rif = __ldcg(v.tA + i);
      row_lift<T>(g, L, a.lift_order, a.time_elim == 1, 1, sm, m, wrow, lane);
      row_store<T>(g, gin0 + (size_t)i * nv, lane, nv);
    } else {
      row_load<T>(g, v.ga + (size_t)i * nv, lane, nv);
      if (gin0 != v.ga) row_store<T>(g, gin0 + (size_t)i * nv, lane, nv);
    }
    double bx, bsq;
    row_moments<T>(g, sm, m, wrow, lane, bx, bsq);
    if (lane == 0) {
      v.fl[i] = bx;
      v.sq[i] = bsq;
    }
  }
}

// Window-start lift scalars (parareal.py:171-178: lift(rho_in, E) with
// dE_dt = None, i.e. dtE_c = 0).
__device__ bool lift_scalars(const FineArgs& a, const SliceView& v, const Smem& sm) {
  const MeshDev& m = a.m;
  const int nx = m.nx, tid = threadIdx.x, nt = blockDim.x;
  if (a.lift_order != 1 && a.lift_order != 2) return false;
  if (a.lift_order == 2 && a.time_elim != 0 && a.time_elim != 1) return false;
  for (int i = tid; i < nx; i += nt) {
    const int ip = wrap(i - 1, nx);
    v.tB[i] = 0.5 * (__ldcg(v.J + ip) + __ldcg(v.J + i));  // J_c
  }
  __syncthreads();
  const double three_rb = 3.0 * v.rb;
  for (int i = tid; i < nx; i += nt) {
    const double d1J = stencil_at(v.tB, i, nx, m, 1);
    v.tD[i] = d1J;
    if (a.lift_order == 2 && a.time_elim == 1) {
      const int ip = wrap(i - 1, nx);
      const double Ec = 0.5 * (__ldcg(v.E + ip) + __ldcg(v.E + i));
      const double d2J = stencil_at(v.tB, i, nx, m, 2);
      const double d3J = stencil_at(v.tB, i, nx, m, 3);
      const double d1r = stencil_at(v.rho, i, nx, m, 1);
      const double rho = __ldcg(v.rho + i);
      const double Jc = __ldcg(v.tB + i);
      const double dtEc = 0.0;
      v.tC[i] = -d3J + Ec * d2J + (2.0 * rho - three_rb) * d1J + 2.0 * Jc * d1r - d1r * dtEc;
    }
  }
  __syncthreads();
  for (int i = tid; i < nx; i += nt) {
    const int in_ = wrap(i + 1, nx);
    const double dJ = 0.5 * (__ldcg(v.tD + i) + __ldcg(v.tD + in_));
    v.tE[i] = dJ - __ldcg(v.E + i) * __ldcg(v.J + i);
    v.tA[i] = (a.lift_order == 2 && a.time_elim == 1) ? 0.5 * (__ldcg(v.tC + i) + __ldcg(v.tC + in_))
                                                     : 0.0;
  }
  __syncthreads();
  return true;
}

__device__ __forceinline__ void cluster_barrier(int C) {
  if (C > 1) {
    cg::this_cluster().sync();
  } else {
    __syncthreads();
  }
}

template <int T, int D>
__global__ void __launch_bounds__(256, 2) fine_kernel(const FineArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const MeshDev& m = a.m;
  const int nx = m.nx, nv = m.nv;
  int C = 1;
  int crank = 0;
  {
    cg::cluster_group cl = cg::this_cluster();
    C = (int)cl.num_blocks();
    crank = (int)cl.block_rank();
  }
  const int b = blockIdx.x / C;
  const bool leader = crank == 0;
  // shared memory carve-up
  Smem sm;
  {
    unsigned char* p = smem_raw;
    sm.plan = reinterpret_cast<PwPlan*>(p);
    p += (sizeof(PwPlan) + 15) / 16 * 16;
    sm.vx = reinterpret_cast<double*>(p); p += nv * 8;
    sm.M = reinterpret_cast<double*>(p); p += nv * 8;
    sm.xiM = reinterpret_cast<double*>(p); p += nv * 8;
    sm.w2 = reinterpret_cast<double*>(p); p += nv * 8;
    sm.red = reinterpret_cast<double*>(p); p += (MAX_LEAF + MAX_NODE) * 8;
    sm.wrow = reinterpret_cast<double*>(p); p += (blockDim.x >> 5) * nv * 8;
    sm.misc = reinterpret_cast<int*>(p);
  }
  {
    const int* src = reinterpret_cast<const int*>(m.plan_x);
    int* dst = reinterpret_cast<int*>(sm.plan);
    for (int i = threadIdx.x; i < (int)(sizeof(PwPlan) / 4); i += blockDim.x) dst[i] = src[i];
    for (int j = threadIdx.x; j < nv; j += blockDim.x) {
      sm.vx[j] = m.vx[j];
      sm.M[j] = m.M[j];
      sm.xiM[j] = m.xiM[j];
      sm.w2[j] = m.w2[j];
    }
  }
  __syncthreads();
  if (b >= a.B) return;  // never: grid is exactly B clusters

  const SliceView v = make_view(a, b);
  const int n0 = a.ph[0].nsteps[b], n1 = a.ph[1].nsteps[b];
  const int nst = n0 + n1;
  const int nwpc = blockDim.x >> 5;
  const int wg = crank * nwpc + (threadIdx.x >> 5);
  const int nwg = C * nwpc;
  const int initf = a.init_flags ? a.init_flags[b] : 0;
  const bool lift0 = (initf & 1) != 0;       // g := lift(rho, E)   (parareal.py:171-178)
  const bool eprev0 = (initf & 2) != 0;      // E_prev := E         (hybrid.py:68-72)
  // step s reads buf(s) and writes buf(s+1); the last output lands in ga.
  auto buf = [&](int s) { return ((s + (nst & 1)) & 1) ? v.gb : v.ga; };
  auto nzf = [&](int s) { return ((s + (nst & 1)) & 1) ? v.nzb : v.nza; };
  int* abort_flag = v.abort_;

  // ---- prologue ----
  if (leader) {
    for (int i = threadIdx.x; i < nx; i += blockDim.x) {
      v.nza[i] = 1;
      v.nzb[i] = 1;
    }
    if (threadIdx.x == 0) *abort_flag = 0;
    bool ok = slice_field(m, v.rho, v.rb, v.tA, v.E, a.rtol, a.exact_scan, sm);
    if (!ok) {
      if (threadIdx.x == 0) {
        set_status(a.status, PK_ERR_SOLVABILITY, b, 0);
        *abort_flag = 1;
      }
    } else {
      for (int i = threadIdx.x; i < nx; i += blockDim.x) {
        const int in_ = wrap(i + 1, nx);
        v.J[i] = flux_J(__ldcg(v.rho + i), __ldcg(v.rho + in_), __ldcg(v.E + i), m.dx);
      }
      __syncthreads();
      if (lift0 && !lift_scalars(a, v, sm)) {
        if (threadIdx.x == 0) {
          set_status(a.status, PK_ERR_BAD_LIFT, b, 0);
          *abort_flag = 1;
        }
      }
    }
    __syncthreads();
    if (eprev0 && !*abort_flag) {
      for (int i = threadIdx.x; i < nx; i += blockDim.x) v.Eprev[i] = v.E[i];
    }
  }
  cluster_barrier(C);
  if (__ldcg(abort_flag)) return;
  prologue_rows<T>(a, v, sm, buf(0), lift0, wg, nwg);
  cluster_barrier(C);
  if (leader) {
    const double dt0 = (n0 > 0 ? a.ph[0].dt : a.ph[1].dt)[b];
    if (!prepare_step<T>(a, v, sm, dt0, 1, buf(0), buf(1), nzf(0), nzf(1), 0)) {
      if (threadIdx.x == 0) *abort_flag = 1;
    }
  }
  cluster_barrier(C);
  if (__ldcg(abort_flag)) return;

  // ---- steps ----
  for (int s = 0; s < nst; ++s) {
    const int ph = s < n0 ? 0 : 1;
    micro_phase<T, D>(a, v, sm, ph, buf(s), buf(s + 1), wg, nwg);
    cluster_barrier(C);
    if (leader) {
      bool ok = finish_step(a, v, sm, ph, s);
      if (ok && s + 1 < nst) {
        // step s+1 reads buf(s+1) and writes buf(s+2) == buf(s); after step
        // s the rows of buf(s+1) hold data exactly on step s's kinetic rows.
        uint8_t* nzn = nzf(s + 1);
        for (int i = threadIdx.x; i < nx; i += blockDim.x) nzn[i] = v.ki[i];
        __syncthreads();
        const int phn = (s + 1) < n0 ? 0 : 1;
        ok = prepare_step<T>(a, v, sm, a.ph[phn].dt[b], 0, buf(s + 1), buf(s), nzn, nzf(s), s + 1);
      }
      if (!ok && threadIdx.x == 0) *abort_flag = 1;
    }
    cluster_barrier(C);
    if (__ldcg(abort_flag)) return;
  }
}

// ---------------------------------------------------------------------------
// Standalone operators: lift (lifting.py:38-105) and solve_field
// (poisson.py:21-54) over B slices, one CTA per slice.

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
    sm.vx = reinterpret_cast<double*>(p); p += nv * 8;
    sm.M = reinterpret_cast<double*>(p); p += nv * 8;
    sm.xiM = reinterpret_cast<double*>(p); p += nv * 8;
    sm.w2 = reinterpret_cast<double*>(p); p += nv * 8;
    sm.wrow = reinterpret_cast<double*>(p); p += (blockDim.x >> 5) * nv * 8;
    sm.red = nullptr;
    sm.misc = nullptr;
  }
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
  for (int i = tid; i < nx; i += nt)
    J[i] = flux_J(rho[i], rho[wrap(i + 1, nx)], E[i], m.dx);
  __syncthreads();
  const bool higher = a.order >= 2 && a.time_elim == 1;
  if (a.order >= 2) {
    for (int i = tid; i < nx; i += nt) Jc[i] = 0.5 * (__ldcg(J + wrap(i - 1, nx)) + __ldcg(J + i));
    __syncthreads();
    const double three_rb = 3.0 * a.rho_bar[b];
    for (int i = tid; i < nx; i += nt) {
      d1[i] = stencil_at(Jc, i, nx, m, 1);
      if (higher) {
        const int ip = wrap(i - 1, nx);
        const double Ec = 0.5 * (E[ip] + E[i]);
        const double dtEc = a.dE_dt ? 0.5 * (a.dE_dt[o + ip] + a.dE_dt[o + i]) : 0.0;
        const double d2J = stencil_at(Jc, i, nx, m, 2);
        const double d3J = stencil_at(Jc, i, nx, m, 3);
        const double d1r = stencil_at(rho, i, nx, m, 1);
        const double d1J = __ldcg(d1 + i);
        R[i] = -d3J + Ec * d2J + (2.0 * rho[i] - three_rb) * d1J + 2.0 * __ldcg(Jc + i) * d1r -
               d1r * dtEc;
      }
    }
    __syncthreads();
    for (int i = tid; i < nx; i += nt) {
      const int in_ = wrap(i + 1, nx);
      const double dJ = 0.5 * (__ldcg(d1 + i) + __ldcg(d1 + in_));
      drift[i] = dJ - E[i] * __ldcg(J + i);
      Rif[i] = higher ? 0.5 * (__ldcg(R + i) + __ldcg(R + in_)) : 0.0;
    }
  }
  __syncthreads();
  const int nwarp = nt >> 5;
  double* wrow = sm.wrow + warp * nv;
  for (int i = warp; i < nx; i += nwarp) {
    LiftRow L;
    L.negJ = a.neg_eps[o + i] * __ldcg(J + i);
    L.e2 = a.eps2[o + i];
    L.drift = a.order >= 2 ? __ldcg(drift + i) : 0.0;
    L.Rif = a.order >= 2 ? __ldcg(Rif + i) : 0.0;
    double g[Layout<T>::S];
    row_lift<T>(g, L, a.order, higher, a.project, sm, m, wrow, lane);
    row_store<T>(g, a.g_out + (o + i) * nv, lane, nv);
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
                   a.exact_scan, sm)) {
    if (threadIdx.x == 0) set_status(a.status, PK_ERR_SOLVABILITY, blockIdx.x, 0);
  }
}

// ---------------------------------------------------------------------------
// Host-side launch.

size_t fine_smem_bytes(int nv, int threads) {
  return (sizeof(PwPlan) + 15) / 16 * 16 + 4 * nv * 8 + (MAX_LEAF + MAX_NODE) * 8 +
         (threads / 32) * nv * 8 + 64 * 4;
}

template <int T, int D>
static cudaError_t launch_T(const FineArgs& a, int C, cudaStream_t st) {
  const int threads = 256;
  const size_t smem = fine_smem_bytes(a.m.nv, threads);
  auto kern = fine_kernel<T, D>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (C > 8) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(a.B * C);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, a);
}

template <int T>
static cudaError_t launch_lift_T(const LiftArgs& a, cudaStream_t st) {
  const int threads = 256;
  const size_t smem = 4 * a.m.nv * 8 + (threads / 32) * a.m.nv * 8;
  cudaError_t e =
      cudaFuncSetAttribute(lift_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  lift_kernel<T><<<a.B, threads, smem, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_lift(const LiftArgs& a, cudaStream_t st) {
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

cudaError_t launch_field(const FieldArgs& a, cudaStream_t st) {
  const size_t smem = (sizeof(PwPlan) + 15) / 16 * 16 + (MAX_LEAF + MAX_NODE) * 8;
  cudaError_t e =
      cudaFuncSetAttribute(field_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  field_kernel<<<a.B, 256, smem, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_fine(const FineArgs& a, int C, cudaStream_t st) {
  switch (a.m.nv) {
    case 64: return launch_T<2, 4>(a, C, st);
    case 128: return launch_T<4, 3>(a, C, st);
    case 256: return launch_T<8, 2>(a, C, st);
    case 512: return launch_T<16, 1>(a, C, st);
    default:
      if (a.m.nv <= 32 * GT) return launch_T<0, 1>(a, C, st);
      return cudaErrorInvalidValue;
  }
}

}  // namespace pk
