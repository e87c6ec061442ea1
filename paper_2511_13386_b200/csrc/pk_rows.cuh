// Row-level (one warp per interface row g[i, 0..nv)) device math shared by
// the fine-propagator and lift kernels: register layouts, the folded
// pairwise velocity bracket, the micro update and the Chapman-Enskog row.
#pragma once

#include "pk_args.h"

namespace pk {

// Per-CTA shared-memory velocity constants and scratch.
struct Smem {
  double* vx;
  double* M;
  double* xiM;
  double* w2;
  PwPlan* plan;
  double* red;    // pairwise scratch (2 (MAX_LEAF + MAX_NODE))
  double* wrow;   // generic rows: one nv-row per warp
  int* misc;      // small ints
  double* scan = nullptr;   // field scan buffer (global-memory slice vectors), or null
  int scan_cap = 0;         // its capacity in doubles (chunks of it when < nx)
};

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
// fold and the pairwise sum go through a per-warp shared-memory row.  A row is
// (nvx, nvy, nvz) in C order; S = nvy * nvz is the stride of the xi axis
// (S = 1: the 1D-x/1D-v reduction).
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

// <q>: fold the xi mirror pairs (jx, nvx-1-jx) of every (vy, vz) column, one
// pairwise sum over the folded (nvx/2, nvy, nvz) block in memory order, plus
// the middle xi plane's own pairwise sum for odd nvx (mesh.py:95-133; numpy
// reduces the trailing contiguous axes as one flattened pairwise sum).  The
// folded block has nv/2 <= 128 terms: one leaf.
__device__ __forceinline__ double gen_bracket(const double (&q)[GT], double* wrow, int lane,
                                              int nv, int S, double dv3) {
#pragma unroll
  for (int s = 0; s < GT; ++s) {
    const int c = 32 * s + lane;
    if (c < nv) wrow[c] = q[s];
  }
  __syncwarp();
  const int nvx = nv / S, h = nvx / 2, F = h * S;
  // the middle plane [F, F + S) is never overwritten below
  const double mid = (nvx & 1) ? warp_leaf([&](int j) { return wrow[j]; }, F, S, lane) : 0.0;
  double f[GT];
#pragma unroll
  for (int s = 0; s < GT; ++s) {
    const int j = 32 * s + lane;
    const int jx = j / S;
    f[s] = j < F ? wrow[j] + wrow[(nvx - 1 - jx) * S + (j - jx * S)] : 0.0;
  }
  __syncwarp();
#pragma unroll
  for (int s = 0; s < GT; ++s) {
    const int j = 32 * s + lane;
    if (j < F) wrow[j] = f[s];
  }
  __syncwarp();
  double tot = warp_leaf([&](int j) { return wrow[j]; }, 0, F, lane);
  if (nvx & 1) tot = tot + mid;
  __syncwarp();
  return tot * dv3;
}

__device__ __forceinline__ void gen_micro(const double (&gp)[GT], const double (&gc)[GT],
                                          const double (&gn)[GT], double (&out)[GT],
                                          const double* svx, const double* sM, const double* sxiM,
                                          const RowCoef& rc, int nv, int S, double* wrow,
                                          double dx, double rdx, int lane) {
  // xi neighbours (c - S, c + S); edge planes have zero inflow (kinetic.py:176-187)
  double lfix[GT], rfix[GT];
  if (S == 1) {  // neighbouring lanes: shuffles
    double left[GT], right[GT];
#pragma unroll
    for (int s = 0; s < GT; ++s) {
      left[s] = __shfl_sync(FULL, gc[s], (lane + 31) & 31);
      right[s] = __shfl_sync(FULL, gc[s], (lane + 1) & 31);
    }
#pragma unroll
    for (int s = 0; s < GT; ++s) {
      // column c-1 for lane 0 is lane 31 of slot s-1; column c+1 for lane 31 is lane 0 of slot s+1
      lfix[s] = lane >= 1 ? left[s] : (s >= 1 ? left[s >= 1 ? s - 1 : 0] : 0.0);
      rfix[s] = lane <= 30 ? right[s] : (s + 1 < GT ? right[s + 1 < GT ? s + 1 : 0] : 0.0);
    }
  } else {  // 1D-3V: through the warp's shared row
#pragma unroll
    for (int s = 0; s < GT; ++s) {
      const int c = 32 * s + lane;
      if (c < nv) wrow[c] = gc[s];
    }
    __syncwarp();
#pragma unroll
    for (int s = 0; s < GT; ++s) {
      const int c = 32 * s + lane;
      lfix[s] = c >= S && c < nv ? wrow[c - S] : 0.0;
      rfix[s] = c + S < nv ? wrow[c + S] : 0.0;
    }
    __syncwarp();
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
    const double dm = (c < S) ? g : g - lfix[s];
    o = o + dm * Ep;
    const double dp = (c >= nv - S) ? -g : rfix[s] - g;
    o = o + dp * Em;
    o = o - sM[c] * rc.dc;
    const double forcing = o + sxiM[c] * rc.J;
    out[s] = rc.k1 * g - rc.k2 * forcing;
  }
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

static __device__ void gen_lift_row(double (&g)[GT], const LiftRow& L, int order, int higher, int project,
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
      const double bb = gen_bracket(g, wrow, lane, nv, m.nvyz, m.dv3) / m.m0;
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

__device__ __forceinline__ void gen_moments(const double (&g)[GT], const Smem& sm, int nv, int S,
                                            double dv3, double* wrow, int lane, double& bx,
                                            double& bsq) {
  double q[GT], r[GT];
#pragma unroll
  for (int s = 0; s < GT; ++s) {
    const int c = 32 * s + lane;
    q[s] = c < nv ? sm.vx[c] * g[s] : 0.0;
    r[s] = g[s] * g[s];
  }
  bx = gen_bracket(q, wrow, lane, nv, S, dv3);
  bsq = gen_bracket(r, wrow, lane, nv, S, dv3);
}

// Layout dispatch: T == 0 selects the generic layout, T < 0 the big-row
// layout (pk_big.cuh: the row stays in global memory; callers branch on it).
template <int T>
struct Layout {
  static constexpr int S = T == 0 ? GT : (T < 0 ? 1 : T);
};

template <int T>
__device__ __forceinline__ void row_load(double (&v)[Layout<T>::S], const double* row, int lane,
                                         int nv) {
  if constexpr (T < 0) return;  // big rows: the callers work on global rows (pk_big.cuh)
  else if constexpr (T == 0) gen_load(v, row, lane, nv);
  else fast_load<T>(v, row, lane);
}

template <int T>
__device__ __forceinline__ void row_store(const double (&v)[Layout<T>::S], double* row, int lane,
                                          int nv) {
  if constexpr (T < 0) return;
  else if constexpr (T == 0) gen_store(v, row, lane, nv);
  else fast_store<T>(v, row, lane);
}

template <int T>
__device__ __forceinline__ void row_zero_store(double* row, int lane, int nv) {
  if constexpr (T < 0) {
    for (int c = lane; c < nv; c += 32) __stcg(row + c, 0.0);
    __syncwarp();
  } else {
    double z[Layout<T>::S];
#pragma unroll
    for (int s = 0; s < Layout<T>::S; ++s) z[s] = 0.0;
    row_store<T>(z, row, lane, nv);
  }
}

template <int T>
__device__ __forceinline__ void row_moments(const double (&g)[Layout<T>::S], const Smem& sm,
                                            const MeshDev& m, double* wrow, int lane, double& bx,
                                            double& bsq) {
  if constexpr (T < 0) return;
  else if constexpr (T == 0) gen_moments(g, sm, m.nv, m.nvyz, m.dv3, wrow, lane, bx, bsq);
  else fast_moments<T>(g, sm, m.dv3, lane, bx, bsq);
}

template <int T>
__device__ __forceinline__ void row_lift(double (&g)[Layout<T>::S], const LiftRow& L, int order,
                                         int higher, int project, const Smem& sm,
                                         const MeshDev& m, double* wrow, int lane) {
  if constexpr (T < 0) return;
  else if constexpr (T == 0) gen_lift_row(g, L, order, higher, project, sm, m, wrow, lane);
  else fast_lift_row<T>(g, L, order, higher, project, sm, m, lane);
}

}  // namespace pk
