// Rows too long for one warp's registers: 1D-3V grids beyond 256 velocity
// nodes (the reference's default grid, nvx x nvy x nvz = 32 x 16 x 16, has
// 8192 per interface).  One warp per row; the row stays in global memory
// (L1/L2-resident while the warp works on it), velocity constants are read
// from global, and the brackets run a host-built pairwise plan over the folded
// row: the folded block of (nvx/2) * nvy * nvz terms in memory order and, for
// odd nvx, the middle xi plane's nvy * nvz terms (mesh.py:95-133; numpy
// reduces trailing contiguous axes as one flattened pairwise sum).  Same
// operations, in the same order, as the generic layout (pk_rows.cuh).
#pragma once

#include "pk_args.h"
#include "pk_rows.cuh"

namespace pk {

constexpr int BIG_SCR = MAX_LEAF + MAX_NODE;  // per-warp plan scratch (doubles)

// Pairwise sum of x(0 .. P.n) following plan P, by one warp: 8-lane groups
// take the leaves four at a time, lanes take the nodes of each level.
// `scr`: this warp's shared scratch, >= nleaf + nnode doubles.
template <class F>
__device__ double warp_plan_sum(F x, const PwPlan& P, double* scr) {
  const int lane = threadIdx.x & 31;
  const int nleaf = P.nleaf, nnode = P.nnode;
  for (int l0 = 0; l0 < nleaf; l0 += 4) {
    const int l = l0 + (lane >> 3);
    const bool act = l < nleaf;
    const double v = group_leaf(x, act ? P.leaf_off[l] : 0, act ? P.leaf_len[l] : 0, act);
    if (act && (lane & 7) == 0) scr[l] = v;
  }
  __syncwarp();
  int start = 0;
  for (int lev = 0; lev < P.nlevel; ++lev) {
    const int end = P.level_end[lev];
    for (int j = start + lane; j < end; j += 32)
      scr[nleaf + j] = scr[P.node_a[j]] + scr[P.node_b[j]];
    __syncwarp();
    start = end;
  }
  const double r = scr[nnode == 0 ? 0 : nleaf + nnode - 1];
  __syncwarp();
  return r;
}

// <q> of a row given element access q(c), c in [0, nv).
template <class Q>
__device__ double big_bracket(Q q, const MeshDev& m, double* scr) {
  const int S = m.nvyz, nvx = m.nv / S, F = (nvx / 2) * S;
  double tot = warp_plan_sum(
      [&](int j) {
        const int jx = j / S;
        return q(j) + q((nvx - 1 - jx) * S + (j - jx * S));
      },
      *m.plan_f, scr);
  if (nvx & 1) tot = tot + warp_plan_sum([&](int j) { return q(F + j); }, *m.plan_s, scr);
  return tot * m.dv3;
}

// One kinetic micro step of row i (kinetic.py:148-224, generic-layout order):
// gp/gc/gn the rows i-1, i, i+1 of the input buffer, out the output row.
__device__ __forceinline__ void big_micro_row(const double* gp, const double* gc, const double* gn,
                                              double* out, const MeshDev& m, const RowCoef& rc,
                                              int lane) {
  const int nv = m.nv, S = m.nvyz;
  const double Ep = rc.vsg > 0 ? rc.vco : 0.0;
  const double Em = rc.vsg < 0 ? rc.vco : 0.0;
  for (int c = lane; c < nv; c += 32) {
    const double xi = m.vx[c];
    const double xp = xi > 0.0 ? xi : 0.0;
    const double xm = xi < 0.0 ? xi : 0.0;
    const double g = __ldcg(gc + c);
    double o = xp * (g - __ldcg(gp + c));
    o = o + xm * (__ldcg(gn + c) - g);
    o = qdiv(o, m.dx, m.rdx);
    const double dm = (c < S) ? g : g - __ldcg(gc + c - S);
    o = o + dm * Ep;
    const double dp = (c >= nv - S) ? -g : __ldcg(gc + c + S) - g;
    o = o + dp * Em;
    o = o - m.M[c] * rc.dc;
    const double forcing = o + m.xiM[c] * rc.J;
    __stcg(out + c, rc.k1 * g - rc.k2 * forcing);
  }
  __syncwarp();
}

// Row moments <xi g> and (when sq) <g^2> of a row in global memory.
__device__ __forceinline__ void big_row_moments(const double* row, const MeshDev& m, double* scr,
                                                bool sq, double& bx, double& bsq) {
  bx = big_bracket([&](int c) { return m.vx[c] * __ldcg(row + c); }, m, scr);
  bsq = 0.0;
  if (sq)
    bsq = big_bracket(
        [&](int c) {
          const double g = __ldcg(row + c);
          return g * g;
        },
        m, scr);
}

// lifting.py:63-105 for one row, written into dst: g = xi M (-eps J)
// [+ (eps^2 w) drift] [+ (eps^2 M) R_if]; two zero-mass projections.
static __device__ void big_row_lift(double* dst, const LiftRow& L, int order, int higher, int project,
                             const MeshDev& m, double* scr, int lane) {
  const int nv = m.nv;
  for (int c = lane; c < nv; c += 32) {
    double v = m.xiM[c] * L.negJ;
    if (order >= 2) {
      v = v + (L.e2 * m.w2[c]) * L.drift;
      if (higher) v = v + (L.e2 * m.M[c]) * L.Rif;
    }
    __stcg(dst + c, v);
  }
  __syncwarp();
  if (project) {
    for (int pass = 0; pass < 2; ++pass) {
      const double bb = big_bracket([&](int c) { return __ldcg(dst + c); }, m, scr) / m.m0;
      for (int c = lane; c < nv; c += 32) __stcg(dst + c, __ldcg(dst + c) - bb * m.M[c]);
      __syncwarp();
    }
  }
}

__device__ __forceinline__ void big_row_copy(const double* src, double* dst, int nv, int lane) {
  for (int c = lane; c < nv; c += 32) __stcg(dst + c, __ldcg(src + c));
  __syncwarp();
}

__device__ __forceinline__ void big_row_zero(double* dst, int nv, int lane) {
  for (int c = lane; c < nv; c += 32) __stcg(dst + c, 0.0);
  __syncwarp();
}

}  // namespace pk
