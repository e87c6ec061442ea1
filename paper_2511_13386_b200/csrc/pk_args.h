// Kernel argument blocks (host <-> device), internal to libpk.
#pragma once

#include <stdint.h>

#include "pk_device.cuh"

namespace pk {

// Velocity-grid constants uploaded once per context (host numpy values,
// uploaded verbatim: mesh.py:167,211-235; lifting.py:88).
struct MeshDev {
  int nx, nv;
  int nvyz;            // nvy * nvz: stride of the xi axis within a row (1: 1D-x/1D-v)
  int xplane;          // xi constant on each xi plane: vx[c] == vx[(c / nvyz) nvyz] bit for bit
  int mirror;          // vx[nv-1-j] == -vx[j], M[nv-1-j] == M[j] and xiM[j] == vx[j]*M[j]
                       // bit for bit (the reference's mirrored grid, mesh.py:31-44,136)
  double dx, rdx, two_dx, dvx, dv3, m0, m2;
  double rtwo_dx, rdvx;  // RN(1 / (2 dx)), RN(1 / dvx): qdiv's reciprocals
  int stc_std;         // the stencil table has the reference's zero pattern (only
                       // orders 1 and 3 have a zero, at offset 0): skip statically
  double three_rb_unused;
  const double* vx;    // [nv] velocity centres xi_j
  const double* M;     // [nv] discrete Maxwellian
  const double* xiM;   // [nv] xi_j * M_j
  const double* w2;    // [nv] (xi_j^2 - 1) * M_j
  double stc[4][7];    // 7-point stencil coefficients, offsets -3..3 (adaptation.py:29-34)
  double sts[4];       // dx ** (-order)
  const PwPlan* plan_x;  // pairwise plan for nx-term reductions
  const PwPlan* plan_f;  // folded velocity row ((nvx/2) * nvyz terms)   (big rows)
  const PwPlan* plan_s;  // middle xi plane (nvyz terms, odd nvx)        (big rows)
};

// One run of identical steps, per slice.
struct PhaseDev {
  const int* nsteps;    // [B]
  const double* dt;     // [B]
  const double* cflu;   // [B]   m2 * (dt / dx)            (fluid.py:57)
  const double* k1;     // [B*nx] exp(-dt/eps_i^2)          (kinetic.py:141-145)
  const double* k2;     // [B*nx] eps_i * -expm1(-dt/eps_i^2)
  const double* cmac;   // [B*nx] dt / (eps_i * dx)         (kinetic.py:240)
  const double* cmacs;  // [B] the common value when uniform in x, else NaN
  const double* k1s;    // [B] likewise for k1 (or null)
  const double* k2s;    // [B] likewise for k2 (or null)
};

struct FineArgs {
  MeshDev m;
  int B;
  int nwarp_total;       // warps per slice (cluster CTAs x warps per CTA)
  int kps;               // slices per cluster (set by the launcher; 1 unless all-kinetic)
  int sg;                // > 1: the "cluster" is a software group of sg CTAs (no hardware
                         // cluster; moments through global memory, barriers on sg_cnt)
  unsigned* sg_cnt;      // [B] per-group arrival counters (zeroed by the launcher)
  int bigc;              // big rows, one CTA per row through shared-memory row buffers (launcher)
  const int* cancel;     // host cancel request (pk_fine_cancel): the slice owners abort at the next step
  int pass_prepare;      // hybrid slice phase of one CTA: the pass-by-pass form instead of
                         // prepare_step_cta (A/B switch PK_PASS_PREPARE=1)
  // state
  double* rho;           // [B*nx] in/out
  double* E;             // [B*nx] out: field at the end (also working E)
  double* Eprev;         // [B*nx] in/out
  uint8_t* kc;           // [B*nx] in/out kinetic cells
  uint8_t* ki;           // [B*nx] in/out kinetic interfaces
  double* ga;            // [B*nx*nv] in/out (result always lands here)
  double* gb;            // [B*nx*nv] scratch
  const double* rho_bar; // [B]
  const uint8_t* init_flags; // [B] bit0: g := lift(rho, E) at entry (parareal.py:171-178)
                             //     bit1: E_prev := E at entry (HybridState.initial)
  // schedule
  PhaseDev ph[2];
  // hybrid options (hybrid.py:45-55)
  int adaptation, combine_and, reinit, lift_order, time_elim, exact_scan;
  int local_smem;         // leader slice vectors in shared memory (set by the launcher)
  int scan_smem;          // else: doubles of the field scan buffer in shared memory (launcher)
  double delta0, eta0, rtol;
  const double* rscale;  // [B*nx] eps_c^2 for scale_remainder, or null
  const double* neg_eps; // [B*nx] -eps_i
  const double* eps2;    // [B*nx] eps_i^2
  // workspace [B*nx] unless noted
  double *J, *fl, *sq, *bm, *dco, *vco, *tA, *tB, *tC, *tD, *tE, *blift, *lJ;
  int8_t* vsg;
  uint8_t *flip, *nza, *nzb, *kcn, *kin;
  int* klist;
  int* kpos;             // [B*nx] row-stream end after each listed row
  int* kstream;          // [B*3nx] row id of each row-stream position
  int* nk;               // [B]
  int* zlist;            // [B*nx] rows the next micro phase zeroes in its output buffer
  int* nzl;              // [B] their count
  int* abort_;           // [B]
  Status* status;
  long long* prof;       // [6] optional phase profile (pk_debug_profile), or null
  long long* rowcnt;     // [2B] optional per-slice row counters (pk_count_rows), or null
};

struct LiftArgs {
  MeshDev m;
  int B, order, time_elim, project;
  const double* rho;      // [B*nx]
  const double* E;        // [B*nx]
  const double* dE_dt;    // [B*nx] or null
  const double* rho_bar;  // [B]
  const double* neg_eps;  // [B*nx]
  const double* eps2;     // [B*nx]
  double* g_out;          // [B*nx*nv]
  double *J, *tA, *tB, *tC, *tD, *tE;  // workspace [B*nx]
};

// Standalone adaptation indicators (adaptation.py:120-181), one CTA per slice.
struct IndArgs {
  MeshDev m;
  int B;
  const double* rho;      // [B*nx]           remainder
  const double* E;        // [B*nx]
  const double* E_prev;   // [B*nx] or null   (E - E_prev) / dt ...
  const double* dtE_c;    // [B*nx] or null   ... or this cell-centred dE/dt
  double dt;
  const double* rho_bar;  // [B]
  double* R;              // [B*nx] out
  const double* g;        // [B*nx*nv]        perturbation norm
  double* gnorm;          // [B*nx] out
  const double* Rin;      // [B*nx]           labels from (R, gnorm)
  const double* gin;      // [B*nx]
  double delta0, eta0;
  int combine_and;
  uint8_t *kc, *ki;       // [B*nx] out
};

struct FieldArgs {
  MeshDev m;
  int B, exact_scan;
  const double* rho;
  const double* rho_bar;
  double* E;
  double* src;            // workspace [B*nx]
  double rtol;
  Status* status;
};

// Coarse drift-diffusion chains (fluid.py:95-118; parareal.py:210-229,276-281).
// Chain c runs windows w = 0..W-1: in = (w == 0 ? rho_in[c] : out[c][w-1]);
// G[c][w] = G(in); out[c][w] = G[c][w] (+ delta[c][w] when delta != null).
struct ChainArgs {
  MeshDev m;
  int nchain, nwin;
  const double* rho_in;  // [nchain*nx]
  const double* E_in;    // [nchain*nx] field of rho_in for window 0, or null (recompute)
  double* gout;          // [nchain*nwin*nx] pure G results (may be null)
  double* out;           // [nchain*nwin*nx]
  double* Eout;          // [nchain*nx] field after the last window (may be null)
  const double* delta;   // [nchain*nwin*nx] or null
  const int* nfull;      // [nchain*nwin]
  const double* rem;     // [nchain*nwin] clipped last step (0: none)
  const double* cflu_full;  // [nchain*nwin]
  const double* cflu_rem;   // [nchain*nwin]
  double dt_full;           // FluidStepParams.dt (stability checked on the host)
  const double* rho_bar;    // [nchain]
  double rtol;
  int exact_scan;
  Status* status;
};

}  // namespace pk
