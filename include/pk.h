/* libpk — B200 (sm_100a) fine/coarse propagators of the space-time hybrid
 * parareal method (arxiv 2511.13386), C ABI.
 *
 * The reference (/root/reference/pkg/src/parakin) is pure Python; it has no
 * FFI.  Its plugin seam for the fine propagator is the module attribute
 * parakin.parareal._fine_window (parareal.py:153-190), monkeypatched by its
 * own tests (tests/test_parareal.py:54-61,124-128), and its public operator
 * API is re-exported by parakin/__init__.py:5-54.  Each entry point below
 * replaces one of those Python operators; the Python drop-in package
 * paper_2511_13386_b200 binds them through ctypes.
 *
 * Conventions
 *  - All array pointers are caller-owned, C-contiguous fp64 (uint8 for
 *    labels) DEVICE memory on the context's device; host pointers are marked.
 *  - Calls are stream-ordered on `stream` (a cudaStream_t, or NULL for the
 *    legacy default stream) and asynchronous: errors detected on the device
 *    are latched in a status record read by pk_status_read().
 *  - A context is not thread-safe: one per (process, device).  Scratch is
 *    owned by the context and grown only by pk_reserve(), never in the hot
 *    loop.
 *  - Return value: PK_OK or a PK_ERR_* code (host-side validation / launch).
 */
#ifndef PK_H
#define PK_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* error taxonomy, mapped by the Python layer onto errors.py:4-26 */
#define PK_OK 0
#define PK_ERR_SOLVABILITY 1   /* SolvabilityViolation (poisson.py:39-48) */
#define PK_ERR_NONFINITE 2     /* NonFiniteState (parareal.py:267-269,283-284) */
#define PK_ERR_STABILITY 3     /* StabilityViolation (fluid.py:40-46, kinetic.py:77-88) */
#define PK_ERR_MESH_TOO_SMALL 4/* MeshTooSmall (mesh.py:58-65) */
#define PK_ERR_BAD_ARG 5       /* ValueError */
#define PK_ERR_CUDA 6          /* CUDA runtime failure */
#define PK_ERR_BAD_REINIT 7    /* ValueError: invalid reinit on a flip (hybrid.py:162-165) */
#define PK_ERR_BAD_LIFT 8      /* ValueError: invalid lift order / time_elim (lifting.py:57-85) */
#define PK_ERR_UNSUPPORTED 9   /* grid shape not supported by this build */

typedef struct pk_ctx pk_ctx;

/* Phase-space mesh, 1D-x / 1D-v (nvy = nvz = 1).  The velocity
 * arrays are HOST pointers holding the reference's own build_mesh values
 * (mesh.py:197-236), uploaded verbatim. */
typedef struct pk_mesh {
  int32_t nx, nv;        /* nv: velocity nodes per interface row, nvx * nvy * nvz */
  double dx, dvx, dv3, m0, m2, x_star, v_star;
  const double* vx;      /* host [nv]  xi of every node of the row (vx[jx] repeated nvy*nvz times) */
  const double* M;       /* host [nv] */
  const double* xi_M;    /* host [nv]  vx * M            (mesh.py:167) */
  const double* w2;      /* host [nv]  (vx**2 - 1) * M   (lifting.py:88) */
  double stencil[4][7];  /* adaptation.py:29-34, as Python floats */
  double stencil_scale[4]; /* dx ** -order (adaptation.py:51) */
  int32_t nvyz;          /* nvy * nvz: stride of the xi axis in a row (1: 1D-x/1D-v) */
} pk_mesh;

/* One run of identical steps.  Device arrays, per slice b (and per
 * interface i for the relaxation coefficients, so eps may vary in x). */
typedef struct pk_phase {
  const int32_t* nsteps; /* [B] */
  const double* dt;      /* [B] */
  const double* cflu;    /* [B]     m2 * (dt / dx)                  fluid.py:57 */
  const double* kappa1;  /* [B*nx]  exp(-dt/eps_i**2)               kinetic.py:141-145 */
  const double* kappa2;  /* [B*nx]  eps_i * -expm1(-dt/eps_i**2) */
  const double* cmac;    /* [B*nx]  dt / (eps_i * dx)               kinetic.py:240 */
  const double* cmac_scalar; /* [B] cmac when uniform in x (constant eps), else NaN */
  const double* kappa1_scalar; /* [B] kappa1 when uniform in x, else NaN (or NULL) */
  const double* kappa2_scalar; /* [B] kappa2 when uniform in x, else NaN (or NULL) */
} pk_phase;

/* Hybrid options (hybrid.py:45-55) and thresholds (adaptation.py:80-90). */
typedef struct pk_hybrid {
  int32_t adaptation;    /* 0: all-kinetic (kinetic_step semantics) */
  int32_t combine_and;   /* 0: "or", 1: "and" */
  int32_t reinit;        /* 0: "lift", 1: "zero", 2: invalid (raises on first flip) */
  int32_t lift_order;    /* 1 or 2 (anything else raises when the lift runs) */
  int32_t time_elim;     /* 0: "leading", 1: "higher_order", 2: invalid */
  int32_t exact_scan;    /* 1: np.cumsum order (bitwise); 0: parallel scan */
  double delta0, eta0;
  const double* rscale;  /* [B*nx] eps_c**2 per cell when scale_remainder, else NULL */
  const double* neg_eps; /* [B*nx] -eps_i  (lift)   */
  const double* eps2;    /* [B*nx] eps_i**2 (lift)  */
} pk_hybrid;

typedef struct pk_status {
  int32_t code, slice, step, pad;
} pk_status;

/* --- context ------------------------------------------------------------ */
pk_ctx* pk_create(int32_t device, const pk_mesh* mesh);           /* NULL on failure */
void pk_destroy(pk_ctx* ctx);
const char* pk_last_error(const pk_ctx* ctx);
int32_t pk_reserve(pk_ctx* ctx, int32_t max_slices);              /* grow scratch */
int32_t pk_status_read(pk_ctx* ctx, pk_status* out, int32_t clear); /* synchronises */
/* Same record, ordered on `stream` only (waits for the work queued on that
   stream, not for the whole device): for contexts driven from several streams. */
int32_t pk_status_read_stream(pk_ctx* ctx, pk_status* out, int32_t clear, void* stream);
/* The same record as two doubles in DEVICE memory, dst[0] = code (0: ok),
   dst[1] = step, stream-ordered without a host synchronisation (the
   multi-rank engine ships a window's status inside its jump's collective);
   clear != 0 re-arms the record. */
int32_t pk_status_store(pk_ctx* ctx, double* dst, int32_t clear, void* stream);
int32_t pk_version(void);
/* diagnostics: accumulate clock64 counters into a device array of
 * 32 + 3 * 1024 int64: [0..5] slice 0's [micro, barrier, slice finish, slice
 * prepare, barrier, steps], [6..31] slice-phase sub-timers and counts,
 * [32 + 3c ..] CTA c's [micro, first-barrier wait, SM id]; NULL disables. */
int32_t pk_debug_profile(pk_ctx* ctx, void* dev_counters);
/* measurement: accumulate, per slice b of every following pk_fine_propagate
 * launch, the interface rows the micro phases streamed (kinetic rows, all
 * steps) at dev_counts[2b] and the rows zeroed (kinetic->fluid) at
 * dev_counts[2b+1] (device int64 [2B]); NULL disables.  The hybrid roofline's
 * algorithmic bytes are 16 B x nv x rows + 8 B x nv x zeroed rows. */
int32_t pk_count_rows(pk_ctx* ctx, void* dev_counts);
/* diagnostics: how the calling thread's last pk_fine_propagate launch was
 * laid out: out[0] CTAs per thread-block cluster (or software group), out[1]
 * slices per cluster, out[2] 1 when the slice vectors were kept in shared
 * memory, out[3] 1 when the group was a software group (cooperative launch,
 * moments through global memory) rather than a hardware cluster, 2 when big
 * 1D-3V rows ran one CTA per row in hardware clusters, 3 when they ran one
 * CTA per row in software groups. */
int32_t pk_fine_last_launch(pk_ctx* ctx, int32_t out[4]);

/* --- fine propagator F --------------------------------------------------
 * B independent slices, each advanced through phases[0] then phases[1]
 * (the reference's n_full steps of dt then the clipped remainder,
 * fluid.py:80-92).  Replaces:
 *   hybrid_propagate  (hybrid.py:191-226)   adaptation on/off
 *   kinetic_propagate (kinetic.py:276-298)  = adaptation off (bitwise, F17)
 *   _fine_window      (parareal.py:153-190) with init_flags[b] = 3 for n >= 2 (lift + E_prev:=E), 2 for n = 1
 * rho, E_prev, kc, ki are read and written; E is written (the field after
 * the last step); g_a holds g on entry and on exit (g_b is scratch of the
 * same size). */
/* Ask the fine launch in flight on `ctx` to stop: its slices return at their
 * next step without writing results (the status record stays as it is).
 * Stream-ordered on `stream`, which must NOT be the stream of that launch
 * (it is busy with it); the request is cleared, in stream order, by the next
 * pk_fine_propagate on this context.  For speculative work that is no longer
 * needed (the overlapped parareal schedule starts the next iteration's windows
 * before convergence is known; the reference has no counterpart).  Slices run
 * as one hardware cluster each honour it; packed ensembles ignore it. */
int32_t pk_fine_cancel(pk_ctx* ctx, void* stream);

int32_t pk_fine_propagate(pk_ctx* ctx, int32_t B,
                          double* rho, double* E, double* E_prev,
                          uint8_t* kc, uint8_t* ki,
                          double* g_a, double* g_b,
                          const double* rho_bar, const uint8_t* init_flags /* [B] bit0 lift g, bit1 E_prev:=E */,
                          const pk_phase* phases /* host [2] */,
                          const pk_hybrid* hyb /* host */,
                          double field_rtol, int32_t cluster_hint,
                          void* stream);

/* --- coarse propagator G ------------------------------------------------
 * nchain independent sequential chains of nwin windows each (fluid.py:95-118
 * per window).  Chain c: x_0 = rho_in[c]; E_in (may be NULL) supplies the
 * field of x_0 (fluid_step semantics, fluid.py:60-77) instead of refreshing
 * it on entry (fluid_propagate, fluid.py:111-113); for w: G_w = G(x_w) over the
 * window's schedule (nfull[c*nwin+w] steps of dt_full, then rem[...] if > 0);
 * x_{w+1} = G_w (+ delta[c][w] if delta != NULL).  out[c][w] = x_{w+1};
 * gout[c][w] = G_w (may be NULL).  Covers fluid_propagate, coarse_sweep
 * (parareal.py:210-229) and the sequential correction (parareal.py:276-281). */
int32_t pk_coarse_chain(pk_ctx* ctx, int32_t nchain, int32_t nwin,
                        const double* rho_in, const double* E_in, double* out, double* gout, double* E_out,
                        const double* delta,
                        const int32_t* nfull, const double* rem,
                        const double* cflu_full, const double* cflu_rem,
                        double dt_full, const double* rho_bar, double field_rtol,
                        int32_t exact_scan, void* stream);

/* --- single operators ---------------------------------------------------- */
/* solve_field (poisson.py:21-54) for B densities. */
int32_t pk_field(pk_ctx* ctx, int32_t B, const double* rho, const double* rho_bar,
                 double* E, double field_rtol, int32_t exact_scan, void* stream);
/* lift (lifting.py:38-105) for B slices; dE_dt may be NULL. */
int32_t pk_lift(pk_ctx* ctx, int32_t B, const double* rho, const double* E,
                const double* dE_dt, const double* rho_bar,
                const double* neg_eps, const double* eps2,
                int32_t order, int32_t time_elim, int32_t project,
                double* g_out, void* stream);

/* --- adaptation indicators (adaptation.py:120-181) ----------------------
 * The public K3 operators as standalone calls, in the arithmetic F uses every
 * step (pk_fine_propagate computes them in-kernel).  Replace:
 *   remainder_indicator / remainder_from_fields (adaptation.py:120-152):
 *     R[B*nx] from rho, E and either E_prev with dt (dE/dt = (E-E_prev)/dt
 *     averaged to cells) or the cell-centred dE/dt dtE_c (E_prev = NULL);
 *   perturbation_indicator (adaptation.py:155-159): gnorm[B*nx] from g;
 *   update_labels (adaptation.py:162-181): kc/ki[B*nx] (uint8 0/1). */
int32_t pk_remainder(pk_ctx* ctx, int32_t B, const double* rho, const double* E,
                     const double* E_prev, const double* dtE_c, double dt, const double* rho_bar,
                     double* R, void* stream);
int32_t pk_perturbation(pk_ctx* ctx, int32_t B, const double* g, double* gnorm, void* stream);
int32_t pk_labels(pk_ctx* ctx, int32_t B, const double* R, const double* gnorm, double delta0,
                  double eta0, int32_t combine_and, uint8_t* kc, uint8_t* ki, void* stream);

/* --- parareal glue (parareal.py:267-289) -------------------------------- */
/* out[i] = a[i] - b[i] over n values; flags non-finite into the status. */
int32_t pk_jump(pk_ctx* ctx, int64_t n, const double* a, const double* b, double* out,
                void* stream);
/* err[0] = max |a - b| over n values (device scalar); flags non-finite. */
int32_t pk_maxdiff(pk_ctx* ctx, int64_t n, const double* a, const double* b, double* err,
                   void* stream);

/* diagnostics: out[i] = x[i] / dx through the kernels' division routine (the
 * Markstein-corrected quotient the transport uses for `out /= dx`,
 * kinetic.py:173), so tests can check it against IEEE division on the device. */
int32_t pk_diag_qdiv(pk_ctx* ctx, int64_t n, const double* x, double* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PK_H */
