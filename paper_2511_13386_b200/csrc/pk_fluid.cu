// Coarse propagator G (explicit drift-diffusion limit scheme) and the small
// parareal glue kernels.
//
// One CTA owns one chain of windows and keeps rho, E and J in shared memory
// for the whole chain: the per-step work is O(nx) and strictly sequential in
// time (fluid.py:60-118), so the kernel is latency-bound; keeping the state
// on-chip removes every global round trip from the step loop.
#include "../../include/pk.h"
#include "pk_args.h"

namespace pk {


// Field of rho into E, up to the zero-mean shift: returns false on a
// solvability violation, else E holds cumsum(src - defect/nx) and `mean` its
// mean, so the field is E[i] - mean (poisson.py:41-54; the subtraction is
// applied where E is read, with the same rounding).  E doubles as src.
// Exact, up to 256 threads: field_exact_onchip.
template <int NT>
__device__ static bool chain_field(const MeshDev& m, const double* rho, double rb, double* E,
                                   double rtol, int exact_scan, const PwPlan& plan, double* red,
                                   double& mean) {
  const int nx = m.nx;
  for (int i = threadIdx.x; i < nx; i += NT) E[i] = (rho[i] - rb) * m.dx;
  __syncthreads();
  if constexpr (NT <= 256) {  // (the 512-thread instantiations spill with it)
    if (exact_scan) {
      const uint32_t rs = (uint32_t)__cvta_generic_to_shared(rho);
      return field_exact_onchip([&](int i) { return fabs(lds64(rs + 8 * i)); }, E, nx, m.dx,
                                rtol, plan, red, mean);
    }
  }
  double defect, abssum;
  block_pairwise2([&](int i) { return E[i]; }, [&](int i) { return fabs(rho[i]); }, plan, red,
                  defect, abssum);
  const double scale = abssum * m.dx;
  if (fabs(defect) > rtol * fmax(scale, 2.2250738585072014e-308)) return false;
  const double corr = defect / (double)nx;
  for (int i = threadIdx.x; i < nx; i += NT) E[i] = E[i] - corr;
  __syncthreads();
  if (exact_scan)
    smem_cumsum(E, E, nx);
  else
    block_scan_fast([&](int i) { return E[i]; }, [&](int i, double v) { E[i] = v; }, nx, red);
  __syncthreads();
  mean = block_pairwise([&](int i) { return E[i]; }, plan, red) / (double)nx;
  return true;
}

// NT threads, PER cells per thread (nx <= PER * NT), so the new-rho registers
// stay unspilled.
template <int PER, int NT>
__global__ void __launch_bounds__(NT) chain_kernel(const ChainArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const MeshDev& m = a.m;
  const int nx = m.nx;
  const int c = blockIdx.x;
  PwPlan* plan = reinterpret_cast<PwPlan*>(smem_raw);
  double* base = reinterpret_cast<double*>(smem_raw + (sizeof(PwPlan) + 15) / 16 * 16);
  double* rho = base;
  double* E = rho + nx;
  double* red = E + nx;
  {
    const int* s = reinterpret_cast<const int*>(m.plan_x);
    int* d = reinterpret_cast<int*>(plan);
    for (int i = threadIdx.x; i < (int)(sizeof(PwPlan) / 4); i += NT) d[i] = s[i];
  }
  for (int i = threadIdx.x; i < nx; i += NT) rho[i] = a.rho_in[(size_t)c * nx + i];
  __syncthreads();
  const double rb = a.rho_bar[c];
  const double dx = m.dx, rdx = m.rdx;
  bool have_E = false;
  double mean = 0.0;  // pending zero-mean shift of E (x - 0.0 == x bitwise)
  for (int w = 0; w < a.nwin; ++w) {
    const size_t cw = (size_t)c * a.nwin + w;
    const int nfull = a.nfull[cw];
    const double rem = a.rem[cw];
    if (nfull > 0 || rem > 0.0) {
      if (w == 0 && a.E_in) {
        // fluid_step: the caller guarantees E matches rho (fluid.py:69-71)
        for (int i = threadIdx.x; i < nx; i += NT) E[i] = a.E_in[(size_t)c * nx + i];
        mean = 0.0;
        __syncthreads();
      } else if (!chain_field<NT>(m, rho, rb, E, a.rtol, a.exact_scan, *plan, red, mean)) {
        // fluid_propagate: the field is refreshed from rho on entry (fluid.py:111-113)
        if (threadIdx.x == 0) set_status(a.status, PK_ERR_SOLVABILITY, c, w);
        return;
      }
      have_E = true;
      const int nstep = nfull + (rem > 0.0 ? 1 : 0);
      for (int s = 0; s < nstep; ++s) {
        const double cflu = s < nfull ? a.cflu_full[cw] : a.cflu_rem[cw];
        // rho_i += cflu (J_{i+1/2} - J_{i-1/2})   (fluid.py:51-57); each J is
        // formed twice (once per neighbour) with identical operands and bits.
        double nr[PER];
#pragma unroll
        for (int k = 0; k < PER; ++k) {
          const int i = threadIdx.x + k * NT;
          if (i < nx) {
            const int ip = i == 0 ? nx - 1 : i - 1, in_ = i + 1 == nx ? 0 : i + 1;
            const double r = rho[i], rp = rho[ip], rn = rho[in_];
            // (.)/dx as the correctly rounded Markstein quotient (qdiv, pk_device.cuh)
            const double Ji = qdiv(rn - r, dx, rdx) - (E[i] - mean) * 0.5 * (r + rn);
            const double Jp = qdiv(r - rp, dx, rdx) - (E[ip] - mean) * 0.5 * (rp + r);
            nr[k] = r + cflu * (Ji - Jp);
          }
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < PER; ++k) {
          const int i = threadIdx.x + k * NT;
          if (i < nx) rho[i] = nr[k];
        }
        __syncthreads();
        if (!chain_field<NT>(m, rho, rb, E, a.rtol, a.exact_scan, *plan, red, mean)) {
          if (threadIdx.x == 0) set_status(a.status, PK_ERR_SOLVABILITY, c, w);
          return;
        }
      }
    }
    if (a.gout)
      for (int i = threadIdx.x; i < nx; i += NT) a.gout[cw * nx + i] = rho[i];
    if (a.delta) {
      // new_row[n] = coarse.rho + deltas[n]   (parareal.py:281)
      for (int i = threadIdx.x; i < nx; i += NT) rho[i] = rho[i] + a.delta[cw * nx + i];
    }
    for (int i = threadIdx.x; i < nx; i += NT) a.out[cw * nx + i] = rho[i];
    __syncthreads();
  }
  if (a.Eout && have_E)
    for (int i = threadIdx.x; i < nx; i += NT) a.Eout[(size_t)c * nx + i] = E[i] - mean;
}


// ---------------------------------------------------------------------------
// Fast mode (exact_scan == 0): the same chain with the field's prefix sum as a
// parallel scan (SURVEY §7 "hard parts": not bitwise -- the prefix differs
// from np.cumsum by O(n u |E|) -- so the defect and mean reductions are plain
// trees too).  The whole state lives in registers: thread t owns the PER
// consecutive cells [t PER, t PER + PER) of rho and E; the only cross-thread
// data are the reductions and each thread's edge cells (first rho, last rho,
// last E) in shared memory.  One step = flux + update in registers, then
// three block barriers: (1) defect and sum|rho| (guard), (2) the scan and,
// folded into the same barrier, the sum of E for the zero-mean gauge
// (sum_t E = sum_w C_w off_w + A_w with per-warp partials), (3) the new edges.
// cfg4's nx = 8192: 1024 threads x 8 cells.
struct FastRed {
  double a[2][32], b[2][32], c[2][32];   // per-warp partials, double-buffered
};

template <int PER>
__global__ void __launch_bounds__(PER >= 8 ? 1024 : 512, 1) chain_fast_kernel(const ChainArgs a) {
  __shared__ FastRed red;
  __shared__ double firstR[1024], lastR[1024], lastE[1024];
  const MeshDev& m = a.m;
  const int nx = m.nx;
  const int c = blockIdx.x;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int nwarp = blockDim.x >> 5;
  const int tl = (nx - 1) / PER;               // last thread that owns cells
  const int i0 = t * PER;
  const int cnt = t <= tl ? min(PER, nx - i0) : 0;
  const double dx = m.dx, rdx = m.rdx;
  const double rb = a.rho_bar[c];
  double r[PER], e[PER];
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    r[k] = k < cnt ? a.rho_in[(size_t)c * nx + i0 + k] : 0.0;
    e[k] = 0.0;
  }
  int par = 0;
  // publish this thread's edge cells, then one barrier
  auto edges = [&]() {
    if (cnt > 0) {
      firstR[t] = r[0];
      double lr = r[0], le = e[0];
#pragma unroll
      for (int k = 1; k < PER; ++k)
        if (k < cnt) { lr = r[k]; le = e[k]; }
      lastR[t] = lr;
      lastE[t] = le;
    }
    __syncthreads();
  };
  auto warp_sum = [&](double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = v + __shfl_xor_sync(FULL, v, o);
    return v;
  };
  // field of r into e (poisson.py:41-54 with a parallel prefix); false on a
  // solvability violation (uniform across the block)
  auto field = [&]() -> bool {
    double ls = 0.0, la = 0.0;
#pragma unroll
    for (int k = 0; k < PER; ++k)
      if (k < cnt) {
        e[k] = (r[k] - rb) * dx;
        ls = ls + e[k];
        la = la + fabs(r[k]);
      }
    ls = warp_sum(ls);
    la = warp_sum(la);
    if (lane == 0) { red.a[par][warp] = ls; red.b[par][warp] = la; }
    __syncthreads();
    const double defect = warp_sum(lane < nwarp ? red.a[par][lane] : 0.0);
    const double abssum = warp_sum(lane < nwarp ? red.b[par][lane] : 0.0);
    if (fabs(defect) > a.rtol * fmax(abssum * dx, 2.2250738585072014e-308)) return false;
    const double corr = defect / (double)nx;
    double acc = 0.0, psum = 0.0;
#pragma unroll
    for (int k = 0; k < PER; ++k)
      if (k < cnt) {
        acc = acc + (e[k] - corr);
        e[k] = acc;          // local inclusive prefix
        psum = psum + acc;
      }
    // warp scan of the thread totals
    double inc = acc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double y = __shfl_up_sync(FULL, inc, o);
      if (lane >= o) inc = inc + y;
    }
    double exc = __shfl_up_sync(FULL, inc, 1);
    if (lane == 0) exc = 0.0;
    // sum of this warp's E values up to the warp offset: A_w = sum_t (cnt exc + psum)
    const double aw = warp_sum((double)cnt * exc + psum);
    const double cw = warp_sum((double)cnt);
    if (lane == 31) red.a[par ^ 1][warp] = inc;   // warp total
    if (lane == 0) { red.b[par ^ 1][warp] = aw; red.c[par ^ 1][warp] = cw; }
    __syncthreads();
    par ^= 1;
    // warp offsets (exclusive scan of the warp totals) and sum(E)
    double tw = lane < nwarp ? red.a[par][lane] : 0.0;
    double wi = tw;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double y = __shfl_up_sync(FULL, wi, o);
      if (lane >= o) wi = wi + y;
    }
    double we = __shfl_up_sync(FULL, wi, 1);
    if (lane == 0) we = 0.0;
    const double tot = warp_sum(lane < nwarp ? red.c[par][lane] * we + red.b[par][lane] : 0.0);
    const double mean = tot / (double)nx;
    const double off = __shfl_sync(FULL, we, warp) + exc;
#pragma unroll
    for (int k = 0; k < PER; ++k)
      if (k < cnt) e[k] = (off + e[k]) - mean;
    return true;
  };

  edges();
  bool have_E = false;
  for (int w = 0; w < a.nwin; ++w) {
    const size_t cw = (size_t)c * a.nwin + w;
    const int nfull = a.nfull[cw];
    const double rem = a.rem[cw];
    if (nfull > 0 || rem > 0.0) {
      if (w == 0 && a.E_in) {
#pragma unroll
        for (int k = 0; k < PER; ++k)
          if (k < cnt) e[k] = a.E_in[(size_t)c * nx + i0 + k];
      } else if (!field()) {
        if (t == 0) set_status(a.status, PK_ERR_SOLVABILITY, c, w);
        return;
      }
      edges();
      have_E = true;
      const int nstep = nfull + (rem > 0.0 ? 1 : 0);
      for (int s = 0; s < nstep; ++s) {
        const double cflu = s < nfull ? a.cflu_full[cw] : a.cflu_rem[cw];
        if (cnt > 0) {
          const int tp = t > 0 ? t - 1 : tl, tn = t < tl ? t + 1 : 0;
          const double rp = lastR[tp], ep = lastE[tp], rn = firstR[tn];
          // J_{i-1/2} of the first cell from the neighbour's last cell (fluid.py:51-57)
          double Jp = qdiv(r[0] - rp, dx, rdx) - ep * 0.5 * (rp + r[0]);
#pragma unroll
          for (int k = 0; k < PER; ++k)
            if (k < cnt) {
              const double rnk = (k + 1 < cnt) ? r[k + 1] : rn;
              const double Ji = qdiv(rnk - r[k], dx, rdx) - e[k] * 0.5 * (r[k] + rnk);
              r[k] = r[k] + cflu * (Ji - Jp);
              Jp = Ji;
            }
        }
        if (!field()) {
          if (t == 0) set_status(a.status, PK_ERR_SOLVABILITY, c, w);
          return;
        }
        edges();
      }
    }
#pragma unroll
    for (int k = 0; k < PER; ++k)
      if (k < cnt) {
        const size_t o = cw * nx + i0 + k;
        if (a.gout) a.gout[o] = r[k];
        if (a.delta) r[k] = r[k] + a.delta[o];   // parareal.py:281
        a.out[o] = r[k];
      }
    if (a.delta) edges();
  }
  if (a.Eout && have_E)
#pragma unroll
    for (int k = 0; k < PER; ++k)
      if (k < cnt) a.Eout[(size_t)c * nx + i0 + k] = e[k];
}

size_t chain_smem_bytes(int nx) {
  return (sizeof(PwPlan) + 15) / 16 * 16 + (size_t)2 * nx * 8 + 2 * (MAX_LEAF + MAX_NODE) * 8;
}

cudaError_t launch_chain(const ChainArgs& a, cudaStream_t st) {
  // The chain is one latency-bound CTA per chain: claim (nearly) a whole SM's
  // shared memory so that no fine-propagator CTA is co-scheduled beside it
  // when the correction overlaps the fine windows (parareal._Overlap).
  const size_t smem = chain_smem_bytes(a.m.nx) > 200 * 1024 ? chain_smem_bytes(a.m.nx) : 200 * 1024;
  const int nx = a.m.nx;
  auto go = [&](auto kern, int nt) {
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<a.nchain, nt, smem, st>>>(a);
    return cudaGetLastError();
  };
  if (!a.exact_scan && nx <= 8192) {
    // fast mode: registers only, PER cells per thread, <= 1024 threads
    auto fast = [&](auto kern, int per) {
      const int nt = ((nx + per - 1) / per + 31) / 32 * 32;
      kern<<<a.nchain, nt, 0, st>>>(a);
      return cudaGetLastError();
    };
    if (nx <= 1024) return fast(chain_fast_kernel<2>, 2);
    if (nx <= 2048) return fast(chain_fast_kernel<4>, 4);
    return fast(chain_fast_kernel<8>, 8);
  }
  // more threads for the element passes at large nx (the scan stays on one)
  if (nx <= 512) return go(chain_kernel<2, 256>, 256);
  if (nx <= 1024) return go(chain_kernel<4, 256>, 256);
  if (nx <= 2048) return go(chain_kernel<4, 512>, 512);
  if (nx <= 4096) return go(chain_kernel<8, 512>, 512);
  if (nx <= 8192) return go(chain_kernel<16, 512>, 512);
  return go(chain_kernel<(MAX_LEAF * 128 + 511) / 512, 512>, 512);
}

// Delta = F - G (parareal.py:429) and the finiteness check of parareal.py:267-269.
__global__ void jump_kernel(int64_t n, const double* __restrict__ a, const double* __restrict__ b,
                            double* __restrict__ out, Status* st) {
  bool bad = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double d = a[i] - b[i];
    out[i] = d;
    bad |= !isfinite(d);
  }
  if (__any_sync(FULL, bad) && (threadIdx.x & 31) == 0) set_status(st, PK_ERR_NONFINITE, -1, -1);
}

cudaError_t launch_jump(int64_t n, const double* a, const double* b, double* out, Status* st,
                        cudaStream_t s) {
  const int64_t want = (n + 255) / 256;
  const int blocks = (int)(want < 148 * 4 ? want : 148 * 4);
  jump_kernel<<<blocks > 0 ? blocks : 1, 256, 0, s>>>(n, a, b, out, st);
  return cudaGetLastError();
}

// pk_status_store: the status record as doubles into device memory (code,
// step), optionally re-armed -- stream-ordered, no host synchronisation, so a
// window's status can travel in the same collective as its jump.
__global__ void status_store_kernel(Status* st, double* dst, int clear) {
  const unsigned long long k = st->key;
  if (k == ~0ull) {
    dst[0] = 0.0;
    dst[1] = 0.0;
  } else {
    dst[0] = (double)(int)(k & 0xFF);
    dst[1] = (double)(int)(unsigned)((k >> 8) & 0xFFFFFFFFull);
  }
  if (clear) st->key = ~0ull;
}

cudaError_t launch_status_store(Status* st, double* dst, int clear, cudaStream_t s) {
  status_store_kernel<<<1, 1, 0, s>>>(st, dst, clear);
  return cudaGetLastError();
}

// pk_diag_qdiv: the kernels' quotient routine over an array (test hook)
__global__ void qdiv_kernel(int64_t n, const double* __restrict__ x, double* __restrict__ out,
                            double dx, double rdx) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = qdiv(x[i], dx, rdx);
}

cudaError_t launch_qdiv(int64_t n, const double* x, double* out, double dx, double rdx,
                        cudaStream_t s) {
  const int64_t want = (n + 255) / 256;
  const int blocks = (int)(want < 148 * 8 ? want : 148 * 8);
  qdiv_kernel<<<blocks > 0 ? blocks : 1, 256, 0, s>>>(n, x, out, dx, rdx);
  return cudaGetLastError();
}

// err = max |a - b| (parareal.py:286); max is order-independent, so a tree is
// exact.  Also flags a non-finite a (parareal.py:283-284).  One CTA.
__global__ void maxdiff_kernel(int64_t n, const double* __restrict__ a,
                               const double* __restrict__ b, double* err, Status* st) {
  __shared__ double sm[32];
  double mx = 0.0;
  bool bad = false;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double d = fabs(a[i] - b[i]);
    bad |= !isfinite(a[i]);
    mx = fmax(mx, d);  // numpy max propagates NaN; non-finite already raises
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(FULL, mx, o));
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = mx;
  if (__any_sync(FULL, bad) && (threadIdx.x & 31) == 0) set_status(st, PK_ERR_NONFINITE, -1, -1);
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? sm[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(FULL, v, o));
    if (threadIdx.x == 0) *err = v;
  }
}

cudaError_t launch_maxdiff(int64_t n, const double* a, const double* b, double* err, Status* st,
                           cudaStream_t s) {
  maxdiff_kernel<<<1, 1024, 0, s>>>(n, a, b, err, st);
  return cudaGetLastError();
}

}  // namespace pk
