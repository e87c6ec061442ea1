// libpk C ABI: context, workspace, pairwise-sum plans and the entry points
// declared in include/pk.h.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <string>
#include <vector>

#include "../../include/pk.h"
#include "pk_args.h"

namespace pk {
cudaError_t launch_fine(const FineArgs& a, int C, cudaStream_t st);
void fine_last_launch(int out[4]);
cudaError_t launch_lift(const LiftArgs& a, cudaStream_t st);
cudaError_t launch_indicators(const IndArgs& a, int which, cudaStream_t st);
cudaError_t launch_field(const FieldArgs& a, cudaStream_t st);
cudaError_t launch_chain(const ChainArgs& a, cudaStream_t st);
cudaError_t launch_jump(int64_t n, const double* a, const double* b, double* out, Status* st,
                        cudaStream_t s);
cudaError_t launch_status_store(Status* st, double* dst, int clear, cudaStream_t s);
cudaError_t launch_qdiv(int64_t n, const double* x, double* out, double dx, double rdx,
                        cudaStream_t s);
cudaError_t launch_maxdiff(int64_t n, const double* a, const double* b, double* err, Status* st,
                           cudaStream_t s);
size_t chain_smem_bytes(int nx);
}  // namespace pk

using pk::PwPlan;

struct pk_ctx {
  int device = 0;
  int num_sms = 148;
  pk::MeshDev m{};
  double* d_const = nullptr;  // vx | M | xiM | w2
  PwPlan* d_plan = nullptr;  // [x: nx terms, folded velocity row, middle xi plane]
  pk::Status* d_status = nullptr;
  int* d_cancel = nullptr;  // cancel request of the fine launch in flight (pk_fine_cancel)
  int cap = 0;
  // workspace
  double* dws = nullptr;  // 16 double arrays of cap*nx
  int8_t* i8ws = nullptr;
  uint8_t* u8ws = nullptr;  // 7 arrays
  int* iws = nullptr;       // klist cap*nx, nk cap, abort cap
  long long* prof = nullptr;  // optional device phase counters (pk_debug_profile)
  long long* rowcnt = nullptr;  // optional per-slice row counters (pk_count_rows)
  std::string err;
};

namespace {

int fail(pk_ctx* c, int code, const std::string& msg) {
  if (c) c->err = msg;
  return code;
}

int cuda_fail(pk_ctx* c, cudaError_t e, const char* where) {
  return fail(c, PK_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

// numpy pairwise_sum recursion -> leaves + level-ordered internal nodes.
struct PlanBuilder {
  std::vector<int> leaf_off, leaf_len;
  struct Node { int a, b, level; };
  std::vector<Node> nodes;  // post-order; operands: >=0 leaf, <0 ~node
  // returns operand id and level
  std::pair<int, int> rec(int off, int n) {
    if (n <= 128) {
      leaf_off.push_back(off);
      leaf_len.push_back(n);
      return {(int)leaf_off.size() - 1, 0};
    }
    int n2 = n / 2;
    n2 -= n2 % 8;
    auto l = rec(off, n2);
    auto r = rec(off + n2, n - n2);
    int lev = std::max(l.second, r.second) + 1;
    nodes.push_back({l.first, r.first, lev});
    return {~((int)nodes.size() - 1), lev};
  }
};

bool build_plan(int n, PwPlan* P) {
  PlanBuilder pb;
  pb.rec(0, n);
  const int nleaf = (int)pb.leaf_off.size(), nnode = (int)pb.nodes.size();
  if (nleaf > pk::MAX_LEAF || nnode > pk::MAX_NODE) return false;
  std::memset(P, 0, sizeof(PwPlan));
  P->n = n;
  P->nleaf = nleaf;
  P->nnode = nnode;
  for (int i = 0; i < nleaf; ++i) {
    P->leaf_off[i] = pb.leaf_off[i];
    P->leaf_len[i] = pb.leaf_len[i];
  }
  int maxlev = 0;
  for (auto& nd : pb.nodes) maxlev = std::max(maxlev, nd.level);
  if (maxlev > pk::MAX_LEVEL) return false;
  // stable order by level; map post-order index -> slot
  std::vector<int> order(nnode), slot(nnode);
  for (int i = 0; i < nnode; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(),
                   [&](int x, int y) { return pb.nodes[x].level < pb.nodes[y].level; });
  for (int i = 0; i < nnode; ++i) slot[order[i]] = i;
  auto opnd = [&](int id) { return id >= 0 ? id : nleaf + slot[~id]; };
  for (int i = 0; i < nnode; ++i) {
    const auto& nd = pb.nodes[order[i]];
    P->node_a[i] = opnd(nd.a);
    P->node_b[i] = opnd(nd.b);
  }
  P->nlevel = maxlev;
  for (int lev = 1; lev <= maxlev; ++lev) {
    int end = 0;
    for (int i = 0; i < nnode; ++i)
      if (pb.nodes[order[i]].level <= lev) end = i + 1;
    P->level_end[lev - 1] = end;
  }
  // perfect: 2^L leaves and level l's q-th node adds items 2q, 2q+1 of level
  // l-1 (the leaves at level 0) -- the xor-butterfly form (pw_perfect)
  bool perf = (nleaf & (nleaf - 1)) == 0 && (1 << maxlev) == nleaf;
  int prev0 = 0, start = 0;  // first operand index of level l-1, first node of level l
  for (int lev = 1; perf && lev <= maxlev; ++lev) {
    const int end = P->level_end[lev - 1];
    if (end - start != nleaf >> lev) perf = false;
    for (int q = 0; perf && q < end - start; ++q)
      perf = P->node_a[start + q] == prev0 + 2 * q && P->node_b[start + q] == prev0 + 2 * q + 1;
    prev0 = nleaf + start;
    start = end;
  }
  P->perfect = perf ? 1 : 0;
  return true;
}

constexpr int NDWS = 16;
constexpr int NU8 = 7;

void free_ws(pk_ctx* c) {
  cudaFree(c->dws);
  cudaFree(c->i8ws);
  cudaFree(c->u8ws);
  cudaFree(c->iws);
  c->dws = nullptr;
  c->i8ws = nullptr;
  c->u8ws = nullptr;
  c->iws = nullptr;
  c->cap = 0;
}

int ensure(pk_ctx* c, int B) {
  if (B <= c->cap) return PK_OK;
  cudaSetDevice(c->device);
  free_ws(c);
  const size_t n = (size_t)B * c->m.nx;
  cudaError_t e;
  if ((e = cudaMalloc(&c->dws, NDWS * n * sizeof(double))) != cudaSuccess) return cuda_fail(c, e, "workspace");
  if ((e = cudaMalloc(&c->i8ws, n)) != cudaSuccess) return cuda_fail(c, e, "workspace");
  if ((e = cudaMalloc(&c->u8ws, NU8 * n)) != cudaSuccess) return cuda_fail(c, e, "workspace");
  // klist [n], nk [B], abort [B], kpos [n], kstream [3n], zlist [n], nzl [B], sg_cnt [B]
  if ((e = cudaMalloc(&c->iws, (6 * n + 4 * (size_t)B) * sizeof(int))) != cudaSuccess)
    return cuda_fail(c, e, "workspace");
  c->cap = B;
  return PK_OK;
}

void bind_ws(pk_ctx* c, pk::FineArgs& a) {
  const size_t n = (size_t)c->cap * c->m.nx;
  double* d = c->dws;
  double** dst[NDWS] = {&a.J, &a.fl, &a.sq, &a.bm, &a.dco, &a.vco, &a.tA, &a.tB,
                        &a.tC, &a.tD, &a.tE, &a.blift, &a.lJ, nullptr, nullptr, nullptr};
  for (int i = 0; i < NDWS; ++i)
    if (dst[i]) *dst[i] = d + i * n;
  a.vsg = c->i8ws;
  uint8_t* u = c->u8ws;
  a.flip = u;
  a.nza = u + n;
  a.nzb = u + 2 * n;
  a.kcn = u + 3 * n;
  a.kin = u + 4 * n;
  a.klist = c->iws;
  a.nk = c->iws + n;
  a.abort_ = c->iws + n + c->cap;
  a.kpos = c->iws + n + 2 * (size_t)c->cap;
  a.kstream = a.kpos + n;
  a.zlist = a.kstream + 3 * n;
  a.nzl = a.zlist + n;
  a.sg_cnt = reinterpret_cast<unsigned*>(a.nzl + c->cap);
  a.status = c->d_status;
  a.prof = c->prof;
  a.rowcnt = c->rowcnt;
}

cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

}  // namespace

extern "C" {

int32_t pk_version(void) { return 1; }

int32_t pk_debug_profile(pk_ctx* c, void* dev_counters) {
  if (!c) return PK_ERR_BAD_ARG;
  c->prof = reinterpret_cast<long long*>(dev_counters);
  return PK_OK;
}

int32_t pk_count_rows(pk_ctx* c, void* dev_counts) {
  if (!c) return PK_ERR_BAD_ARG;
  c->rowcnt = reinterpret_cast<long long*>(dev_counts);
  return PK_OK;
}

int32_t pk_fine_last_launch(pk_ctx* c, int32_t out[4]) {
  if (!c || !out) return PK_ERR_BAD_ARG;
  int v[4];
  pk::fine_last_launch(v);
  for (int i = 0; i < 4; ++i) out[i] = v[i];
  return PK_OK;
}

pk_ctx* pk_create(int32_t device, const pk_mesh* mesh) {
  if (!mesh || mesh->nx < 7 || mesh->nv < 1) return nullptr;
  const int nvyz = mesh->nvyz > 0 ? mesh->nvyz : 1;
  if (mesh->nv % nvyz != 0) return nullptr;
  pk_ctx* c = new pk_ctx();
  c->device = device;
  if (cudaSetDevice(device) != cudaSuccess) {
    delete c;
    return nullptr;
  }
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
  const int nv = mesh->nv, nx = mesh->nx;
  pk::MeshDev& m = c->m;
  m.nx = nx;
  m.nv = nv;
  m.nvyz = nvyz;
  m.dx = mesh->dx;
  m.rdx = 1.0 / mesh->dx;
  m.two_dx = 2.0 * mesh->dx;
  m.rtwo_dx = 1.0 / m.two_dx;
  m.rdvx = 1.0 / mesh->dvx;
  m.dvx = mesh->dvx;
  m.dv3 = mesh->dv3;
  m.m0 = mesh->m0;
  m.m2 = mesh->m2;
  std::memcpy(m.stc, mesh->stencil, sizeof(m.stc));
  std::memcpy(m.sts, mesh->stencil_scale, sizeof(m.sts));
  m.stc_std = 1;
  for (int p = 0; p < 4; ++p)
    for (int o = 0; o < 7; ++o)
      if ((m.stc[p][o] == 0.0) != ((p == 0 || p == 2) && o == 3)) m.stc_std = 0;
  std::vector<double> h(4 * (size_t)nv);
  std::memcpy(h.data(), mesh->vx, nv * 8);
  std::memcpy(h.data() + nv, mesh->M, nv * 8);
  std::memcpy(h.data() + 2 * nv, mesh->xi_M, nv * 8);
  std::memcpy(h.data() + 3 * nv, mesh->w2, nv * 8);
  m.mirror = 1;
  for (int j = 0; j < nv; ++j) {
    const double* vx = h.data();
    const double* M = h.data() + nv;
    const double* xM = h.data() + 2 * nv;
    const double p = vx[j] * M[j];
    if (vx[nv - 1 - j] != -vx[j] || std::memcmp(&M[nv - 1 - j], &M[j], 8) != 0 ||
        std::memcmp(&xM[j], &p, 8) != 0)
      m.mirror = 0;
  }
  m.xplane = 1;
  for (int j = 0; j < nv; ++j)
    if (std::memcmp(&h[j], &h[(size_t)(j / nvyz) * nvyz], 8) != 0) m.xplane = 0;
  // pairwise plans: x sums (nx terms), and for 1D-3V rows the folded velocity
  // block ((nvx/2) nvy nvz terms) and the middle xi plane (nvy nvz terms)
  PwPlan plan[3];
  const int nvx = nv / nvyz;
  if (!build_plan(nx, &plan[0]) || !build_plan((nvx / 2) * nvyz, &plan[1]) ||
      !build_plan(nvyz, &plan[2])) {
    delete c;
    return nullptr;
  }
  if (cudaMalloc(&c->d_const, h.size() * 8) != cudaSuccess ||
      cudaMalloc(&c->d_plan, 3 * sizeof(PwPlan)) != cudaSuccess ||
      cudaMalloc(&c->d_status, sizeof(pk::Status)) != cudaSuccess ||
      cudaMalloc(&c->d_cancel, sizeof(int)) != cudaSuccess) {
    delete c;
    return nullptr;
  }
  cudaMemcpy(c->d_const, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(c->d_plan, plan, 3 * sizeof(PwPlan), cudaMemcpyHostToDevice);
  cudaMemset(c->d_status, 0xFF, sizeof(pk::Status));
  m.vx = c->d_const;
  m.M = c->d_const + nv;
  m.xiM = c->d_const + 2 * nv;
  m.w2 = c->d_const + 3 * nv;
  m.plan_x = c->d_plan;
  m.plan_f = c->d_plan + 1;
  m.plan_s = c->d_plan + 2;
  return c;
}

void pk_destroy(pk_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  free_ws(c);
  cudaFree(c->d_const);
  cudaFree(c->d_plan);
  cudaFree(c->d_status);
  cudaFree(c->d_cancel);
  delete c;
}

const char* pk_last_error(const pk_ctx* c) { return c ? c->err.c_str() : "null context"; }

int32_t pk_reserve(pk_ctx* c, int32_t max_slices) {
  if (!c || max_slices < 1) return PK_ERR_BAD_ARG;
  return ensure(c, max_slices);
}

// pk_device.cuh Status key -> pk_status (all ones = no error)
static void decode_status(const pk::Status& s, pk_status* out) {
  if (s.key == ~0ull) {
    out->code = 0;
    out->slice = 0;
    out->step = 0;
  } else {
    out->code = (int32_t)(s.key & 0xFF);
    out->step = (int32_t)(uint32_t)((s.key >> 8) & 0xFFFFFFFFull);
    out->slice = (int32_t)(s.key >> 40) - 1;
  }
  out->pad = 0;
}

int32_t pk_status_read_stream(pk_ctx* c, pk_status* out, int32_t clear, void* stream) {
  if (!c || !out) return PK_ERR_BAD_ARG;
  cudaSetDevice(c->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  pk::Status s;
  cudaError_t e = cudaMemcpyAsync(&s, c->d_status, sizeof(s), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(c, e, "status copy");
  decode_status(s, out);
  if (clear) cudaMemsetAsync(c->d_status, 0xFF, sizeof(pk::Status), st);
  return PK_OK;
}

int32_t pk_status_read(pk_ctx* c, pk_status* out, int32_t clear) {
  if (!c || !out) return PK_ERR_BAD_ARG;
  cudaSetDevice(c->device);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return cuda_fail(c, e, "synchronize");
  pk::Status s;
  e = cudaMemcpy(&s, c->d_status, sizeof(s), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_fail(c, e, "status copy");
  decode_status(s, out);
  if (clear) cudaMemset(c->d_status, 0xFF, sizeof(pk::Status));
  return PK_OK;
}

int32_t pk_fine_propagate(pk_ctx* c, int32_t B, double* rho, double* E, double* E_prev,
                          uint8_t* kc, uint8_t* ki, double* g_a, double* g_b,
                          const double* rho_bar, const uint8_t* init_flags,
                          const pk_phase* phases, const pk_hybrid* hyb, double field_rtol,
                          int32_t cluster_hint, void* stream) {
  if (!c || B < 1 || !phases || !hyb || !rho || !E || !E_prev || !kc || !ki || !g_a || !g_b ||
      !rho_bar)
    return fail(c, PK_ERR_BAD_ARG, "pk_fine_propagate: null argument");
  const int nv = c->m.nv;
  // 1V rows: the fast layouts (64/128/256/512) or the generic one (<= 256);
  // 1D-3V rows of any length (generic up to 256 nodes, big rows beyond)
  if (c->m.nvyz == 1 && !(nv == 512 || nv <= 256))
    return fail(c, PK_ERR_UNSUPPORTED, "pk_fine_propagate: nv not supported");
  cudaSetDevice(c->device);
  int r = ensure(c, B);
  if (r) return r;
  pk::FineArgs a{};
  a.m = c->m;
  a.B = B;
  a.rho = rho;
  a.E = E;
  a.Eprev = E_prev;
  a.kc = kc;
  a.ki = ki;
  a.ga = g_a;
  a.gb = g_b;
  a.rho_bar = rho_bar;
  a.init_flags = init_flags;
  for (int p = 0; p < 2; ++p) {
    a.ph[p].nsteps = phases[p].nsteps;
    a.ph[p].dt = phases[p].dt;
    a.ph[p].cflu = phases[p].cflu;
    a.ph[p].k1 = phases[p].kappa1;
    a.ph[p].k2 = phases[p].kappa2;
    a.ph[p].cmac = phases[p].cmac;
    a.ph[p].cmacs = phases[p].cmac_scalar;
    a.ph[p].k1s = phases[p].kappa1_scalar;
    a.ph[p].k2s = phases[p].kappa2_scalar;
    if (!a.ph[p].nsteps || !a.ph[p].dt || !a.ph[p].cflu || !a.ph[p].k1 || !a.ph[p].k2 ||
        !a.ph[p].cmac)
      return fail(c, PK_ERR_BAD_ARG, "pk_fine_propagate: incomplete phase");
  }
  a.adaptation = hyb->adaptation;
  a.combine_and = hyb->combine_and;
  a.reinit = hyb->reinit;
  a.lift_order = hyb->lift_order;
  a.time_elim = hyb->time_elim;
  a.exact_scan = hyb->exact_scan;
  a.delta0 = hyb->delta0;
  a.eta0 = hyb->eta0;
  a.rscale = hyb->rscale;
  a.neg_eps = hyb->neg_eps;
  a.eps2 = hyb->eps2;
  a.rtol = field_rtol;
  bind_ws(c, a);
  // a cancel request is for the launch in flight: cleared in stream order
  static const bool no_cancel = getenv("PK_NO_CANCEL") != nullptr;  // (A/B switch)
  a.cancel = no_cancel ? nullptr : c->d_cancel;
  if (cudaMemsetAsync(c->d_cancel, 0, sizeof(int), S(stream)) != cudaSuccess)
    return cuda_fail(c, cudaGetLastError(), "cancel flag");
  // cluster size: enough CTAs to fill the chip, >= 4 rows per warp
  int C = cluster_hint;
  if (C <= 0) {
    C = 1;
    if (c->m.nvyz > 1 && c->m.nv > 256) {  // (the big-row layout, launch_fine)
      // big rows: one CTA per row at one CTA per SM, >= 2 rows per CTA
      while (C < 8 && B * C * 2 <= c->num_sms && c->m.nx >= (C * 2) * 2) C *= 2;
    } else {
      const int slots = 2 * c->num_sms;
      while (C < 8 && B * C * 2 <= slots && c->m.nx >= (C * 2) * 8 * 4) C *= 2;
    }
  }
  a.nwarp_total = C * 8;
  a.kps = cluster_hint > 0 ? 1 : 0;  // 0: the launcher may pack slices per cluster
  cudaError_t e = pk::launch_fine(a, C, S(stream));
  while (e != cudaSuccess && C > 1) {  // cluster too large for this device: shrink
    cudaGetLastError();
    C /= 2;
    a.nwarp_total = C * 8;
    e = pk::launch_fine(a, C, S(stream));
  }
  if (e != cudaSuccess) return cuda_fail(c, e, "fine launch");
  return PK_OK;
}

int32_t pk_coarse_chain(pk_ctx* c, int32_t nchain, int32_t nwin, const double* rho_in,
                        const double* E_in, double* out, double* gout, double* E_out, const double* delta,
                        const int32_t* nfull, const double* rem, const double* cflu_full,
                        const double* cflu_rem, double dt_full, const double* rho_bar,
                        double field_rtol, int32_t exact_scan, void* stream) {
  if (!c || nchain < 1 || nwin < 1 || !rho_in || !out || !nfull || !rem || !cflu_full ||
      !cflu_rem || !rho_bar)
    return fail(c, PK_ERR_BAD_ARG, "pk_coarse_chain: bad argument");
  if (pk::chain_smem_bytes(c->m.nx) > 227 * 1024)
    return fail(c, PK_ERR_UNSUPPORTED, "pk_coarse_chain: nx too large for on-chip state");
  cudaSetDevice(c->device);
  pk::ChainArgs a{};
  a.m = c->m;
  a.nchain = nchain;
  a.nwin = nwin;
  a.rho_in = rho_in;
  a.E_in = E_in;
  a.out = out;
  a.gout = gout;
  a.Eout = E_out;
  a.delta = delta;
  a.nfull = nfull;
  a.rem = rem;
  a.cflu_full = cflu_full;
  a.cflu_rem = cflu_rem;
  a.dt_full = dt_full;
  a.rho_bar = rho_bar;
  a.rtol = field_rtol;
  a.exact_scan = exact_scan;
  a.status = c->d_status;
  cudaError_t e = pk::launch_chain(a, S(stream));
  if (e != cudaSuccess) return cuda_fail(c, e, "chain launch");
  return PK_OK;
}

int32_t pk_field(pk_ctx* c, int32_t B, const double* rho, const double* rho_bar, double* E,
                 double field_rtol, int32_t exact_scan, void* stream) {
  if (!c || B < 1 || !rho || !rho_bar || !E) return fail(c, PK_ERR_BAD_ARG, "pk_field: bad argument");
  cudaSetDevice(c->device);
  int r = ensure(c, B);
  if (r) return r;
  pk::FineArgs w{};
  bind_ws(c, w);
  pk::FieldArgs a{};
  a.m = c->m;
  a.B = B;
  a.exact_scan = exact_scan;
  a.rho = rho;
  a.rho_bar = rho_bar;
  a.E = E;
  a.src = w.tA;
  a.rtol = field_rtol;
  a.status = c->d_status;
  cudaError_t e = pk::launch_field(a, S(stream));
  if (e != cudaSuccess) return cuda_fail(c, e, "field launch");
  return PK_OK;
}

int32_t pk_lift(pk_ctx* c, int32_t B, const double* rho, const double* E, const double* dE_dt,
                const double* rho_bar, const double* neg_eps, const double* eps2, int32_t order,
                int32_t time_elim, int32_t project, double* g_out, void* stream) {
  if (!c || B < 1 || !rho || !E || !rho_bar || !neg_eps || !eps2 || !g_out)
    return fail(c, PK_ERR_BAD_ARG, "pk_lift: bad argument");
  if (order != 1 && order != 2) return fail(c, PK_ERR_BAD_LIFT, "lift order must be 1 or 2");
  if (order == 2 && time_elim != 0 && time_elim != 1)
    return fail(c, PK_ERR_BAD_LIFT, "time_elim must be 'leading' or 'higher_order'");
  cudaSetDevice(c->device);
  int r = ensure(c, B);
  if (r) return r;
  pk::FineArgs w{};
  bind_ws(c, w);
  pk::LiftArgs a{};
  a.m = c->m;
  a.B = B;
  a.order = order;
  a.time_elim = time_elim;
  a.project = project;
  a.rho = rho;
  a.E = E;
  a.dE_dt = dE_dt;
  a.rho_bar = rho_bar;
  a.neg_eps = neg_eps;
  a.eps2 = eps2;
  a.g_out = g_out;
  a.J = w.J;
  a.tA = w.tA;
  a.tB = w.tB;
  a.tC = w.tC;
  a.tD = w.tD;
  a.tE = w.tE;
  cudaError_t e = pk::launch_lift(a, S(stream));
  if (e != cudaSuccess) return cuda_fail(c, e, "lift launch");
  return PK_OK;
}

int32_t pk_jump(pk_ctx* c, int64_t n, const double* a, const double* b, double* out, void* stream) {
  if (!c || n < 1 || !a || !b || !out) return fail(c, PK_ERR_BAD_ARG, "pk_jump: bad argument");
  cudaSetDevice(c->device);
  cudaError_t e = pk::launch_jump(n, a, b, out, c->d_status, S(stream));
  if (e != cudaSuccess) return cuda_fail(c, e, "jump launch");
  return PK_OK;
}

int32_t pk_fine_cancel(pk_ctx* c, void* stream) {
  if (!c) return PK_ERR_BAD_ARG;
  cudaSetDevice(c->device);
  // (bytes 0x01: a non-zero int) in the order of `stream` -- NOT the stream of
  // the launch to cancel, which is busy with it
  if (cudaMemsetAsync(c->d_cancel, 1, sizeof(int), S(stream)) != cudaSuccess)
    return cuda_fail(c, cudaGetLastError(), "pk_fine_cancel");
  return PK_OK;
}

int32_t pk_status_store(pk_ctx* c, double* dst, int32_t clear, void* stream) {
  if (!c || !dst) return fail(c, PK_ERR_BAD_ARG, "pk_status_store: bad argument");
  cudaSetDevice(c->device);
  cudaError_t e = pk::launch_status_store(c->d_status, dst, clear, S(stream));
  if (e != cudaSuccess) return cuda_fail(c, e, "status store launch");
  return PK_OK;
}

int32_t pk_remainder(pk_ctx* c, int32_t B, const double* rho, const double* E,
                     const double* E_prev, const double* dtE_c, double dt, const double* rho_bar,
                     double* R, void* stream) {
  if (!c || B < 1 || !rho || !E || !rho_bar || !R || (!E_prev && !dtE_c))
    return fail(c, PK_ERR_BAD_ARG, "pk_remainder: bad argument");
  if (c->m.nx < 7) return fail(c, PK_ERR_MESH_TOO_SMALL, "stencils need at least 7 points");
  cudaSetDevice(c->device);
  pk::IndArgs a{};
  a.m = c->m;
  a.B = B;
  a.rho = rho;
  a.E = E;
  a.E_prev = E_prev;
  a.dtE_c = dtE_c;
  a.dt = dt;
  a.rho_bar = rho_bar;
  a.R = R;
  cudaError_t e = pk::launch_indicators(a, 0, S(stream));
  if (e != cudaSuccess) return cuda_fail(c, e, "remainder launch");
  return PK_OK;
}

int32_t pk_perturbation(pk_ctx* c, int32_t B, const double* g, double* gnorm, void* stream) {
  if (!c || B < 1 || !g || !gnorm) return fail(c, PK_ERR_BAD_ARG, "pk_perturbation: bad argument");
  cudaSetDevice(c->device);
  pk::IndArgs a{};
  a.m = c->m;
  a.B = B;
  a.g = g;
  a.gnorm = gnorm;
  cudaError_t e = pk::launch_indicators(a, 1, S(stream));
  if (e != cudaSuccess) return cuda_fail(c, e, "perturbation launch");
  return PK_OK;
}

int32_t pk_labels(pk_ctx* c, int32_t B, const double* R, const double* gnorm, double delta0,
                  double eta0, int32_t combine_and, uint8_t* kc, uint8_t* ki, void* stream) {
  if (!c || B < 1 || !R || !gnorm || !kc || !ki)
    return fail(c, PK_ERR_BAD_ARG, "pk_labels: bad argument");
  cudaSetDevice(c->device);
  pk::IndArgs a{};
  a.m = c->m;
  a.B = B;
  a.Rin = R;
  a.gin = gnorm;
  a.delta0 = delta0;
  a.eta0 = eta0;
  a.combine_and = combine_and;
  a.kc = kc;
  a.ki = ki;
  cudaError_t e = pk::launch_indicators(a, 2, S(stream));
  if (e != cudaSuccess) return cuda_fail(c, e, "labels launch");
  return PK_OK;
}

int32_t pk_diag_qdiv(pk_ctx* c, int64_t n, const double* x, double* out, void* stream) {
  if (!c || n < 1 || !x || !out) return fail(c, PK_ERR_BAD_ARG, "pk_diag_qdiv: bad argument");
  cudaSetDevice(c->device);
  cudaError_t e = pk::launch_qdiv(n, x, out, c->m.dx, c->m.rdx, S(stream));
  if (e != cudaSuccess) return cuda_fail(c, e, "qdiv launch");
  return PK_OK;
}

int32_t pk_maxdiff(pk_ctx* c, int64_t n, const double* a, const double* b, double* err,
                   void* stream) {
  if (!c || n < 1 || !a || !b || !err) return fail(c, PK_ERR_BAD_ARG, "pk_maxdiff: bad argument");
  cudaSetDevice(c->device);
  cudaError_t e = pk::launch_maxdiff(n, a, b, err, c->d_status, S(stream));
  if (e != cudaSuccess) return cuda_fail(c, e, "maxdiff launch");
  return PK_OK;
}

}  // extern "C"
