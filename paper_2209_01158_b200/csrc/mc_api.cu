// mc_api.cu — host side of libmc: the C ABI of include/mc.h.
//
// Setup (mc_set_continuum / mc_set_coupling, finalised lazily before the first step)
// derives the operator arrays of Eq. app-mc from the physical
// inputs in native C++ and uploads them once; every step is one cooperative launch
// of the sm_100a step kernel (mc_kernels.cu).  Readings C1-C15 of DESIGN.md §3.
#ifndef MC_NVTX
#define MC_NVTX 1                          // NVTX ranges `mc_step`, `mc_run` and per-solve marks `pcg[a]`
#endif
#if MC_NVTX
#include <nvtx3/nvToolsExt.h>
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
#else
struct NvtxRange {
  explicit NvtxRange(const char*) {}
};
#endif
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "mc_internal.h"
#include "mc_nlmc.h"

using namespace mc;

namespace {

constexpr int64_t kLargeRows = int64_t(2) << 20;   // "bandwidth-bound" solve
#if MC_CHECK
constexpr size_t kGuardBytes = 256;
constexpr int kGuardByte = 0xA5;
#endif
constexpr int kPlanSteps = 3;                        // D-scheme steps after which the CTA plan is frozen
constexpr int kRunBatch = 256;                       // mc_run: steps enqueued per synchronisation
constexpr int64_t kOneCtaWork = 0;                   // rows + stored entries below which a solve gets one CTA

struct HostCont {
  bool set = false;
  int32_t kind = 0;
  int64_t n = 0;
  int32_t nx = 0, ny = 0;
  double h = 0.0;
  std::vector<double> mtau, dbase, F, u0, tsum, measure;
  std::vector<double> mass, dbd, dwell;        // m = c|cell|; non-edge diagonal of D; well terms (NLMC)
  std::vector<double> Tx, Ty;                  // grid
  std::vector<int32_t> rowptr, col;            // graph, local columns
  std::vector<double> val;                     // graph per-entry T (empty -> uniform)
  double Tconst = 0.0;
  double rtol = 0.0;                           // per-continuum CG tolerance (D-scheme)
  int64_t col_count = 0;                       // graph: stored off-diagonal entries
  int64_t estride = 0;                         // graph: ELL stride
  bool bj = false;                             // graph: block-Jacobi preconditioner (mc_set_preconditioner)
  std::vector<int32_t> perm, inv;              // graph: internal position -> caller index, inverse
  int maxdeg = 0;                              // graph: largest neighbour count
  bool anyfixed = false;                       // graph: has fixed (Dirichlet) cells
  std::vector<uint8_t> fixed;                  // graph Dirichlet DOFs
  std::vector<double> gfix;
};

struct HostCoupling {
  int32_t a = 0, b = 0;
  std::vector<int32_t> i, j;
  std::vector<double> s;
};

struct Plan {
  int nphases = 0, ngroups = 0;
  Group grp[MC_MAX_CONTINUA];
  std::vector<Item> items;
  bool valid = false;
};

}  // namespace

struct mc_ctx {
  mc_options opt{};
  int32_t L = 0;
  std::string err;
  HostCont hc[MC_MAX_CONTINUA];
  std::vector<HostCoupling> cpl;
  bool finalized = false;
  cudaStream_t stream = nullptr;
  int sms = 0, occ = 0, total_ctas = 0;
  // device
  int64_t off[MC_MAX_CONTINUA + 1] = {0};
  int64_t N = 0;
  double* u[2] = {nullptr, nullptr};
  double* r[2] = {nullptr, nullptr};
  double* p[2] = {nullptr, nullptr};
  double* q[2] = {nullptr, nullptr};
  double *dinv = nullptr, *dsD = nullptr, *dsC = nullptr, *mtau = nullptr, *F = nullptr;
  int32_t *cptr = nullptr, *cidx = nullptr;
  double* cval = nullptr;
  double* Tx[MC_MAX_CONTINUA] = {nullptr};
  double* Ty[MC_MAX_CONTINUA] = {nullptr};
  int32_t* rowptr[MC_MAX_CONTINUA] = {nullptr};
  int32_t* col[MC_MAX_CONTINUA] = {nullptr};
  double* val[MC_MAX_CONTINUA] = {nullptr};
  int32_t* ecol[MC_MAX_CONTINUA] = {nullptr};
  int32_t* perm[MC_MAX_CONTINUA] = {nullptr};   // graph: internal -> caller numbering
  double* bstat[MC_MAX_CONTINUA] = {nullptr};                // chunk-blocked streaming ELL pass: static blocks
  double* rrec[MC_MAX_CONTINUA][2] = {{nullptr, nullptr}};   // resident pass: published records (allocated on first use)
  double* bdyn[MC_MAX_CONTINUA][2] = {{nullptr, nullptr}};   //   and CG-state blocks (allocated on first use)
  double* tinv[MC_MAX_CONTINUA] = {nullptr};    // bj: chunk Thomas factors
  double* tcp[MC_MAX_CONTINUA] = {nullptr};
  double* tem[MC_MAX_CONTINUA] = {nullptr};
  int32_t precond = 0;                           // MC_PRECOND_*
  double* scratch = nullptr;                     // state I/O staging (max graph n)
  double* partials = nullptr;
  SyncBlock* sync = nullptr;
  GroupOut* gout = nullptr;
  int32_t* cur = nullptr;
  int32_t* fail = nullptr;
  mc_step_report* rep = nullptr;
  Item* items = nullptr;
  size_t items_cap = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  int32_t cur_host = 0;
  int32_t step_no = 0;
  int64_t last_iters[MC_MAX_CONTINUA] = {0};
  // D-scheme CTA plan: re-chosen from the last step's iteration counts until every solve
  // has a history (at most kPlanSteps steps), then frozen, so that mc_run can enqueue
  // steps without reading anything back and mc_step follows bitwise the same path
  int64_t plan_iters[MC_MAX_CONTINUA] = {0};
  int32_t d_steps = 0;
  int32_t path_mask = 0;                       // MC_PATH_* per continuum of the last enqueued step
  bool d_frozen = false;
  // mc_run: reports and events of one batch of back-to-back steps
  mc_step_report* rep_run = nullptr;
  std::vector<cudaEvent_t> run_ev;
  Plan plan[4];                                 // by scheme
  int32_t korder[MC_MAX_CONTINUA] = {0};        // continua by ascending permeability
  bool has_korder = false;
  int uploaded_plan = -1;                       // scheme whose items are on device
  std::vector<void*> allocs;
  std::vector<std::pair<void*, size_t>> guards;   // MC_CHECK builds: (array, bytes) with guard bytes behind
};

static std::string g_create_err;

namespace {

mc_status fail(mc_ctx* c, mc_status st, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (c) c->err = buf;
  else g_create_err = buf;
  return st;
}

#define CUDA_TRY(c, call)                                                                     \
  do {                                                                                        \
    cudaError_t e_ = (call);                                                                  \
    if (e_ != cudaSuccess)                                                                    \
      return fail((c), e_ == cudaErrorMemoryAllocation ? MC_ERR_NOMEM : MC_ERR_CUDA,          \
                  "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__);       \
  } while (0)

template <class T>
mc_status dev_alloc(mc_ctx* c, T** p, size_t count) {
  void* v = nullptr;
  const size_t bytes = std::max<size_t>(count, 1) * sizeof(T);
#if MC_CHECK
  // checked build: 256 guard bytes after every device array, verified by mc_debug_check
  CUDA_TRY(c, cudaMalloc(&v, bytes + kGuardBytes));
  CUDA_TRY(c, cudaMemset(static_cast<char*>(v) + bytes, kGuardByte, kGuardBytes));
  c->guards.emplace_back(v, bytes);
#else
  CUDA_TRY(c, cudaMalloc(&v, bytes));
#endif
  c->allocs.push_back(v);
  *p = static_cast<T*>(v);
  return MC_OK;
}

// copy `count` elements from a host or device pointer into a host vector
template <class T>
mc_status fetch(mc_ctx* c, std::vector<T>& dst, const T* src, int64_t count) {
  dst.resize((size_t)count);
  if (count == 0) return MC_OK;
  CUDA_TRY(c, cudaMemcpy(dst.data(), src, (size_t)count * sizeof(T), cudaMemcpyDefault));
  return MC_OK;
}

template <class T>
mc_status upload(mc_ctx* c, T** dst, const std::vector<T>& src) {
  mc_status st = dev_alloc(c, dst, src.size());
  if (st != MC_OK) return st;
  if (!src.empty())
    CUDA_TRY(c, cudaMemcpyAsync(*dst, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice,
                                c->stream));
  return MC_OK;
}

bool finite_nonneg(double v) { return std::isfinite(v) && v >= 0.0; }

mc_status field(mc_ctx* c, std::vector<double>& out, const double* ptr, double cst, int64_t n,
                const char* name, bool positive) {
  if (ptr) {
    mc_status st = fetch(c, out, ptr, n);
    if (st != MC_OK) return st;
  } else {
    out.assign((size_t)n, cst);
  }
  for (int64_t i = 0; i < n; ++i) {
    const double v = out[(size_t)i];
    if (!finite_nonneg(v) || (positive && !(v > 0.0)))
      return fail(c, MC_ERR_ARG, "%s[%lld] = %g is not %s", name, (long long)i, v,
                  positive ? "finite and > 0" : "finite and >= 0");
  }
  return MC_OK;
}

double harmonic(double a, double b) { return (a + b) > 0.0 ? 2.0 * a * b / (a + b) : 0.0; }

}  // namespace

// ====================================================================== create / destroy
extern "C" int32_t mc_abi_version(void) { return MC_ABI_VERSION; }

extern "C" const char* mc_error_string(const mc_ctx* ctx) {
  return ctx ? ctx->err.c_str() : g_create_err.c_str();
}

extern "C" mc_status mc_create(mc_ctx** out, int32_t n_continua, const mc_options* opt) {
  if (!out) return fail(nullptr, MC_ERR_ARG, "out is NULL");
  *out = nullptr;
  if (n_continua < 1 || n_continua > MC_MAX_CONTINUA)
    return fail(nullptr, MC_ERR_ARG, "n_continua = %d not in [1, %d]", n_continua, MC_MAX_CONTINUA);
  if (!opt) return fail(nullptr, MC_ERR_ARG, "opt is NULL");
  if (!(std::isfinite(opt->tau) && opt->tau > 0.0))
    return fail(nullptr, MC_ERR_ARG, "tau = %g must be finite and > 0", opt->tau);
  if (!std::isfinite(opt->rtol) || opt->rtol >= 1.0)
    return fail(nullptr, MC_ERR_ARG, "rtol = %g must be < 1", opt->rtol);
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0)
    return fail(nullptr, MC_ERR_CUDA, "no CUDA device: %s", cudaGetErrorString(e));
  if (opt->device < 0 || opt->device >= ndev)
    return fail(nullptr, MC_ERR_ARG, "device %d not in [0, %d)", opt->device, ndev);
  mc_ctx* c = new mc_ctx();
  c->opt = *opt;
  if (!(c->opt.rtol > 0.0)) c->opt.rtol = 1e-12;
  c->L = n_continua;
  c->stream = static_cast<cudaStream_t>(opt->stream);
  e = cudaSetDevice(opt->device);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, opt->device);
  if (e == cudaSuccess) e = step_kernel_occupancy(&c->occ);
  if (e == cudaSuccess) e = cudaEventCreate(&c->ev0);
  if (e == cudaSuccess) e = cudaEventCreate(&c->ev1);
  if (e != cudaSuccess) {
    fail(nullptr, MC_ERR_CUDA, "device setup: %s", cudaGetErrorString(e));
    delete c;
    return MC_ERR_CUDA;
  }
  int coop = 0;
  cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, opt->device);
  if (!coop || c->occ < 1) {
    fail(nullptr, MC_ERR_CUDA, "device lacks cooperative launch (occupancy %d)", c->occ);
    delete c;
    return MC_ERR_CUDA;
  }
  const int maxc = c->sms * c->occ;
  c->total_ctas = (opt->ctas > 0) ? std::min(opt->ctas, maxc) : maxc;
  *out = c;
  return MC_OK;
}

extern "C" mc_status mc_destroy(mc_ctx* c) {
  if (!c) return MC_OK;
  cudaStreamSynchronize(c->stream);
  for (void* v : c->allocs) cudaFree(v);
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->ev1) cudaEventDestroy(c->ev1);
  for (cudaEvent_t e : c->run_ev) cudaEventDestroy(e);
  delete c;
  return MC_OK;
}

#if MC_CHECK
// checked build only (libmc_check.so, not declared in include/mc.h): number of device arrays
// whose guard bytes were overwritten -- an out-of-bounds write of some kernel
extern "C" int32_t mc_debug_check(mc_ctx* c) {
  if (!c) return -1;
  if (cudaStreamSynchronize(c->stream) != cudaSuccess) return -2;
  int32_t bad = 0;
  std::vector<unsigned char> h(kGuardBytes);
  for (auto& g : c->guards) {
    if (cudaMemcpy(h.data(), static_cast<char*>(g.first) + g.second, kGuardBytes, cudaMemcpyDeviceToHost) != cudaSuccess)
      return -2;
    for (unsigned char b : h)
      if (b != (unsigned char)kGuardByte) {
        ++bad;
        break;
      }
  }
  return bad;
}
#endif

extern "C" int64_t mc_size(const mc_ctx* c, int32_t alpha) {
  if (!c) return -1;
  if (alpha < 0) {
    int64_t s = 0;
    for (int a = 0; a < c->L; ++a) s += c->hc[a].n;
    return s;
  }
  if (alpha >= c->L) return -1;
  return c->hc[alpha].n;
}

// ====================================================================== continua
// wells f = q_w (p_w - p): q_w |cell| on the diagonal (both schemes), q_w p_w |cell| in F
static mc_status add_wells(mc_ctx* c, HostCont& H, const mc_continuum_desc* d, double meas_const) {
  if (!d->well_q) return MC_OK;
  if (!std::isfinite(d->well_p)) return fail(c, MC_ERR_ARG, "well_p not finite");
  std::vector<double> q;
  mc_status st = field(c, q, d->well_q, 0.0, H.n, "well_q", false);
  if (st != MC_OK) return st;
  for (int64_t i = 0; i < H.n; ++i) {
    const size_t s = (size_t)i;
    if (!H.fixed.empty() && H.fixed[s]) continue;
    const double w = q[s] * (meas_const > 0.0 ? meas_const : H.measure[s]);
    H.dbase[s] += w;
    H.dwell[s] += w;
    H.F[s] += w * d->well_p;
  }
  return MC_OK;
}

static mc_status set_grid(mc_ctx* c, HostCont& H, const mc_continuum_desc* d) {
  const int64_t n = d->n;
  if (d->nx < 1 || d->ny < 1 || (int64_t)d->nx * d->ny != n)
    return fail(c, MC_ERR_ARG, "grid nx*ny = %d*%d != n = %lld", d->nx, d->ny, (long long)n);
  if (!(std::isfinite(d->h) && d->h > 0.0)) return fail(c, MC_ERR_ARG, "grid h = %g must be > 0", d->h);
  if ((d->bc_left != 0 && d->bc_left != 1) || (d->bc_right != 0 && d->bc_right != 1))
    return fail(c, MC_ERR_ARG, "bc_left/bc_right must be 0 (no-flow) or 1 (Dirichlet)");
  if ((d->bc_left && !std::isfinite(d->g_left)) || (d->bc_right && !std::isfinite(d->g_right)))
    return fail(c, MC_ERR_ARG, "Dirichlet value not finite");
  const int nx = d->nx, ny = d->ny;
  const double h = d->h, tau = c->opt.tau, area = h * h;   // |cell| = h^2 (reading C1)
  std::vector<double> k, cc, f;
  mc_status st;
  if ((st = field(c, k, d->k, d->k_const, n, "k", false)) != MC_OK) return st;
  if ((st = field(c, cc, d->c, d->c_const, n, "c", false)) != MC_OK) return st;
  if (d->f) {
    if ((st = fetch(c, f, d->f, n)) != MC_OK) return st;
    for (double v : f)
      if (!std::isfinite(v)) return fail(c, MC_ERR_ARG, "source f not finite");
  }
  H.kind = KIND_GRID;
  H.n = n;
  H.nx = nx;
  H.ny = ny;
  H.h = h;
  H.Tx.assign((size_t)n, 0.0);
  H.Ty.assign((size_t)n, 0.0);
  H.tsum.assign((size_t)n, 0.0);
  H.mtau.resize((size_t)n);
  H.dbase.resize((size_t)n);
  H.F.assign((size_t)n, 0.0);
  H.measure.assign((size_t)n, area);
  H.mass.assign((size_t)n, 0.0);
  H.dbd.assign((size_t)n, 0.0);
  H.dwell.assign((size_t)n, 0.0);
  const bool kc = (d->k == nullptr);
  // T = k |E|/d, |E| = d = h; harmonic mean for a k field (reading C2)
  for (int iy = 0; iy < ny; ++iy)
    for (int ix = 0; ix < nx; ++ix) {
      const int64_t i = (int64_t)iy * nx + ix;
      if (ix + 1 < nx) H.Tx[(size_t)i] = kc ? d->k_const : harmonic(k[(size_t)i], k[(size_t)i + 1]);
      if (iy + 1 < ny) H.Ty[(size_t)i] = kc ? d->k_const : harmonic(k[(size_t)i], k[(size_t)(i + nx)]);
    }
  for (int iy = 0; iy < ny; ++iy)
    for (int ix = 0; ix < nx; ++ix) {
      const size_t i = (size_t)iy * nx + ix;
      double ts = H.Tx[i] + H.Ty[i];
      if (ix > 0) ts += H.Tx[i - 1];
      if (iy > 0) ts += H.Ty[i - nx];
      H.tsum[i] = ts;
      const double m = cc[i] * area;                       // m = c |cell|
      H.mtau[i] = m / tau;
      double db = 0.0, Fi = f.empty() ? 0.0 : f[i] * area;  // F = f |cell|
      // Dirichlet face, half-cell distance: T_b = k h / (h/2) (reading C3)
      if (ix == 0 && d->bc_left) {
        const double tb = k[i] * h / (h / 2.0);
        db += tb;
        Fi += tb * d->g_left;
      }
      if (ix == nx - 1 && d->bc_right) {
        const double tb = k[i] * h / (h / 2.0);
        db += tb;
        Fi += tb * d->g_right;
      }
      H.dbase[i] = H.mtau[i] + db;
      H.F[i] = Fi;
      H.mass[i] = m;
      H.dbd[i] = db;
    }
  return add_wells(c, H, d, area);
}

static mc_status set_graph(mc_ctx* c, HostCont& H, const mc_continuum_desc* d) {
  const int64_t n = d->n, E = d->n_edges;
  if (n > INT32_MAX - 1) return fail(c, MC_ERR_ARG, "graph n too large for int32 indices");
  if (E < 0) return fail(c, MC_ERR_ARG, "n_edges < 0");
  if (E > 0 && (!d->edge_i || !d->edge_j)) return fail(c, MC_ERR_ARG, "edge_i / edge_j NULL");
  if (E > 0 && !d->edge_t && !(std::isfinite(d->edge_geom) && d->edge_geom >= 0.0))
    return fail(c, MC_ERR_ARG, "edge_geom = %g must be finite and >= 0", d->edge_geom);
  const double tau = c->opt.tau;
  std::vector<double> k, cc, f, meas, et, dir;
  std::vector<int32_t> ei, ej;
  mc_status st;
  if ((st = field(c, k, d->k, d->k_const, n, "k", false)) != MC_OK) return st;
  if ((st = field(c, cc, d->c, d->c_const, n, "c", false)) != MC_OK) return st;
  if ((st = field(c, meas, d->measure, d->measure_const, n, "measure", true)) != MC_OK) return st;
  if (d->f) {
    if ((st = fetch(c, f, d->f, n)) != MC_OK) return st;
    for (double v : f)
      if (!std::isfinite(v)) return fail(c, MC_ERR_ARG, "source f not finite");
  }
  if ((st = fetch(c, ei, d->edge_i, E)) != MC_OK) return st;
  if ((st = fetch(c, ej, d->edge_j, E)) != MC_OK) return st;
  if (d->edge_t) {
    if ((st = fetch(c, et, d->edge_t, E)) != MC_OK) return st;
  }
  if (d->dirichlet) {
    if ((st = fetch(c, dir, d->dirichlet, n)) != MC_OK) return st;
    for (double v : dir)
      if (std::isinf(v)) return fail(c, MC_ERR_ARG, "dirichlet value infinite");
  }
  // edges: range, self-loops, duplicates
  std::vector<int64_t> key((size_t)E);
  for (int64_t e = 0; e < E; ++e) {
    const int32_t a = ei[(size_t)e], b = ej[(size_t)e];
    if (a < 0 || b < 0 || a >= n || b >= n || a == b)
      return fail(c, MC_ERR_ARG, "edge %lld = (%d, %d) out of range or self-loop", (long long)e, a, b);
    key[(size_t)e] = (int64_t)std::min(a, b) * n + std::max(a, b);
    if (d->edge_t && !(d->signed_edges ? std::isfinite(et[(size_t)e]) : finite_nonneg(et[(size_t)e])))
      return fail(c, MC_ERR_ARG, "edge_t[%lld] = %g must be finite%s", (long long)e, et[(size_t)e],
                  d->signed_edges ? "" : " and >= 0");
  }
  {
    std::vector<int64_t> ks(key);
    std::sort(ks.begin(), ks.end());
    if (std::adjacent_find(ks.begin(), ks.end()) != ks.end())
      return fail(c, MC_ERR_ARG, "duplicate edge in graph continuum");
  }
  H.kind = KIND_GRAPH;
  H.n = n;
  H.measure = meas;
  H.mtau.resize((size_t)n);
  H.dbase.resize((size_t)n);
  H.F.assign((size_t)n, 0.0);
  H.tsum.assign((size_t)n, 0.0);
  H.fixed.assign((size_t)n, 0);
  H.gfix.assign((size_t)n, 0.0);
  H.mass.assign((size_t)n, 0.0);
  H.dbd.assign((size_t)n, 0.0);
  H.dwell.assign((size_t)n, 0.0);
  std::vector<double> dx;
  if (d->diag_extra) {
    if ((st = fetch(c, dx, d->diag_extra, n)) != MC_OK) return st;
    for (double v : dx)
      if (!std::isfinite(v)) return fail(c, MC_ERR_ARG, "diag_extra not finite");
  }
  for (int64_t i = 0; i < n; ++i) {
    const size_t s = (size_t)i;
    H.mass[s] = cc[s] * meas[s];
    H.mtau[s] = cc[s] * meas[s] / tau;                       // m = c |cell|
    H.dbase[s] = H.mtau[s];
    if (!dx.empty()) {                                       // explicit diagonal term (ABI 2)
      H.dbase[s] += dx[s];
      H.dbd[s] += dx[s];
    }
    H.F[s] = f.empty() ? 0.0 : f[s] * meas[s];
    if (!dir.empty() && !std::isnan(dir[s])) {                // fixed DOF: identity row (C12)
      H.fixed[s] = 1;
      H.gfix[s] = dir[s];
      H.mtau[s] = 0.0;
      H.mass[s] = 0.0;
      H.dbase[s] = 1.0;
      H.F[s] = dir[s];
    }
  }
  // edge transmissibilities T_e = k |E|/d, harmonic k for a field
  std::vector<double> T((size_t)E);
  const bool kc = (d->k == nullptr);
  for (int64_t e = 0; e < E; ++e) {
    const int32_t a = ei[(size_t)e], b = ej[(size_t)e];
    T[(size_t)e] = d->edge_t ? et[(size_t)e]
                             : (kc ? d->k_const : harmonic(k[(size_t)a], k[(size_t)b])) * d->edge_geom;
  }
  // CSR of free-free edges; edges to fixed DOFs eliminated into diagonal and F (C12)
  std::vector<int32_t> cnt((size_t)n + 1, 0);
  for (int64_t e = 0; e < E; ++e) {
    const int32_t a = ei[(size_t)e], b = ej[(size_t)e];
    const bool fa = H.fixed[(size_t)a], fb = H.fixed[(size_t)b];
    if (!fa && !fb) {
      cnt[(size_t)a + 1]++;
      cnt[(size_t)b + 1]++;
    } else if (!fa && fb) {
      H.dbase[(size_t)a] += T[(size_t)e];
      H.dbd[(size_t)a] += T[(size_t)e];
      H.F[(size_t)a] += T[(size_t)e] * H.gfix[(size_t)b];
    } else if (fa && !fb) {
      H.dbase[(size_t)b] += T[(size_t)e];
      H.dbd[(size_t)b] += T[(size_t)e];
      H.F[(size_t)b] += T[(size_t)e] * H.gfix[(size_t)a];
    }
  }
  for (size_t i = 0; i < (size_t)n; ++i) cnt[i + 1] += cnt[i];
  if (cnt[(size_t)n] > INT32_MAX / 2) return fail(c, MC_ERR_ARG, "graph too large for int32 CSR");
  H.rowptr = cnt;
  H.col.assign((size_t)cnt[(size_t)n], 0);
  std::vector<double> vals((size_t)cnt[(size_t)n]);
  std::vector<int32_t> pos(cnt.begin(), cnt.end() - 1);
  bool uniform = true;
  double t0 = E > 0 ? T[0] : 0.0;
  for (int64_t e = 0; e < E; ++e) {
    const int32_t a = ei[(size_t)e], b = ej[(size_t)e];
    if (H.fixed[(size_t)a] || H.fixed[(size_t)b]) continue;
    const double t = T[(size_t)e];
    if (t != t0) uniform = false;
    H.col[(size_t)pos[(size_t)a]] = b;
    vals[(size_t)pos[(size_t)a]++] = t;
    H.col[(size_t)pos[(size_t)b]] = a;
    vals[(size_t)pos[(size_t)b]++] = t;
    H.tsum[(size_t)a] += t;
    H.tsum[(size_t)b] += t;
  }
  // sort each row by column (deterministic, cache-friendlier gathers)
  for (int64_t i = 0; i < n; ++i) {
    const int32_t b0 = H.rowptr[(size_t)i], b1 = H.rowptr[(size_t)i + 1];
    std::vector<std::pair<int32_t, double>> row;
    row.reserve((size_t)(b1 - b0));
    for (int32_t e = b0; e < b1; ++e) row.emplace_back(H.col[(size_t)e], vals[(size_t)e]);
    std::sort(row.begin(), row.end());
    for (int32_t e = b0; e < b1; ++e) {
      H.col[(size_t)e] = row[(size_t)(e - b0)].first;
      vals[(size_t)e] = row[(size_t)(e - b0)].second;
    }
  }
  if (uniform) {
    H.val.clear();
    H.Tconst = t0;
  } else {
    H.val = std::move(vals);
    H.Tconst = 0.0;
  }
  return add_wells(c, H, d, 0.0);
}

// Internal numbering of a graph continuum: walk the connection graph in
// chains — start at every endpoint / junction (degree != 2) in caller order, follow
// unvisited neighbours until the chain ends, then sweep what is left (cycles, isolated
// cells).  Along a fracture segment consecutive cells become consecutive rows, so most
// neighbours of a row sit in the same 64-row chunk of the CG pass.
static void chain_order(const HostCont& H, std::vector<int32_t>& perm) {
  const int64_t n = H.n;
  perm.clear();
  perm.reserve((size_t)n);
  std::vector<uint8_t> seen((size_t)n, 0);
  auto deg = [&](int64_t i) { return H.rowptr[(size_t)i + 1] - H.rowptr[(size_t)i]; };
  auto walk = [&](int32_t start) {
    int32_t cur = start;
    while (cur >= 0 && !seen[(size_t)cur]) {
      seen[(size_t)cur] = 1;
      perm.push_back(cur);
      int32_t nxt = -1;
      for (int32_t e = H.rowptr[(size_t)cur]; e < H.rowptr[(size_t)cur + 1]; ++e)
        if (!seen[(size_t)H.col[(size_t)e]]) {
          nxt = H.col[(size_t)e];
          break;
        }
      cur = nxt;
    }
  };
  for (int64_t i = 0; i < n; ++i)
    if (!seen[(size_t)i] && deg(i) != 2) walk((int32_t)i);
  for (int64_t i = 0; i < n; ++i)
    if (!seen[(size_t)i]) walk((int32_t)i);
}

// renumber every per-row array and the CSR of graph continuum H into chain order
// Block-Jacobi (MC_PRECOND_BLOCK) packing: reorder the chains of `perm` (maximal runs of
// connected consecutive cells) so that 64-cell chunks end where chains end: each chunk
// is filled with the longest remaining chain that fits, the longest overall when none
// does.  Fewer chain links cut by chunk boundaries = fewer CG iterations.
static void pack_chains(const HostCont& H, std::vector<int32_t>& perm) {
  const int64_t n = H.n;
  auto linked = [&](int32_t a, int32_t b) {
    for (int32_t e = H.rowptr[(size_t)a]; e < H.rowptr[(size_t)a + 1]; ++e)
      if (H.col[(size_t)e] == b) return true;
    return false;
  };
  std::vector<int64_t> start;
  for (int64_t t = 0; t < n; ++t)
    if (t == 0 || !linked(perm[(size_t)t - 1], perm[(size_t)t])) start.push_back(t);
  start.push_back(n);
  const int nc = (int)start.size() - 1;
  // chains by length (longest first), ties in order of appearance
  std::vector<std::vector<int>> bylen(65);          // 1..64; index 0 unused
  std::vector<int> longer;                           // > 64, longest first
  for (int c = 0; c < nc; ++c) {
    const int64_t L = start[(size_t)c + 1] - start[(size_t)c];
    if (L <= 64) bylen[(size_t)L].push_back(c);
    else longer.push_back(c);
  }
  std::stable_sort(longer.begin(), longer.end(), [&](int x, int y) {
    return start[(size_t)x + 1] - start[(size_t)x] > start[(size_t)y + 1] - start[(size_t)y];
  });
  for (auto& v : bylen) std::reverse(v.begin(), v.end());   // pop_back = first appearance
  std::vector<int32_t> out;
  out.reserve((size_t)n);
  size_t li = 0;
  while ((int64_t)out.size() < n) {
    const int space = 64 - (int)(out.size() % 64);
    int c = -1;
    for (int L = space; L >= 1 && c < 0; --L)
      if (!bylen[(size_t)L].empty()) {
        c = bylen[(size_t)L].back();
        bylen[(size_t)L].pop_back();
      }
    if (c < 0) {                                     // nothing fits: the longest chain left
      if (li < longer.size()) {
        c = longer[li++];
      } else {
        for (int L = 64; L >= 1 && c < 0; --L)
          if (!bylen[(size_t)L].empty()) {
            c = bylen[(size_t)L].back();
            bylen[(size_t)L].pop_back();
          }
      }
    }
    for (int64_t t = start[(size_t)c]; t < start[(size_t)c + 1]; ++t) out.push_back(perm[(size_t)t]);
  }
  perm.swap(out);
}

static void apply_chain_order(HostCont& H) {
  const int64_t n = H.n;
  chain_order(H, H.perm);
  if (H.bj) pack_chains(H, H.perm);
  H.inv.assign((size_t)n, 0);
  for (int64_t t = 0; t < n; ++t) H.inv[(size_t)H.perm[(size_t)t]] = (int32_t)t;
  auto pv = [&](std::vector<double>& v) {
    if (v.empty()) return;
    std::vector<double> w((size_t)n);
    for (int64_t t = 0; t < n; ++t) w[(size_t)t] = v[(size_t)H.perm[(size_t)t]];
    v.swap(w);
  };
  pv(H.mtau);
  pv(H.dbase);
  pv(H.mass);
  pv(H.dbd);
  pv(H.dwell);
  pv(H.F);
  pv(H.u0);
  pv(H.tsum);
  pv(H.measure);
  pv(H.gfix);
  {
    std::vector<uint8_t> w((size_t)n);
    for (int64_t t = 0; t < n; ++t) w[(size_t)t] = H.fixed[(size_t)H.perm[(size_t)t]];
    H.fixed.swap(w);
  }
  std::vector<int32_t> rp((size_t)n + 1, 0), col;
  std::vector<double> val;
  col.reserve(H.col.size());
  if (!H.val.empty()) val.reserve(H.val.size());
  for (int64_t t = 0; t < n; ++t) {
    const int32_t i = H.perm[(size_t)t];
    std::vector<std::pair<int32_t, double>> row;
    for (int32_t e = H.rowptr[(size_t)i]; e < H.rowptr[(size_t)i + 1]; ++e)
      row.emplace_back(H.inv[(size_t)H.col[(size_t)e]], H.val.empty() ? 0.0 : H.val[(size_t)e]);
    std::sort(row.begin(), row.end());
    for (auto& pr : row) {
      col.push_back(pr.first);
      if (!H.val.empty()) val.push_back(pr.second);
    }
    rp[(size_t)t + 1] = (int32_t)col.size();
  }
  H.rowptr.swap(rp);
  H.col.swap(col);
  if (!H.val.empty()) H.val.swap(val);
}

extern "C" mc_status mc_set_continuum(mc_ctx* c, int32_t alpha, const mc_continuum_desc* d) {
  if (!c || !d) return fail(c, MC_ERR_ARG, "NULL argument");
  if (alpha < 0 || alpha >= c->L) return fail(c, MC_ERR_ARG, "alpha = %d not in [0, %d)", alpha, c->L);
  if (c->finalized) return fail(c, MC_ERR_STATE, "continuum %d set after the first step", alpha);
  if (c->hc[alpha].set) return fail(c, MC_ERR_STATE, "continuum %d already set", alpha);
  if (d->n < 1) return fail(c, MC_ERR_ARG, "continuum %d: n = %lld < 1", alpha, (long long)d->n);
  if (d->n > (int64_t)INT32_MAX / 2) return fail(c, MC_ERR_ARG, "continuum %d too large", alpha);
  HostCont H;
  mc_status st;
  if (d->kind == MC_GRID2D) st = set_grid(c, H, d);
  else if (d->kind == MC_GRAPH) st = set_graph(c, H, d);
  else return fail(c, MC_ERR_ARG, "continuum %d: unknown kind %d", alpha, (int)d->kind);
  if (st != MC_OK) {
    c->err = "continuum " + std::to_string(alpha) + ": " + c->err;
    return st;
  }
  if (d->u0) {
    if ((st = fetch(c, H.u0, d->u0, d->n)) != MC_OK) return st;
    for (double v : H.u0)
      if (!std::isfinite(v)) return fail(c, MC_ERR_ARG, "continuum %d: u0 not finite", alpha);
  } else {
    H.u0.assign((size_t)d->n, 0.0);
  }
  if (!std::isfinite(d->rtol) || d->rtol >= 1.0)
    return fail(c, MC_ERR_ARG, "continuum %d: rtol = %g must be < 1", alpha, d->rtol);
  H.rtol = d->rtol > 0.0 ? d->rtol : c->opt.rtol;
  if (H.kind == KIND_GRAPH) {
    for (size_t i = 0; i < H.fixed.size(); ++i)
      if (H.fixed[i]) H.u0[i] = H.gfix[i];                     // fixed DOF starts at g (C12)
    // optional internal chain numbering for sparse (<= 4 neighbours) graphs, MC_CHAIN=1.
    // Off by default: measured slower on the config-1/4 fracture networks than the
    // caller's host-cell order.
    int maxdeg = 0;
    for (int64_t i = 0; i < H.n; ++i) maxdeg = std::max(maxdeg, H.rowptr[(size_t)i + 1] - H.rowptr[(size_t)i]);
    const char* ch = getenv("MC_CHAIN");
    H.maxdeg = maxdeg;
    H.anyfixed = std::any_of(H.fixed.begin(), H.fixed.end(), [](uint8_t f) { return f != 0; });
    H.bj = (c->precond == MC_PRECOND_BLOCK) && maxdeg <= 4 && H.val.empty();
    if (maxdeg <= 4 && ((ch && ch[0] == '1') || H.bj)) apply_chain_order(H);
  }
  H.set = true;
  c->hc[alpha] = std::move(H);
  return MC_OK;
}

// ====================================================================== couplings
extern "C" mc_status mc_set_coupling(mc_ctx* c, const mc_coupling_desc* d) {
  if (!c || !d) return fail(c, MC_ERR_ARG, "NULL argument");
  if (c->finalized) return fail(c, MC_ERR_STATE, "coupling set after the first step");
  if (d->a < 0 || d->b < 0 || d->a >= c->L || d->b >= c->L || d->a == d->b)
    return fail(c, MC_ERR_ARG, "coupling pair (%d, %d) invalid", d->a, d->b);
  for (int a = 0; a < c->L; ++a)
    if (!c->hc[a].set) return fail(c, MC_ERR_STATE, "coupling before continuum %d was set", a);
  if (d->nnz < 0) return fail(c, MC_ERR_ARG, "coupling nnz < 0");
  const HostCont& A = c->hc[d->a];
  const HostCont& B = c->hc[d->b];
  HostCoupling hcp;
  hcp.a = d->a;
  hcp.b = d->b;
  mc_status st;
  const int64_t m = d->nnz;
  if (d->i_a) {
    if ((st = fetch(c, hcp.i, d->i_a, m)) != MC_OK) return st;
  } else {
    if (m > A.n) return fail(c, MC_ERR_ARG, "identity coupling nnz %lld > n_a", (long long)m);
    hcp.i.resize((size_t)m);
    std::iota(hcp.i.begin(), hcp.i.end(), 0);
  }
  if (d->j_b) {
    if ((st = fetch(c, hcp.j, d->j_b, m)) != MC_OK) return st;
  } else {
    if (m > B.n) return fail(c, MC_ERR_ARG, "identity coupling nnz %lld > n_b", (long long)m);
    hcp.j.resize((size_t)m);
    std::iota(hcp.j.begin(), hcp.j.end(), 0);
  }
  if (d->signed_sigma) {                                    // ABI 2: any finite sigma (NLMC)
    if (d->sigma) {
      if ((st = fetch(c, hcp.s, d->sigma, m)) != MC_OK) return st;
    } else {
      hcp.s.assign((size_t)m, d->sigma_const);
    }
    for (double v : hcp.s)
      if (!std::isfinite(v)) return fail(c, MC_ERR_ARG, "sigma not finite");
  } else if ((st = field(c, hcp.s, d->sigma, d->sigma_const, m, "sigma", false)) != MC_OK) {
    return st;
  }
  for (int64_t e = 0; e < m; ++e) {
    const int32_t i = hcp.i[(size_t)e], j = hcp.j[(size_t)e];
    if (i < 0 || i >= A.n || j < 0 || j >= B.n)
      return fail(c, MC_ERR_ARG, "coupling entry %lld = (%d, %d) out of range", (long long)e, i, j);
    if (!A.inv.empty()) hcp.i[(size_t)e] = A.inv[(size_t)i];              // internal numbering
    if (!B.inv.empty()) hcp.j[(size_t)e] = B.inv[(size_t)j];
    if (d->scale_by_measure) hcp.s[(size_t)e] *= A.measure[(size_t)hcp.i[(size_t)e]];   // sigma |cell| (C9)
  }
  c->cpl.push_back(std::move(hcp));
  return MC_OK;
}

// ====================================================================== finalize
static mc_status finalize(mc_ctx* c) {
  if (c->finalized) return MC_OK;
  for (int a = 0; a < c->L; ++a)
    if (!c->hc[a].set) return fail(c, MC_ERR_STATE, "continuum %d not set", a);
  // padded offsets (256 B) so no cache line is shared by two continua
  int64_t o = 0;
  for (int a = 0; a < c->L; ++a) {
    c->off[a] = o;
    o += (c->hc[a].n + kPadDofs - 1) / kPadDofs * kPadDofs;
  }
  c->off[c->L] = o;
  c->N = o;
  const int64_t N = c->N;
  if (N + 1 > INT32_MAX) return fail(c, MC_ERR_ARG, "total size exceeds int32 indexing");
  const size_t NS = (size_t)N + kSlack;          // staged loads may read up to kSlack past N
  std::vector<double> mtau(NS, 0.0), dbase(NS, 0.0), F(NS, 0.0), u0(NS, 0.0), tsum(NS, 0.0),
      sig(NS, 0.0);
  for (int a = 0; a < c->L; ++a) {
    HostCont& H = c->hc[a];
    const size_t off = (size_t)c->off[a];
    std::copy(H.mtau.begin(), H.mtau.end(), mtau.begin() + off);
    std::copy(H.dbase.begin(), H.dbase.end(), dbase.begin() + off);
    std::copy(H.F.begin(), H.F.end(), F.begin() + off);
    std::copy(H.u0.begin(), H.u0.end(), u0.begin() + off);
    std::copy(H.tsum.begin(), H.tsum.end(), tsum.begin() + off);
  }
  // couplings -> global CSR (both directions); fixed endpoints eliminated (C12)
  std::vector<int32_t> cnt((size_t)N + 1, 0);
  auto fixed = [&](int a, int32_t i) {
    return c->hc[a].kind == KIND_GRAPH && c->hc[a].fixed[(size_t)i];
  };
  for (const HostCoupling& h : c->cpl)
    for (size_t e = 0; e < h.i.size(); ++e) {
      const bool fa = fixed(h.a, h.i[e]), fb = fixed(h.b, h.j[e]);
      if (!fa && !fb) {
        cnt[(size_t)(c->off[h.a] + h.i[e]) + 1]++;
        cnt[(size_t)(c->off[h.b] + h.j[e]) + 1]++;
      }
    }
  for (size_t i = 0; i < (size_t)N; ++i) cnt[i + 1] += cnt[i];
  std::vector<int32_t> cidx((size_t)cnt[(size_t)N]);
  std::vector<double> cval((size_t)cnt[(size_t)N]);
  std::vector<int32_t> pos(cnt.begin(), cnt.end() - 1);
  for (const HostCoupling& h : c->cpl)
    for (size_t e = 0; e < h.i.size(); ++e) {
      const int64_t gi = c->off[h.a] + h.i[e], gj = c->off[h.b] + h.j[e];
      const double s = h.s[e];
      const bool fa = fixed(h.a, h.i[e]), fb = fixed(h.b, h.j[e]);
      if (!fa && !fb) {
        cidx[(size_t)pos[(size_t)gi]] = (int32_t)gj;
        cval[(size_t)pos[(size_t)gi]++] = s;
        cidx[(size_t)pos[(size_t)gj]] = (int32_t)gi;
        cval[(size_t)pos[(size_t)gj]++] = s;
        sig[(size_t)gi] += s;
        sig[(size_t)gj] += s;
      } else if (!fa && fb) {
        dbase[(size_t)gi] += s;
        F[(size_t)gi] += s * c->hc[h.b].gfix[(size_t)h.j[e]];
      } else if (fa && !fb) {
        dbase[(size_t)gj] += s;
        F[(size_t)gj] += s * c->hc[h.a].gfix[(size_t)h.i[e]];
      }
    }
  std::vector<double> dsD(NS, 0.0), dinv(NS, 0.0);
  for (int a = 0; a < c->L; ++a)
    for (int64_t i = 0; i < c->hc[a].n; ++i) {
      const size_t g = (size_t)(c->off[a] + i);
      dsD[g] = dbase[g] + sig[g];
      const double diag = dsD[g] + tsum[g];            // diag(K), Jacobi (reading C14)
      if (!(diag > 0.0) || !std::isfinite(diag))
        return fail(c, MC_ERR_ARG, "continuum %d row %lld: diagonal %g of M/tau + A is not > 0", a,
                    (long long)i, diag);
      dinv[g] = 1.0 / diag;
    }
  mc_status st;
#define UP(dst, src) \
  if ((st = upload(c, &(dst), (src))) != MC_OK) return st
  UP(c->mtau, mtau);
  UP(c->dsC, dbase);
  UP(c->dsD, dsD);
  UP(c->dinv, dinv);
  UP(c->F, F);
  UP(c->cptr, cnt);
  UP(c->cidx, cidx);
  UP(c->cval, cval);
  UP(c->u[0], u0);
  for (int a = 0; a < c->L; ++a) {
    HostCont& H = c->hc[a];
    if (H.kind == KIND_GRID) {
      UP(c->Tx[a], H.Tx);
      UP(c->Ty[a], H.Ty);
    } else {
      std::vector<int32_t> gcol(H.col);
      for (auto& v : gcol) v += (int32_t)c->off[a];
      H.col_count = (int64_t)H.col.size();
      // ELL copy (width 4, k-major) when every row has <= 4 neighbours: one coalesced
      // trip for the structure instead of rowptr -> col
      int maxdeg = 0;
      for (int64_t i = 0; i < H.n; ++i) maxdeg = std::max(maxdeg, H.rowptr[(size_t)i + 1] - H.rowptr[(size_t)i]);
      if (maxdeg <= 4 && H.val.empty()) {
        const int64_t es = (H.n + 63) / 64 * 64 + 64;          // staged 64-row chunks may over-read
        H.estride = es;
        // ELL entries pre-classified against the static 64-row chunk of their row:
        //   -1 none; -2-w: window slot w = j - chunk_start + 2 in [0, 68) (the chunk and its
        //   2-row halo on each side, staged in shared memory); >= 0: global index (far)
        std::vector<int32_t> ell((size_t)(4 * es), -1);
        for (int64_t i = 0; i < H.n; ++i) {
          const int64_t b = i / 64 * 64;
          for (int32_t e = H.rowptr[(size_t)i], k = 0; e < H.rowptr[(size_t)i + 1]; ++e, ++k) {
            const int64_t j = H.col[(size_t)e], w = j - b + 2;
            ell[(size_t)(k * es + i)] = (w >= 0 && w < 68) ? (int32_t)(-2 - w) : (int32_t)(j + c->off[a]);
          }
        }
        UP(c->ecol[a], ell);
        {
          // chunk-blocked static data of the streaming passes (iter_ellb, bjs_pass_s2): per 64-row chunk
          // D^-1 (64) | D-scheme shift (64) | int32 codes [64][4], far neighbours first
          const int64_t nchk = (H.n + 63) / 64;
          std::vector<double> bst((size_t)nchk * kBStat, 0.0);
          for (int64_t m = 0; m < nchk; ++m) {
            int32_t* cp = reinterpret_cast<int32_t*>(&bst[(size_t)(m * kBStat + 128)]);
            for (int q = 0; q < 256; ++q) cp[q] = -1;
          }
          for (int64_t i = 0; i < H.n; ++i) {
            const int64_t m = i >> 6, w = i & 63;
            const size_t g = (size_t)(c->off[a] + i);
            bst[(size_t)(m * kBStat + w)] = dinv[g];
            bst[(size_t)(m * kBStat + 64 + w)] = dsD[g];
            int32_t* cp = reinterpret_cast<int32_t*>(&bst[(size_t)(m * kBStat + 128)]) + 4 * w;
            int k = 0;
            for (int pass = 0; pass < 2; ++pass)                 // far neighbours first
              for (int32_t e = H.rowptr[(size_t)i]; e < H.rowptr[(size_t)i + 1]; ++e) {
                const int64_t j = H.col[(size_t)e];
                const bool far = (j >> 6) != m;
                if (far == (pass == 0)) cp[k++] = far ? (int32_t)j : (int32_t)(-2 - (j & 63));
              }
          }
          UP(c->bstat[a], bst);
        }
        if (H.bj) {
          // block-Jacobi: tridiagonal part of every 64-row chunk (rows i, i+1 of the
          // chunk connected along the chain-ordered network), factored once (Thomas)
          std::vector<double> inv(NS, 1.0), cpv(NS, 0.0), em(NS, 0.0);
          auto linked = [&](int64_t i) {            // i -- i+1 connected
            for (int32_t e = H.rowptr[(size_t)i]; e < H.rowptr[(size_t)i + 1]; ++e)
              if (H.col[(size_t)e] == i + 1) return true;
            return false;
          };
          for (int64_t i0 = 0; i0 < H.n; i0 += 64) {
            const int64_t i1 = std::min<int64_t>(H.n, i0 + 64);
            double cprev = 0.0, eprev = 0.0;
            for (int64_t i = i0; i < i1; ++i) {
              const size_t gi = (size_t)(c->off[a] + i);
              const double ai = dsD[gi] + tsum[gi];
              const double den = ai - eprev * cprev;
              if (!(den > 0.0)) return fail(c, MC_ERR_ARG, "continuum %d: block-Jacobi pivot %g not > 0", a, den);
              const double ei = (i + 1 < i1 && linked(i)) ? -H.Tconst : 0.0;
              inv[gi] = 1.0 / den;
              em[gi] = eprev;
              cprev = ei * inv[gi];                   // = em[i+1] * inv[i]: bjs recomputes it
              cpv[gi] = cprev;
              eprev = ei;
            }
          }
          UP(c->tinv[a], inv);
          UP(c->tcp[a], cpv);
          UP(c->tem[a], em);
        }
      }
      if (!H.perm.empty()) UP(c->perm[a], H.perm);
      UP(c->rowptr[a], H.rowptr);
      UP(c->col[a], gcol);
      if (!H.val.empty()) UP(c->val[a], H.val);
    }
  }
#undef UP
  for (int k = 0; k < 2; ++k) {
    if (k == 1 && (st = dev_alloc(c, &c->u[1], NS)) != MC_OK) return st;
    if ((st = dev_alloc(c, &c->r[k], NS)) != MC_OK) return st;
    if ((st = dev_alloc(c, &c->p[k], NS)) != MC_OK) return st;
    if ((st = dev_alloc(c, &c->q[k], NS)) != MC_OK) return st;
    CUDA_TRY(c, cudaMemsetAsync(c->r[k], 0, NS * 8, c->stream));
    CUDA_TRY(c, cudaMemsetAsync(c->p[k], 0, NS * 8, c->stream));
    CUDA_TRY(c, cudaMemsetAsync(c->q[k], 0, NS * 8, c->stream));
  }
  CUDA_TRY(c, cudaMemcpyAsync(c->u[1], c->u[0], NS * 8, cudaMemcpyDeviceToDevice, c->stream));
  {
    int64_t mx = 1;
    for (int a = 0; a < c->L; ++a)
      if (c->hc[a].kind == KIND_GRAPH) mx = std::max(mx, c->hc[a].n);
    if ((st = dev_alloc(c, &c->scratch, (size_t)mx)) != MC_OK) return st;
  }
  if ((st = dev_alloc(c, &c->partials, (size_t)2 * kNPart * c->total_ctas)) != MC_OK) return st;
  if ((st = dev_alloc(c, &c->sync, 1)) != MC_OK) return st;
  if ((st = dev_alloc(c, &c->gout, MC_MAX_CONTINUA)) != MC_OK) return st;
  if ((st = dev_alloc(c, &c->cur, 1)) != MC_OK) return st;
  if ((st = dev_alloc(c, &c->fail, 1)) != MC_OK) return st;
  if ((st = dev_alloc(c, &c->rep, 1)) != MC_OK) return st;
  CUDA_TRY(c, cudaMemsetAsync(c->cur, 0, 4, c->stream));
  CUDA_TRY(c, cudaMemsetAsync(c->fail, 0, 4, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  c->cur_host = 0;
  // host copies no longer needed
  for (int a = 0; a < c->L; ++a) {
    HostCont& H = c->hc[a];
    std::vector<double>().swap(H.mtau);
    std::vector<double>().swap(H.dbase);
    std::vector<double>().swap(H.F);
    std::vector<double>().swap(H.u0);
    std::vector<double>().swap(H.tsum);
    std::vector<double>().swap(H.Tx);
    std::vector<double>().swap(H.Ty);
    std::vector<int32_t>().swap(H.col);
    std::vector<double>().swap(H.val);
  }
  c->cpl.clear();
  c->finalized = true;
  return MC_OK;
}

// ====================================================================== work plan
// Work items of continuum a for `warps` warps: about one item per warp, equal sizes.
static void add_items(const mc_ctx* c, int a, int warps, std::vector<Item>& items) {
  const HostCont& H = c->hc[a];
  warps = std::max(warps, 1);
  if (H.kind == KIND_GRAPH && c->ecol[a] != nullptr && c->val[a] == nullptr) return;   // round-robin (rr)
  if (H.kind == KIND_GRID) {
    const int w = (H.nx % 2 == 0) ? 64 : 32;       // 2 columns per lane when rows stay 16-B aligned
    const int strips = (H.nx + w - 1) / w;
    // distribute `warps` segments over the strips (+-1), heights as equal as possible
    const int base = std::max(1, warps / strips), extra = (warps >= strips) ? warps % strips : 0;
    // segment-major order: consecutive warps (one CTA) take adjacent strips of the same
    // rows, so a CTA streams contiguous 8 x 512 B of every array per row step
    const int smax = std::min(H.ny, base + (extra > 0 ? 1 : 0));
    for (int k = 0; k < smax; ++k)
      for (int s = 0; s < strips; ++s) {
        const int segs = std::min(H.ny, base + (s < extra ? 1 : 0));
        if (k >= segs) continue;
        Item it{};
        it.cont = a;
        it.kind = ITEM_GRID;
        it.a = s * w;
        it.b = (int)((int64_t)H.ny * k / segs);
        it.c = (int)((int64_t)H.ny * (k + 1) / segs);
        it.w = w;
        if (it.c > it.b) items.push_back(it);
      }
  } else {
    int64_t chunk = (H.n + warps - 1) / warps;
    const int64_t q = (H.col_count > 8 * H.n) ? 4 : 64;   // rows per warp-step (LPR 8) / staged chunk
    chunk = std::max<int64_t>(q, (chunk + q - 1) / q * q);
    for (int64_t r0 = 0; r0 < H.n; r0 += chunk) {
      Item it{};
      it.cont = a;
      it.kind = ITEM_GRAPH;
      it.a = (int32_t)r0;
      it.b = (int32_t)std::min<int64_t>(H.n, r0 + chunk);
      items.push_back(it);
    }
  }
}

static int64_t default_maxit(const mc_ctx* c, int64_t n) {
  if (c->opt.maxit > 0) return c->opt.maxit;
  return std::min<int64_t>(10 * n, 2000000);
}

// CTAs a latency-bound solve of n rows can use with >= 2 rows per thread
// A solve whose pass is this small runs on ONE CTA: its reduction is a CTA barrier
// (~0.1 us) instead of a grid-wide one (>= 1.8 us, profiles/r01_barrier.txt).
static int64_t one_cta_work() {
  static const int64_t w = [] {
    const char* e = getenv("MC_ONE_CTA_WORK");
    return e ? (int64_t)atoll(e) : (int64_t)kOneCtaWork;
  }();
  return w;
}

// MC_BLOCKED=0 (dev, A/B): keep the streaming ELL pass on the separate r, q, p arrays
static bool use_blocked() {
  static const bool v = [] {
    const char* e = getenv("MC_BLOCKED");
    return !(e && e[0] == '0');
  }();
  return v;
}

static int useful_ctas(const HostCont& H) {
  const int64_t work = H.kind == KIND_GRID ? 5 * H.n : H.n + H.col_count;
  if (work <= one_cta_work()) return 1;
  const int64_t lanes = (H.kind == KIND_GRAPH && H.col_count > 8 * H.n) ? 8 * H.n : H.n;
  return (int)std::max<int64_t>(1, (lanes + 2 * kThreads - 1) / (2 * kThreads));
}

static Plan make_plan(const mc_ctx* c, int scheme) {
  Plan P;
  const int T = c->total_ctas;
  double rmin = c->opt.rtol;
  for (int a = 0; a < c->L; ++a) rmin = std::min(rmin, c->hc[a].rtol > 0.0 ? c->hc[a].rtol : c->opt.rtol);
  const double tol2 = rmin * rmin;                 // coupled: the tightest tolerance
  if (scheme == MC_COUPLED) {
    P.ngroups = 1;
    P.nphases = 1;
    Group& g = P.grp[0];
    g.cta_begin = 0;
    g.cta_count = T;
    g.phase = 0;
    g.tol2 = tol2;
    int64_t ntot = 0;
    for (int a = 0; a < c->L; ++a) ntot += c->hc[a].n;
    g.maxit = default_maxit(c, ntot);
    g.cont_mask = (1 << c->L) - 1;
    g.item_begin = 0;
    for (int a = 0; a < c->L; ++a)
      add_items(c, a, (int)std::max<int64_t>(1, (int64_t)T * kWarps * c->hc[a].n / ntot), P.items);
    g.item_count = (int32_t)P.items.size();
    P.valid = true;
    return P;
  }
  const int L = c->L;
  P.ngroups = L;
  if (scheme == MC_DECOUPLED_L || scheme == MC_DECOUPLED_U) {
    // sequential: one phase per continuum in permeability order, all CTAs each
    P.nphases = L;
    for (int pos = 0; pos < L; ++pos) {
      const int a = scheme == MC_DECOUPLED_L ? c->korder[pos] : c->korder[L - 1 - pos];
      Group& g = P.grp[a];
      g.phase = pos;
      g.cta_begin = 0;
      // a latency-bound solve pays for every CTA in its barrier: use what it can use
      g.cta_count = c->hc[a].n >= kLargeRows ? T : std::min(T, useful_ctas(c->hc[a]));
      g.tol2 = c->hc[a].rtol * c->hc[a].rtol;
      g.maxit = default_maxit(c, c->hc[a].n);
      g.cont_mask = 1 << a;
    }
    for (int a = 0; a < L; ++a) {
      P.grp[a].item_begin = (int32_t)P.items.size();
      add_items(c, a, P.grp[a].cta_count * kWarps, P.items);
      P.grp[a].item_count = (int32_t)P.items.size() - P.grp[a].item_begin;
    }
    P.valid = true;
    return P;
  }
  bool all_large = true, hist = true;
  // a solve that can keep every CTA busy (bandwidth- or chunk-latency-bound: >= 2 rows per
  // thread on all CTAs) gains nothing from running beside another one -- the streams contend
  // and the split is never exactly balanced (config 2: 426 ms concurrent, 379 ms in phases);
  // only solves too small for the whole grid (config 1's fracture network: 143 CTAs) run
  // concurrently with the rest
  for (int a = 0; a < L; ++a) {
    if (c->hc[a].n < kLargeRows && useful_ctas(c->hc[a]) < T) all_large = false;
    if (c->plan_iters[a] <= 0) hist = false;
  }
  int ctas[MC_MAX_CONTINUA] = {0};
  if (all_large || !hist || L == 1 || T < 4 * L) {
    // sequential phases, every solve on all CTAs (bandwidth-bound, or no iteration history)
    P.nphases = L;
    for (int a = 0; a < L; ++a) {
      P.grp[a].phase = a;
      P.grp[a].cta_begin = 0;
      ctas[a] = c->hc[a].n >= kLargeRows ? T : std::min(T, useful_ctas(c->hc[a]));
    }
  } else {
    // one phase: CTAs split by work (rows x last iterations), each solve guaranteed the
    // CTAs its latency-bound loop can use (capped at an equal share)
    P.nphases = 1;
    double w[MC_MAX_CONTINUA], wsum = 0.0;
    int used = 0;
    for (int a = 0; a < L; ++a) {
      w[a] = (double)c->hc[a].n * (double)c->plan_iters[a];
      wsum += w[a];
      ctas[a] = std::min(useful_ctas(c->hc[a]), std::max(1, T / (2 * L)));
      used += ctas[a];
    }
    // a block-Jacobi network needs one warp per 64-row chunk (resident layout): give it
    // all its useful CTAs when they fit beside the others' shares, else it runs Jacobi
    for (int a = 0; a < L; ++a)
      if (c->tinv[a]) {
        const int want = useful_ctas(c->hc[a]);
        const int others = used - ctas[a];
        if (want > ctas[a] && others + want <= T) {
          used += want - ctas[a];
          ctas[a] = want;
        }
      }
    int rest = std::max(0, T - used);
    // distribute by work, never beyond what a solve can use (latency-bound solves pay
    // for every extra CTA in their per-iteration barrier)
    for (int round = 0; round < 4 && rest > 0; ++round) {
      double wl = 0.0;
      for (int a = 0; a < L; ++a)
        if (ctas[a] < useful_ctas(c->hc[a])) wl += w[a];
      if (wl <= 0.0) break;
      int given = 0;
      for (int a = 0; a < L; ++a) {
        if (ctas[a] >= useful_ctas(c->hc[a])) continue;
        int add = (int)std::floor(rest * (w[a] / wl));
        add = std::min(add, useful_ctas(c->hc[a]) - ctas[a]);
        ctas[a] += add;
        given += add;
      }
      if (given == 0) {
        int amax = -1;
        for (int a = 0; a < L; ++a)
          if (ctas[a] < useful_ctas(c->hc[a]) && (amax < 0 || w[a] > w[amax])) amax = a;
        if (amax < 0) break;
        const int add = std::min(rest, useful_ctas(c->hc[amax]) - ctas[amax]);
        ctas[amax] += add;
        given = add;
      }
      rest -= given;
    }
    int b = 0;
    for (int a = 0; a < L; ++a) {
      P.grp[a].phase = 0;
      P.grp[a].cta_begin = b;
      b += ctas[a];
    }
  }
  for (int a = 0; a < L; ++a) {
    Group& g = P.grp[a];
    g.cta_count = ctas[a];
    g.tol2 = c->hc[a].rtol * c->hc[a].rtol;
    g.maxit = default_maxit(c, c->hc[a].n);
    g.cont_mask = 1 << a;
    g.item_begin = (int32_t)P.items.size();
    add_items(c, a, ctas[a] * kWarps, P.items);
    g.item_count = (int32_t)P.items.size() - g.item_begin;
  }
  P.valid = true;
  return P;
}

static bool same_plan(const Plan& a, const Plan& b) {
  if (!a.valid || !b.valid || a.ngroups != b.ngroups || a.nphases != b.nphases) return false;
  for (int g = 0; g < a.ngroups; ++g)
    if (a.grp[g].cta_begin != b.grp[g].cta_begin || a.grp[g].cta_count != b.grp[g].cta_count ||
        a.grp[g].phase != b.grp[g].phase)
      return false;
  return true;
}

// ====================================================================== stepping
static mc_status enqueue_step(mc_ctx* c, int scheme, mc_step_report* rep_dev, cudaEvent_t ev0, cudaEvent_t ev1,
                              int32_t step_no) {
  Plan np = make_plan(c, scheme);
  Plan& cp = c->plan[scheme];
  if (!same_plan(np, cp) || c->uploaded_plan != scheme) {
    cp = np;
    if (cp.items.size() > c->items_cap) {
      if (c->items) {
        cudaStreamSynchronize(c->stream);
        cudaFree(c->items);
        c->allocs.erase(std::find(c->allocs.begin(), c->allocs.end(), (void*)c->items));
        for (size_t gi = 0; gi < c->guards.size(); ++gi)
          if (c->guards[gi].first == (void*)c->items) {
            c->guards.erase(c->guards.begin() + (long)gi);
            break;
          }
        c->items = nullptr;
      }
      mc_status st = dev_alloc(c, &c->items, cp.items.size() * 2);
      if (st != MC_OK) return st;
      c->items_cap = cp.items.size() * 2;
    }
    CUDA_TRY(c, cudaMemcpyAsync(c->items, cp.items.data(), cp.items.size() * sizeof(Item),
                                cudaMemcpyHostToDevice, c->stream));
    c->uploaded_plan = scheme;
  }
  StepParams P{};
  for (int a = 0; a < c->L; ++a) {
    ContDev& C = P.cont[a];
    const HostCont& H = c->hc[a];
    C.kind = H.kind;
    C.nx = H.nx;
    C.ny = H.ny;
    C.off = c->off[a];
    C.n = H.n;
    C.Tx = c->Tx[a];
    C.Ty = c->Ty[a];
    C.rowptr = c->rowptr[a];
    C.col = c->col[a];
    C.val = c->val[a];
    C.Tconst = H.Tconst;
    C.ecol = c->ecol[a];
    C.ell = c->ecol[a] ? 4 : 0;
    C.estride = H.estride;
    C.rr = (c->ecol[a] != nullptr && c->val[a] == nullptr) ? 1 : 0;
    C.lpr = 1;
    if (H.kind == KIND_GRAPH && H.n > 0 && H.col_count > 8 * H.n) C.lpr = 8;   // > 8 neighbours per row
  }
  for (int g = 0; g < cp.ngroups; ++g) P.grp[g] = cp.grp[g];
  // resident fracture solves: alone in their group, every warp owns <= kStages chunks
  for (int g = 0; g < cp.ngroups; ++g) {
    const Group& G = cp.grp[g];
    int nconts = 0;
    for (int a = 0; a < c->L; ++a) nconts += (G.cont_mask >> a) & 1;
    for (int a = 0; a < c->L; ++a)
      if (((G.cont_mask >> a) & 1) && P.cont[a].rr) {
        const int64_t nch = (c->hc[a].n + 63) / 64;
        P.cont[a].resident = (nconts == 1 && nch <= (int64_t)kStages * G.cta_count * kWarps) ? 1 : 0;
        P.cont[a].bj = (nconts == 1 && nch <= (int64_t)G.cta_count * kWarps && c->tinv[a] != nullptr &&
                        scheme != MC_COUPLED) ? 1 : 0;
        P.cont[a].bjs = (!P.cont[a].bj && nconts == 1 && c->tinv[a] != nullptr && scheme != MC_COUPLED) ? 1 : 0;
        // streaming Jacobi pass of a decoupled solve: chunk-blocked workspace (the CG-state
        // blocks are allocated the first time a plan streams this network)
        if (use_blocked() && c->bstat[a] && nconts == 1 && scheme != MC_COUPLED && P.cont[a].resident) {
          // resident pass on the blocked static data, publishing 32-byte records
          if (!c->rrec[a][0]) {
            const size_t cnt = (size_t)4 * ((size_t)c->hc[a].n + 64);
            for (int k = 0; k < 2; ++k) {
              mc_status st = dev_alloc(c, &c->rrec[a][k], cnt);
              if (st != MC_OK) return st;
              CUDA_TRY(c, cudaMemsetAsync(c->rrec[a][k], 0, cnt * 8, c->stream));
            }
          }
          P.cont[a].bstat = c->bstat[a];
          P.cont[a].rrec[0] = c->rrec[a][0];
          P.cont[a].rrec[1] = c->rrec[a][1];
        }
        if (use_blocked() && c->bstat[a] && nconts == 1 && scheme != MC_COUPLED && !P.cont[a].resident &&
            !P.cont[a].bj && !P.cont[a].bjs) {
          if (!c->bdyn[a][0]) {
            const size_t cnt = (size_t)((c->hc[a].n + 63) / 64) * kBDyn;
            for (int k = 0; k < 2; ++k) {
              mc_status st = dev_alloc(c, &c->bdyn[a][k], cnt);
              if (st != MC_OK) return st;
              CUDA_TRY(c, cudaMemsetAsync(c->bdyn[a][k], 0, cnt * 8, c->stream));
            }
          }
          P.cont[a].bstat = c->bstat[a];
          P.cont[a].bdyn[0] = c->bdyn[a][0];
          P.cont[a].bdyn[1] = c->bdyn[a][1];
        }
      }
  }
  c->path_mask = 0;
  for (int a = 0; a < c->L; ++a) {
    const ContDev& C = P.cont[a];
    const int path = C.bj ? MC_PATH_BJ_RESIDENT : C.bjs ? MC_PATH_BJ_STREAM : C.resident ? MC_PATH_ELL_RESIDENT
                     : C.rr ? MC_PATH_ELL_STREAM : MC_PATH_STREAM;
    c->path_mask |= path << (4 * a);
  }
  for (int a = 0; a < c->L; ++a) {
    if (P.cont[a].bjs && use_blocked()) P.cont[a].bstat = c->bstat[a];   // pass S on the blocked codes
    P.cont[a].tinv = c->tinv[a];
    P.cont[a].tcp = c->tcp[a];
    P.cont[a].tem = c->tem[a];
  }
  P.L = c->L;
  P.ngroups = cp.ngroups;
  P.nphases = cp.nphases;
  P.coupled = (scheme == MC_COUPLED);
  P.gs = (scheme == MC_DECOUPLED_L || scheme == MC_DECOUPLED_U) ? 1 : 0;
  P.total_ctas = c->total_ctas;
  P.N = c->N;
  for (int k = 0; k < 2; ++k) {
    P.u[k] = c->u[k];
    P.r[k] = c->r[k];
    P.p[k] = c->p[k];
    P.q[k] = c->q[k];
  }
  P.dinv = c->dinv;
  P.dsD = c->dsD;
  P.dsC = c->dsC;
  P.mtau = c->mtau;
  P.F = c->F;
  P.cptr = c->cptr;
  P.cidx = c->cidx;
  P.cval = c->cval;
  P.items = c->items;
  P.partials = c->partials;
  P.sync = c->sync;
  P.gout = c->gout;
  P.cur = c->cur;
  P.fail = c->fail;
  P.rep = rep_dev;
  P.step_no = step_no;
  P.scheme = scheme;
  CUDA_TRY(c, cudaMemsetAsync(c->sync, 0, sizeof(SyncBlock), c->stream));
  CUDA_TRY(c, cudaEventRecord(ev0, c->stream));
  CUDA_TRY(c, launch_step(&P, c->total_ctas, c->stream));
  CUDA_TRY(c, cudaEventRecord(ev1, c->stream));
  return MC_OK;
}

static const char* scheme_name(int scheme) {
  return scheme == MC_COUPLED ? "coupled" : scheme == MC_DECOUPLED_D ? "D-scheme"
         : scheme == MC_DECOUPLED_L ? "L-scheme" : "U-scheme";
}

// host mirrors after a completed step whose report is `rep`
static mc_status account_step(mc_ctx* c, int scheme, const mc_step_report& rep) {
#if MC_NVTX
  for (int g = 0; g < rep.nsolves; ++g) {
    char buf[96];
    snprintf(buf, sizeof buf, "pcg[%d] step %d: %lld iterations, %.3f ms", g, rep.step, (long long)rep.iters[g],
             rep.ms_solve[g]);
    nvtxMarkA(buf);
  }
#endif
  if (rep.status == MC_OK) {
    c->cur_host ^= 1;
    c->step_no += 1;
    if (scheme == MC_DECOUPLED_D) {
      for (int a = 0; a < c->L; ++a) c->last_iters[a] = rep.iters[a];
      if (!c->d_frozen) {
        // the plan of the next D step is chosen from this step's counts; frozen once every
        // solve has iterated (or after kPlanSteps steps), DESIGN.md §5.4
        bool hist = true;
        for (int a = 0; a < c->L; ++a) {
          c->plan_iters[a] = rep.iters[a];
          if (rep.iters[a] <= 0) hist = false;
        }
        c->d_steps += 1;
        if (hist || c->d_steps >= kPlanSteps) c->d_frozen = true;
      }
    }
    return MC_OK;
  }
  const char* what = rep.status == MC_ERR_NOCONV ? "no convergence within maxit"
                     : rep.status == MC_ERR_BREAKDOWN ? "CG breakdown (p.q <= 0)"
                                                      : "step skipped after an earlier failure";
  return fail(c, (mc_status)rep.status, "step %d (%s), solve %d: %s after %lld iterations; state not advanced",
              c->step_no + 1, scheme_name(scheme), rep.failed_solve, what,
              rep.failed_solve >= 0 ? (long long)rep.iters[rep.failed_solve] : 0LL);
}

// wait for the step, read its report, update host mirrors
static mc_status complete_step(mc_ctx* c, int scheme, mc_step_report* out) {
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  mc_step_report rep;
  CUDA_TRY(c, cudaMemcpy(&rep, c->rep, sizeof rep, cudaMemcpyDeviceToHost));
  float ms = 0.f;
  CUDA_TRY(c, cudaEventElapsedTime(&ms, c->ev0, c->ev1));
  rep.ms = ms;
  rep.paths = c->path_mask;
  if (out) *out = rep;
  return account_step(c, scheme, rep);
}

static mc_status check_scheme(mc_ctx* c, int scheme) {
  if (!c) return fail(c, MC_ERR_ARG, "NULL context");
  if (scheme < MC_COUPLED || scheme > MC_DECOUPLED_U) return fail(c, MC_ERR_ARG, "unknown scheme %d", scheme);
  if ((scheme == MC_DECOUPLED_L || scheme == MC_DECOUPLED_U) && !c->has_korder)
    return fail(c, MC_ERR_STATE, "L/U scheme before mc_set_permeability_order");
  return finalize(c);
}

static mc_status do_step(mc_ctx* c, int scheme, mc_step_report* rep) {
  mc_status st = check_scheme(c, scheme);
  if (st != MC_OK) return st;
  NvtxRange range("mc_step");
  CUDA_TRY(c, cudaMemsetAsync(c->fail, 0, 4, c->stream));
  if ((st = enqueue_step(c, scheme, c->rep, c->ev0, c->ev1, c->step_no + 1)) != MC_OK) return st;
  return complete_step(c, scheme, rep);
}

extern "C" mc_status mc_step_decoupled(mc_ctx* c, mc_step_report* rep) {
  return do_step(c, MC_DECOUPLED_D, rep);
}

extern "C" mc_status mc_step_coupled(mc_ctx* c, mc_step_report* rep) {
  return do_step(c, MC_COUPLED, rep);
}

extern "C" mc_status mc_step(mc_ctx* c, int32_t scheme, mc_step_report* rep) { return do_step(c, scheme, rep); }

extern "C" mc_status mc_set_preconditioner(mc_ctx* c, int32_t kind) {
  if (!c) return fail(c, MC_ERR_ARG, "NULL context");
  if (kind != MC_PRECOND_JACOBI && kind != MC_PRECOND_BLOCK) return fail(c, MC_ERR_ARG, "preconditioner %d unknown", kind);
  for (int a = 0; a < c->L; ++a)
    if (c->hc[a].set) return fail(c, MC_ERR_STATE, "mc_set_preconditioner after mc_set_continuum");
  c->precond = kind;
  return MC_OK;
}

extern "C" mc_status mc_set_permeability_order(mc_ctx* c, const int32_t* order) {
  if (!c || !order) return fail(c, MC_ERR_ARG, "NULL argument");
  std::vector<int32_t> o;
  mc_status st = fetch(c, o, order, c->L);
  if (st != MC_OK) return st;
  std::vector<int32_t> srt(o);
  std::sort(srt.begin(), srt.end());
  for (int a = 0; a < c->L; ++a)
    if (srt[(size_t)a] != a) return fail(c, MC_ERR_ARG, "permeability order is not a permutation of 0..%d", c->L - 1);
  for (int a = 0; a < c->L; ++a) c->korder[a] = o[(size_t)a];
  c->has_korder = true;
  for (auto& pl : c->plan) pl.valid = false;
  c->uploaded_plan = -1;
  return MC_OK;
}

static mc_status copy_out(mc_ctx* c, int a, double* dst);

static void mark_skipped(mc_step_report* reps, int32_t from, int32_t n) {
  for (int32_t t = from; t < n && reps; ++t) {
    std::memset(&reps[t], 0, sizeof(mc_step_report));
    reps[t].status = MC_ERR_STATE;
    reps[t].failed_solve = -1;
  }
}

extern "C" mc_status mc_run(mc_ctx* c, int32_t scheme, int32_t n_steps, mc_step_report* reps,
                            double* const* snapshots) {
  mc_status st = check_scheme(c, scheme);
  if (st != MC_OK) return st;
  if (n_steps < 0) return fail(c, MC_ERR_ARG, "n_steps < 0");
  NvtxRange range("mc_run");
  auto snap = [&](int32_t s) -> mc_status {
    if (!snapshots) return MC_OK;
    for (int a = 0; a < c->L; ++a) {
      double* dst = snapshots[(size_t)s * c->L + a];
      mc_status e = dst ? copy_out(c, a, dst) : MC_OK;
      if (e != MC_OK) return e;
    }
    return MC_OK;
  };
  int32_t s = 0;
  // planning steps: while the D-scheme's CTA plan still follows the iteration counts of
  // the previous step (at most kPlanSteps steps of a context's life) each step is completed
  // before the next one is planned -- exactly what mc_step does
  for (; s < n_steps && scheme == MC_DECOUPLED_D && !c->d_frozen; ++s) {
    mc_step_report rep;
    st = do_step(c, scheme, &rep);
    if (reps) reps[s] = rep;
    if (st != MC_OK) {
      mark_skipped(reps, s + 1, n_steps);
      return st;
    }
    if ((st = snap(s)) != MC_OK) return st;
  }
  if (s == n_steps) {
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    return MC_OK;
  }
  // the rest: enqueued back to back (fixed plan, reports and the ping-pong index stay on
  // the device), one synchronisation per batch of kRunBatch steps
  if (!c->rep_run && (st = dev_alloc(c, &c->rep_run, (size_t)kRunBatch)) != MC_OK) return st;
  while ((int)c->run_ev.size() < 2 * kRunBatch) {
    cudaEvent_t e = nullptr;
    CUDA_TRY(c, cudaEventCreate(&e));
    c->run_ev.push_back(e);
  }
  std::vector<mc_step_report> hrep((size_t)kRunBatch);
  CUDA_TRY(c, cudaMemsetAsync(c->fail, 0, 4, c->stream));
  while (s < n_steps) {
    const int32_t nb = std::min<int32_t>(kRunBatch, n_steps - s);
    const int32_t cur0 = c->cur_host;
    for (int32_t k = 0; k < nb; ++k) {
      if ((st = enqueue_step(c, scheme, c->rep_run + k, c->run_ev[2 * (size_t)k], c->run_ev[2 * (size_t)k + 1],
                             c->step_no + 1 + k)) != MC_OK)
        return st;
      c->cur_host ^= 1;                       // optimistic mirror for the snapshot copies
      if ((st = snap(s + k)) != MC_OK) return st;
    }
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    CUDA_TRY(c, cudaMemcpy(hrep.data(), c->rep_run, (size_t)nb * sizeof(mc_step_report), cudaMemcpyDeviceToHost));
    c->cur_host = cur0;
    for (int32_t k = 0; k < nb; ++k) {
      float ms = 0.f;
      CUDA_TRY(c, cudaEventElapsedTime(&ms, c->run_ev[2 * (size_t)k], c->run_ev[2 * (size_t)k + 1]));
      hrep[(size_t)k].ms = ms;
      hrep[(size_t)k].paths = c->path_mask;
      if (reps) reps[s + k] = hrep[(size_t)k];
      if ((st = account_step(c, scheme, hrep[(size_t)k])) != MC_OK) {
        // the device skipped every later step of the batch (sticky failure flag)
        mark_skipped(reps, s + k + 1, n_steps);
        return st;
      }
    }
    // the last step's events are what mc_last_kernel_ms reports
    std::swap(c->ev0, c->run_ev[2 * (size_t)(nb - 1)]);
    std::swap(c->ev1, c->run_ev[2 * (size_t)(nb - 1) + 1]);
    s += nb;
  }
  return MC_OK;
}

// copy p_alpha (internal numbering) to dst in the caller's numbering, stream-ordered
static mc_status copy_out(mc_ctx* c, int a, double* dst) {
  const double* src = c->u[c->cur_host] + c->off[a];
  const size_t bytes = (size_t)c->hc[a].n * 8;
  if (c->perm[a]) {
    CUDA_TRY(c, launch_to_caller(c->scratch, src, c->perm[a], c->hc[a].n, c->stream));
    src = c->scratch;
  }
  CUDA_TRY(c, cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, c->stream));
  return MC_OK;
}

extern "C" mc_status mc_get_state(mc_ctx* c, int32_t alpha, double* dst) {
  if (!c || !dst) return fail(c, MC_ERR_ARG, "NULL argument");
  if (alpha < 0 || alpha >= c->L) return fail(c, MC_ERR_ARG, "alpha = %d out of range", alpha);
  mc_status st = finalize(c);
  if (st != MC_OK) return st;
  if ((st = copy_out(c, alpha, dst)) != MC_OK) return st;
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return MC_OK;
}

extern "C" mc_status mc_set_state(mc_ctx* c, int32_t alpha, const double* src) {
  if (!c || !src) return fail(c, MC_ERR_ARG, "NULL argument");
  if (alpha < 0 || alpha >= c->L) return fail(c, MC_ERR_ARG, "alpha = %d out of range", alpha);
  mc_status st = finalize(c);
  if (st != MC_OK) return st;
  double* dst = c->u[c->cur_host] + c->off[alpha];
  const size_t bytes = (size_t)c->hc[alpha].n * 8;
  if (c->perm[alpha]) {
    CUDA_TRY(c, cudaMemcpyAsync(c->scratch, src, bytes, cudaMemcpyDefault, c->stream));
    CUDA_TRY(c, launch_from_caller(dst, c->scratch, c->perm[alpha], c->hc[alpha].n, c->stream));
  } else {
    CUDA_TRY(c, cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, c->stream));
  }
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return MC_OK;
}

extern "C" mc_status mc_last_kernel_ms(mc_ctx* c, double* ms_out) {
  if (!c || !ms_out) return fail(c, MC_ERR_ARG, "NULL argument");
  float ms = 0.f;
  CUDA_TRY(c, cudaEventElapsedTime(&ms, c->ev0, c->ev1));
  *ms_out = ms;
  return MC_OK;
}

// ====================================================================== NLMC export
namespace mc {

mc_status ctx_error(mc_ctx* c, mc_status st, const char* msg) { return fail(c, st, "%s", msg); }

mc_status export_fine(mc_ctx* c, const int32_t* const* host, FineSystem& fs) {
  if (!c) return MC_ERR_ARG;
  if (c->finalized) return fail(c, MC_ERR_STATE, "NLMC build after the first step (setup data released)");
  fs = FineSystem();
  fs.L = c->L;
  fs.device = c->opt.device;
  fs.off.assign((size_t)c->L + 1, 0);
  for (int a = 0; a < c->L; ++a) {
    const HostCont& H = c->hc[a];
    if (!H.set) return fail(c, MC_ERR_STATE, "continuum %d not set", a);
    fs.off[(size_t)a + 1] = fs.off[(size_t)a] + H.n;
    fs.kind.push_back(H.kind);
    if (H.kind == KIND_GRID) {
      if (fs.nx == 0) {
        fs.nx = H.nx;
        fs.ny = H.ny;
      } else if (fs.nx != H.nx || fs.ny != H.ny) {
        return fail(c, MC_ERR_ARG, "NLMC: grid continua on different grids");
      }
    } else {
      for (uint8_t f : H.fixed)
        if (f) return fail(c, MC_ERR_ARG, "NLMC: continuum %d has fixed (Dirichlet) cells", a);
    }
  }
  if (fs.nx == 0) return fail(c, MC_ERR_ARG, "NLMC needs a grid continuum");
  const int64_t N = fs.off[(size_t)c->L];
  fs.cont.resize((size_t)N);
  fs.host.resize((size_t)N);
  fs.meas.resize((size_t)N);
  fs.mass.resize((size_t)N);
  fs.F.resize((size_t)N);
  fs.u0.resize((size_t)N);
  fs.ddiag.resize((size_t)N);
  fs.wdiag.resize((size_t)N);
  auto caller = [&](int a, int64_t t) -> int64_t {      // internal position -> caller index
    const HostCont& H = c->hc[a];
    return H.perm.empty() ? t : (int64_t)H.perm[(size_t)t];
  };
  for (int a = 0; a < c->L; ++a) {
    const HostCont& H = c->hc[a];
    const int64_t o = fs.off[(size_t)a];
    std::vector<int32_t> hc;
    if (H.kind == KIND_GRAPH) {
      if (!host || !host[a]) return fail(c, MC_ERR_ARG, "NLMC: host cells of graph continuum %d missing", a);
      mc_status st = fetch(c, hc, host[a], H.n);
      if (st != MC_OK) return st;
      for (int32_t v : hc)
        if (v < 0 || (int64_t)v >= (int64_t)fs.nx * fs.ny)
          return fail(c, MC_ERR_ARG, "NLMC: host cell %d of continuum %d out of range", v, a);
    }
    for (int64_t t = 0; t < H.n; ++t) {
      const int64_t i = caller(a, t);
      const size_t g = (size_t)(o + i);
      fs.cont[g] = a;
      fs.host[g] = H.kind == KIND_GRID ? (int32_t)i : hc[(size_t)i];
      fs.meas[g] = H.measure[(size_t)t];
      fs.mass[g] = H.mass[(size_t)t];
      fs.F[g] = H.F[(size_t)t];
      fs.u0[g] = H.u0[(size_t)t];
      fs.ddiag[g] = H.dbd[(size_t)t];
      fs.wdiag[g] = H.dwell[(size_t)t];
    }
    if (H.kind == KIND_GRID) {
      for (int iy = 0; iy < H.ny; ++iy)
        for (int ix = 0; ix < H.nx; ++ix) {
          const int64_t i = (int64_t)iy * H.nx + ix;
          if (ix + 1 < H.nx && H.Tx[(size_t)i] != 0.0) {
            fs.ei.push_back((int32_t)(o + i));
            fs.ej.push_back((int32_t)(o + i + 1));
            fs.et.push_back(H.Tx[(size_t)i]);
          }
          if (iy + 1 < H.ny && H.Ty[(size_t)i] != 0.0) {
            fs.ei.push_back((int32_t)(o + i));
            fs.ej.push_back((int32_t)(o + i + H.nx));
            fs.et.push_back(H.Ty[(size_t)i]);
          }
        }
    } else {
      for (int64_t t = 0; t < H.n; ++t)
        for (int32_t e = H.rowptr[(size_t)t]; e < H.rowptr[(size_t)t + 1]; ++e) {
          const int32_t u = H.col[(size_t)e];
          if (u <= t) continue;                               // each connection once
          fs.ei.push_back((int32_t)(o + caller(a, t)));
          fs.ej.push_back((int32_t)(o + caller(a, u)));
          fs.et.push_back(H.val.empty() ? H.Tconst : H.val[(size_t)e]);
        }
    }
  }
  for (const HostCoupling& h : c->cpl)
    for (size_t e = 0; e < h.i.size(); ++e) {
      fs.qi.push_back((int32_t)(fs.off[(size_t)h.a] + caller(h.a, h.i[e])));
      fs.qj.push_back((int32_t)(fs.off[(size_t)h.b] + caller(h.b, h.j[e])));
      fs.qs.push_back(h.s[e]);
    }
  return MC_OK;
}

}  // namespace mc
