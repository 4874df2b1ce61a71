// mc_nlmc.cu — NLMC multiscale space on the GPU (§4.1, :591-729; include/mc.h).
//
// Host (native C++, setup): coarse DOFs (continuum, coarse cell, piece; reading C30),
// per oversampled region K_i^+ the local DOF list in host-cell order (small bandwidth),
// the lower band of D + Q restricted to K_i^+ (zero Dirichlet outside),
// the constraint rows.
// Device (sm_100a):
//   nlmc_basis_kernel   one CTA per K_i^+ (persistent, as many per SM as shared memory allows):
//                       banded Cholesky D + Q = L L^T (right-looking, ring of b+1+8 rows
//                       in shared memory, cp.async prefetch), Z = (D+Q)^{-1} C^T by banded forward / backward
//                       substitution for all constraint columns at once, Schur complement
//                       S = C Z and its dense Cholesky, psi^{i,beta} = Z S^{-1} e_(i,beta)
//                       -- Eq. eq:basis by block elimination of the multipliers.
//   nlmc_project_kernel one warp per pair of overlapping bases: psi_r^T D psi_s in flux
//                       form (sum over connections T (dpsi_r)(dpsi_s) + boundary terms),
//                       read from the per-region sparse storage the basis kernel wrote
//                       (O(sum |K_i^+|) doubles; a window map per region finds psi_r(g)).
// Host: Dbar in flux form (reading C32), Qbar, Wbar, Mbar, Fbar aggregated.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <numeric>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "mc_nlmc.h"


namespace mc {

constexpr int kNlThreads = 512;      // max threads of the CTA that factors one region K_i^+
constexpr int kWP = 8;               // cp.async prefetch distance (rows)
constexpr int kNlMaxCons = 128;      // constraint rows per K_i^+ (4 per lane)
constexpr int kNlSmemDoubles = 27000;   // 216 KB dynamic shared memory per CTA

struct NlDomain {
  int32_t n, b, kc, nown;       // local DOFs, bandwidth, constraints, own coarse DOFs
  int32_t cx0, cx1, cy0, cy1;   // coarse-cell box of K_i^+ (inclusive)
  int64_t dof0;                 // first local DOF in the per-DOF arrays
  int64_t ent0, nent;           // lower off-diagonal entries
  int64_t cons0;                // constraint -> local DOF lists (CSR over kc rows)
  int32_t own0;                 // first own entry
  int32_t pad;
  int64_t woff;                 // window map of K_i^+: (layer, fine y, fine x) -> local DOF or -1
};

struct NlParams {
  const NlDomain* dom;
  int32_t ndom;
  const int32_t* lglob;         // local DOF -> global fine DOF
  const int32_t* lcon;          // local DOF -> constraint index within the domain
  const double* lw;             // local DOF -> constraint weight |cell| / |K_j^alpha|
  const double* ldiag;          // diagonal of D + Q restricted (incl. connections leaving K_i^+)
  const int32_t* erow;          // lower entries: row l1, offset d = l1 - l2 > 0, value
  const int32_t* eoff;
  const double* eval;
  const int32_t* cptr;          // per domain: kc + 1 offsets (relative to cons0) into cidx
  const int32_t* cidx;          // local DOFs of each constraint (ascending)
  const int32_t* own_con;       // own coarse DOF -> constraint index within its domain
  const int64_t* own_psi;       // own coarse DOF -> offset of its psi (n values) in psi
  double* band;                 // [gridDim][nmax * (bmax + 1)] workspace
  double* Z;                    // [gridDim][nmax * kcmax] workspace
  double* psi;                  // output
  int64_t band_stride, z_stride;
  int32_t* err;                 // first failing domain + 1 (0 = ok)
  int32_t wpb;                  // warps per CTA
  int32_t spw;                  // shared-memory doubles per warp
};

// ---------------------------------------------------------------- basis kernel
// One CTA per region K_i^+ at a time (persistent over regions; a one-warp-per-region
// version measured 6x slower).  Global rows the next steps need are
// prefetched kWP rows ahead with cp.async into shared-memory rings.
__device__ __forceinline__ unsigned nl_smem(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void nl_cp8(double* dst, const double* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(nl_smem(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void nl_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void nl_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int NT>
__global__ void __launch_bounds__(NT) nlmc_basis_kernel(const NlParams P) {
  extern __shared__ __align__(16) double sm[];
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  constexpr int NW = NT / 32;
  double* ws = sm;
  double* band = P.band + (size_t)blockIdx.x * P.band_stride;
  double* Z = P.Z + (size_t)blockIdx.x * P.z_stride;
  for (int di = blockIdx.x; di < P.ndom; di += gridDim.x) {
    const NlDomain D = P.dom[di];
    const int n = D.n, b = D.b, kc = D.kc, bw = b + 1, R = bw + kWP;
    const int32_t* lcon = P.lcon + D.dof0;
    const double* lw = P.lw + D.dof0;
    // ---- lower band of D + Q in global (row r: entry d = A(r, r - d))
    for (int64_t q = t; q < (int64_t)n * bw; q += NT) band[q] = 0.0;
    __syncthreads();
    for (int r = t; r < n; r += NT) band[(size_t)r * bw] = P.ldiag[D.dof0 + r];
    for (int64_t e = t; e < D.nent; e += NT)
      band[(size_t)P.erow[D.ent0 + e] * bw + P.eoff[D.ent0 + e]] = P.eval[D.ent0 + e];
    __syncthreads();
    // ---- banded Cholesky; ring of R = bw + kWP rows (slot r % R): rows k..k+b live,
    //      the next kWP rows in flight (cp.async issued kWP columns before they are used)
    double* W = ws;
    double* lv = ws + (size_t)R * bw;
    for (int q = t; q < bw * bw; q += NT) {
      const int r = q / bw;
      W[(size_t)(r % R) * bw + q % bw] = r < n ? band[(size_t)r * bw + q % bw] : 0.0;
    }
#pragma unroll 1
    for (int pq = 0; pq < kWP - 1; ++pq) {               // rows bw .. R-2
      const int r = bw + pq;
      if (r < n)
        for (int q = t; q < bw; q += NT) nl_cp8(W + (size_t)(r % R) * bw + q, band + (size_t)r * bw + q);
      nl_commit();
    }
    bool bad = false;
    for (int k = 0; k < n; ++k) {
      const int rn = k + R - 1;                          // into row k-1's slot
      if (rn < n)
        for (int q = t; q < bw; q += NT) nl_cp8(W + (size_t)(rn % R) * bw + q, band + (size_t)rn * bw + q);
      nl_commit();
      const double akk = __ldg(P.ldiag + D.dof0 + k);   // unfactored diagonal
      nl_wait<kWP>();                                    // rows up to k+b landed
      __syncthreads();
      const int s0 = k % R;
      const double dk = W[(size_t)s0 * bw];
      if (!(dk > 1e-13 * akk)) {                         // (numerically) singular region
        bad = true;
        break;
      }
      const double s = sqrt(dk);
      const int bk = min(b, n - 1 - k);
      if (t == 0) band[(size_t)k * bw] = s;
      for (int i = 1 + t; i <= bk; i += NT) {
        const int si = s0 + i >= R ? s0 + i - R : s0 + i;
        const double li = W[(size_t)si * bw + i] / s;
        lv[i] = li;
        band[(size_t)(k + i) * bw + i] = li;
      }
      __syncthreads();
      // A(k+i, k+i-d) -= l_i l_{i-d}: warp per row i, lanes over d (contiguous in the row)
      for (int i = 1 + wid; i <= bk; i += NW) {
        const int si = s0 + i >= R ? s0 + i - R : s0 + i;
        double* row = W + (size_t)si * bw;
        const double li = lv[i];
#pragma unroll 4
        for (int d = lane; d < i; d += 32) row[d] = __fma_rn(-li, lv[i - d], row[d]);
      }
    }
    nl_wait<0>();
    __syncthreads();
    if (__syncthreads_or(bad)) {
      if (t == 0) atomicCAS(P.err, 0, di + 1);
      continue;
    }
    // ---- Z = L^{-T} L^{-1} C^T for all kc columns: thread (c, g), G = NT / kc groups
    //      split the band offsets; one barrier for the partial sums, one for the result
    double* Lr = ws;                                     // kWP rows (forward) / columns (backward) of L
    double* Zw = ws + (size_t)kWP * bw;                  // last bw rows of Z, slot r % bw
    double* part = Zw + (size_t)bw * kc;                 // G * kc partial sums
    const int G = NT / kc;
    const int c = t % kc, g = t / kc;
    const bool act = g < G;
#pragma unroll 1
    for (int pq = 0; pq < kWP - 1; ++pq) {
      if (pq < n)
        for (int q = t; q < bw; q += NT) nl_cp8(Lr + (size_t)pq * bw + q, band + (size_t)pq * bw + q);
      nl_commit();
    }
    for (int r = 0; r < n; ++r) {
      const int rn = r + kWP - 1;
      if (rn < n)
        for (int q = t; q < bw; q += NT) nl_cp8(Lr + (size_t)(rn % kWP) * bw + q, band + (size_t)rn * bw + q);
      nl_commit();
      nl_wait<kWP - 1>();
      __syncthreads();
      const double* lr = Lr + (size_t)(r % kWP) * bw;
      const int rs = r % bw;
      if (act) {
        double a0 = 0.0, a1 = 0.0;
        const int dm = min(b, r);
        int d = 1 + g;
        int sl = rs - d;                                 // ring slot of row r - d
        if (sl < 0) sl += bw;
        for (; d + G <= dm; d += 2 * G) {
          int s2 = sl - G;
          if (s2 < 0) s2 += bw;
          a0 = __fma_rn(lr[d], Zw[sl * kc + c], a0);
          a1 = __fma_rn(lr[d + G], Zw[s2 * kc + c], a1);
          sl = s2 - G;
          if (sl < 0) sl += bw;
        }
        if (d <= dm) a0 = __fma_rn(lr[d], Zw[sl * kc + c], a0);
        part[g * kc + c] = a0 + a1;
      }
      const double piv = lr[0];                          // read before the ring slot is reused
      __syncthreads();
      if (t < kc) {
        double sacc = 0.0;
        for (int q = 0; q < G; ++q) sacc += part[q * kc + t];
        const double rhs = (lcon[r] == t) ? lw[r] : 0.0;
        const double y = (rhs - sacc) / piv;
        Zw[rs * kc + t] = y;
        Z[(size_t)r * kc + t] = y;
      }
    }
    nl_wait<0>();
    __syncthreads();
    // backward: z_r = (y_r - sum_d L(r+d, r) z_{r+d}) / L(r, r); column r of L gathered
#pragma unroll 1
    for (int pq = 0; pq < kWP - 1; ++pq) {
      const int r = n - 1 - pq;
      if (r >= 0)
        for (int q = t; q < bw; q += NT)
          if (r + q < n) nl_cp8(Lr + (size_t)(pq % kWP) * bw + q, band + (size_t)(r + q) * bw + q);
      nl_commit();
    }
    for (int tt = 0; tt < n; ++tt) {
      const int r = n - 1 - tt;
      const int tn = tt + kWP - 1, rn = n - 1 - tn;
      if (rn >= 0)
        for (int q = t; q < bw; q += NT)
          if (rn + q < n) nl_cp8(Lr + (size_t)(tn % kWP) * bw + q, band + (size_t)(rn + q) * bw + q);
      nl_commit();
      nl_wait<kWP - 1>();
      __syncthreads();
      const double* lc = Lr + (size_t)(tt % kWP) * bw;
      const int rs = r % bw;
      if (act) {
        double a0 = 0.0, a1 = 0.0;
        const int dm = min(b, n - 1 - r);
        int d = 1 + g;
        int sl = rs + d;                                 // ring slot of row r + d
        if (sl >= bw) sl -= bw;
        for (; d + G <= dm; d += 2 * G) {
          int s2 = sl + G;
          if (s2 >= bw) s2 -= bw;
          a0 = __fma_rn(lc[d], Zw[sl * kc + c], a0);
          a1 = __fma_rn(lc[d + G], Zw[s2 * kc + c], a1);
          sl = s2 + G;
          if (sl >= bw) sl -= bw;
        }
        if (d <= dm) a0 = __fma_rn(lc[d], Zw[sl * kc + c], a0);
        part[g * kc + c] = a0 + a1;
      }
      const double piv = lc[0];
      __syncthreads();
      if (t < kc) {
        double sacc = 0.0;
        for (int q = 0; q < G; ++q) sacc += part[q * kc + t];
        const double z = (Z[(size_t)r * kc + t] - sacc) / piv;
        Zw[rs * kc + t] = z;
        Z[(size_t)r * kc + t] = z;
      }
    }
    nl_wait<0>();
    __syncthreads();
    // ---- S = C Z (kc x kc) in shared memory; S(c1, c2) = sum_{l in c1} w_l Z(l, c2)
    double* S = ws;
    double* y = ws + (size_t)kc * kc;
    const int32_t* cp = P.cptr + D.cons0;
    for (int q = t; q < kc * kc; q += NT) {
      const int c1 = q / kc, c2 = q % kc;
      double acc = 0.0;
      for (int32_t e = cp[c1]; e < cp[c1 + 1]; ++e) {
        const int l = P.cidx[e];
        acc = __fma_rn(lw[l], Z[(size_t)l * kc + c2], acc);
      }
      S[q] = acc;
    }
    __syncthreads();
    for (int q = t; q < kc * kc; q += NT) {              // symmetrise (S = S^T exactly)
      const int c1 = q / kc, c2 = q % kc;
      if (c2 > c1) {
        const double v = 0.5 * (S[q] + S[c2 * kc + c1]);
        S[q] = v;
        S[c2 * kc + c1] = v;
      }
    }
    __syncthreads();
    for (int k = 0; k < kc; ++k) {                       // dense Cholesky, lower
      const double dk = S[k * kc + k];
      if (!(dk > 0.0)) {
        bad = true;
        break;
      }
      const double s = sqrt(dk);
      __syncthreads();
      for (int i = k + 1 + t; i < kc; i += NT) S[i * kc + k] /= s;
      if (t == 0) S[k * kc + k] = s;
      __syncthreads();
      for (int i = k + 1 + wid; i < kc; i += NW) {
        const double lik = S[i * kc + k];
        for (int j = k + 1 + lane; j <= i; j += 32) S[i * kc + j] = __fma_rn(-lik, S[j * kc + k], S[i * kc + j]);
      }
      __syncthreads();
    }
    if (__syncthreads_or(bad)) {
      if (t == 0) atomicCAS(P.err, 0, di + 1);
      continue;
    }
    // ---- psi = Z S^{-1} e_own for every coarse DOF of cell i
    for (int o = 0; o < D.nown; ++o) {
      const int ce = P.own_con[D.own0 + o];
      if (t == 0) {                                      // kc <= 128: serial triangular solves
        for (int i = 0; i < kc; ++i) {
          double sacc = (i == ce) ? 1.0 : 0.0;
          for (int j = 0; j < i; ++j) sacc = __fma_rn(-S[i * kc + j], y[j], sacc);
          y[i] = sacc / S[i * kc + i];
        }
        for (int i = kc - 1; i >= 0; --i) {
          double sacc = y[i];
          for (int j = i + 1; j < kc; ++j) sacc = __fma_rn(-S[j * kc + i], y[j], sacc);
          y[i] = sacc / S[i * kc + i];
        }
      }
      __syncthreads();
      double* out = P.psi + P.own_psi[D.own0 + o];
      for (int l = t; l < n; l += NT) {
        double acc = 0.0;
        for (int q = 0; q < kc; ++q) acc = __fma_rn(Z[(size_t)l * kc + q], y[q], acc);
        out[l] = acc;
      }
      __syncthreads();
    }
  }
}

// ---------------------------------------------------------------- projection kernel
// Dbar(r, s) = psi_r^T D psi_s = sum over connections (a, b) T (psi_r(a) - psi_r(b)) *
// (psi_s(a) - psi_s(b)) + sum_g ddiag_g psi_r(g) psi_s(g): one warp per pair, the
// connections of the fine DOFs of K_{i(s)}^+ (each connection counted at its lower end
// when both ends are inside, at the inside end otherwise).
//
// The bases stay in the per-region sparse storage the basis kernel wrote (psi[psi_off[r] +
// l], l = local DOF of K_{i(r)}^+): O(sum |K_i^+|) doubles.  psi_r(g) for a global fine DOF
// g is found through the region's window map: K_i^+ is a rectangle of fine cells, every
// fine DOF has a host cell and a layer (its continuum; several graph cells of one continuum
// in one host cell take successive layers), wmap[woff + (layer * wy + y) * wx + x] = l or -1.
struct NlProj {
  int64_t npair;
  const int32_t* pr;            // pair -> coarse DOF r, s
  const int32_t* ps;
  const int32_t* dom_of;        // coarse DOF -> domain
  const NlDomain* dom;
  const int32_t* lglob;
  const double* psi;            // bases, per-region local numbering
  const int64_t* psi_off;
  const int32_t* wmap;
  const int32_t* host;          // fine DOF -> host grid cell
  const int32_t* layer;         // fine DOF -> window layer
  int32_t nx, bx, by;
  const int32_t* arow;          // fine D in CSR (global): connections
  const int32_t* acol;
  const double* aval;
  const double* ddiag;
  double* out;                  // [npair]
};

// local DOF of fine DOF (host cell (hx, hy), layer) in region D, or -1 when outside K_i^+
__device__ __forceinline__ int nl_wloc(const NlProj& P, const NlDomain& D, int hx, int hy, int layer) {
  const int x = hx - D.cx0 * P.bx, y = hy - D.cy0 * P.by;
  const int wx = (D.cx1 - D.cx0 + 1) * P.bx, wy = (D.cy1 - D.cy0 + 1) * P.by;
  if ((unsigned)x >= (unsigned)wx || (unsigned)y >= (unsigned)wy) return -1;
  return P.wmap[D.woff + ((int64_t)layer * wy + y) * wx + x];
}

__global__ void nlmc_project_kernel(const NlProj P) {
  const int lane = threadIdx.x & 31;
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t pi = w; pi < P.npair; pi += nwarps) {
    const int r = P.pr[pi], s = P.ps[pi];
    const NlDomain Ds = P.dom[P.dom_of[s]];
    const NlDomain Dr = P.dom[P.dom_of[r]];
    const double* xr = P.psi + P.psi_off[r];
    const double* xs = P.psi + P.psi_off[s];
    double acc = 0.0;
    for (int l = lane; l < Ds.n; l += 32) {
      const int g = P.lglob[Ds.dof0 + l];
      const int hc = P.host[g], gy = hc / P.nx, gx = hc - gy * P.nx;
      const int lr = nl_wloc(P, Dr, gx, gy, P.layer[g]);
      const double rg = lr >= 0 ? xr[lr] : 0.0, sg = xs[l];
      double v = P.ddiag[g] * rg * sg;
      for (int32_t e = P.arow[g]; e < P.arow[g + 1]; ++e) {
        const int h = P.acol[e];
        const int hh = P.host[h], hy = hh / P.nx, hx = hh - hy * P.nx, hl = P.layer[h];
        const int ls = nl_wloc(P, Ds, hx, hy, hl);
        // count each connection once: at g if the other end h lies outside K_{i(s)}^+
        // (psi_s(h) = 0 there) or h > g
        if (ls < 0 || h > g) {
          const int lrh = nl_wloc(P, Dr, hx, hy, hl);
          const double d1 = rg - (lrh >= 0 ? xr[lrh] : 0.0), d2 = sg - (ls >= 0 ? xs[ls] : 0.0);
          v = __fma_rn(P.aval[e] * d1, d2, v);
        }
      }
      acc += v;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) P.out[pi] = acc;
  }
}

}  // namespace mc

using namespace mc;

struct mc_nlmc {
  ~mc_nlmc() {
    if (d_psi) cudaFree(d_psi);
  }
  std::string err;
  int L = 0;
  int64_t nH = 0, N = 0;
  int64_t n_alpha[MC_MAX_CONTINUA] = {0};
  std::vector<int32_t> key;          // 3 per coarse DOF
  std::vector<int32_t> fine_dof;
  std::vector<int32_t> rowptr, col;
  std::vector<double> val, mass, rhs, u0;
  double* d_psi = nullptr;           // bases in per-region local numbering (device), sum |K_i^+| x own DOFs
  std::vector<int64_t> psi_off;      // coarse DOF -> its basis in d_psi
  std::vector<int32_t> psi_dof0, psi_n;   // coarse DOF -> its region's slice of lglob
  std::vector<int32_t> lglob;        // region-local DOF -> global fine DOF
  double ms_basis = 0.0, ms_project = 0.0;
  double flops_basis = 0.0;          // fp64 operations of the basis kernel (Cholesky, substitutions, Schur)
  double bytes_bases = 0.0;          // device bytes that hold the bases and their window maps
};

namespace {

template <class T>
cudaError_t up(T** d, const std::vector<T>& h) {
  cudaError_t e = cudaMalloc(d, std::max<size_t>(h.size(), 1) * sizeof(T));
  if (e == cudaSuccess && !h.empty()) e = cudaMemcpy(*d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice);
  return e;
}

struct DevBufs {
  std::vector<void*> p;
  ~DevBufs() {
    for (void* v : p) cudaFree(v);
  }
  template <class T>
  cudaError_t put(T** d, const std::vector<T>& h) {
    cudaError_t e = up(d, h);
    if (e == cudaSuccess) p.push_back(*d);
    return e;
  }
  template <class T>
  cudaError_t alloc(T** d, size_t n) {
    cudaError_t e = cudaMalloc(d, std::max<size_t>(n, 1) * sizeof(T));
    if (e == cudaSuccess) p.push_back(*d);
    return e;
  }
};

struct UF {
  std::vector<int64_t> p;
  explicit UF(int64_t n) : p((size_t)n) { std::iota(p.begin(), p.end(), 0); }
  int64_t f(int64_t x) {
    while (p[(size_t)x] != x) x = p[(size_t)x] = p[(size_t)p[(size_t)x]];
    return x;
  }
  void u(int64_t a, int64_t b) {
    a = f(a);
    b = f(b);
    if (a != b) p[(size_t)std::max(a, b)] = std::min(a, b);   // root = smallest index
  }
};

}  // namespace

#define NL_CUDA(call)                                                                          \
  do {                                                                                         \
    cudaError_t e_ = (call);                                                                   \
    if (e_ != cudaSuccess) {                                                                   \
      char b_[512];                                                                            \
      snprintf(b_, sizeof b_, "NLMC: %s: %s", #call, cudaGetErrorString(e_));                 \
      delete nl;                                                                               \
      return ctx_error(fine, e_ == cudaErrorMemoryAllocation ? MC_ERR_NOMEM : MC_ERR_CUDA, b_); \
    }                                                                                          \
  } while (0)

extern "C" mc_status mc_nlmc_build(mc_ctx* fine, const mc_nlmc_desc* d, mc_nlmc** out) {
  if (!fine || !d || !out) return MC_ERR_ARG;
  *out = nullptr;
  FineSystem fs;
  mc_status st = export_fine(fine, d->host, fs);
  if (st != MC_OK) return st;
  char msg[512];
  if (d->nHx < 1 || d->nHy < 1 || fs.nx % d->nHx || fs.ny % d->nHy || d->oversample < 0) {
    snprintf(msg, sizeof msg, "NLMC: coarse grid %d x %d / oversampling %d invalid for the %d x %d grid", d->nHx,
             d->nHy, d->oversample, fs.nx, fs.ny);
    return ctx_error(fine, MC_ERR_ARG, msg);
  }
  const int nHx = d->nHx, nHy = d->nHy, m = d->oversample;
  const int bx = fs.nx / nHx, by = fs.ny / nHy;
  const int64_t N = fs.off[(size_t)fs.L];
  const int L = fs.L;
  // coarse cell of every fine DOF
  std::vector<int32_t> cell((size_t)N);
  for (int64_t g = 0; g < N; ++g) {
    const int32_t hc = fs.host[(size_t)g];
    cell[(size_t)g] = (hc / fs.nx / by) * nHx + (hc % fs.nx) / bx;
  }
  // pieces (C30): connected parts of each graph continuum inside one coarse cell
  UF uf(N);
  for (size_t e = 0; e < fs.ei.size(); ++e) {
    const int32_t a = fs.ei[e], b = fs.ej[e];
    if (fs.kind[(size_t)fs.cont[(size_t)a]] == 1 && cell[(size_t)a] == cell[(size_t)b]) uf.u(a, b);
  }
  std::vector<std::array<int64_t, 3>> keys;
  keys.reserve((size_t)N);
  std::vector<std::array<int64_t, 3>> fkey((size_t)N);
  for (int64_t g = 0; g < N; ++g) {
    const int a = fs.cont[(size_t)g];
    const int64_t piece = fs.kind[(size_t)a] == 1 ? uf.f(g) - fs.off[(size_t)a] : 0;
    fkey[(size_t)g] = {a, cell[(size_t)g], piece};
  }
  keys = fkey;
  std::sort(keys.begin(), keys.end());
  keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
  const int64_t nH = (int64_t)keys.size();
  std::vector<int32_t> fdof((size_t)N);
  for (int64_t g = 0; g < N; ++g)
    fdof[(size_t)g] = (int32_t)(std::lower_bound(keys.begin(), keys.end(), fkey[(size_t)g]) - keys.begin());
  mc_nlmc* nl = new mc_nlmc();
  nl->L = L;
  nl->nH = nH;
  nl->N = N;
  nl->fine_dof = fdof;
  for (auto& k : keys) {
    nl->n_alpha[k[0]]++;
    nl->key.push_back((int32_t)k[0]);
    nl->key.push_back((int32_t)k[1]);
    nl->key.push_back((int32_t)k[2]);
  }
  std::vector<double> kmeas((size_t)nH, 0.0), u0w((size_t)nH, 0.0);
  nl->mass.assign((size_t)nH, 0.0);
  nl->rhs.assign((size_t)nH, 0.0);
  std::vector<double> wbar((size_t)nH, 0.0), dbar1((size_t)nH, 0.0);
  for (int64_t g = 0; g < N; ++g) {
    const size_t r = (size_t)fdof[(size_t)g];
    kmeas[r] += fs.meas[(size_t)g];
    nl->mass[r] += fs.mass[(size_t)g];                 // c |K_j^alpha|
    nl->rhs[r] += fs.F[(size_t)g];                     // f |K_j^alpha|
    u0w[r] += fs.meas[(size_t)g] * fs.u0[(size_t)g];
    wbar[r] += fs.wdiag[(size_t)g];                    // wells (reading C31)
    dbar1[r] += fs.ddiag[(size_t)g];                   // P (D 1): boundary faces (reading C32)
  }
  nl->u0.resize((size_t)nH);
  for (int64_t r = 0; r < nH; ++r) nl->u0[(size_t)r] = u0w[(size_t)r] / kmeas[(size_t)r];
  // fine D (global CSR of connections) and D + Q adjacency
  std::vector<int32_t> arow((size_t)N + 1, 0), acol;
  std::vector<double> aval;
  {
    for (size_t e = 0; e < fs.ei.size(); ++e) {
      arow[(size_t)fs.ei[e] + 1]++;
      arow[(size_t)fs.ej[e] + 1]++;
    }
    for (int64_t g = 0; g < N; ++g) arow[(size_t)g + 1] += arow[(size_t)g];
    acol.resize((size_t)arow[(size_t)N]);
    aval.resize((size_t)arow[(size_t)N]);
    std::vector<int32_t> pos(arow.begin(), arow.end() - 1);
    for (size_t e = 0; e < fs.ei.size(); ++e) {
      acol[(size_t)pos[(size_t)fs.ei[e]]] = fs.ej[e];
      aval[(size_t)pos[(size_t)fs.ei[e]]++] = fs.et[e];
      acol[(size_t)pos[(size_t)fs.ej[e]]] = fs.ei[e];
      aval[(size_t)pos[(size_t)fs.ej[e]]++] = fs.et[e];
    }
  }
  std::vector<int32_t> qrow((size_t)N + 1, 0), qcol;
  std::vector<double> qval;
  {
    for (size_t e = 0; e < fs.qi.size(); ++e) {
      qrow[(size_t)fs.qi[e] + 1]++;
      qrow[(size_t)fs.qj[e] + 1]++;
    }
    for (int64_t g = 0; g < N; ++g) qrow[(size_t)g + 1] += qrow[(size_t)g];
    qcol.resize((size_t)qrow[(size_t)N]);
    qval.resize((size_t)qrow[(size_t)N]);
    std::vector<int32_t> pos(qrow.begin(), qrow.end() - 1);
    for (size_t e = 0; e < fs.qi.size(); ++e) {
      qcol[(size_t)pos[(size_t)fs.qi[e]]] = fs.qj[e];
      qval[(size_t)pos[(size_t)fs.qi[e]]++] = fs.qs[e];
      qcol[(size_t)pos[(size_t)fs.qj[e]]] = fs.qi[e];
      qval[(size_t)pos[(size_t)fs.qj[e]]++] = fs.qs[e];
    }
  }
  // diagonal of D + Q (connections leaving K_i^+ stay on the diagonal: zero Dirichlet)
  std::vector<double> fdiag((size_t)N);
  for (int64_t g = 0; g < N; ++g) {
    double s = fs.ddiag[(size_t)g];
    for (int32_t e = arow[(size_t)g]; e < arow[(size_t)g + 1]; ++e) s += aval[(size_t)e];
    for (int32_t e = qrow[(size_t)g]; e < qrow[(size_t)g + 1]; ++e) s += qval[(size_t)e];
    fdiag[(size_t)g] = s;
  }
  // fine DOFs of every coarse cell, in host-cell order
  std::vector<std::vector<int32_t>> incell((size_t)nHx * nHy);
  {
    std::vector<int32_t> order((size_t)N);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int32_t x, int32_t y) {
      if (fs.host[(size_t)x] != fs.host[(size_t)y]) return fs.host[(size_t)x] < fs.host[(size_t)y];
      return fs.cont[(size_t)x] < fs.cont[(size_t)y];
    });
    for (int32_t g : order) incell[(size_t)cell[(size_t)g]].push_back(g);
  }
  std::vector<std::vector<int32_t>> owned((size_t)nHx * nHy);
  for (int64_t r = 0; r < nH; ++r) owned[(size_t)keys[(size_t)r][1]].push_back((int32_t)r);
  // ---- per-domain data
  std::vector<NlDomain> dom;
  std::vector<int32_t> lglob, lcon, erow, eoff, cptr, cidx, own_con, dom_of((size_t)nH, -1);
  std::vector<double> lw, ldiag, eval;
  std::vector<int64_t> own_psi((size_t)0);
  std::vector<int64_t> psi_off((size_t)nH, -1);
  int64_t psi_len = 0;
  std::vector<int32_t> loc((size_t)N, -1);
  int nmax = 1, bmax = 0, kcmax = 1;
  int64_t spw_need = 1;
  // window layers: one per grid continuum; a graph continuum takes as many as its busiest
  // host cell holds cells of it (1 when the host map is injective, e.g. merged fracture cells)
  std::vector<int32_t> layer((size_t)N, 0), wmap;
  int nlayers = 0;
  {
    std::vector<int32_t> seen;
    for (int a = 0; a < L; ++a) {
      int mult = 1;
      if (fs.kind[(size_t)a] == 1) {
        seen.assign((size_t)fs.nx * fs.ny, 0);
        for (int64_t g = fs.off[(size_t)a]; g < fs.off[(size_t)a + 1]; ++g) {
          const int32_t k = seen[(size_t)fs.host[(size_t)g]]++;
          layer[(size_t)g] = nlayers + k;
          mult = std::max(mult, k + 1);
        }
      } else {
        for (int64_t g = fs.off[(size_t)a]; g < fs.off[(size_t)a + 1]; ++g) layer[(size_t)g] = nlayers;
      }
      nlayers += mult;
    }
  }
  for (int i = 0; i < nHx * nHy; ++i) {
    if (owned[(size_t)i].empty()) continue;
    const int iy = i / nHx, ix = i % nHx;
    // S: fine DOFs of K_i^+ sorted by host cell (then continuum): small bandwidth
    std::vector<int32_t> S;
    for (int jy = std::max(0, iy - m); jy <= std::min(nHy - 1, iy + m); ++jy)
      for (int jx = std::max(0, ix - m); jx <= std::min(nHx - 1, ix + m); ++jx)
        for (int32_t g : incell[(size_t)(jy * nHx + jx)]) S.push_back(g);
    std::stable_sort(S.begin(), S.end(), [&](int32_t x, int32_t y) {
      if (fs.host[(size_t)x] != fs.host[(size_t)y]) return fs.host[(size_t)x] < fs.host[(size_t)y];
      if (fs.cont[(size_t)x] != fs.cont[(size_t)y]) return fs.cont[(size_t)x] < fs.cont[(size_t)y];
      return x < y;
    });
    NlDomain D{};
    D.n = (int32_t)S.size();
    D.cx0 = std::max(0, ix - m);
    D.cx1 = std::min(nHx - 1, ix + m);
    D.cy0 = std::max(0, iy - m);
    D.cy1 = std::min(nHy - 1, iy + m);
    D.dof0 = (int64_t)lglob.size();
    D.ent0 = (int64_t)erow.size();
    for (int l = 0; l < D.n; ++l) loc[(size_t)S[(size_t)l]] = l;
    {
      const int wx = (D.cx1 - D.cx0 + 1) * bx, wy = (D.cy1 - D.cy0 + 1) * by;
      D.woff = (int64_t)wmap.size();
      wmap.resize(wmap.size() + (size_t)nlayers * wx * wy, -1);
      for (int l = 0; l < D.n; ++l) {
        const int32_t g = S[(size_t)l], hc = fs.host[(size_t)g];
        const int x = hc % fs.nx - D.cx0 * bx, y = hc / fs.nx - D.cy0 * by;
        wmap[(size_t)(D.woff + ((int64_t)layer[(size_t)g] * wy + y) * wx + x)] = l;
      }
    }
    // constraints: coarse DOFs present in K_i^+ (ascending)
    std::vector<int32_t> cons;
    for (int32_t g : S) cons.push_back(fdof[(size_t)g]);
    std::sort(cons.begin(), cons.end());
    cons.erase(std::unique(cons.begin(), cons.end()), cons.end());
    D.kc = (int32_t)cons.size();
    int b = 0;
    // singularity check (exact, structural): every connected part of the region's graph
    // needs a sink -- a connection leaving K_i^+ (zero Dirichlet) or a boundary term
    UF luf(D.n);
    std::vector<uint8_t> sink((size_t)D.n, 0);
    for (int l = 0; l < D.n; ++l) {
      const int32_t g = S[(size_t)l];
      if (fs.ddiag[(size_t)g] > 0.0) sink[(size_t)l] = 1;
      auto look = [&](int32_t h) {
        const int32_t lh = loc[(size_t)h];
        if (lh < 0) sink[(size_t)l] = 1;
        else luf.u(l, lh);
      };
      for (int32_t e = arow[(size_t)g]; e < arow[(size_t)g + 1]; ++e) look(acol[(size_t)e]);
      for (int32_t e = qrow[(size_t)g]; e < qrow[(size_t)g + 1]; ++e) look(qcol[(size_t)e]);
    }
    {
      std::vector<uint8_t> rs((size_t)D.n, 0);
      for (int l = 0; l < D.n; ++l)
        if (sink[(size_t)l]) rs[(size_t)luf.f(l)] = 1;
      for (int l = 0; l < D.n; ++l)
        if (!rs[(size_t)luf.f(l)]) {
          snprintf(msg, sizeof msg, "NLMC: local operator of coarse cell %d is not positive definite (a part of "
                   "K_i^+ has no connection out of the region and no boundary term)", i);
          delete nl;
          return ctx_error(fine, MC_ERR_ARG, msg);
        }
    }
    for (int l = 0; l < D.n; ++l) {
      const int32_t g = S[(size_t)l];
      lglob.push_back(g);
      lcon.push_back((int32_t)(std::lower_bound(cons.begin(), cons.end(), fdof[(size_t)g]) - cons.begin()));
      lw.push_back(fs.meas[(size_t)g] / kmeas[(size_t)fdof[(size_t)g]]);
      ldiag.push_back(fdiag[(size_t)g]);
      auto add = [&](int32_t h, double v) {
        const int32_t lh = loc[(size_t)h];
        if (lh < 0 || lh >= l) return;                  // outside K_i^+, or upper triangle
        erow.push_back(l);
        eoff.push_back(l - lh);
        eval.push_back(-v);
        b = std::max(b, l - lh);
      };
      for (int32_t e = arow[(size_t)g]; e < arow[(size_t)g + 1]; ++e) add(acol[(size_t)e], aval[(size_t)e]);
      for (int32_t e = qrow[(size_t)g]; e < qrow[(size_t)g + 1]; ++e) add(qcol[(size_t)e], qval[(size_t)e]);
    }
    D.b = b;
    D.nent = (int64_t)erow.size() - D.ent0;
    // constraint -> local DOFs (CSR, ascending local index)
    D.cons0 = (int64_t)cptr.size();
    {
      std::vector<int32_t> cnt((size_t)D.kc + 1, 0);
      for (int l = 0; l < D.n; ++l) cnt[(size_t)lcon[(size_t)(D.dof0 + l)] + 1]++;
      for (int q = 0; q < D.kc; ++q) cnt[(size_t)q + 1] += cnt[(size_t)q];
      const int32_t base = (int32_t)cidx.size();
      std::vector<int32_t> pos(cnt.begin(), cnt.end() - 1);
      cidx.resize(cidx.size() + (size_t)D.n);
      for (int l = 0; l < D.n; ++l) cidx[(size_t)(base + pos[(size_t)lcon[(size_t)(D.dof0 + l)]]++)] = l;
      for (int q = 0; q <= D.kc; ++q) cptr.push_back(base + cnt[(size_t)q]);
    }
    D.own0 = (int32_t)own_con.size();
    D.nown = (int32_t)owned[(size_t)i].size();
    for (int32_t r : owned[(size_t)i]) {
      own_con.push_back((int32_t)(std::lower_bound(cons.begin(), cons.end(), r) - cons.begin()));
      own_psi.push_back(psi_len);
      psi_off[(size_t)r] = psi_len;
      psi_len += D.n;
      dom_of[(size_t)r] = (int32_t)dom.size();
    }
    for (int32_t g : S) loc[(size_t)g] = -1;
    nmax = std::max(nmax, D.n);
    bmax = std::max(bmax, b);
    kcmax = std::max(kcmax, D.kc);
    const int64_t need = std::max<int64_t>((int64_t)(b + 1 + kWP) * (b + 1) + b + 1,
                                           std::max<int64_t>((int64_t)kWP * (b + 1) + (int64_t)(b + 1) * D.kc +
                                                                 (int64_t)(kNlThreads / std::max(1, D.kc)) * D.kc,
                                                             (int64_t)D.kc * D.kc + D.kc));
    spw_need = std::max<int64_t>(spw_need, need);
    if (D.kc > kNlMaxCons || need > kNlSmemDoubles) {
      snprintf(msg, sizeof msg, "NLMC: region of coarse cell %d too large for one CTA (bandwidth %d, %d constraints)",
               i, b, D.kc);
      delete nl;
      return ctx_error(fine, MC_ERR_ARG, msg);
    }
    {
      // fp64 operations of this region: banded Cholesky n (b+1)^2, forward + backward
      // substitution of kc columns 4 n (b+1) kc, S = C Z 2 n kc, dense Cholesky kc^3 / 3,
      // psi = Z S^-1 e per own DOF 2 kc^2 + 2 n kc
      const double n_ = D.n, b_ = b + 1, k_ = D.kc;
      nl->flops_basis += n_ * b_ * b_ + 4.0 * n_ * b_ * k_ + 2.0 * n_ * k_ + k_ * k_ * k_ / 3.0 +
                         (double)D.nown * (2.0 * k_ * k_ + 2.0 * n_ * k_);
    }
    dom.push_back(D);
  }
  // ---- device: bases
  int sms = 0;
  NL_CUDA(cudaSetDevice(fs.device));                  // the fine context's device
  NL_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, fs.device));
  // one region per CTA; as many CTAs per SM as their shared memory allows (<= 8)
  const int spw = (int)((spw_need + 1) & ~int64_t(1));
  const int wpb = 1;
  const int per_sm = std::max(1, std::min<int>(8, (228 * 1024) / (spw * 8 + 2048)));
  const int grid = std::max(1, std::min<int>((int)dom.size(), sms * per_sm));
  DevBufs B;
  NlParams P{};
  NlDomain* ddom;
  int32_t *dlglob, *dlcon, *derow, *deoff, *dcptr, *dcidx, *down_con, *derr;
  double *dlw, *dldiag, *deval, *dband, *dZ, *dpsi;
  int64_t* down_psi;
  NL_CUDA(B.put(&ddom, dom));
  NL_CUDA(B.put(&dlglob, lglob));
  NL_CUDA(B.put(&dlcon, lcon));
  NL_CUDA(B.put(&dlw, lw));
  NL_CUDA(B.put(&dldiag, ldiag));
  NL_CUDA(B.put(&derow, erow));
  NL_CUDA(B.put(&deoff, eoff));
  NL_CUDA(B.put(&deval, eval));
  NL_CUDA(B.put(&dcptr, cptr));
  NL_CUDA(B.put(&dcidx, cidx));
  NL_CUDA(B.put(&down_con, own_con));
  NL_CUDA(B.put(&down_psi, own_psi));
  P.band_stride = (int64_t)nmax * (bmax + 1);
  P.z_stride = (int64_t)nmax * kcmax;
  NL_CUDA(B.alloc(&dband, (size_t)grid * wpb * P.band_stride));
  NL_CUDA(B.alloc(&dZ, (size_t)grid * wpb * P.z_stride));
  NL_CUDA(cudaMalloc(&dpsi, std::max<size_t>((size_t)psi_len, 1) * sizeof(double)));   // kept: the bases
  nl->d_psi = dpsi;
  NL_CUDA(B.alloc(&derr, 1));
  NL_CUDA(cudaMemset(derr, 0, sizeof(int32_t)));
  P.dom = ddom;
  P.ndom = (int32_t)dom.size();
  P.lglob = dlglob;
  P.lcon = dlcon;
  P.lw = dlw;
  P.ldiag = dldiag;
  P.erow = derow;
  P.eoff = deoff;
  P.eval = deval;
  P.cptr = dcptr;
  P.cidx = dcidx;
  P.own_con = down_con;
  P.own_psi = down_psi;
  P.band = dband;
  P.Z = dZ;
  P.psi = dpsi;
  P.err = derr;
  P.wpb = wpb;
  P.spw = spw;
  const size_t smem = (size_t)wpb * spw * sizeof(double);
  // large regions (<= 2 per SM) take 512 threads, small ones 256 (measured)
  const bool wide = per_sm <= 2;
  if (wide) NL_CUDA(cudaFuncSetAttribute(nlmc_basis_kernel<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  else NL_CUDA(cudaFuncSetAttribute(nlmc_basis_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaEvent_t e0, e1, e2;
  NL_CUDA(cudaEventCreate(&e0));
  NL_CUDA(cudaEventCreate(&e1));
  NL_CUDA(cudaEventCreate(&e2));
  NL_CUDA(cudaEventRecord(e0));
  if (wide) nlmc_basis_kernel<512><<<grid, 512, smem>>>(P);
  else nlmc_basis_kernel<256><<<grid, 256, smem>>>(P);
  NL_CUDA(cudaGetLastError());
  NL_CUDA(cudaEventRecord(e1));
  int32_t herr = 0;
  NL_CUDA(cudaMemcpy(&herr, derr, sizeof herr, cudaMemcpyDeviceToHost));
  if (herr) {
    int ci = 0, k = 0;
    for (int i = 0; i < nHx * nHy; ++i)
      if (!owned[(size_t)i].empty() && k++ == herr - 1) ci = i;
    snprintf(msg, sizeof msg, "NLMC: local operator of coarse cell %d is not positive definite (singular K_i^+ "
             "system: no-flow region without sink?)", ci);
    delete nl;
    return ctx_error(fine, MC_ERR_ARG, msg);
  }
  // ---- the bases stay in their per-region storage (dpsi); project from it
  nl->psi_off = psi_off;
  nl->lglob = lglob;
  nl->bytes_bases = 8.0 * (double)psi_len + 4.0 * (double)wmap.size();
  nl->psi_dof0.resize((size_t)nH);
  nl->psi_n.resize((size_t)nH);
  for (int64_t r = 0; r < nH; ++r) {
    const NlDomain& Dr = dom[(size_t)dom_of[(size_t)r]];
    nl->psi_dof0[(size_t)r] = (int32_t)Dr.dof0;
    nl->psi_n[(size_t)r] = Dr.n;
  }
  // pairs (r <= s) whose regions overlap
  std::vector<int32_t> pr, ps;
  for (int64_t r = 0; r < nH; ++r)
    for (int64_t s = r; s < nH; ++s) {
      const int ci = keys[(size_t)r][1], cj = keys[(size_t)s][1];
      if (std::abs(ci / nHx - cj / nHx) <= 2 * m + 1 && std::abs(ci % nHx - cj % nHx) <= 2 * m + 1) {
        pr.push_back((int32_t)r);
        ps.push_back((int32_t)s);
      }
    }
  NlProj Q{};
  int32_t *dpr, *dps, *ddom_of, *darow, *dacol, *dwmap, *dhost, *dlayer;
  int64_t* dpoff;
  double *daval, *dddiag, *dout;
  NL_CUDA(B.put(&dpr, pr));
  NL_CUDA(B.put(&dps, ps));
  NL_CUDA(B.put(&ddom_of, dom_of));
  NL_CUDA(B.put(&darow, arow));
  NL_CUDA(B.put(&dacol, acol));
  NL_CUDA(B.put(&daval, aval));
  NL_CUDA(B.put(&dddiag, fs.ddiag));
  NL_CUDA(B.put(&dwmap, wmap));
  NL_CUDA(B.put(&dhost, fs.host));
  NL_CUDA(B.put(&dlayer, layer));
  NL_CUDA(B.put(&dpoff, psi_off));
  NL_CUDA(B.alloc(&dout, pr.size()));
  Q.npair = (int64_t)pr.size();
  Q.pr = dpr;
  Q.ps = dps;
  Q.dom_of = ddom_of;
  Q.dom = ddom;
  Q.lglob = dlglob;
  Q.psi = dpsi;
  Q.psi_off = dpoff;
  Q.wmap = dwmap;
  Q.host = dhost;
  Q.layer = dlayer;
  Q.nx = fs.nx;
  Q.bx = bx;
  Q.by = by;
  Q.arow = darow;
  Q.acol = dacol;
  Q.aval = daval;
  Q.ddiag = dddiag;
  Q.out = dout;
  cudaEvent_t e3;
  NL_CUDA(cudaEventCreate(&e3));
  NL_CUDA(cudaEventRecord(e3));
  nlmc_project_kernel<<<std::max(1, std::min<int>((int)((pr.size() + 7) / 8), 8 * sms)), 256>>>(Q);
  NL_CUDA(cudaGetLastError());
  NL_CUDA(cudaEventRecord(e2));
  std::vector<double> dv(pr.size());
  NL_CUDA(cudaMemcpy(dv.data(), dout, dv.size() * sizeof(double), cudaMemcpyDeviceToHost));
  float t1 = 0.f, t2 = 0.f;
  NL_CUDA(cudaEventElapsedTime(&t1, e0, e1));
  NL_CUDA(cudaEventElapsedTime(&t2, e3, e2));
  cudaEventDestroy(e3);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaEventDestroy(e2);
  nl->ms_basis = t1;
  nl->ms_project = t2;
  // ---- Abar = Dbar (flux form, C32) + Qbar + Wbar (aggregated, C31), CSR
  std::vector<std::vector<std::pair<int32_t, double>>> rows((size_t)nH);
  for (size_t q = 0; q < pr.size(); ++q) {
    if (pr[q] == ps[q]) continue;
    rows[(size_t)pr[q]].emplace_back(ps[q], dv[q]);
    rows[(size_t)ps[q]].emplace_back(pr[q], dv[q]);
  }
  for (size_t e = 0; e < fs.qi.size(); ++e) {
    const int32_t r1 = fdof[(size_t)fs.qi[e]], r2 = fdof[(size_t)fs.qj[e]];
    rows[(size_t)r1].emplace_back(r1, fs.qs[e]);
    rows[(size_t)r2].emplace_back(r2, fs.qs[e]);
    rows[(size_t)r1].emplace_back(r2, -fs.qs[e]);
    rows[(size_t)r2].emplace_back(r1, -fs.qs[e]);
  }
  nl->rowptr.assign((size_t)nH + 1, 0);
  for (int64_t r = 0; r < nH; ++r) {
    auto& row = rows[(size_t)r];
    std::stable_sort(row.begin(), row.end(),
                     [](const std::pair<int32_t, double>& x, const std::pair<int32_t, double>& y) {
                       return x.first < y.first;
                     });
    std::vector<std::pair<int32_t, double>> merged;
    for (auto& pv : row) {
      if (!merged.empty() && merged.back().first == pv.first) merged.back().second += pv.second;
      else merged.push_back(pv);
    }
    row.swap(merged);
  }
  // flux-form diagonal of Dbar: P(D 1) - sum_{s != r} Dbar(r, s)
  std::vector<double> doff((size_t)nH, 0.0);
  for (size_t q = 0; q < pr.size(); ++q) {
    if (pr[q] == ps[q]) continue;
    doff[(size_t)pr[q]] += dv[q];
    doff[(size_t)ps[q]] += dv[q];
  }
  for (int64_t r = 0; r < nH; ++r) {
    auto& row = rows[(size_t)r];
    const double dd = dbar1[(size_t)r] - doff[(size_t)r] + wbar[(size_t)r];
    auto it = std::lower_bound(row.begin(), row.end(), std::make_pair((int32_t)r, -(double)INFINITY));
    if (it != row.end() && it->first == r) it->second += dd;
    else row.insert(it, std::make_pair((int32_t)r, dd));
    for (auto& pv : row) {
      nl->col.push_back(pv.first);
      nl->val.push_back(pv.second);
    }
    nl->rowptr[(size_t)r + 1] = (int32_t)nl->col.size();
  }
  *out = nl;
  return MC_OK;
}

extern "C" mc_status mc_nlmc_sizes(const mc_nlmc* nl, int64_t* n_alpha, int64_t* nnz, int64_t* n_fine) {
  if (!nl) return MC_ERR_ARG;
  if (n_alpha)
    for (int a = 0; a < MC_MAX_CONTINUA; ++a) n_alpha[a] = nl->n_alpha[a];
  if (nnz) *nnz = (int64_t)nl->col.size();
  if (n_fine) *n_fine = nl->N;
  return MC_OK;
}

template <class T>
static mc_status put_out(T* dst, const std::vector<T>& src) {
  if (!dst || src.empty()) return MC_OK;
  return cudaMemcpy(dst, src.data(), src.size() * sizeof(T), cudaMemcpyDefault) == cudaSuccess ? MC_OK
                                                                                                : MC_ERR_CUDA;
}

extern "C" mc_status mc_nlmc_get(const mc_nlmc* nl, int32_t* rowptr, int32_t* col, double* val, double* mass,
                                 double* rhs, double* u0, int32_t* key, int32_t* fine_dof) {
  if (!nl) return MC_ERR_ARG;
  mc_status st = MC_OK;
  if (st == MC_OK) st = put_out(rowptr, nl->rowptr);
  if (st == MC_OK) st = put_out(col, nl->col);
  if (st == MC_OK) st = put_out(val, nl->val);
  if (st == MC_OK) st = put_out(mass, nl->mass);
  if (st == MC_OK) st = put_out(rhs, nl->rhs);
  if (st == MC_OK) st = put_out(u0, nl->u0);
  if (st == MC_OK) st = put_out(key, nl->key);
  if (st == MC_OK) st = put_out(fine_dof, nl->fine_dof);
  return st;
}

extern "C" mc_status mc_nlmc_basis(const mc_nlmc* nl, int64_t r, double* psi) {
  if (!nl || !psi || r < 0 || r >= nl->nH) return MC_ERR_ARG;
  // expand the region-local basis into a fine vector (zero outside K_i^+)
  const int32_t n = nl->psi_n[(size_t)r];
  std::vector<double> loc((size_t)n), out((size_t)nl->N, 0.0);
  if (cudaMemcpy(loc.data(), nl->d_psi + nl->psi_off[(size_t)r], (size_t)n * sizeof(double), cudaMemcpyDeviceToHost) !=
      cudaSuccess)
    return MC_ERR_CUDA;
  const int32_t* lg = nl->lglob.data() + nl->psi_dof0[(size_t)r];
  for (int32_t l = 0; l < n; ++l) out[(size_t)lg[l]] = loc[(size_t)l];
  return cudaMemcpy(psi, out.data(), (size_t)nl->N * sizeof(double), cudaMemcpyDefault) == cudaSuccess ? MC_OK
                                                                                                      : MC_ERR_CUDA;
}

extern "C" mc_status mc_nlmc_cost(const mc_nlmc* nl, double* flops_basis, double* bytes_bases) {
  if (!nl) return MC_ERR_ARG;
  if (flops_basis) *flops_basis = nl->flops_basis;
  if (bytes_bases) *bytes_bases = nl->bytes_bases;
  return MC_OK;
}

extern "C" mc_status mc_nlmc_times(const mc_nlmc* nl, double* ms_basis, double* ms_project) {
  if (!nl) return MC_ERR_ARG;
  if (ms_basis) *ms_basis = nl->ms_basis;
  if (ms_project) *ms_project = nl->ms_project;
  return MC_OK;
}

extern "C" const char* mc_nlmc_error_string(const mc_nlmc* nl) { return nl ? nl->err.c_str() : ""; }

extern "C" mc_status mc_nlmc_destroy(mc_nlmc* nl) {
  delete nl;
  return MC_OK;
}
