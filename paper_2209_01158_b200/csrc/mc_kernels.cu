// mc_kernels.cu — the sm_100a step kernel of libmc.
//
// One persistent, cooperatively launched kernel advances the whole system by one time
// layer.  Its CTAs are partitioned into groups; each group runs one
// Jacobi-preconditioned CG solve:
//   D-scheme: one group per continuum, all groups concurrently; the
//            inter-continuum transfer enters only the right-hand side, from layer n-1.
//   coupled: one group over all continua, transfer in the operator.
//
// Per step:   init pass   b = (m/tau) u^{n-1} + F [+ sum_b Q_ab u_b^{n-1}],  r0 = b - K x0,
//                         x0 = u^{n-1} (warm start);  one group reduction.
//             CG passes   one fused pass and ONE group reduction per iteration:
//                         r_j = r_{j-1} - a q_{j-1};  x_j = x_{j-1} + a p_{j-1};
//                         p_j = D^{-1} r_j + b p_{j-1};  q_j = K p_j;
//                         partials (p.q, r.r, r.z, z.q, q.D^{-1}q) -> a = (r.z)/(p.q),
//                         (r.z)_{j+1} = r.z - 2a z.q + a^2 q.D^{-1}q,  b = (r.z)_{j+1}/(r.z).
//   This is CG in exact arithmetic with the recursive residual computed exactly
//   (reading C13 stop rule), reorganised so each iteration reads every vector once
//   (single-reduction form).  Neighbour values of p_j needed by the
//   SpMV are recomputed from r, q, p of the previous iteration (bitwise identical
//   to what the owner stores), so no barrier separates the update from the SpMV.
//
// Operators (flux form, reading C15):
//   grid: q_i = ds_i p_i + sum_faces T_f (p_i - p_nb)
//   graph: q_i = ds_i p_i + sum_e T_e (p_i - p_j)
//   coupled adds sum_cpl sigma (p_i - p_other).
#include <algorithm>

#include "mc_internal.h"

namespace mc {

__device__ __forceinline__ double ldro(const double* p) { return __ldg(p); }
__device__ __forceinline__ int32_t ldro(const int32_t* p) { return __ldg(p); }
__device__ __forceinline__ double ldmut(const double* p) { return __ldcg(p); }
// L1-cached load of a vector written in the previous pass: safe because every CTA's
// barrier acquire (ld.acquire.gpu) invalidates its SM's L1 before the next pass reads.
__device__ __forceinline__ double ldnb(const double* p) { return *p; }
__device__ __forceinline__ void stmut(double* p, double v) { __stcg(p, v); }

__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void red_release_add(unsigned long long* p, unsigned long long v) {
  asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ long long globaltimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// p_j = D^{-1}(r_{j-1} - a q_{j-1}) + b p_{j-1}; one definition used by owners and by
// neighbours so the recomputed halo value is bitwise identical to the stored one.
__device__ __forceinline__ double pnew(double ro, double qo, double po, double di, double a,
                                       double b) {
  const double rn = __fma_rn(-a, qo, ro);
  return __fma_rn(di, rn, __dmul_rn(b, po));
}

// 32-byte records {r, q, p, D^-1} published by the resident ELL pass: one 256-bit access each
__device__ __forceinline__ void st_rec(double* rec, double r, double q, double p, double d) {
  asm volatile("st.global.cg.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(rec), "d"(r), "d"(q), "d"(p), "d"(d) : "memory");
}
__device__ __forceinline__ double pn_rec(const double* rec, double a, double b) {
  double r, q, p, d;
  asm volatile("ld.global.cg.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(r), "=d"(q), "=d"(p), "=d"(d) : "l"(rec) : "memory");
  return pnew(r, q, p, d, a, b);
}

#if MC_PROF
// dev instrumentation (-DMC_PROF=1 builds only): clock64 per phase of the CG loop,
// summed over iterations by thread 0 of each group's first CTA
__device__ long long g_prof[MC_MAX_CONTINUA][8];
#define PROF_T(v) long long v = clock64()
#define PROF_ADD(g, k, d) atomicAdd((unsigned long long*)&g_prof[g][k], (unsigned long long)(d))
#else
#define PROF_T(v)
#define PROF_ADD(g, k, d)
#endif

struct Ctx {
  const StepParams* P;
  const double* rs;
  const double* qs;
  const double* ps;
  double* rd;
  double* pd;
  double* qd;
  double* x;
  const double* ds;
  double a, b;

  __device__ __forceinline__ double pn_at(int64_t gi) const {
    MC_ASSERT(gi >= 0 && gi < P->N + kSlack);   // rows past n of a last chunk read the zeroed slack, discarded
    return pnew(ldnb(rs + gi), ldnb(qs + gi), ldnb(ps + gi), ldro(P->dinv + gi), a, b);
  }
  // owner update of row gi: x, r, p stored; returns p_j, r_j, D^{-1}_ii
  __device__ __forceinline__ void own(int64_t gi, double& pn, double& rn, double& di) const {
    MC_ASSERT(gi >= 0 && gi < P->N + kSlack);   // rows past n of a last chunk read the zeroed slack, discarded
    const double ro = ldmut(rs + gi), qo = ldmut(qs + gi), po = ldmut(ps + gi);
    di = ldro(P->dinv + gi);
    const double xo = x[gi];
    rn = __fma_rn(-a, qo, ro);
    pn = __fma_rn(di, rn, __dmul_rn(b, po));
    x[gi] = __fma_rn(a, po, xo);
    stmut(rd + gi, rn);
    stmut(pd + gi, pn);
  }
  __device__ __forceinline__ double couple_q(int64_t gi, double pc) const {
    double acc = 0.0;
    const int32_t e0 = ldro(P->cptr + gi), e1 = ldro(P->cptr + gi + 1);
    MC_ASSERT(e0 <= e1);
    for (int32_t e = e0; e < e1; ++e) {
      const int32_t j = ldro(P->cidx + e);
      acc += ldro(P->cval + e) * (pc - pn_at(j));
    }
    return acc;
  }
  // the same sum with the row's entry range [e0, e1) already loaded (grid strips load the
  // range before they wait for the staged row, so the first of the three dependent trips
  // -- range, entry, neighbour -- is off the critical path)
  __device__ __forceinline__ double couple_q_range(int32_t e0, int32_t e1, double pc) const {
    double acc = 0.0;
    for (int32_t e = e0; e < e1; ++e) {
      const int32_t j = ldro(P->cidx + e);
      acc += ldro(P->cval + e) * (pc - pn_at(j));
    }
    return acc;
  }
  __device__ __forceinline__ void accum(double (&acc)[kNPart], double pc, double rc, double dc,
                                        double qv) const {
    acc[0] += pc * qv;        // p.q
    acc[1] += rc * rc;        // r.r   (exact recursive residual norm)
    acc[2] += dc * rc * rc;   // r.z   (z = D^{-1} r)
    acc[3] += dc * rc * qv;   // z.q
    acc[4] += dc * qv * qv;   // q.D^{-1}q
  }
};

// ---------------------------------------------------------------- CG pass, grid strip
template <bool CPL>
__device__ void iter_grid(const Ctx& c, const ContDev& C, int x0, int y0, int y1,
                          double (&acc)[kNPart]) {
  const int lane = threadIdx.x & 31;
  const int nx = C.nx, ny = C.ny;
  const int col = x0 + lane;
  const bool valid = col < nx;
  const int64_t off = C.off;
  double pm = 0.0, tym = 0.0;
  if (valid && y0 > 0) {
    const int64_t i = (int64_t)(y0 - 1) * nx + col;
    pm = c.pn_at(off + i);
    tym = ldro(C.Ty + i);
  }
  double pc = 0.0, rc = 0.0, dc = 0.0;
  if (valid) c.own(off + (int64_t)y0 * nx + col, pc, rc, dc);
  for (int y = y0; y < y1; ++y) {
    const int64_t i = (int64_t)y * nx + col;
    const int64_t gi = off + i;
    double pp = 0.0, rp = 0.0, dp = 0.0;
    if (valid && y + 1 < ny) {
      if (y + 1 < y1) c.own(gi + nx, pp, rp, dp);
      else pp = c.pn_at(gi + nx);
    }
    const double txc = valid ? ldro(C.Tx + i) : 0.0;
    double pl = __shfl_up_sync(0xffffffffu, pc, 1);
    double pr = __shfl_down_sync(0xffffffffu, pc, 1);
    double txl = __shfl_up_sync(0xffffffffu, txc, 1);
    if (lane == 0) {
      if (valid && col > 0) {
        pl = c.pn_at(gi - 1);
        txl = ldro(C.Tx + i - 1);
      } else {
        pl = 0.0;
        txl = 0.0;
      }
    }
    if (lane == 31) pr = (valid && col + 1 < nx) ? c.pn_at(gi + 1) : 0.0;
    if (valid) {
      const double tyc = ldro(C.Ty + i);
      double qv = ldro(c.ds + gi) * pc;
      qv += txc * (pc - pr);
      qv += txl * (pc - pl);
      qv += tyc * (pc - pp);
      qv += tym * (pc - pm);
      if (CPL) qv += c.couple_q(gi, pc);
      stmut(c.qd + gi, qv);
      c.accum(acc, pc, rc, dc, qv);
      tym = tyc;
    }
    pm = pc;
    pc = pp;
    rc = rp;
    dc = dp;
  }
}

// ---------------------------------------------------------------- CG pass, grid strip, 2 columns per lane
// (even nx): every load and store is a 16-byte double2, a warp covers 64 columns.
__device__ __forceinline__ double2 ld2ro(const double* p) { return __ldg(reinterpret_cast<const double2*>(p)); }
__device__ __forceinline__ double2 ld2mut(const double* p) { return __ldcg(reinterpret_cast<const double2*>(p)); }
__device__ __forceinline__ void st2mut(double* p, double2 v) { __stcg(reinterpret_cast<double2*>(p), v); }

struct Row2 {
  double2 p, r, d;
};

__device__ __forceinline__ double2 pnew2(const Ctx& c, int64_t gi) {
  const double2 ro = ld2mut(c.rs + gi), qo = ld2mut(c.qs + gi), po = ld2mut(c.ps + gi);
  const double2 di = ld2ro(c.P->dinv + gi);
  return make_double2(pnew(ro.x, qo.x, po.x, di.x, c.a, c.b), pnew(ro.y, qo.y, po.y, di.y, c.a, c.b));
}

__device__ __forceinline__ Row2 own2(const Ctx& c, int64_t gi) {
  const double2 ro = ld2mut(c.rs + gi), qo = ld2mut(c.qs + gi), po = ld2mut(c.ps + gi);
  const double2 di = ld2ro(c.P->dinv + gi);
  const double2 xo = *reinterpret_cast<const double2*>(c.x + gi);
  Row2 o;
  o.d = di;
  o.r = make_double2(__fma_rn(-c.a, qo.x, ro.x), __fma_rn(-c.a, qo.y, ro.y));
  o.p = make_double2(__fma_rn(di.x, o.r.x, __dmul_rn(c.b, po.x)), __fma_rn(di.y, o.r.y, __dmul_rn(c.b, po.y)));
  *reinterpret_cast<double2*>(c.x + gi) = make_double2(__fma_rn(c.a, po.x, xo.x), __fma_rn(c.a, po.y, xo.y));
  st2mut(c.rd + gi, o.r);
  st2mut(c.pd + gi, o.p);
  return o;
}

template <bool CPL>
__device__ void iter_grid2(const Ctx& c, const ContDev& C, int x0, int y0, int y1,
                           double (&acc)[kNPart]) {
  const int lane = threadIdx.x & 31;
  const int nx = C.nx, ny = C.ny;
  const int c0 = x0 + 2 * lane;
  const bool valid = c0 < nx;              // nx even: c0 + 1 < nx as well
  const int64_t off = C.off;
  double2 pm = make_double2(0.0, 0.0), tym = make_double2(0.0, 0.0);
  if (valid && y0 > 0) {
    const int64_t i = (int64_t)(y0 - 1) * nx + c0;
    pm = pnew2(c, off + i);
    tym = ld2ro(C.Ty + i);
  }
  Row2 cur;
  cur.p = cur.r = cur.d = make_double2(0.0, 0.0);
  if (valid) cur = own2(c, off + (int64_t)y0 * nx + c0);
  for (int y = y0; y < y1; ++y) {
    const int64_t i = (int64_t)y * nx + c0;
    const int64_t gi = off + i;
    Row2 nxt;
    nxt.p = nxt.r = nxt.d = make_double2(0.0, 0.0);
    if (valid && y + 1 < ny) {
      if (y + 1 < y1) nxt = own2(c, gi + nx);
      else nxt.p = pnew2(c, gi + nx);
    }
    const double2 tx = valid ? ld2ro(C.Tx + i) : make_double2(0.0, 0.0);
    double pl = __shfl_up_sync(0xffffffffu, cur.p.y, 1);
    double pr = __shfl_down_sync(0xffffffffu, cur.p.x, 1);
    double txl = __shfl_up_sync(0xffffffffu, tx.y, 1);
    if (lane == 0) {
      if (valid && c0 > 0) {
        pl = c.pn_at(gi - 1);
        txl = ldro(C.Tx + i - 1);
      } else {
        pl = 0.0;
        txl = 0.0;
      }
    }
    if (lane == 31) pr = (valid && c0 + 2 < nx) ? c.pn_at(gi + 2) : 0.0;
    if (valid) {
      const double2 ty = ld2ro(C.Ty + i);
      const double2 ds = ld2ro(c.ds + gi);
      const double2 pc = cur.p;
      double q0 = ds.x * pc.x;
      q0 += tx.x * (pc.x - pc.y);
      q0 += txl * (pc.x - pl);
      q0 += ty.x * (pc.x - nxt.p.x);
      q0 += tym.x * (pc.x - pm.x);
      double q1 = ds.y * pc.y;
      q1 += tx.y * (pc.y - pr);
      q1 += tx.x * (pc.y - pc.x);
      q1 += ty.y * (pc.y - nxt.p.y);
      q1 += tym.y * (pc.y - pm.y);
      if (CPL) {
        q0 += c.couple_q(gi, pc.x);
        q1 += c.couple_q(gi + 1, pc.y);
      }
      st2mut(c.qd + gi, make_double2(q0, q1));
      c.accum(acc, pc.x, cur.r.x, cur.d.x, q0);
      c.accum(acc, pc.y, cur.r.y, cur.d.y, q1);
      tym = ty;
    }
    pm = cur.p;
    cur = nxt;
  }
}

// ---------------------------------------------------------------- cp.async staging
__device__ __forceinline__ void cp16(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// TMA bulk copies (cp.async.bulk, one issuing lane per warp) tracked by an mbarrier per
// staging slot; the parity of every slot's barrier lives in a per-warp word (`ph`).
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  MC_ASSERT((reinterpret_cast<uintptr_t>(src) & 15) == 0 && (smem_u32(dst) & 15) == 0 && (bytes & 15) == 0 && bytes > 0);
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT%=;\n}" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_shared_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

// per-warp staging state: slots of doubles, one mbarrier per slot, slot parities
struct Stage {
  double* wsm;
  uint64_t* bars;
  unsigned* ph;
  // lane 0 of the warp: begin filling slot t with `bytes` of bulk copies
  __device__ __forceinline__ void begin(int t, unsigned bytes) const {
    fence_proxy_async();
    mbar_expect_tx(bars + t, bytes);
  }
  // all lanes: wait until slot t is filled, flip its parity
  __device__ __forceinline__ void wait(int t) const {
    const unsigned par = (*ph >> t) & 1u;
    mbar_wait(bars + t, par);
    __syncwarp();
    if ((threadIdx.x & 31) == 0) *ph ^= (1u << t);
    __syncwarp();
  }
};

// Grid strip, 2 columns per lane, operands of the next row streamed into shared memory
// with cp.async one row ahead, so each warp keeps a row of loads in flight while it
// computes the current one.  Slot k (of 2) holds: r, q, p, D^-1, x of row k+1 (own
// columns), Tx, Ty, shift of row k, and for the strip's edge lanes the neighbouring
// column pair (r, q, p, D^-1 of row k+1; Tx of row k).  Same arithmetic as iter_grid2.
template <bool CPL>
__device__ void iter_grid2s(const Ctx& c, const ContDev& C, int x0, int y0, int y1, const Stage& st,
                            double (&acc)[kNPart]) {
  double* wsm = st.wsm;
  const int lane = threadIdx.x & 31;
  const int nx = C.nx, ny = C.ny;
  const int c0 = x0 + 2 * lane;
  const bool valid = c0 < nx;
  const bool hasL = valid && lane == 0 && c0 > 0;
  const bool hasR = valid && lane == 31 && c0 + 2 < nx;
  const int64_t off = C.off;
#if MC_TMA
  const int vl = (nx - x0) / 2 < 32 ? (nx - x0) / 2 : 32;      // valid lanes of this strip
  const unsigned rowb = 16u * (unsigned)vl;
  const bool sL = x0 > 0, sR = x0 + 64 < nx;                    // strip has left / right neighbours
  auto prefetch = [&](int k) {
    const int t = k % kStages;
    double* sl = wsm + t * kSlotG;
    __syncwarp();
    if (lane == 0) {
      const int64_t ik = (int64_t)k * nx + x0;
      const bool nxt = k + 1 < ny;
      const unsigned bytes = 3u * rowb + (sL ? 16u : 0u) +
                             (nxt ? 5u * rowb + (sL ? 64u : 0u) + (sR ? 64u : 0u) : 0u);
      st.begin(t, bytes);
      uint64_t* bar = st.bars + t;
      bulk_g2s(sl + 5 * 64, C.Tx + ik, rowb, bar);
      bulk_g2s(sl + 6 * 64, C.Ty + ik, rowb, bar);
      bulk_g2s(sl + 7 * 64, c.ds + off + ik, rowb, bar);
      if (sL) bulk_g2s(sl + 512 + 8, C.Tx + ik - 2, 16, bar);
      if (nxt) {
        const int64_t g1 = off + ik + nx;
        bulk_g2s(sl + 0 * 64, c.rs + g1, rowb, bar);
        bulk_g2s(sl + 1 * 64, c.qs + g1, rowb, bar);
        bulk_g2s(sl + 2 * 64, c.ps + g1, rowb, bar);
        bulk_g2s(sl + 3 * 64, c.P->dinv + g1, rowb, bar);
        bulk_g2s(sl + 4 * 64, c.x + g1, rowb, bar);
        if (sL) {
          bulk_g2s(sl + 512 + 0, c.rs + g1 - 2, 16, bar);
          bulk_g2s(sl + 512 + 2, c.qs + g1 - 2, 16, bar);
          bulk_g2s(sl + 512 + 4, c.ps + g1 - 2, 16, bar);
          bulk_g2s(sl + 512 + 6, c.P->dinv + g1 - 2, 16, bar);
        }
        if (sR) {
          bulk_g2s(sl + 512 + 10, c.rs + g1 + 64, 16, bar);
          bulk_g2s(sl + 512 + 12, c.qs + g1 + 64, 16, bar);
          bulk_g2s(sl + 512 + 14, c.ps + g1 + 64, 16, bar);
          bulk_g2s(sl + 512 + 16, c.P->dinv + g1 + 64, 16, bar);
        }
      }
    }
  };
#else
  auto prefetch = [&](int k) {
    double* sl = wsm + (k % kStages) * kSlotG;
    if (valid) {
      const int64_t ik = (int64_t)k * nx + c0;
      cp16(sl + 5 * 64 + 2 * lane, C.Tx + ik);
      cp16(sl + 6 * 64 + 2 * lane, C.Ty + ik);
      cp16(sl + 7 * 64 + 2 * lane, c.ds + off + ik);
      if (hasL) cp16(sl + 512 + 8, C.Tx + ik - 2);
      if (k + 1 < ny) {
        const int64_t g1 = off + ik + nx;
        cp16(sl + 0 * 64 + 2 * lane, c.rs + g1);
        cp16(sl + 1 * 64 + 2 * lane, c.qs + g1);
        cp16(sl + 2 * 64 + 2 * lane, c.ps + g1);
        cp16(sl + 3 * 64 + 2 * lane, c.P->dinv + g1);
        cp16(sl + 4 * 64 + 2 * lane, c.x + g1);
        if (hasL) {
          cp16(sl + 512 + 0, c.rs + g1 - 2);
          cp16(sl + 512 + 2, c.qs + g1 - 2);
          cp16(sl + 512 + 4, c.ps + g1 - 2);
          cp16(sl + 512 + 6, c.P->dinv + g1 - 2);
        }
        if (hasR) {
          cp16(sl + 512 + 10, c.rs + g1 + 2);
          cp16(sl + 512 + 12, c.qs + g1 + 2);
          cp16(sl + 512 + 14, c.ps + g1 + 2);
          cp16(sl + 512 + 16, c.P->dinv + g1 + 2);
        }
      }
    }
    cp_commit();
  };
#endif
  // prologue (synchronous): halo row above, own row y0, its edge neighbours
  double2 pm = make_double2(0.0, 0.0), tym = make_double2(0.0, 0.0);
  if (valid && y0 > 0) {
    const int64_t i = (int64_t)(y0 - 1) * nx + c0;
    pm = pnew2(c, off + i);
    tym = ld2ro(C.Ty + i);
  }
  Row2 cur;
  cur.p = cur.r = cur.d = make_double2(0.0, 0.0);
  double eL = 0.0, eR = 0.0;
  if (valid) {
    const int64_t g0 = off + (int64_t)y0 * nx + c0;
    cur = own2(c, g0);
    if (hasL) eL = c.pn_at(g0 - 1);
    if (hasR) eR = c.pn_at(g0 + 2);
  }
#pragma unroll
  for (int d = 0; d < kStages - 1; ++d) {
    if (y0 + d < y1) prefetch(y0 + d);
#if !MC_TMA
    else cp_commit();
#endif
  }
  for (int y = y0; y < y1; ++y) {
    if (y + kStages - 1 < y1) prefetch(y + kStages - 1);
    int32_t ce0 = 0, ce1 = 0, ce2 = 0;                             // coupled: entry ranges of this lane's two cells
    if (CPL && valid) {
      const int32_t* cp = c.P->cptr + off + (int64_t)y * nx + c0;
      ce0 = ldro(cp);
      ce1 = ldro(cp + 1);
      ce2 = ldro(cp + 2);
    }
#if MC_TMA
    st.wait(y % kStages);
#else
    else cp_commit();
    cp_wait<kStages - 1>();
#endif
    const double* sl = wsm + (y % kStages) * kSlotG;
    const int64_t i = (int64_t)y * nx + c0;
    const int64_t gi = off + i;
    Row2 nxt;
    nxt.p = nxt.r = nxt.d = make_double2(0.0, 0.0);
    double nL = 0.0, nR = 0.0;
    if (valid && y + 1 < ny) {
      const double2 ro = *reinterpret_cast<const double2*>(sl + 0 * 64 + 2 * lane);
      const double2 qo = *reinterpret_cast<const double2*>(sl + 1 * 64 + 2 * lane);
      const double2 po = *reinterpret_cast<const double2*>(sl + 2 * 64 + 2 * lane);
      const double2 di = *reinterpret_cast<const double2*>(sl + 3 * 64 + 2 * lane);
      nxt.d = di;
      nxt.r = make_double2(__fma_rn(-c.a, qo.x, ro.x), __fma_rn(-c.a, qo.y, ro.y));
      nxt.p = make_double2(__fma_rn(di.x, nxt.r.x, __dmul_rn(c.b, po.x)),
                           __fma_rn(di.y, nxt.r.y, __dmul_rn(c.b, po.y)));
      if (y + 1 < y1) {
        const double2 xo = *reinterpret_cast<const double2*>(sl + 4 * 64 + 2 * lane);
        const int64_t g1 = gi + nx;
        *reinterpret_cast<double2*>(c.x + g1) =
            make_double2(__fma_rn(c.a, po.x, xo.x), __fma_rn(c.a, po.y, xo.y));
        st2mut(c.rd + g1, nxt.r);
        st2mut(c.pd + g1, nxt.p);
      }
      if (hasL) nL = pnew(sl[512 + 1], sl[512 + 3], sl[512 + 5], sl[512 + 7], c.a, c.b);
      if (hasR) nR = pnew(sl[512 + 10], sl[512 + 12], sl[512 + 14], sl[512 + 16], c.a, c.b);
    }
    const double2 tx = valid ? *reinterpret_cast<const double2*>(sl + 5 * 64 + 2 * lane) : make_double2(0.0, 0.0);
    double pl = __shfl_up_sync(0xffffffffu, cur.p.y, 1);
    double pr = __shfl_down_sync(0xffffffffu, cur.p.x, 1);
    double txl = __shfl_up_sync(0xffffffffu, tx.y, 1);
    if (lane == 0) {
      pl = hasL ? eL : 0.0;
      txl = hasL ? sl[512 + 9] : 0.0;
    }
    if (lane == 31) pr = hasR ? eR : 0.0;
    if (valid) {
      const double2 ty = *reinterpret_cast<const double2*>(sl + 6 * 64 + 2 * lane);
      const double2 ds = *reinterpret_cast<const double2*>(sl + 7 * 64 + 2 * lane);
      const double2 pc = cur.p;
      double q0 = ds.x * pc.x;
      q0 += tx.x * (pc.x - pc.y);
      q0 += txl * (pc.x - pl);
      q0 += ty.x * (pc.x - nxt.p.x);
      q0 += tym.x * (pc.x - pm.x);
      double q1 = ds.y * pc.y;
      q1 += tx.y * (pc.y - pr);
      q1 += tx.x * (pc.y - pc.x);
      q1 += ty.y * (pc.y - nxt.p.y);
      q1 += tym.y * (pc.y - pm.y);
      if (CPL) {
        q0 += c.couple_q_range(ce0, ce1, pc.x);
        q1 += c.couple_q_range(ce1, ce2, pc.y);
      }
      st2mut(c.qd + gi, make_double2(q0, q1));
      c.accum(acc, pc.x, cur.r.x, cur.d.x, q0);
      c.accum(acc, pc.y, cur.r.y, cur.d.y, q1);
      tym = ty;
    }
    pm = cur.p;
    cur = nxt;
    eL = nL;
    eR = nR;
  }
  cp_wait<0>();
}

// ELL rows in 64-row chunks swept round-robin by the group's warps (lane l owns rows
// 2l, 2l+1 of a chunk).  Per chunk: TMA bulk copies of the NEXT chunk's r, q, p, D^-1
// over the chunk and a 2-row halo on each side (68-row window), x, shift and the 4 ELL
// codes are issued; this chunk's "far" neighbours (code >= 0: neither in the chunk nor
// its halo, at most 2 per lane per batch) are gathered, p_j recomputed from the previous
// iteration's r, q, p; the new p of every window row goes to a per-warp buffer and q is
// formed from it.  (A three-stage load / gather / compute pipeline measured no faster.)
// ELL codes are pre-classified on the host against the static chunk (mc_api.cu).
// Neighbours in another chunk were (or are about to be) streamed by another warp of
// the sweep, so the far gathers hit L2.
struct FarG {
  double w0, w1, w2, w3;   // p_j of the (at most 4) far neighbours of this lane, in (h, k) order
  int s0, s1, s2, s3;      // 4*h + k slot each value belongs to, -1 = none
};

__device__ __forceinline__ void ell_codes(const double* sl, int lane, int32_t (&j)[2][4]) {
  const int32_t* si = reinterpret_cast<const int32_t*>(sl + 400);
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int k = 0; k < 4; ++k) j[h][k] = si[k * 64 + 2 * lane + h];
}

// far neighbours of this lane's two rows: up to 4 gathered in one batch, each load issued
// only by the lanes that have that neighbour (no dummy own-row loads)
__device__ __forceinline__ FarG far_gather(const Ctx& c, const double* sl, int lane) {
  int32_t j[2][4];
  ell_codes(sl, lane, j);
  FarG f;
  f.s0 = f.s1 = f.s2 = f.s3 = -1;
  int32_t i0 = -1, i1 = -1, i2 = -1, i3 = -1;
  int nfar = 0;
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (j[h][k] >= 0) {
        if (nfar == 0) {
          i0 = j[h][k];
          f.s0 = 4 * h + k;
        } else if (nfar == 1) {
          i1 = j[h][k];
          f.s1 = 4 * h + k;
        } else if (nfar == 2) {
          i2 = j[h][k];
          f.s2 = 4 * h + k;
        } else if (nfar == 3) {
          i3 = j[h][k];
          f.s3 = 4 * h + k;
        }
        ++nfar;
      }
  f.w0 = f.w1 = f.w2 = f.w3 = 0.0;
  MC_ASSERT(i0 < c.P->N && i1 < c.P->N && i2 < c.P->N && i3 < c.P->N);
  if (i0 >= 0) f.w0 = c.pn_at(i0);
  if (i1 >= 0) f.w1 = c.pn_at(i1);
  if (i2 >= 0) f.w2 = c.pn_at(i2);
  if (i3 >= 0) f.w3 = c.pn_at(i3);
  return f;
}

template <bool CPL>
__device__ void iter_ells(const Ctx& c, const ContDev& C, int wg, int W, const Stage& st,
                          double (&acc)[kNPart]) {
  double* wsm = st.wsm;
  double* pnb = wsm + kWarpSmem - kPnBuf;                      // new p of the window rows
  const int lane = threadIdx.x & 31;
  const int64_t off = C.off, es = C.estride;
  const int r1 = (int)C.n;
  const int nch = (r1 + 63) / 64;
  auto tix = [&](int m) { return (m / W) % kStagesE; };
  auto slot = [&](int m) { return wsm + tix(m) * kSlotE; };
  auto prefetch = [&](int m) {
    const int t = tix(m);
    double* sl = wsm + t * kSlotE;
    __syncwarp();
    if (lane == 0) {
      const int64_t b = 64 * (int64_t)m;
      const int64_t g = off + b;
      const bool full = g >= 2;                                 // window start in bounds
      const unsigned wb = full ? 544u : 528u;
      st.begin(t, 4u * wb + 2u * 512u + 4u * 256u);
      uint64_t* bar = st.bars + t;
      const int64_t g0 = g - (full ? 2 : 0);
      const int d0 = full ? 0 : 2;
      bulk_g2s(sl + d0, c.rs + g0, wb, bar);
      bulk_g2s(sl + 68 + d0, c.qs + g0, wb, bar);
      bulk_g2s(sl + 136 + d0, c.ps + g0, wb, bar);
      bulk_g2s(sl + 204 + d0, c.P->dinv + g0, wb, bar);
      bulk_g2s(sl + 272, c.x + g, 512, bar);
      bulk_g2s(sl + 336, c.ds + g, 512, bar);
      int32_t* si = reinterpret_cast<int32_t*>(sl + 400);
#pragma unroll
      for (int k = 0; k < 4; ++k) bulk_g2s(si + k * 64, C.ecol + k * es + b, 256, bar);
    }
  };
  if (wg >= nch) return;
  prefetch(wg);
  for (int m = wg; m < nch; m += W) {
    if (m + W < nch) prefetch(m + W);                             // next chunk in flight
    int32_t ce0 = 0, ce1 = 0, ce2 = 0;                             // coupled: transfer entry ranges of this lane's two rows,
    if (CPL) {                                                    // loaded before the wait for the staged chunk
      const int64_t gr = off + 64 * (int64_t)m + 2 * lane;
      if (64 * m + 2 * lane < r1) {
        ce0 = ldro(c.P->cptr + gr);
        ce1 = ldro(c.P->cptr + gr + 1);
      }
      ce2 = ce1;
      if (64 * m + 2 * lane + 1 < r1) ce2 = ldro(c.P->cptr + gr + 2);
    }
    st.wait(tix(m));
    const FarG fcur = far_gather(c, slot(m), lane);
    // stage C: chunk m
    const double* sl = slot(m);
    const int base = 64 * m + 2 * lane;
    const int64_t g = off + base;
    const bool ok0 = base < r1, ok1 = base + 1 < r1;
    double pc[2], rc[2], dc[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int w = 2 + 2 * lane + h;
      rc[h] = __fma_rn(-c.a, sl[68 + w], sl[w]);
      dc[h] = sl[204 + w];
      pc[h] = __fma_rn(dc[h], rc[h], __dmul_rn(c.b, sl[136 + w]));
    }
    __syncwarp();                                                 // previous chunk's pnb reads done
    pnb[2 + 2 * lane] = pc[0];
    pnb[3 + 2 * lane] = pc[1];
    if (lane < 4) {                                               // halo rows 0, 1, 66, 67
      const int w = lane < 2 ? lane : 64 + lane;
      pnb[w] = pnew(sl[w], sl[68 + w], sl[136 + w], sl[204 + w], c.a, c.b);
    }
    {
      const double2 xo = *reinterpret_cast<const double2*>(sl + 272 + 2 * lane);
      const double po0 = sl[136 + 2 + 2 * lane], po1 = sl[136 + 3 + 2 * lane];
      const double2 xn = make_double2(__fma_rn(c.a, po0, xo.x), __fma_rn(c.a, po1, xo.y));
      if (ok1) {
        *reinterpret_cast<double2*>(c.x + g) = xn;
        st2mut(c.rd + g, make_double2(rc[0], rc[1]));
        st2mut(c.pd + g, make_double2(pc[0], pc[1]));
      } else if (ok0) {
        c.x[g] = xn.x;
        stmut(c.rd + g, rc[0]);
        stmut(c.pd + g, pc[0]);
      }
    }
    int32_t j[2][4];
    ell_codes(sl, lane, j);
    __syncwarp();
    double qv[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int32_t cd = j[h][k];
        double v = pc[h];                                          // -1: no neighbour
        MC_ASSERT(cd >= -2 - 67);
        if (cd <= -2) v = pnb[-2 - cd];
        else if (cd >= 0) {
          if (fcur.s0 == 4 * h + k) v = fcur.w0;
          else if (fcur.s1 == 4 * h + k) v = fcur.w1;
          else if (fcur.s2 == 4 * h + k) v = fcur.w2;
          else if (fcur.s3 == 4 * h + k) v = fcur.w3;
          else v = c.pn_at(cd);                                    // rare: > 4 far in this lane
        }
        s += pc[h] - v;
      }
      qv[h] = sl[336 + 2 * lane + h] * pc[h] + C.Tconst * s;
      if (CPL && base + h < r1) qv[h] += c.couple_q_range(h == 0 ? ce0 : ce1, h == 0 ? ce1 : ce2, pc[h]);
    }
    if (ok1) st2mut(c.qd + g, make_double2(qv[0], qv[1]));
    else if (ok0) stmut(c.qd + g, qv[0]);
    if (ok0) c.accum(acc, pc[0], rc[0], dc[0], qv[0]);
    if (ok1) c.accum(acc, pc[1], rc[1], dc[1], qv[1]);
  }
}

// Chunk-blocked streaming ELL pass (decoupled Jacobi solve of a network too large to stay
// resident: configs 2 and 4).  Same sweep and arithmetic as iter_ells, on a
// private layout in which everything a 64-row chunk needs is contiguous:
//   bstat[m]   256 doubles  D^-1 (64) | shift (64) | int32 codes [64 rows][4]
//   bdyn[s][m] 192 doubles  r (64) | q (64) | p (64)          (s = iteration parity)
//   x          the state vector itself (64 doubles at the chunk's rows)
// so a chunk arrives with THREE bulk copies (2048 + 1536 + 512 B) instead of ten, and the
// pass issues ~3x fewer instructions per chunk than iter_ells (whose 715 instructions per
// chunk made it co-limited by instruction issue: profiles/r02_fracture_only_soa.txt).
// Codes (host, finalize): -1 none, -2 - w: row w of this chunk, >= 0: continuum-local row
// of a neighbour in another chunk ("far": gathered from the previous iteration's r, q, p).
// Far neighbours come first in a row's four slots, so only slots 0 and 1 are gathered in
// the common batch; rows with three or four far neighbours take a warp-uniform extra step.
__device__ __forceinline__ double pn_blk(const double* dyn, const double* stat, int32_t j, double a, double b) {
  const int64_t blk = j >> 6;
  const int w = j & 63;
  const double* d = dyn + blk * kBDyn + w;
  return pnew(ldnb(d), ldnb(d + 64), ldnb(d + 128), ldro(stat + blk * kBStat + w), a, b);
}

__device__ void iter_ellb(const Ctx& c, const ContDev& C, int wg, int W, const Stage& st, int s,
                          double (&acc)[kNPart]) {
  double* wsm = st.wsm;
  double* pnb = wsm + kWarpSmem - kPnBuf;                      // new p of the chunk's rows
  const int lane = threadIdx.x & 31;
  const int r1 = (int)C.n;
  const int nch = (r1 + 63) / 64;
  const double* stat = C.bstat;
  const double* dyns = C.bdyn[s];
  double* dynd = C.bdyn[s ^ 1];
  double* xg = c.x + C.off;
  auto prefetch = [&](int m, int t) {
    double* sl = wsm + t * kSlotE;
    __syncwarp();
    if (lane == 0) {
      st.begin(t, 8u * (kBStat + kBDyn + 64));
      uint64_t* bar = st.bars + t;
      bulk_g2s(sl, stat + (int64_t)m * kBStat, 8u * kBStat, bar);
      bulk_g2s(sl + kBStat, dyns + (int64_t)m * kBDyn, 8u * kBDyn, bar);
      bulk_g2s(sl + kBStat + kBDyn, xg + 64 * (int64_t)m, 512, bar);
    }
  };
  if (wg >= nch) return;
  prefetch(wg, 0);
  int t = 0;
  for (int m = wg; m < nch; m += W, t ^= 1) {
    if (m + W < nch) prefetch(m + W, t ^ 1);                      // next chunk in flight
    st.wait(t);
    const double* sl = wsm + t * kSlotE;
    // codes of rows 2 lane, 2 lane + 1: 8 consecutive int32
    const int4 c0 = *reinterpret_cast<const int4*>(sl + 128 + 4 * lane);
    const int4 c1 = *reinterpret_cast<const int4*>(sl + 128 + 4 * lane + 2);
    // far neighbours (slots 0, 1 of each row): gathered in one batch, loads predicated per lane
    double f00 = 0.0, f01 = 0.0, f10 = 0.0, f11 = 0.0;
    if (c0.x >= 0) f00 = pn_blk(dyns, stat, c0.x, c.a, c.b);
    if (c0.y >= 0) f01 = pn_blk(dyns, stat, c0.y, c.a, c.b);
    if (c1.x >= 0) f10 = pn_blk(dyns, stat, c1.x, c.a, c.b);
    if (c1.y >= 0) f11 = pn_blk(dyns, stat, c1.y, c.a, c.b);
    const double2 di = *reinterpret_cast<const double2*>(sl + 2 * lane);
    const double2 ds = *reinterpret_cast<const double2*>(sl + 64 + 2 * lane);
    const double2 ro = *reinterpret_cast<const double2*>(sl + kBStat + 2 * lane);
    const double2 qo = *reinterpret_cast<const double2*>(sl + kBStat + 64 + 2 * lane);
    const double2 po = *reinterpret_cast<const double2*>(sl + kBStat + 128 + 2 * lane);
    const double2 xo = *reinterpret_cast<const double2*>(sl + kBStat + kBDyn + 2 * lane);
    const double r0 = __fma_rn(-c.a, qo.x, ro.x), r1n = __fma_rn(-c.a, qo.y, ro.y);
    const double p0 = __fma_rn(di.x, r0, __dmul_rn(c.b, po.x)), p1 = __fma_rn(di.y, r1n, __dmul_rn(c.b, po.y));
    __syncwarp();                                                 // previous chunk's pnb reads done
    *reinterpret_cast<double2*>(pnb + 2 * lane) = make_double2(p0, p1);
    __syncwarp();
    // v(code, far value, own p): the neighbour's new p
    auto nbv = [&](int32_t cd, double far, double own) { return cd >= 0 ? far : (cd <= -2 ? pnb[-2 - cd] : own); };
    double f02 = 0.0, f03 = 0.0, f12 = 0.0, f13 = 0.0;
    if (__any_sync(0xffffffffu, (c0.z >= 0) | (c0.w >= 0) | (c1.z >= 0) | (c1.w >= 0))) {   // rare: > 2 far in a row
      if (c0.z >= 0) f02 = pn_blk(dyns, stat, c0.z, c.a, c.b);
      if (c0.w >= 0) f03 = pn_blk(dyns, stat, c0.w, c.a, c.b);
      if (c1.z >= 0) f12 = pn_blk(dyns, stat, c1.z, c.a, c.b);
      if (c1.w >= 0) f13 = pn_blk(dyns, stat, c1.w, c.a, c.b);
    }
    double s0 = p0 - nbv(c0.x, f00, p0);
    s0 += p0 - nbv(c0.y, f01, p0);
    s0 += p0 - nbv(c0.z, f02, p0);
    s0 += p0 - nbv(c0.w, f03, p0);
    double s1 = p1 - nbv(c1.x, f10, p1);
    s1 += p1 - nbv(c1.y, f11, p1);
    s1 += p1 - nbv(c1.z, f12, p1);
    s1 += p1 - nbv(c1.w, f13, p1);
    const double q0 = __fma_rn(C.Tconst, s0, __dmul_rn(ds.x, p0));
    const double q1 = __fma_rn(C.Tconst, s1, __dmul_rn(ds.y, p1));
    const int base = 64 * m + 2 * lane;
    double* dd = dynd + (int64_t)m * kBDyn + 2 * lane;
    // rows past n in the last chunk: their block slots exist (padded), the state vector's do not
    st2mut(dd, make_double2(r0, r1n));
    st2mut(dd + 64, make_double2(q0, q1));
    st2mut(dd + 128, make_double2(p0, p1));
    const double2 xn = make_double2(__fma_rn(c.a, po.x, xo.x), __fma_rn(c.a, po.y, xo.y));
    if (base + 1 < r1) {
      *reinterpret_cast<double2*>(xg + base) = xn;
      c.accum(acc, p0, r0, di.x, q0);
      c.accum(acc, p1, r1n, di.y, q1);
    } else if (base < r1) {
      xg[base] = xn.x;
      c.accum(acc, p0, r0, di.x, q0);
    }
  }
}

// Resident variant for latency-bound graphs (every warp owns <= kStages chunks,
// DESIGN.md §5.3): the chunks' r, q, p, x, D^-1, shift and codes stay in this warp's
// slots for the whole solve, so an iteration streams nothing; in-chunk neighbours read
// the new p straight from the slot; halo and far neighbours (owned by other warps) are
// gathered from the previous iteration's r, q, p in global memory.  r, p, q are stored
// to global every iteration for those gathers; x is flushed at the end of the solve.
template <bool CPL>
__device__ void iter_ells_res(const Ctx& c, const ContDev& C, int wg, int W, const Stage& st, bool first,
                              double (&acc)[kNPart]) {
  double* wsm = st.wsm;
  const int lane = threadIdx.x & 31;
  const int64_t off = C.off, es = C.estride;
  const int r1 = (int)C.n;
  const int nch = (r1 + 63) / 64;
  if (first) {
    for (int m = wg, t = 0; m < nch; m += W, ++t) {
      double* sl = wsm + t * kSlotE;
      __syncwarp();
      if (lane == 0) {
        const int64_t b = 64 * (int64_t)m, g = off + b;
        st.begin(t, 6u * 512u + 4u * 256u);
        uint64_t* bar = st.bars + t;
        bulk_g2s(sl + 2, c.rs + g, 512, bar);
        bulk_g2s(sl + 68 + 2, c.qs + g, 512, bar);
        bulk_g2s(sl + 136 + 2, c.ps + g, 512, bar);
        bulk_g2s(sl + 204 + 2, c.P->dinv + g, 512, bar);
        bulk_g2s(sl + 272, c.x + g, 512, bar);
        bulk_g2s(sl + 336, c.ds + g, 512, bar);
        int32_t* si = reinterpret_cast<int32_t*>(sl + 400);
  #pragma unroll
      for (int k = 0; k < 4; ++k) bulk_g2s(si + k * 64, C.ecol + k * es + b, 256, bar);
      }
    }
    for (int m = wg, t = 0; m < nch; m += W, ++t) st.wait(t);
    // the slot is this warp's own copy: decode the ELL codes into global column
    // indices once (-1 = none), so the loop below needs one compare per neighbour
    for (int m = wg, t = 0; m < nch; m += W, ++t) {
      int32_t* si = reinterpret_cast<int32_t*>(wsm + t * kSlotE + 400);
      const int64_t cb = off + 64 * (int64_t)m;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = lane + 32 * u, cd = si[e];
        si[e] = cd <= -2 ? (int32_t)(cb + (-2 - cd) - 2) : cd;
      }
    }
    __syncwarp();
  }
  for (int m = wg, t = 0; m < nch; m += W, ++t) {
    double* sl = wsm + t * kSlotE;
    const int32_t* si = reinterpret_cast<const int32_t*>(sl + 400);
    const int base = 64 * m + 2 * lane;
    const int64_t g = off + base;
    const int64_t cb = off + 64 * (int64_t)m;
    const bool ok0 = base < r1, ok1 = base + 1 < r1;
    double pc[2], rc[2], dc[2], dsv[2];
    int32_t j[2][4];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int l2 = 2 * lane + h;
      const double ro = sl[2 + l2], qo = sl[70 + l2], po = sl[138 + l2];
      dc[h] = sl[206 + l2];
      rc[h] = __fma_rn(-c.a, qo, ro);
      pc[h] = __fma_rn(dc[h], rc[h], __dmul_rn(c.b, po));
      dsv[h] = sl[336 + l2];
      sl[272 + l2] = __fma_rn(c.a, po, sl[272 + l2]);           // x (flushed at the end)
#pragma unroll
      for (int k = 0; k < 4; ++k) j[h][k] = si[k * 64 + l2];
    }
    // neighbours outside the chunk: previous iteration's r, q, p from global memory
    // (scalars, not arrays indexed by a runtime count: those would live in local memory)
    int64_t fi0 = g, fi1 = g;
    int fs0 = -1, fs1 = -1;
    int nfar = 0;
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int64_t jj = j[h][k];
        const int64_t li = jj - cb;
        if (jj >= 0 && !(li >= 0 && li < 64)) {
          if (nfar == 0) {
            fi0 = jj;
            fs0 = 4 * h + k;
          } else if (nfar == 1) {
            fi1 = jj;
            fs1 = 4 * h + k;
          }
          ++nfar;
        }
      }
    const int wfar = __reduce_max_sync(0xffffffffu, (unsigned)nfar);
    double v0 = 0.0, v1 = 0.0;
    if (wfar > 0) {
      v0 = c.pn_at(fi0);
      v1 = c.pn_at(fi1);
    }
    // publish: own r_j, p_j into the slot (p_j is what in-chunk neighbours need)
    __syncwarp();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      sl[2 + 2 * lane + h] = rc[h];
      sl[138 + 2 * lane + h] = pc[h];
    }
    if (ok1) {
      st2mut(c.rd + g, make_double2(rc[0], rc[1]));
      st2mut(c.pd + g, make_double2(pc[0], pc[1]));
    } else if (ok0) {
      stmut(c.rd + g, rc[0]);
      stmut(c.pd + g, pc[0]);
    }
    __syncwarp();
    double pj[2][4];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int64_t jj = j[h][k];
        const int64_t li = jj - cb;
        const bool in = jj >= 0 && li >= 0 && li < 64;
        double v = in ? sl[138 + (int)li] : pc[h];
        if (fs0 == 4 * h + k) v = v0;
        else if (fs1 == 4 * h + k) v = v1;
        pj[h][k] = v;
      }
    if (wfar > 2) {
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int64_t jj = j[h][k];
          const int64_t li = jj - cb;
          if (jj >= 0 && !(li >= 0 && li < 64) && fs0 != 4 * h + k && fs1 != 4 * h + k)
            pj[h][k] = c.pn_at(jj);
        }
    }
    double qv[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < 4; ++k) s += pc[h] - pj[h][k];
      qv[h] = dsv[h] * pc[h] + C.Tconst * s;
    }
    sl[70 + 2 * lane] = qv[0];
    sl[70 + 2 * lane + 1] = qv[1];
    if (ok1) st2mut(c.qd + g, make_double2(qv[0], qv[1]));
    else if (ok0) stmut(c.qd + g, qv[0]);
    if (ok0) c.accum(acc, pc[0], rc[0], dc[0], qv[0]);
    if (ok1) c.accum(acc, pc[1], rc[1], dc[1], qv[1]);
  }
}

// Resident pass on the chunk-blocked static data (decoupled solves; same arithmetic as
// iter_ells_res with a third of its instructions): the slot holds the chunk's bstat block
// (D^-1, shift, far-first int32 codes [64][4]) and r, q, p, x (64 doubles each) for the
// whole solve; far neighbours (slots 0 and 1 of a row; rarely 2 and 3) are gathered from
// the previous iteration's r, q, p in global memory, in-chunk neighbours read the new p
// from the slot.  r, p, q are published to global every iteration; x at the end.
__device__ void iter_ells_res2(const Ctx& c, const ContDev& C, int wg, int W, const Stage& st, bool first, int s,
                               double (&acc)[kNPart]) {
  double* wsm = st.wsm;
  const int lane = threadIdx.x & 31;
  const int64_t off = C.off;
  const int r1 = (int)C.n;
  const int nch = (r1 + 63) / 64;
  const double* recs = C.rrec[s];
  double* recd = C.rrec[s ^ 1];
  if (first) {
    for (int m = wg, t = 0; m < nch; m += W, ++t) {
      double* sl = wsm + t * kSlotE;
      __syncwarp();
      if (lane == 0) {
        const int64_t g = off + 64 * (int64_t)m;
        st.begin(t, 8u * kBStat + 4u * 512u);
        uint64_t* bar = st.bars + t;
        bulk_g2s(sl, C.bstat + (int64_t)m * kBStat, 8u * kBStat, bar);
        bulk_g2s(sl + 256, c.rs + g, 512, bar);
        bulk_g2s(sl + 320, c.qs + g, 512, bar);
        bulk_g2s(sl + 384, c.ps + g, 512, bar);
        bulk_g2s(sl + 448, c.x + g, 512, bar);
      }
    }
    for (int m = wg, t = 0; m < nch; m += W, ++t) st.wait(t);
  }
  for (int m = wg, t = 0; m < nch; m += W, ++t) {
    double* sl = wsm + t * kSlotE;
    const int base = 64 * m + 2 * lane;
    const int4 c0 = *reinterpret_cast<const int4*>(sl + 128 + 4 * lane);
    const int4 c1 = *reinterpret_cast<const int4*>(sl + 128 + 4 * lane + 2);
    double f00 = 0.0, f01 = 0.0, f10 = 0.0, f11 = 0.0;
    if (c0.x >= 0) f00 = pn_rec(recs + 4 * (int64_t)c0.x, c.a, c.b);
    if (c0.y >= 0) f01 = pn_rec(recs + 4 * (int64_t)c0.y, c.a, c.b);
    if (c1.x >= 0) f10 = pn_rec(recs + 4 * (int64_t)c1.x, c.a, c.b);
    if (c1.y >= 0) f11 = pn_rec(recs + 4 * (int64_t)c1.y, c.a, c.b);
    const double2 di = *reinterpret_cast<const double2*>(sl + 2 * lane);
    const double2 ds = *reinterpret_cast<const double2*>(sl + 64 + 2 * lane);
    const double2 ro = *reinterpret_cast<const double2*>(sl + 256 + 2 * lane);
    const double2 qo = *reinterpret_cast<const double2*>(sl + 320 + 2 * lane);
    const double2 po = *reinterpret_cast<const double2*>(sl + 384 + 2 * lane);
    const double2 xo = *reinterpret_cast<const double2*>(sl + 448 + 2 * lane);
    const double r0 = __fma_rn(-c.a, qo.x, ro.x), r1n = __fma_rn(-c.a, qo.y, ro.y);
    const double p0 = __fma_rn(di.x, r0, __dmul_rn(c.b, po.x)), p1 = __fma_rn(di.y, r1n, __dmul_rn(c.b, po.y));
    *reinterpret_cast<double2*>(sl + 448 + 2 * lane) = make_double2(__fma_rn(c.a, po.x, xo.x), __fma_rn(c.a, po.y, xo.y));
    *reinterpret_cast<double2*>(sl + 256 + 2 * lane) = make_double2(r0, r1n);
    __syncwarp();                                                 // every lane has read the old p
    *reinterpret_cast<double2*>(sl + 384 + 2 * lane) = make_double2(p0, p1);
    const bool ok0 = base < r1, ok1 = base + 1 < r1;
    __syncwarp();
    const double* pn = sl + 384;
    auto nbv = [&](int32_t cd, double far, double own) { return cd >= 0 ? far : (cd <= -2 ? pn[-2 - cd] : own); };
    double f02 = 0.0, f03 = 0.0, f12 = 0.0, f13 = 0.0;
    if (__any_sync(0xffffffffu, (c0.z >= 0) | (c0.w >= 0) | (c1.z >= 0) | (c1.w >= 0))) {   // rare: > 2 far in a row
      if (c0.z >= 0) f02 = pn_rec(recs + 4 * (int64_t)c0.z, c.a, c.b);
      if (c0.w >= 0) f03 = pn_rec(recs + 4 * (int64_t)c0.w, c.a, c.b);
      if (c1.z >= 0) f12 = pn_rec(recs + 4 * (int64_t)c1.z, c.a, c.b);
      if (c1.w >= 0) f13 = pn_rec(recs + 4 * (int64_t)c1.w, c.a, c.b);
    }
    double s0 = p0 - nbv(c0.x, f00, p0);
    s0 += p0 - nbv(c0.y, f01, p0);
    s0 += p0 - nbv(c0.z, f02, p0);
    s0 += p0 - nbv(c0.w, f03, p0);
    double s1 = p1 - nbv(c1.x, f10, p1);
    s1 += p1 - nbv(c1.y, f11, p1);
    s1 += p1 - nbv(c1.z, f12, p1);
    s1 += p1 - nbv(c1.w, f13, p1);
    const double q0 = __fma_rn(C.Tconst, s0, __dmul_rn(ds.x, p0));
    const double q1 = __fma_rn(C.Tconst, s1, __dmul_rn(ds.y, p1));
    *reinterpret_cast<double2*>(sl + 320 + 2 * lane) = make_double2(q0, q1);
    // publish this iteration's records for the other warps' far gathers
    if (ok0) st_rec(recd + 4 * (int64_t)base, r0, q0, p0, di.x);
    if (ok1) st_rec(recd + 4 * (int64_t)(base + 1), r1n, q1, p1, di.y);
    if (ok0) c.accum(acc, p0, r0, di.x, q0);
    if (ok1) c.accum(acc, p1, r1n, di.y, q1);
  }
}

__device__ void flush_ells_res2(const ContDev& C, int wg, int W, const double* wsm, double* x) {
  const int lane = threadIdx.x & 31;
  const int nch = (int)((C.n + 63) / 64);
  for (int m = wg, t = 0; m < nch; m += W, ++t) {
    const double* sl = wsm + t * kSlotE;
    for (int h = 0; h < 2; ++h) {
      const int64_t i = 64 * (int64_t)m + 2 * lane + h;
      if (i < C.n) x[C.off + i] = sl[448 + 2 * lane + h];
    }
  }
}

__device__ void flush_ells_res(const ContDev& C, int wg, int W, const double* wsm, double* x) {
  const int lane = threadIdx.x & 31;
  const int nch = (int)((C.n + 63) / 64);
  for (int m = wg, t = 0; m < nch; m += W, ++t) {
    const double* sl = wsm + t * kSlotE;
    for (int h = 0; h < 2; ++h) {
      const int64_t i = 64 * (int64_t)m + 2 * lane + h;
      if (i < C.n) x[C.off + i] = sl[272 + 2 * lane + h];
    }
  }
}

// ---------------------------------------------------------------- CG pass, graph rows
// lane-per-row; the edge loop gathers 4 neighbours at a time (fixed summation order)
template <bool CPL>
__device__ void iter_graph(const Ctx& c, const ContDev& C, int r0, int r1,
                           double (&acc)[kNPart]) {
  const int lane = threadIdx.x & 31;
  for (int i = r0 + lane; i < r1; i += 32) {
    const int64_t gi = C.off + i;
    double pc, rc, dc;
    c.own(gi, pc, rc, dc);
    const int32_t e0 = ldro(C.rowptr + i), e1 = ldro(C.rowptr + i + 1);
    double s = 0.0;
    int32_t e = e0;
    if (C.val) {
      for (; e + 4 <= e1; e += 4) {
        const int32_t j0 = ldro(C.col + e), j1 = ldro(C.col + e + 1), j2 = ldro(C.col + e + 2),
                      j3 = ldro(C.col + e + 3);
        const double v0 = ldro(C.val + e), v1 = ldro(C.val + e + 1), v2 = ldro(C.val + e + 2),
                     v3 = ldro(C.val + e + 3);
        const double q0 = c.pn_at(j0), q1 = c.pn_at(j1), q2 = c.pn_at(j2), q3 = c.pn_at(j3);
        s += v0 * (pc - q0);
        s += v1 * (pc - q1);
        s += v2 * (pc - q2);
        s += v3 * (pc - q3);
      }
      for (; e < e1; ++e) s += ldro(C.val + e) * (pc - c.pn_at(ldro(C.col + e)));
    } else {
      for (; e + 4 <= e1; e += 4) {
        const int32_t j0 = ldro(C.col + e), j1 = ldro(C.col + e + 1), j2 = ldro(C.col + e + 2),
                      j3 = ldro(C.col + e + 3);
        const double q0 = c.pn_at(j0), q1 = c.pn_at(j1), q2 = c.pn_at(j2), q3 = c.pn_at(j3);
        s += pc - q0;
        s += pc - q1;
        s += pc - q2;
        s += pc - q3;
      }
      for (; e < e1; ++e) s += pc - c.pn_at(ldro(C.col + e));
      s *= C.Tconst;
    }
    double qv = ldro(c.ds + gi) * pc + s;
    if (CPL) qv += c.couple_q(gi, pc);
    stmut(c.qd + gi, qv);
    c.accum(acc, pc, rc, dc, qv);
  }
}

// 8 lanes per row (wide rows, e.g. the NLMC operator's ~24 neighbours): each lane sums
// every 8th edge, then a fixed xor tree combines the 8 partial sums.
template <bool CPL>
__device__ void iter_graph8(const Ctx& c, const ContDev& C, int r0, int r1,
                            double (&acc)[kNPart]) {
  // lane `sub` of a row's 8 lanes takes edges (and, coupled, transfer entries) sub,
  // sub+8, sub+16, sub+24: all their column / value loads issue together, then all
  // neighbour gathers, so a row costs ~3 memory trips however long it is (<= 32 entries
  // per list in one batch; longer lists loop)
  const int lane = threadIdx.x & 31, sub = lane & 7, grp = lane >> 3;
  // the row pointers of a batch are loaded one batch ahead, so a batch costs two memory
  // trips (entries, then neighbour gathers) instead of three
  int32_t e0 = 0, e1 = 0, f0 = 0, f1 = 0;
  if (r0 + grp < r1) {
    e0 = ldro(C.rowptr + r0 + grp);
    e1 = ldro(C.rowptr + r0 + grp + 1);
    if (CPL) {
      f0 = ldro(c.P->cptr + C.off + r0 + grp);
      f1 = ldro(c.P->cptr + C.off + r0 + grp + 1);
    }
  }
  for (int base = r0; base < r1; base += 4) {
    const int i = base + grp;
    const bool ok = i < r1;
    const int64_t gi = C.off + (ok ? i : r0);
    int32_t e0n = 0, e1n = 0, f0n = 0, f1n = 0;
    if (i + 4 < r1) {
      e0n = ldro(C.rowptr + i + 4);
      e1n = ldro(C.rowptr + i + 5);
      if (CPL) {
        f0n = ldro(c.P->cptr + gi + 4);
        f1n = ldro(c.P->cptr + gi + 5);
      }
    }
    double pc = 0.0, rc = 0.0, dc = 0.0;
    if (ok && sub == 0) c.own(gi, pc, rc, dc);
    // first batch (<= 32 entries per list): every load issues before pc is needed
    double pj[4], tj[4], pf[4], tf[4];
    // unconditional loads (an unused slot reads entry 0 / this row and is discarded):
    // no branch separates the loads, so they all issue in one batch
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int32_t e = e0 + sub + 8 * k;
      const bool use = e < e1;
      const int32_t ee = use ? e : 0;
      const int32_t jr = ldro(C.col + ee);
      const double tv = C.val ? ldro(C.val + ee) : C.Tconst;
      tj[k] = use ? tv : 0.0;
      pj[k] = c.pn_at(use ? (int64_t)jr : gi);
      if (CPL) {
        const int32_t f = f0 + sub + 8 * k;
        const bool usef = f < f1;
        const int32_t ff = usef ? f : 0;
        const int32_t jf = ldro(c.P->cidx + ff);
        const double tv2 = ldro(c.P->cval + ff);
        tf[k] = usef ? tv2 : 0.0;
        pf[k] = c.pn_at(usef ? (int64_t)jf : gi);
      }
    }
    pc = __shfl_sync(0xffffffffu, pc, lane & ~7);                 // all lanes, uniform
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 4; ++k) s += tj[k] * (pc - pj[k]);
    if (CPL) {
#pragma unroll
      for (int k = 0; k < 4; ++k) s += tf[k] * (pc - pf[k]);
    }
    // rare: longer lists
    for (int32_t e = e0 + 32 + sub; e < e1; e += 8)
      s += (C.val ? ldro(C.val + e) : C.Tconst) * (pc - c.pn_at(ldro(C.col + e)));
    if (CPL)
      for (int32_t f = f0 + 32 + sub; f < f1; f += 8) s += ldro(c.P->cval + f) * (pc - c.pn_at(ldro(c.P->cidx + f)));
    s += __shfl_xor_sync(0xffffffffu, s, 4);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    if (ok && sub == 0) {
      const double qv = ldro(c.ds + gi) * pc + s;
      stmut(c.qd + gi, qv);
      c.accum(acc, pc, rc, dc, qv);
    }
    e0 = e0n;
    e1 = e1n;
    f0 = f0n;
    f1 = f1n;
  }
}

// ---------------------------------------------------------------- init pass
// b = (m/tau) u + F + [D: sum sigma u_other];  r0 = b - K u;  x = u;  p0 = q0 = 0
// bw: nullptr, or this row's r slot in the chunk-blocked workspace (q, p follow 64 and 128 doubles on)
template <bool CPL>
__device__ __forceinline__ void init_row(const StepParams& P, int64_t gi, double Ku_nb,
                                         const double* uo, double* x, int myphase, double (&acc)[3],
                                         double* bw = nullptr, double* rw = nullptr) {
  const double u = uo[gi];
  double b = ldro(P.mtau + gi) * u + ldro(P.F + gi);
  double Ku = ldro((CPL ? P.dsC : P.dsD) + gi) * u + Ku_nb;
  const int32_t e0 = ldro(P.cptr + gi), e1 = ldro(P.cptr + gi + 1);
  for (int32_t e = e0; e < e1; ++e) {
    const int32_t j = ldro(P.cidx + e);
    MC_ASSERT(j >= 0 && j < P.N);
    const double s = ldro(P.cval + e);
    if (CPL) {
      Ku += s * (u - uo[j]);
    } else {
      // D-scheme: Q_ab u_b^{n-1}.  L/U schemes: continua solved
      // earlier in this step contribute their layer-n value.
      const double* src = uo;
      if (P.gs) {
        int bc = 0;
        while (bc + 1 < P.L && j >= P.cont[bc + 1].off) ++bc;
        if (P.grp[bc].phase < myphase) src = x;
      }
      b += s * src[j];
    }
  }
  const double r = b - Ku;
  const double di = ldro(P.dinv + gi);
  x[gi] = u;
  if (rw) st_rec(rw, r, 0.0, 0.0, di);       // resident pass: record for the first iteration's far gathers
  if (bw) {
    stmut(bw, r);
    stmut(bw + 64, 0.0);
    stmut(bw + 128, 0.0);
  } else {
    stmut(P.r[0] + gi, r);
    stmut(P.p[0] + gi, 0.0);
    stmut(P.q[0] + gi, 0.0);
  }
  acc[0] += b * b;
  acc[1] += r * r;
  acc[2] += di * r * r;
}

template <bool CPL>
__device__ void init_item(const StepParams& P, const Item& it, const double* uo, double* x, int myphase,
                          double (&acc)[3]) {
  MC_ASSERT(it.cont >= 0 && it.cont < P.L);
  const ContDev& C = P.cont[it.cont];
  MC_ASSERT(it.kind == ITEM_GRID ? (it.a >= 0 && it.b >= 0 && it.c <= C.ny && it.b <= it.c) : (it.a >= 0 && it.b <= C.n));
  const int lane = threadIdx.x & 31;
  if (it.kind == ITEM_GRID) {
    const int nx = C.nx, ny = C.ny;
    for (int col = it.a + lane; col < it.a + it.w && col < nx; col += 32)
    for (int y = it.b; y < it.c; ++y) {
      const int64_t i = (int64_t)y * nx + col, gi = C.off + i;
      const double u = uo[gi];
      double s = 0.0;
      if (col > 0) s += ldro(C.Tx + i - 1) * (u - uo[gi - 1]);
      if (col + 1 < nx) s += ldro(C.Tx + i) * (u - uo[gi + 1]);
      if (y > 0) s += ldro(C.Ty + i - nx) * (u - uo[gi - nx]);
      if (y + 1 < ny) s += ldro(C.Ty + i) * (u - uo[gi + nx]);
      init_row<CPL>(P, gi, s, uo, x, myphase, acc);
    }
  } else {
    for (int i = it.a + lane; i < it.b; i += 32) {
      const int64_t gi = C.off + i;
      const double u = uo[gi];
      const int32_t e0 = ldro(C.rowptr + i), e1 = ldro(C.rowptr + i + 1);
      double s = 0.0;
      for (int32_t e = e0; e < e1; ++e) {
        const double t = C.val ? ldro(C.val + e) : C.Tconst;
        s += t * (u - uo[ldro(C.col + e)]);
      }
      init_row<CPL>(P, gi, s, uo, x, myphase, acc, (!CPL && C.bdyn[0]) ? C.bdyn[0] + (int64_t)(i >> 6) * kBDyn + (i & 63) : nullptr,
               (!CPL && C.rrec[0]) ? C.rrec[0] + 4 * (int64_t)i : nullptr);
    }
  }
}

__device__ void zero_item(const StepParams& P, const Item& it, double* x) {
  const ContDev& C = P.cont[it.cont];
  const int lane = threadIdx.x & 31;
  if (it.kind == ITEM_GRID) {
    for (int col = it.a + lane; col < it.a + it.w && col < C.nx; col += 32)
      for (int y = it.b; y < it.c; ++y) x[C.off + (int64_t)y * C.nx + col] = 0.0;
  } else {
    for (int i = it.a + lane; i < it.b; i += 32) x[C.off + i] = 0.0;
  }
}

// ---------------------------------------------------------------- group all-reduce + barrier
// Deterministic: CTA partial = fixed-order warp/CTA tree; group total = fixed-order sum
// over the group's CTAs, computed redundantly (identically) by every CTA of the group.
template <int NP>
__device__ __forceinline__ void group_allreduce(const StepParams& P, int g, int cl,
                                                unsigned long long& epoch, const double (&v)[NP],
                                                double (&out)[NP]) {
  __shared__ double sh[2][kWarps][kNPart];
  __shared__ double tot[kNPart];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int G = P.grp[g].cta_count, base = P.grp[g].cta_begin;
  MC_ASSERT(cl >= 0 && cl < G && base + G <= P.total_ctas);
  const int eb = (int)(epoch & 1ull);
#pragma unroll
  for (int k = 0; k < NP; ++k) {
    double s = v[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) sh[eb][w][k] = s;
  }
  if (G == 1) {
    // one-CTA group: the CTA barrier orders this pass's global writes before the next
    // pass's reads (bar.sync), the proxy fence makes them visible to the TMA copies;
    // every thread sums the warp partials in the same fixed order, so the result is
    // bitwise the multi-CTA path's at G = 1.  sh is parity-buffered: one barrier.
    asm volatile("fence.proxy.async.global;" ::: "memory");
    __syncthreads();
#pragma unroll
    for (int k = 0; k < NP; ++k) {
      double s = 0.0;
#pragma unroll
      for (int i = 0; i < kWarps; ++i) s += sh[eb][i][k];
      out[k] = s + 0.0;
    }
    ++epoch;
    return;
  }
  __syncthreads();
  double* part = P.partials + (size_t)(epoch & 1ull) * kNPart * P.total_ctas;
  PROF_T(ta);
  if (w == 0) {
    if (lane < NP) {                                   // lane k: CTA partial of value k, fixed order
      double s = 0.0;
#pragma unroll
      for (int i = 0; i < kWarps; ++i) s += sh[eb][i][lane];
      __stcg(part + (size_t)lane * P.total_ctas + base + cl, s);
    }
    __syncwarp();
    // release: this CTA's r/p/q stores (ordered before by bar.sync) and its partials
    if (lane == 0) red_release_add(&P.sync->arrive[(g * kNSub + cl % kNSub) * kCtrStride], 1ull);
    PROF_T(tb);
    // lane s polls sub-counter s: the CTAs cl = s, s + kNSub, ... of the group arrive there
    if (lane < kNSub) {
      const unsigned long long cnt = (unsigned long long)((G - lane + kNSub - 1) / kNSub);
      const unsigned long long target = (epoch + 1ull) * cnt;
      const unsigned long long* ctr = &P.sync->arrive[(g * kNSub + lane) * kCtrStride];
      while (ld_acquire(ctr) < target) {
      }
    }
    __syncwarp();
#if MC_PROF
    if (cl == 0 && lane == 0) {
      PROF_T(tc);
      PROF_ADD(g, 1, tb - ta);
      PROF_ADD(g, 2, tc - tb);
    }
#endif
  }
  __syncthreads();
  PROF_T(td);
  if (w < NP) {
    double s = 0.0;
    const double* src = part + (size_t)w * P.total_ctas + base;
    for (int i = lane; i < G; i += 32) s += __ldcg(src + i);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) tot[w] = s;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < NP; ++k) out[k] = tot[k];
  __syncthreads();
#if MC_PROF
  if (cl == 0 && threadIdx.x == 0) {
    PROF_T(te);
    PROF_ADD(g, 3, te - td);
  }
#endif
  ++epoch;
}


// ---------------------------------------------------------------- block-Jacobi PCG (bj)
// Optional preconditioner (mc_set_preconditioner): M = the
// tridiagonal part of each 64-row chunk of a chain-ordered graph continuum (consecutive
// rows of a chunk connected along the network), solved exactly in shared memory with the
// chunk's precomputed Thomas factors.  Standard PCG, two reductions per iteration:
//   pass S:  p_j = z_j + beta p_{j-1} (own rows; far neighbours recomputed from their
//            published z, p_{j-1}), q = K p_j, partial p.q            -> alpha
//   pass U:  x += alpha p_j, r -= alpha q, z = M^{-1} r, partials r.z, r.r -> beta, stop
// The iterates solve the same SPD system; only the iteration count changes.

// z = M^{-1} r over a 64-row chunk by the whole warp (lane l: rows 2l, 2l+1): both Thomas
// sweeps are affine recurrences, d_i = (r_i - e_{i-1} d_{i-1}) / pivot_i forward and
// z_i = d_i - c'_i z_{i+1} backward, evaluated as 5-level shuffle scans of the composed
// affine maps instead of 64 serial steps each.
__device__ __forceinline__ void bj_scan_solve(const double* r, const double* inv, const double* cp,
                                              const double* em, int lane, double& z0, double& z1) {
  const int i0 = 2 * lane, i1 = i0 + 1;
  // forward: d_i = a_i d_{i-1} + b_i
  const double a0 = -em[i0] * inv[i0], b0 = r[i0] * inv[i0];
  const double a1 = -em[i1] * inv[i1], b1 = r[i1] * inv[i1];
  double A = a1 * a0, B = __fma_rn(a1, b0, b1);
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const double Ap = __shfl_up_sync(0xffffffffu, A, off), Bp = __shfl_up_sync(0xffffffffu, B, off);
    if (lane >= off) {
      B = __fma_rn(A, Bp, B);
      A = A * Ap;
    }
  }
  double dprev = __shfl_up_sync(0xffffffffu, B, 1);     // d_{2l-1}
  if (lane == 0) dprev = 0.0;
  const double d0 = __fma_rn(a0, dprev, b0), d1 = B;
  // backward: z_i = g_i z_{i+1} + h_i, g = -c', h = d.  cp == nullptr: c'_i = e_i / pivot_i
  // recomputed as em[i+1] * inv[i] (bitwise the stored factor; e_63 = 0 at the chunk's end)
  const double g0 = cp ? -cp[i0] : -(em[i1] * inv[i0]);
  const double g1 = cp ? -cp[i1] : (lane == 31 ? -0.0 : -(em[i1 + 1] * inv[i1]));
  double Ab = g0 * g1, Bb = __fma_rn(g0, d1, d0);
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const double An = __shfl_down_sync(0xffffffffu, Ab, off), Bn = __shfl_down_sync(0xffffffffu, Bb, off);
    if (lane + off < 32) {
      Bb = __fma_rn(Ab, Bn, Bb);
      Ab = Ab * An;
    }
  }
  double znext = __shfl_down_sync(0xffffffffu, Bb, 1);  // z_{2l+2}
  if (lane == 31) znext = 0.0;
  z0 = Bb;
  z1 = __fma_rn(g1, znext, d1);
}

__device__ __forceinline__ void bj_solve(const double* sl, double* zc, int lane) {
  // z = M^{-1} r over the chunk (r at sl + 2, 1/pivot at sl + 206, c' at zc + 64, e at zc + 128)
  double z0, z1;
  bj_scan_solve(sl + 2, sl + 206, zc + 64, zc + 128, lane, z0, z1);
  __syncwarp();
  zc[2 * lane] = z0;
  zc[2 * lane + 1] = z1;
  __syncwarp();
}

__device__ __noinline__ void run_group_bj(const StepParams& P, int g, int cl, double* x, const double* uo) {
  const Group& G = P.grp[g];
  const int W = G.cta_count * kWarps;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int wg = cl * kWarps + wid;
  const bool leader = (cl == 0 && threadIdx.x == 0);
  const long long t0 = leader ? globaltimer() : 0;
  const ContDev& C = P.cont[__ffs(G.cont_mask) - 1];
  extern __shared__ __align__(16) double dsm[];
  Stage st;
  st.wsm = dsm + wid * kWarpSmem;
  st.bars = reinterpret_cast<uint64_t*>(dsm + kWarps * kWarpSmem) + wid * kNBars;
  st.ph = reinterpret_cast<unsigned*>(dsm + kWarps * kWarpSmem + kWarps * kNBars) + 2 * wid;
  double* sl = st.wsm;                 // slot 0: r, q, p, 1/pivot, x, shift, codes
  double* zc = st.wsm + kSlotE;        // slot 1: z, c', e_{i-1}
  const int64_t off = C.off, es = C.estride;
  const int r1 = (int)C.n, nch = (r1 + 63) / 64;
  const int m = wg;                    // this warp's chunk (one per warp)
  const bool own = m < nch;
  const int base = 64 * m + 2 * lane;
  const int64_t g0 = off + base;
  const bool ok0 = own && base < r1, ok1 = own && base + 1 < r1;
  double* zg = P.q[0];                 // published z (global), read by far neighbours
  // init (a1, a2): lagged right-hand side, r0 = b - K x0, x0 = u^{n-1}
  double a3[3] = {0.0, 0.0, 0.0};
  for (int mm = wg; 32 * mm < r1; mm += W) {
    Item rit{};
    rit.cont = __ffs(G.cont_mask) - 1;
    rit.kind = ITEM_GRAPH;
    rit.a = 32 * mm;
    rit.b = min(32 * mm + 32, r1);
    init_item<false>(P, rit, uo, x, G.phase, a3);
  }
  unsigned long long epoch = 0;
  double t3[3];
  group_allreduce<3>(P, g, cl, epoch, a3, t3);
  const double bb = t3[0];
  double rr = t3[1];
  int64_t iters = 0;
  int status = MC_OK;
  bool zero = false, ran = false;
  if (bb == 0.0) {
    zero = true;
    rr = 0.0;
  } else if (!(rr <= G.tol2 * bb)) {
    ran = true;
    // own chunk -> shared memory: r, p (= 0), 1/pivot, x, shift, codes; z factors
    fence_proxy_async_shared_global();
    if (own) {
      __syncwarp();
      if (lane == 0) {
        const int64_t b0 = 64 * (int64_t)m, gg = off + b0;
        st.begin(0, 4u * 512u + 4u * 256u);
        uint64_t* bar = st.bars;
        bulk_g2s(sl + 2, P.r[0] + gg, 512, bar);
        bulk_g2s(sl + 206, C.tinv + gg, 512, bar);
        bulk_g2s(sl + 272, x + gg, 512, bar);
        bulk_g2s(sl + 336, P.dsD + gg, 512, bar);
        int32_t* si = reinterpret_cast<int32_t*>(sl + 400);
#pragma unroll
        for (int k = 0; k < 4; ++k) bulk_g2s(si + k * 64, C.ecol + k * es + b0, 256, bar);
        st.begin(1, 2u * 512u);
        bulk_g2s(zc + 64, C.tcp + gg, 512, st.bars + 1);
        bulk_g2s(zc + 128, C.tem + gg, 512, st.bars + 1);
      }
      st.wait(0);
      st.wait(1);
      // decode ELL codes into global columns (-1 none); p_{-1} = 0
      int32_t* si = reinterpret_cast<int32_t*>(sl + 400);
      const int64_t cb = off + 64 * (int64_t)m;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = lane + 32 * u, cd = si[e];
        si[e] = cd <= -2 ? (int32_t)(cb + (-2 - cd) - 2) : cd;
      }
      sl[138 + 2 * lane] = 0.0;
      sl[139 + 2 * lane] = 0.0;
      __syncwarp();
    }
    // U_0: z_0 = M^{-1} r_0, publish, r.z
    double rz = 0.0;
    {
      double a2[2] = {0.0, 0.0};
      if (own) {
        bj_solve(sl, zc, lane);
#pragma unroll
        for (int h = 0; h < 2; ++h)
          if (base + h < r1) {
            const double rv = sl[2 + 2 * lane + h], zv = zc[2 * lane + h];
            stmut(zg + g0 + h, zv);
            stmut(P.p[1] + g0 + h, 0.0);
            a2[0] += rv * zv;
            a2[1] += rv * rv;
          }
      }
      double t2[2];
      group_allreduce<2>(P, g, cl, epoch, a2, t2);
      rz = t2[0];
    }
    double beta = 0.0;
    const int32_t* si = reinterpret_cast<const int32_t*>(sl + 400);
    for (int64_t j = 0;; ++j) {
      // ---- pass S: p_j = z_j + beta p_{j-1}; q = K p_j; p.q
      const double* pold = P.p[(j + 1) & 1];
      double* pnew_g = P.p[j & 1];
      double a1[1] = {0.0};
      if (own) {
        double pc[2];
        int32_t jc[2][4];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int l2 = 2 * lane + h;
          pc[h] = __fma_rn(beta, sl[138 + l2], zc[l2]);
#pragma unroll
          for (int k = 0; k < 4; ++k) jc[h][k] = si[k * 64 + l2];
        }
        // far neighbours: recompute p from their published z and p_{j-1}
        double pf[2][4];
        const int64_t cb = off + 64 * (int64_t)m;
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int64_t jj = jc[h][k];
            const int64_t li = jj - cb;
            pf[h][k] = 0.0;
            if (jj >= 0 && !(li >= 0 && li < 64)) pf[h][k] = __fma_rn(beta, ldnb(pold + jj), ldnb(zg + jj));
          }
        __syncwarp();
        sl[138 + 2 * lane] = pc[0];
        sl[139 + 2 * lane] = pc[1];
        if (ok1) st2mut(pnew_g + g0, make_double2(pc[0], pc[1]));
        else if (ok0) stmut(pnew_g + g0, pc[0]);
        __syncwarp();
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          double s = 0.0;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int64_t jj = jc[h][k];
            const int64_t li = jj - cb;
            const bool in = jj >= 0 && li >= 0 && li < 64;
            const double v = jj < 0 ? pc[h] : (in ? sl[138 + (int)li] : pf[h][k]);
            s += pc[h] - v;
          }
          const double qv = sl[336 + 2 * lane + h] * pc[h] + C.Tconst * s;
          sl[70 + 2 * lane + h] = qv;
          if (base + h < r1) a1[0] += pc[h] * qv;
        }
      }
      double t1[1];
      group_allreduce<1>(P, g, cl, epoch, a1, t1);
      if (!(t1[0] > 0.0)) {
        iters = j;
        status = MC_ERR_BREAKDOWN;
        break;
      }
      const double alpha = rz / t1[0];
      // ---- pass U: x += alpha p; r -= alpha q; z = M^{-1} r; r.z, r.r
      double a2[2] = {0.0, 0.0};
      if (own) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int l2 = 2 * lane + h;
          sl[272 + l2] = __fma_rn(alpha, sl[138 + l2], sl[272 + l2]);
          sl[2 + l2] = __fma_rn(-alpha, sl[70 + l2], sl[2 + l2]);
        }
        __syncwarp();
        bj_solve(sl, zc, lane);
#pragma unroll
        for (int h = 0; h < 2; ++h)
          if (base + h < r1) {
            const double rv = sl[2 + 2 * lane + h], zv = zc[2 * lane + h];
            stmut(zg + g0 + h, zv);
            a2[0] += rv * zv;
            a2[1] += rv * rv;
          }
      }
      double t2[2];
      group_allreduce<2>(P, g, cl, epoch, a2, t2);
      rr = t2[1];
      iters = j + 1;
      if (rr <= G.tol2 * bb) break;
      if (j + 1 >= G.maxit) {
        status = MC_ERR_NOCONV;
        break;
      }
      if (!(t2[0] > 0.0)) {
        status = MC_ERR_BREAKDOWN;
        break;
      }
      beta = t2[0] / rz;
      rz = t2[0];
    }
  }
  if (ran && own)
    for (int h = 0; h < 2; ++h)
      if (base + h < r1) x[g0 + h] = sl[272 + 2 * lane + h];
  if (zero)
    for (int64_t i = (int64_t)wg * 32 + lane; i < C.n; i += (int64_t)W * 32) x[C.off + i] = 0.0;
  if (leader) {
    GroupOut o;
    o.iters = iters;
    o.status = status;
    o.pad = 0;
    o.bb = bb;
    o.rr = rr;
    o.t0 = t0;
    o.t1 = globaltimer();
    P.gout[g] = o;
  }
}


// ---------------------------------------------------------------- streaming block-Jacobi (bjs)
// The block-Jacobi PCG of run_group_bj for networks too large to stay resident (configs
// 2 and 4): both passes stream 64-row chunks round-robin over the group's warps, TMA
// staging kStagesB - 1 chunks ahead (MC_BJS_STAGES).
//   pass U:  x += alpha p, r -= alpha q, z = M^{-1} r (in-chunk Thomas from 1/pivot and e;
//            c' recomputed), r.z, r.r
//   pass S:  p = z + beta p_old on the chunk's 68-row window and its far neighbours
//            (gathered z, p_old), q = K p, p.q
// r, q, z single buffers (each written and read by the owner, z read by neighbours only
// after the reduction); p double-buffered (neighbours read p_old while owners write p).
__device__ void bjs_pass_u(const StepParams& P, const ContDev& C, int wg, int W, const Stage& st, double* x,
                           const double* pj, double* zg, double* pzero, double alpha, double (&a2)[2]) {
  const int lane = threadIdx.x & 31;
  double* wsm = st.wsm;
  const int64_t off = C.off;
  const int r1 = (int)C.n, nch = (r1 + 63) / 64;
  auto prefetch = [&](int m, int t) {
    double* sl = wsm + t * kSlotE;
    __syncwarp();
    if (lane == 0) {
      const int64_t g = off + 64 * (int64_t)m;
      st.begin(t, 6u * 512u);
      uint64_t* bar = st.bars + t;
      bulk_g2s(sl + 0, P.r[0] + g, 512, bar);
      bulk_g2s(sl + 64, P.q[0] + g, 512, bar);
      bulk_g2s(sl + 128, pj + g, 512, bar);
      bulk_g2s(sl + 192, x + g, 512, bar);
      bulk_g2s(sl + 256, C.tinv + g, 512, bar);
      bulk_g2s(sl + 384, C.tem + g, 512, bar);       // c' recomputed from e and 1/pivot
    }
  };
  if (wg >= nch) return;
#pragma unroll
  for (int k = 0; k < kStagesB - 1; ++k)
    if (wg + k * W < nch) prefetch(wg + k * W, k);
  int t = 0;
  for (int m = wg; m < nch; m += W, t = (t + 1 == kStagesB ? 0 : t + 1)) {
    if (m + (kStagesB - 1) * W < nch) prefetch(m + (kStagesB - 1) * W, t == 0 ? kStagesB - 1 : t - 1);
    st.wait(t);
    double* sl = wsm + t * kSlotE;
    const int base = 64 * m + 2 * lane;
    const int64_t g = off + base;
    double rn[2], xn[2];
    {
      const double2 r2 = *reinterpret_cast<const double2*>(sl + 2 * lane);
      const double2 q2 = *reinterpret_cast<const double2*>(sl + 64 + 2 * lane);
      const double2 p2 = *reinterpret_cast<const double2*>(sl + 128 + 2 * lane);
      const double2 x2 = *reinterpret_cast<const double2*>(sl + 192 + 2 * lane);
      xn[0] = __fma_rn(alpha, p2.x, x2.x);
      xn[1] = __fma_rn(alpha, p2.y, x2.y);
      rn[0] = __fma_rn(-alpha, q2.x, r2.x);
      rn[1] = __fma_rn(-alpha, q2.y, r2.y);
    }
    __syncwarp();
    *reinterpret_cast<double2*>(sl + 2 * lane) = make_double2(rn[0], rn[1]);
    __syncwarp();
    double z0, z1;                                      // z = M^{-1} r over the chunk
    bj_scan_solve(sl, sl + 256, nullptr, sl + 384, lane, z0, z1);
    if (base + 1 < r1) {
      *reinterpret_cast<double2*>(x + g) = make_double2(xn[0], xn[1]);
      st2mut(P.r[0] + g, make_double2(rn[0], rn[1]));
      st2mut(zg + g, make_double2(z0, z1));
      if (pzero) st2mut(pzero + g, make_double2(0.0, 0.0));
      a2[0] += rn[0] * z0;
      a2[1] += rn[0] * rn[0];
      a2[0] += rn[1] * z1;
      a2[1] += rn[1] * rn[1];
    } else if (base < r1) {
      x[g] = xn[0];
      stmut(P.r[0] + g, rn[0]);
      stmut(zg + g, z0);
      if (pzero) stmut(pzero + g, 0.0);
      a2[0] += rn[0] * z0;
      a2[1] += rn[0] * rn[0];
    }
  }
}

__device__ void bjs_pass_s(const StepParams& P, const ContDev& C, int wg, int W, const Stage& st,
                           const double* zg, const double* pold, double* pnew_g, double beta, double (&a1)[1]) {
  const int lane = threadIdx.x & 31;
  double* wsm = st.wsm;
  double* pnb = wsm + kWarpSmem - kPnBuf;
  const int64_t off = C.off, es = C.estride;
  const int r1 = (int)C.n, nch = (r1 + 63) / 64;
  auto tix = [&](int m) { return (m / W) % kStagesB; };
  auto prefetch = [&](int m) {
    const int t = tix(m);
    double* sl = wsm + t * kSlotE;
    __syncwarp();
    if (lane == 0) {
      const int64_t b = 64 * (int64_t)m;
      const int64_t g = off + b;
      const bool full = g >= 2;
      const unsigned wb = full ? 544u : 528u;
      st.begin(t, 2u * wb + 512u + 4u * 256u);
      uint64_t* bar = st.bars + t;
      const int64_t g0 = g - (full ? 2 : 0);
      const int d0 = full ? 0 : 2;
      bulk_g2s(sl + d0, zg + g0, wb, bar);
      bulk_g2s(sl + 68 + d0, pold + g0, wb, bar);
      bulk_g2s(sl + 136, P.dsD + g, 512, bar);
      int32_t* si = reinterpret_cast<int32_t*>(sl + 200);
#pragma unroll
      for (int k = 0; k < 4; ++k) bulk_g2s(si + k * 64, C.ecol + k * es + b, 256, bar);
    }
  };
  if (wg >= nch) return;
#pragma unroll
  for (int k = 0; k < kStagesB - 1; ++k)
    if (wg + k * W < nch) prefetch(wg + k * W);
  for (int m = wg; m < nch; m += W) {
    if (m + (kStagesB - 1) * W < nch) prefetch(m + (kStagesB - 1) * W);
    const int t = tix(m);
    st.wait(t);
    const double* sl = wsm + t * kSlotE;
    const int base = 64 * m + 2 * lane;
    const int64_t g = off + base;
    const bool ok0 = base < r1, ok1 = base + 1 < r1;
    // codes and far gathers (z, p_old of rows outside the window)
    int32_t j[2][4];
    {
      const int32_t* si = reinterpret_cast<const int32_t*>(sl + 200);
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int k = 0; k < 4; ++k) j[h][k] = si[k * 64 + 2 * lane + h];
    }
    int fs0 = -1, fs1 = -1, fs2 = -1, fs3 = -1;
    int32_t i0 = -1, i1 = -1, i2 = -1, i3 = -1;
    int nfar = 0;
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (j[h][k] >= 0) {
          if (nfar == 0) { i0 = j[h][k]; fs0 = 4 * h + k; }
          else if (nfar == 1) { i1 = j[h][k]; fs1 = 4 * h + k; }
          else if (nfar == 2) { i2 = j[h][k]; fs2 = 4 * h + k; }
          else if (nfar == 3) { i3 = j[h][k]; fs3 = 4 * h + k; }
          ++nfar;
        }
    double w0 = 0.0, w1 = 0.0, w2 = 0.0, w3 = 0.0;
    if (i0 >= 0) w0 = __fma_rn(beta, ldnb(pold + i0), ldnb(zg + i0));
    if (i1 >= 0) w1 = __fma_rn(beta, ldnb(pold + i1), ldnb(zg + i1));
    if (i2 >= 0) w2 = __fma_rn(beta, ldnb(pold + i2), ldnb(zg + i2));
    if (i3 >= 0) w3 = __fma_rn(beta, ldnb(pold + i3), ldnb(zg + i3));
    // p on the window (own rows and the 2-row halos)
    double pc[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int w = 2 + 2 * lane + h;
      pc[h] = __fma_rn(beta, sl[68 + w], sl[w]);
    }
    __syncwarp();
    pnb[2 + 2 * lane] = pc[0];
    pnb[3 + 2 * lane] = pc[1];
    if (lane < 4) {
      const int w = lane < 2 ? lane : 64 + lane;
      pnb[w] = __fma_rn(beta, sl[68 + w], sl[w]);
    }
    if (ok1) st2mut(pnew_g + g, make_double2(pc[0], pc[1]));
    else if (ok0) stmut(pnew_g + g, pc[0]);
    __syncwarp();
    double qv[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      double sum = 0.0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int32_t cd = j[h][k];
        double v = pc[h];
        if (cd <= -2) v = pnb[-2 - cd];
        else if (cd >= 0) {
          if (fs0 == 4 * h + k) v = w0;
          else if (fs1 == 4 * h + k) v = w1;
          else if (fs2 == 4 * h + k) v = w2;
          else if (fs3 == 4 * h + k) v = w3;
          else v = __fma_rn(beta, ldnb(pold + cd), ldnb(zg + cd));     // rare: > 4 far
        }
        sum += pc[h] - v;
      }
      qv[h] = sl[136 + 2 * lane + h] * pc[h] + C.Tconst * sum;
    }
    if (ok1) st2mut(P.q[0] + g, make_double2(qv[0], qv[1]));
    else if (ok0) stmut(P.q[0] + g, qv[0]);
    if (ok0) a1[0] += pc[0] * qv[0];
    if (ok1) a1[0] += pc[1] * qv[1];
  }
}

// Pass S on the chunk-blocked static data (the shift and the far-first int32 codes of C.bstat;
// no halo window: neighbours in other chunks are gathered, z and p_old from global).  Same
// arithmetic as bjs_pass_s with three bulk copies per chunk instead of seven and without the
// far-slot search cascades (the instruction diet of iter_ellb).
__device__ void bjs_pass_s2(const StepParams& P, const ContDev& C, int wg, int W, const Stage& st,
                            const double* zg, const double* pold, double* pnew_g, double beta, double (&a1)[1]) {
  const int lane = threadIdx.x & 31;
  double* wsm = st.wsm;
  double* pnb = wsm + kWarpSmem - kPnBuf;
  const int64_t off = C.off;
  const int r1 = (int)C.n, nch = (r1 + 63) / 64;
  const double* zo = zg + off;
  const double* po_g = pold + off;
  auto prefetch = [&](int m, int t) {
    double* sl = wsm + t * kSlotE;
    __syncwarp();
    if (lane == 0) {
      const int64_t g = off + 64 * (int64_t)m;
      st.begin(t, 2u * 512u + 8u * 192u);
      uint64_t* bar = st.bars + t;
      bulk_g2s(sl, zg + g, 512, bar);
      bulk_g2s(sl + 64, pold + g, 512, bar);
      bulk_g2s(sl + 128, C.bstat + (int64_t)m * kBStat + 64, 8u * 192u, bar);   // shift (64) | codes (128)
    }
  };
  if (wg >= nch) return;
  prefetch(wg, 0);
  int t = 0;
  auto pfar = [&](int32_t j) { return __fma_rn(beta, ldnb(po_g + j), ldnb(zo + j)); };
  for (int m = wg; m < nch; m += W, t ^= 1) {
    if (m + W < nch) prefetch(m + W, t ^ 1);
    st.wait(t);
    const double* sl = wsm + t * kSlotE;
    const int4 c0 = *reinterpret_cast<const int4*>(sl + 192 + 4 * lane);
    const int4 c1 = *reinterpret_cast<const int4*>(sl + 192 + 4 * lane + 2);
    double f00 = 0.0, f01 = 0.0, f10 = 0.0, f11 = 0.0;
    if (c0.x >= 0) f00 = pfar(c0.x);
    if (c0.y >= 0) f01 = pfar(c0.y);
    if (c1.x >= 0) f10 = pfar(c1.x);
    if (c1.y >= 0) f11 = pfar(c1.y);
    const double2 z2 = *reinterpret_cast<const double2*>(sl + 2 * lane);
    const double2 po = *reinterpret_cast<const double2*>(sl + 64 + 2 * lane);
    const double2 ds = *reinterpret_cast<const double2*>(sl + 128 + 2 * lane);
    const double p0 = __fma_rn(beta, po.x, z2.x), p1 = __fma_rn(beta, po.y, z2.y);
    __syncwarp();                                                 // previous chunk's pnb reads done
    *reinterpret_cast<double2*>(pnb + 2 * lane) = make_double2(p0, p1);
    __syncwarp();
    auto nbv = [&](int32_t cd, double far, double own) { return cd >= 0 ? far : (cd <= -2 ? pnb[-2 - cd] : own); };
    double f02 = 0.0, f03 = 0.0, f12 = 0.0, f13 = 0.0;
    if (__any_sync(0xffffffffu, (c0.z >= 0) | (c0.w >= 0) | (c1.z >= 0) | (c1.w >= 0))) {   // rare: > 2 far in a row
      if (c0.z >= 0) f02 = pfar(c0.z);
      if (c0.w >= 0) f03 = pfar(c0.w);
      if (c1.z >= 0) f12 = pfar(c1.z);
      if (c1.w >= 0) f13 = pfar(c1.w);
    }
    double s0 = p0 - nbv(c0.x, f00, p0);
    s0 += p0 - nbv(c0.y, f01, p0);
    s0 += p0 - nbv(c0.z, f02, p0);
    s0 += p0 - nbv(c0.w, f03, p0);
    double s1 = p1 - nbv(c1.x, f10, p1);
    s1 += p1 - nbv(c1.y, f11, p1);
    s1 += p1 - nbv(c1.z, f12, p1);
    s1 += p1 - nbv(c1.w, f13, p1);
    const double q0 = __fma_rn(C.Tconst, s0, __dmul_rn(ds.x, p0));
    const double q1 = __fma_rn(C.Tconst, s1, __dmul_rn(ds.y, p1));
    const int base = 64 * m + 2 * lane;
    const int64_t g = off + base;
    if (base + 1 < r1) {
      st2mut(pnew_g + g, make_double2(p0, p1));
      st2mut(P.q[0] + g, make_double2(q0, q1));
      a1[0] += p0 * q0;
      a1[0] += p1 * q1;
    } else if (base < r1) {
      stmut(pnew_g + g, p0);
      stmut(P.q[0] + g, q0);
      a1[0] += p0 * q0;
    }
  }
}

__device__ __noinline__ void run_group_bjs(const StepParams& P, int g, int cl, double* x, const double* uo) {
  const Group& G = P.grp[g];
  const int W = G.cta_count * kWarps;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int wg = cl * kWarps + wid;
  const bool leader = (cl == 0 && threadIdx.x == 0);
  const long long t0 = leader ? globaltimer() : 0;
  const int ca = __ffs(G.cont_mask) - 1;
  const ContDev& C = P.cont[ca];
  extern __shared__ __align__(16) double dsm[];
  Stage st;
  st.wsm = dsm + wid * kWarpSmem;
  st.bars = reinterpret_cast<uint64_t*>(dsm + kWarps * kWarpSmem) + wid * kNBars;
  st.ph = reinterpret_cast<unsigned*>(dsm + kWarps * kWarpSmem + kWarps * kNBars) + 2 * wid;
  const int r1 = (int)C.n;
  double* zg = P.q[1];
  double a3[3] = {0.0, 0.0, 0.0};
  for (int mm = wg; 32 * mm < r1; mm += W) {
    Item rit{};
    rit.cont = ca;
    rit.kind = ITEM_GRAPH;
    rit.a = 32 * mm;
    rit.b = min(32 * mm + 32, r1);
    init_item<false>(P, rit, uo, x, G.phase, a3);
  }
  unsigned long long epoch = 0;
  double t3[3];
  group_allreduce<3>(P, g, cl, epoch, a3, t3);
  const double bb = t3[0];
  double rr = t3[1];
  int64_t iters = 0;
  int status = MC_OK;
  bool zero = false;
  if (bb == 0.0) {
    zero = true;
    rr = 0.0;
  } else if (!(rr <= G.tol2 * bb)) {
    fence_proxy_async_shared_global();
    double rz;
    {
      double a2[2] = {0.0, 0.0};
      bjs_pass_u(P, C, wg, W, st, x, P.p[0], zg, P.p[1], 0.0, a2);     // U_0: z_0, p_{-1} = 0
      double t2[2];
      group_allreduce<2>(P, g, cl, epoch, a2, t2);
      rz = t2[0];
    }
    double beta = 0.0;
    for (int64_t j = 0;; ++j) {
      double* pj = P.p[j & 1];
      const double* pold = P.p[(j + 1) & 1];
      double a1[1] = {0.0};
      fence_proxy_async_shared_global();
      if (C.bstat) bjs_pass_s2(P, C, wg, W, st, zg, pold, pj, beta, a1);
      else bjs_pass_s(P, C, wg, W, st, zg, pold, pj, beta, a1);
      double t1[1];
      group_allreduce<1>(P, g, cl, epoch, a1, t1);
      if (!(t1[0] > 0.0)) {
        iters = j;
        status = MC_ERR_BREAKDOWN;
        break;
      }
      const double alpha = rz / t1[0];
      double a2[2] = {0.0, 0.0};
      fence_proxy_async_shared_global();
      bjs_pass_u(P, C, wg, W, st, x, pj, zg, nullptr, alpha, a2);
      double t2[2];
      group_allreduce<2>(P, g, cl, epoch, a2, t2);
      rr = t2[1];
      iters = j + 1;
      if (rr <= G.tol2 * bb) break;
      if (j + 1 >= G.maxit) {
        status = MC_ERR_NOCONV;
        break;
      }
      if (!(t2[0] > 0.0)) {
        status = MC_ERR_BREAKDOWN;
        break;
      }
      beta = t2[0] / rz;
      rz = t2[0];
    }
  }
  if (zero)
    for (int64_t i = (int64_t)wg * 32 + lane; i < C.n; i += (int64_t)W * 32) x[C.off + i] = 0.0;
  if (leader) {
    GroupOut o;
    o.iters = iters;
    o.status = status;
    o.pad = 0;
    o.bb = bb;
    o.rr = rr;
    o.t0 = t0;
    o.t1 = globaltimer();
    P.gout[g] = o;
  }
}

// ---------------------------------------------------------------- the step kernel
template <bool CPL>
__device__ void run_group(const StepParams& P, int g, int cl, double* x, const double* uo) {
  const Group& G = P.grp[g];
  const int W = G.cta_count * kWarps;
  const int wg = cl * kWarps + (threadIdx.x >> 5);
  const int ib = G.item_begin, ie = G.item_begin + G.item_count;
  const bool leader = (cl == 0 && threadIdx.x == 0);
  long long t0 = leader ? globaltimer() : 0;
  extern __shared__ __align__(16) double dsm[];
  const int wid = threadIdx.x >> 5;
  Stage st;
  st.wsm = dsm + wid * kWarpSmem;                            // this warp's staging slots
  st.bars = reinterpret_cast<uint64_t*>(dsm + kWarps * kWarpSmem) + wid * kNBars;
  st.ph = reinterpret_cast<unsigned*>(dsm + kWarps * kWarpSmem + kWarps * kNBars) + 2 * wid;
  double* wsm = st.wsm;

  double a3[3] = {0.0, 0.0, 0.0};
  for (int k = 0; k < P.L; ++k)
    if (((G.cont_mask >> k) & 1) && P.cont[k].rr)
      for (int m = wg; 32 * m < P.cont[k].n; m += W) {
        Item rit{};
        rit.cont = k;
        rit.kind = ITEM_GRAPH;
        rit.a = 32 * m;
        rit.b = (int32_t)min((int64_t)(32 * m + 32), P.cont[k].n);
        init_item<CPL>(P, rit, uo, x, G.phase, a3);
      }
  for (int it = ib + wg; it < ie; it += W) init_item<CPL>(P, P.items[it], uo, x, G.phase, a3);
  unsigned long long epoch = 0;
  double t3[3];
  group_allreduce<3>(P, g, cl, epoch, a3, t3);
  const double bb = t3[0];
  double rr = t3[1];
  int64_t iters = 0;
  int64_t passes = 0;
  int status = MC_OK;
  bool zero = false;
  if (bb == 0.0) {
    zero = true;       // b = 0  =>  x = 0 after 0 iterations
    rr = 0.0;
  } else if (!(rr <= G.tol2 * bb)) {
    Item it0{};
    if (ib + wg < ie) it0 = P.items[ib + wg];     // most warps own exactly one item
    Ctx c;
    c.P = &P;
    c.x = x;
    c.ds = CPL ? P.dsC : P.dsD;
    c.a = 0.0;
    c.b = 0.0;
    for (int64_t j = 0;; ++j) {
      const int s = (int)(j & 1);
      c.rs = P.r[s];
      c.qs = P.q[s];
      c.ps = P.p[s];
      c.rd = P.r[s ^ 1];
      c.pd = P.p[s ^ 1];
      c.qd = P.q[s ^ 1];
      double a5[kNPart] = {0.0, 0.0, 0.0, 0.0, 0.0};
      PROF_T(tp0);
      for (int k = 0; k < P.L; ++k)
        if (((G.cont_mask >> k) & 1) && P.cont[k].rr) {
          if (P.cont[k].resident) {
            if (!CPL && P.cont[k].bstat) iter_ells_res2(c, P.cont[k], wg, W, st, j == 0, s, a5);
            else iter_ells_res<CPL>(c, P.cont[k], wg, W, st, j == 0, a5);
          } else if (!CPL && P.cont[k].bdyn[0]) iter_ellb(c, P.cont[k], wg, W, st, s, a5);
          else iter_ells<CPL>(c, P.cont[k], wg, W, st, a5);
        }
      for (int it = ib + wg; it < ie; it += W) {
        const Item item = (it == ib + wg) ? it0 : P.items[it];
        const ContDev& C = P.cont[item.cont];
        if (item.kind == ITEM_GRID) {
          if (item.w == 64) iter_grid2s<CPL>(c, C, item.a, item.b, item.c, st, a5);
          else iter_grid<CPL>(c, C, item.a, item.b, item.c, a5);
        } else if (C.lpr == 8) {
          iter_graph8<CPL>(c, C, item.a, item.b, a5);
        } else {
          iter_graph<CPL>(c, C, item.a, item.b, a5);
        }
      }
      double t5[kNPart];
#if MC_PROF
      if (cl == 0 && threadIdx.x == 0) {
        PROF_T(tp1);
        PROF_ADD(g, 0, tp1 - tp0);
        PROF_ADD(g, 4, 1);
      }
#endif
      group_allreduce<kNPart>(P, g, cl, epoch, a5, t5);
      passes = j + 1;
      rr = t5[1];
      if (j > 0 && rr <= G.tol2 * bb) {
        iters = j;
        break;
      }
      if (j >= G.maxit) {
        iters = j;
        status = MC_ERR_NOCONV;
        break;
      }
      if (!(t5[0] > 0.0) || !(t5[2] > 0.0)) {
        iters = j;
        status = MC_ERR_BREAKDOWN;
        break;
      }
      const double rz = t5[2];
      const double alpha = rz / t5[0];
      const double rz_next = __fma_rn(alpha * alpha, t5[4], __fma_rn(-2.0 * alpha, t5[3], rz));
      c.a = alpha;
      c.b = rz_next / rz;
    }
  }
  if (passes > 0)
    for (int k = 0; k < P.L; ++k)
      if (((G.cont_mask >> k) & 1) && P.cont[k].rr && P.cont[k].resident) {
        if (!CPL && P.cont[k].bstat) flush_ells_res2(P.cont[k], wg, W, wsm, x);
        else flush_ells_res(P.cont[k], wg, W, wsm, x);
      }
  if (zero)
    for (int it = ib + wg; it < ie; it += W) zero_item(P, P.items[it], x);
  if (zero)
    for (int k = 0; k < P.L; ++k)
      if (((G.cont_mask >> k) & 1) && P.cont[k].rr)
        for (int64_t i = (int64_t)wg * 32 + (threadIdx.x & 31); i < P.cont[k].n; i += (int64_t)W * 32)
          x[P.cont[k].off + i] = 0.0;
  if (leader) {
    GroupOut o;
    o.iters = iters;
    o.status = status;
    o.pad = 0;
    o.bb = bb;
    o.rr = rr;
    o.t0 = t0;
    o.t1 = globaltimer();
    P.gout[g] = o;
  }
}

__device__ __forceinline__ void grid_barrier(const StepParams& P, unsigned long long target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    red_release_add(&P.sync->phase_arrive, 1ull);
    while (ld_acquire(&P.sync->phase_arrive) < target) {
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kThreads, kMinBlocks) step_kernel(const __grid_constant__ StepParams P) {
  {  // staging barriers: one mbarrier per slot per warp (arrival count 1: the issuing lane)
    extern __shared__ __align__(16) double dsm[];
    if ((threadIdx.x & 31) == 0) {
      const int wid = threadIdx.x >> 5;
      uint64_t* bars = reinterpret_cast<uint64_t*>(dsm + kWarps * kWarpSmem) + wid * kNBars;
      for (int t = 0; t < kNBars; ++t) mbar_init(bars + t, 1);
      *(reinterpret_cast<unsigned*>(dsm + kWarps * kWarpSmem + kWarps * kNBars) + 2 * wid) = 0u;
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
  }
  const int failed = *(volatile const int32_t*)P.fail;
  const int cur = *(volatile const int32_t*)P.cur;
  if (!failed) {
    const double* uo = P.u[cur];
    double* x = P.u[cur ^ 1];
    for (int ph = 0; ph < P.nphases; ++ph) {
      for (int g = 0; g < P.ngroups; ++g) {
        const Group& G = P.grp[g];
        if (G.phase != ph || (int)blockIdx.x < G.cta_begin || (int)blockIdx.x >= G.cta_begin + G.cta_count)
          continue;
        const int cl = (int)blockIdx.x - G.cta_begin;
        const int a0 = __ffs(G.cont_mask) - 1;
        if (P.coupled) run_group<true>(P, g, cl, x, uo);
        else if ((G.cont_mask & (G.cont_mask - 1)) == 0 && P.cont[a0].bj) run_group_bj(P, g, cl, x, uo);
        else if ((G.cont_mask & (G.cont_mask - 1)) == 0 && P.cont[a0].bjs) run_group_bjs(P, g, cl, x, uo);
        else run_group<false>(P, g, cl, x, uo);
      }
      if (ph + 1 < P.nphases) grid_barrier(P, (unsigned long long)(ph + 1) * gridDim.x);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned prev = atomicAdd(&P.sync->finished, 1u);
    if (prev == gridDim.x - 1) {
      __threadfence();
      mc_step_report* rep = P.rep;
      rep->step = P.step_no;
      rep->scheme = P.scheme;
      rep->nsolves = P.ngroups;
      rep->failed_solve = -1;
      rep->paths = 0;
      if (failed) {
        rep->status = MC_ERR_STATE;    // an earlier step of this run failed: skipped
        for (int k = 0; k < MC_MAX_CONTINUA; ++k) {
          rep->iters[k] = 0;
          rep->relres[k] = 0.0;
          rep->bnorm[k] = 0.0;
          rep->ms_solve[k] = 0.0;
        }
      } else {
        int st = MC_OK;
        for (int k = 0; k < MC_MAX_CONTINUA; ++k) {
          if (k < P.ngroups) {
            volatile GroupOut* o = P.gout + k;
            rep->iters[k] = o->iters;
            const double bb = o->bb, rr = o->rr;
            rep->bnorm[k] = sqrt(bb);
            rep->relres[k] = bb > 0.0 ? sqrt(rr / bb) : 0.0;
            rep->ms_solve[k] = (double)(o->t1 - o->t0) * 1e-6;
            if (o->status != MC_OK && st == MC_OK) {
              st = o->status;
              rep->failed_solve = k;
            }
          } else {
            rep->iters[k] = 0;
            rep->relres[k] = 0.0;
            rep->bnorm[k] = 0.0;
            rep->ms_solve[k] = 0.0;
          }
        }
        rep->status = st;
        if (st == MC_OK) *(volatile int32_t*)P.cur = cur ^ 1;   // commit p^n (all solves converged)
        else *(volatile int32_t*)P.fail = 1;
      }
      rep->ms = 0.0;
      __threadfence();
    }
  }
}

// state I/O between the caller's numbering and the internal chain numbering
__global__ void to_caller_kernel(double* __restrict__ dst, const double* __restrict__ src,
                                 const int32_t* __restrict__ perm, int64_t n) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    dst[perm[t]] = src[t];
}
__global__ void from_caller_kernel(double* __restrict__ dst, const double* __restrict__ src,
                                   const int32_t* __restrict__ perm, int64_t n) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    dst[t] = src[perm[t]];
}
static int io_blocks(int64_t n) { return (int)std::min<int64_t>(4 * 148, (n + 255) / 256 + 1); }
cudaError_t launch_to_caller(double* dst, const double* src, const int32_t* perm, int64_t n, cudaStream_t s) {
  to_caller_kernel<<<io_blocks(n), 256, 0, s>>>(dst, src, perm, n);
  return cudaGetLastError();
}
cudaError_t launch_from_caller(double* dst, const double* src, const int32_t* perm, int64_t n, cudaStream_t s) {
  from_caller_kernel<<<io_blocks(n), 256, 0, s>>>(dst, src, perm, n);
  return cudaGetLastError();
}

cudaError_t launch_step(const StepParams* params, int total_ctas, cudaStream_t s) {
  void* args[] = {(void*)params};
  return cudaLaunchCooperativeKernel((const void*)step_kernel, dim3(total_ctas), dim3(kThreads),
                                     args, kDynSmem, s);
}

#if MC_PROF
extern "C" int mc_prof_read(long long* out, int reset) {
  cudaError_t e = cudaMemcpyFromSymbol(out, g_prof, sizeof(g_prof));
  if (reset) {
    static long long z[MC_MAX_CONTINUA][8] = {};
    cudaMemcpyToSymbol(g_prof, z, sizeof(z));
  }
  return (int)e;
}
#endif

cudaError_t step_kernel_occupancy(int* blocks_per_sm) {
  cudaError_t e = cudaFuncSetAttribute((const void*)step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kDynSmem);
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, step_kernel, kThreads, kDynSmem);
}

}  // namespace mc
