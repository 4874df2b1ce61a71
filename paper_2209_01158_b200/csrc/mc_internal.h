// mc_internal.h — structures shared by the host API (mc_api.cu) and the sm_100a
// kernels (mc_kernels.cu).  Not part of the public ABI (include/mc.h).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "../../include/mc.h"

namespace mc {

constexpr int kThreads = 256;          // threads per CTA of the step kernel
constexpr int kWarps = kThreads / 32;
#ifndef MC_MINBLOCKS
#define MC_MINBLOCKS 2
#endif
#ifndef MC_STAGES
#define MC_STAGES 2
#endif
#ifndef MC_PROF
#define MC_PROF 0                          // dev: per-phase clock64 instrumentation (mc_prof_read)
#endif
#ifndef MC_CHECK
#define MC_CHECK 0                         // checked build (libmc_check.so): device-side bounds asserts on every
#endif                                     // gather index, staged window and work item; guard words after every
                                           // device array verified at mc_destroy.  compute-sanitizer is closed
                                           // on the B200 pool, this is its stand-in.
#if MC_CHECK
#include <cassert>
#define MC_ASSERT(c) assert(c)
#else
#define MC_ASSERT(c) ((void)0)
#endif
#ifndef MC_TMA
#define MC_TMA 1                           // stage with TMA bulk copies (1) or per-lane cp.async (0)
#endif
constexpr int kMinBlocks = MC_MINBLOCKS;   // __launch_bounds__ residency target (CTAs of 256 per SM)
constexpr int kStages = MC_STAGES;         // cp.async staging slots per warp (prefetch distance - 1)
constexpr int kNPart = 5;              // reduction slots per barrier (pq, rr, rz, rq, qq)
constexpr int kPadDofs = 32;           // continuum offsets padded to 32 doubles (256 B)
constexpr int kCtrStride = 32;         // barrier counters 256 B apart (own L2 line / slice)
#ifndef MC_NSUB
#define MC_NSUB 1
#endif
constexpr int kNSub = MC_NSUB;         // arrival sub-counters per group barrier (CTA cl arrives on counter
                                       // cl % kNSub, lanes 0..kNSub-1 of warp 0 poll one each).  Measured
                                       // with 8: no gain (config-1 fracture 5.4 vs 5.3 us per iteration,
                                       // profiles/r02_barrier_subcounters.txt), so the default is one
constexpr int kSlack = 128;            // extra doubles after every per-DOF array (staged over-reads)
// cp.async staging: per warp, two slots of the next rows' operands
constexpr int kSlotG = 536;            // grid strip slot: 8 arrays x 64 doubles + 18 edge doubles
constexpr int kSlotE = 528;            // ELL chunk slot: r, q, p, D^-1 windows (68), x, shift (64), 4 x 64 int32 codes
constexpr int kStagesE = 2;                // ELL pass: chunk in flight + chunk computed
constexpr int kBStat = 256;                // chunk-blocked pass: doubles of static data per chunk
constexpr int kBDyn = 192;                 //                     doubles of CG state per chunk and parity
constexpr int kPnBuf = 72;                 // ELL pass: new p of the chunk window (68) per warp
#ifndef MC_BJS_STAGES
#define MC_BJS_STAGES 2
#endif
constexpr int kStagesB = MC_BJS_STAGES;    // streaming block-Jacobi passes: chunks in flight + 1
constexpr int kStagesEB = (kStagesE > kStagesB) ? kStagesE : kStagesB;
constexpr int kMaxI(int a, int b) { return a > b ? a : b; }
constexpr int kWarpSmem = kMaxI(kStages * kSlotG, kStagesEB * kSlotE) + kPnBuf;
// bytes per CTA: staging slots, then one mbarrier per slot per warp, then a parity word per warp
constexpr int kNBars = kMaxI(kStages, kStagesEB);   // mbarriers per warp
constexpr int kDynSmem = kWarps * kWarpSmem * 8 + kWarps * kNBars * 8 + kWarps * 8;

enum ContKind : int32_t { KIND_GRID = 0, KIND_GRAPH = 1 };
enum ItemKind : int32_t { ITEM_GRID = 0, ITEM_GRAPH = 1 };

// one continuum as the kernels see it
struct ContDev {
  int32_t kind;
  int32_t nx, ny;          // grid
  int64_t off, n;          // global DOF offset and count
  const double* Tx;        // grid: face (iy,ix)-(iy,ix+1); 0 on the last column
  const double* Ty;        // grid: face (iy,ix)-(iy+1,ix); 0 on the last row
  const int32_t* rowptr;   // graph: [n+1], local
  const int32_t* col;      // graph: GLOBAL column indices
  const double* val;       // graph: per-entry T, or nullptr -> Tconst
  const int32_t* ecol;     // graph: ELL codes [4][estride] (k-major): -1 none, -2-w window slot, >=0 global
  double Tconst;
  int32_t lpr;             // graph: lanes per row (1 or 8)
  int32_t ell;             // graph: ELL width (4) when ecol != nullptr
  int64_t estride;         // graph: ELL row stride (n rounded up to 64, + 64)
  int32_t rr;              // 1: processed by the whole group, 64-row chunks round-robin over warps
  int32_t resident;        // rr + every warp owns <= kStages chunks: state stays in shared memory
  int32_t bj;              // resident, one chunk per warp, block-Jacobi preconditioner (§8(f) rank 4)
  int32_t bjs;             // block-Jacobi, streaming passes (network too large to stay resident)
  // chunk-blocked workspace of the streaming ELL pass of a decoupled Jacobi solve:
  const double* bstat;     // per 64-row chunk 256 doubles: D^-1 (64), shift (64), 4 int32 codes per row (128)
  double* rrec[2];         // resident pass: published 32-byte records {r, q, p, D^-1} per row (far gathers:
                           // one 256-bit load of one sector instead of four 8-byte loads), by iteration parity
  double* bdyn[2];         // per chunk 192 doubles: r (64), q (64), p (64); double-buffered by iteration parity
  const double* tinv;      // bj: Thomas factors of each 64-row chunk's tridiagonal block:
  const double* tcp;       //     1 / pivot, super-diagonal multiplier c', sub-diagonal e_{i-1}
  const double* tem;
};

// a work item: a 32-column strip segment of a grid, or a row range of a graph
struct Item {
  int32_t cont;
  int32_t kind;
  int32_t a, b, c;         // grid: x0, y0, y1   graph: r0, r1, -
  int32_t w;               // grid: strip width (32 scalar lanes, or 64 = 2 columns per lane)
};

// one CG solve (D-scheme: one continuum; coupled: all)
struct Group {
  int32_t cta_begin, cta_count;
  int32_t item_begin, item_count;
  int64_t maxit;
  double tol2;             // rtol^2
  int32_t cont_mask;       // continua solved by this group
  int32_t phase;           // groups of one phase run concurrently; phases run in order
};

// per-group device results of one step
struct GroupOut {
  int64_t iters;
  int32_t status;          // mc_status
  int32_t pad;
  double bb, rr;           // ||b||^2, final ||r||^2
  long long t0, t1;        // %globaltimer ns
};

struct SyncBlock {         // zeroed before every step launch
  unsigned long long arrive[MC_MAX_CONTINUA * kNSub * kCtrStride];
  unsigned long long phase_arrive;
  unsigned long long pad0[kCtrStride - 1];
  unsigned int finished;
  unsigned int pad[3];
};

struct StepParams {
  ContDev cont[MC_MAX_CONTINUA];
  Group grp[MC_MAX_CONTINUA];
  int32_t L, ngroups, nphases, coupled, total_ctas;
  int32_t gs;              // L/U schemes: transfer from continua of earlier phases at layer n
  int64_t N;               // padded global size
  // state and CG work vectors (global DOF space, padded)
  double* u[2];            // ping-pong state: u[cur] = p^{n-1}, u[cur^1] = iterate x
  double* r[2];
  double* p[2];
  double* q[2];
  // operator data
  const double* dinv;      // 1 / diag(K) (Jacobi; identical for both schemes, reading C14)
  const double* dsD;       // D-scheme shift  m/tau + boundary + sum_b sigma
  const double* dsC;       // coupled shift   m/tau + boundary
  const double* mtau;      // m / tau
  const double* F;         // time-constant source incl. Dirichlet terms
  const int32_t* cptr;     // coupling CSR over global rows [N+1]
  const int32_t* cidx;     // global column
  const double* cval;      // sigma
  const Item* items;
  double* partials;        // [2][kNPart][total_ctas]
  SyncBlock* sync;
  GroupOut* gout;          // [ngroups]
  int32_t* cur;            // device ping-pong index
  int32_t* fail;           // sticky failure flag (mc_run)
  mc_step_report* rep;     // report slot of this launch
  int32_t step_no;
  int32_t scheme;
};

// caller order <-> internal (chain) order of a graph continuum's state, perm[t] = caller index
cudaError_t launch_to_caller(double* dst, const double* src, const int32_t* perm, int64_t n, cudaStream_t s);
cudaError_t launch_from_caller(double* dst, const double* src, const int32_t* perm, int64_t n, cudaStream_t s);

// kernel launch (mc_kernels.cu)
cudaError_t launch_step(const StepParams* dparams, int total_ctas, cudaStream_t s);
cudaError_t step_kernel_occupancy(int* blocks_per_sm);

}  // namespace mc
