/*
 * mc.h — C ABI of libmc: one time step of the multicontinuum flow system
 *
 *     M dp/dt + A p = F,   A = D + Q                         (Eq. app-mc)
 *
 * advanced either by the coupled backward-Euler scheme
 *
 *     (M/tau + A) p^n = M/tau p^{n-1} + F                    (Eq. ct-mc)
 *
 * or by the decoupled D-scheme (A0 = blockdiag(A), A1 = A - A0, the inter-continuum
 * transfer lagged to time layer n-1), one independent SPD solve per continuum:
 *
 *     (M_a/tau + D_a + sum_b Q_ab) p_a^n = M_a/tau p_a^{n-1} + F_a + sum_b Q_ab p_b^{n-1}
 *                                                            (Eq. si-mc, D-scheme)
 *
 * Every linear system is solved on the GPU by Jacobi-preconditioned CG (the paper's
 * solver is CG) in fp64, stopping at the first iterate whose recursive
 * residual satisfies ||r_k||_2 <= rtol ||b||_2 (reading C13), warm-started
 * from p^{n-1}.  All kernels are hand-written for sm_100a.
 *
 * Conventions
 *  - No exceptions cross this ABI; every call returns mc_status and mc_error_string()
 *    returns a message for the last failure on that context (continuum and step named).
 *  - Array arguments may be HOST or DEVICE pointers (unified addressing; the library
 *    inspects each pointer).  The library copies everything it keeps during the call,
 *    so the caller may free its arrays as soon as the call returns.  No pointer passed
 *    in is ever written, except the documented output arguments.
 *  - Indices are 0-based int32; counts are int64.  fp64 everywhere.
 *  - All device work is ordered on mc_options.stream (the caller's cudaStream_t, or the
 *    legacy default stream when NULL).
 *  - A context is not thread-safe; use one context per host thread.
 */
#ifndef MC_H
#define MC_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MC_ABI_VERSION 2
#define MC_MAX_CONTINUA 4

typedef struct mc_ctx mc_ctx;

typedef enum {
  MC_OK = 0,
  MC_ERR_ARG = 1,        /* invalid argument (range, sign, CSR/index structure, sizes)      */
  MC_ERR_STATE = 2,      /* call out of order (coupling before continuum, step before setup) */
  MC_ERR_NOMEM = 3,      /* device or host allocation failed                                 */
  MC_ERR_CUDA = 4,       /* a CUDA runtime call failed (message carries cudaGetErrorString)  */
  MC_ERR_NOCONV = 5,     /* a CG solve hit maxit; the state is NOT advanced    */
  MC_ERR_BREAKDOWN = 6   /* CG breakdown (p.q <= 0): operator not SPD                        */
} mc_status;

typedef enum {
  MC_GRID2D = 0,  /* d-dimensional continuum on a structured nx x ny grid of h x h cells
                     (PAPER.md:247-248), TPFA 5-point operator   */
  MC_GRAPH = 1    /* continuum given by its cells and symmetric two-point connections:
                     the (d-1)-dimensional fracture mesh or an
                     NLMC coarse operator                              */
} mc_kind;

typedef enum {
  MC_COUPLED = 0,      /* Eq. ct-mc: one CG solve over all continua per step            */
  MC_DECOUPLED_D = 1,  /* Eq. si-mc, D-scheme: one CG solve per continuum per step      */
  MC_DECOUPLED_L = 2,  /* L-scheme: continua solved in ascending permeability, each
                          taking the transfer from continua already solved at layer n
                          (block lower-triangular A0)                 */
  MC_DECOUPLED_U = 3   /* U-scheme: descending permeability (block upper-triangular A0,
                          PAPER.md:562-580); needs mc_set_permeability_order            */
} mc_scheme;

typedef struct {
  double tau;        /* time step tau > 0                                     */
  double rtol;       /* CG stop ||r_k|| <= rtol ||b||; <= 0 selects 1e-12 (BASELINE.json:5)   */
  int64_t maxit;     /* per solve; <= 0 selects min(10 N_solve, 2e6)                          */
  int32_t ctas;      /* persistent CTAs per step kernel; 0 = all co-resident (148 x occupancy) */
  int32_t device;    /* CUDA device ordinal                                                    */
  void* stream;      /* cudaStream_t for all work, NULL = legacy default stream               */
} mc_options;

/*
 * One continuum alpha.  Storage m_i = c_i |cell_i|; source
 * F_i = f_i |cell_i|; initial state p_alpha^0 = u0.
 *
 * MC_GRID2D: n = nx*ny cells, row-major (i = iy*nx + ix), |cell| = h^2.  Interior faces
 *   carry T = k|E|/d = k (|E| = d = h); with a per-cell k field the face
 *   value is the harmonic mean 2 k_i k_j / (k_i + k_j) (reading C2).  All outer faces
 *   are no-flow unless bc_left / bc_right = 1: then the left
 *   (ix = 0) / right (ix = nx-1) faces are Dirichlet faces with value g_left / g_right,
 *   half-cell transmissibility T_b = k_i h / (h/2) = 2 k_i (reading C3).
 * MC_GRAPH: n cells, |cell_i| = measure[i] (or measure_const); n_edges undirected
 *   connections (edge_i[e], edge_j[e]), 0 <= i,j < n, i != j, each pair at most once,
 *   with flux T_e (p_i - p_j).  T_e = edge_t[e] if edge_t != NULL,
 *   else T_e = k_e * edge_geom where k_e = k_const, or the harmonic mean of k[i], k[j]
 *   when k != NULL, and edge_geom = |E|/d.  dirichlet (optional): per cell, NaN = free,
 *   otherwise the cell is a fixed-value DOF: identity row with m = 0, F = g, u0 = g,
 *   and every connection / coupling touching it is eliminated into the free cell's
 *   diagonal and F (reading C12).
 * Scalars *_const are used when the corresponding pointer is NULL.
 */
typedef struct {
  mc_kind kind;
  int64_t n;
  const double* c;        double c_const;        /* storage coefficient c >= 0            */
  const double* k;        double k_const;        /* permeability k >= 0                   */
  const double* f;                               /* volumetric source, NULL = 0           */
  const double* u0;                              /* initial state, NULL = 0               */
  /* MC_GRID2D */
  int32_t nx, ny;
  double h;                                      /* cell edge length > 0                  */
  int32_t bc_left, bc_right;                     /* 0 = no-flow, 1 = Dirichlet            */
  double g_left, g_right;
  /* MC_GRAPH */
  const double* measure;  double measure_const;  /* |cell| > 0                            */
  int64_t n_edges;
  const int32_t* edge_i;
  const int32_t* edge_j;
  const double* edge_t;                          /* explicit T_e >= 0, or NULL            */
  double edge_geom;                              /* |E|/d when edge_t == NULL             */
  const double* dirichlet;                       /* NULL, or per cell NaN / fixed value   */
  double rtol;                                   /* this continuum's D-scheme CG tolerance;
                                                    <= 0: mc_options.rtol.  The coupled solve
                                                    uses the smallest over all continua.    */
  const double* well_q;                          /* NULL, or per cell well index q_w >= 0:
                                                    source f = q_w (p_w - p) (PAPER.md:834,
                                                    injection sign of SPEC.md:154), i.e.
                                                    q_w|cell| on the diagonal and
                                                    q_w p_w |cell| in F                     */
  double well_p;                                 /* p_w                                    */
  /* since ABI 2 — general symmetric operators such as the NLMC coarse system
     (PAPER.md:667-729), whose transmissibilities may have either sign: */
  const double* diag_extra;                      /* MC_GRAPH: NULL, or per cell a term added
                                                    to the diagonal of A (any sign)          */
  int32_t signed_edges;                          /* MC_GRAPH: 1 = edge_t may be negative    */
} mc_continuum_desc;

/*
 * Transfer between continua a != b: Q_ab has entries q_{i j} = sigma_e at
 * (i = i_a[e], j = j_b[e]), e < nnz; Q_ba = Q_ab^T.
 * The library adds sum_j q_ij to diagonal row i of a and sum_i q_ij to row j of b and
 * uses -q_ij off the diagonal.  i_a == NULL (j_b == NULL) means the
 * identity map i = e (j = e) — co-located continua.  sigma == NULL
 * uses sigma_const.  scale_by_measure = 1 multiplies sigma by |cell_i| of continuum a
 * (co-located field coefficient integrated over the cell, reading C9).  Several
 * couplings may name the same pair; entries with the same (i, j) add.
 */
typedef struct {
  int32_t a, b;
  int64_t nnz;
  const int32_t* i_a;
  const int32_t* j_b;
  const double* sigma;  double sigma_const;     /* sigma >= 0                             */
  int32_t scale_by_measure;
  int32_t signed_sigma;                          /* since ABI 2: 1 = sigma may be negative
                                                    (NLMC between-continuum entries)        */
} mc_coupling_desc;

/* Kernel path of a continuum in a step (mc_step_report.paths; informational). */
enum { MC_PATH_STREAM = 0,            /* grid strips / CSR rows streamed from HBM every iteration   */
       MC_PATH_ELL_STREAM = 1,        /* fracture network, 64-row ELL chunks streamed               */
       MC_PATH_ELL_RESIDENT = 2,      /* fracture network resident in shared memory (small network) */
       MC_PATH_BJ_RESIDENT = 3,       /* block-Jacobi, resident                                     */
       MC_PATH_BJ_STREAM = 4 };       /* block-Jacobi, two streaming passes                         */

/* Per-step report.  For MC_COUPLED there is one solve (nsolves = 1, index 0). */
typedef struct {
  int32_t step;                        /* time layer n reached (1-based)                  */
  int32_t scheme;                      /* mc_scheme                                        */
  int32_t nsolves;
  int32_t status;                      /* mc_status of the step                            */
  int32_t failed_solve;                /* -1, or the solve index that failed               */
  int32_t paths;                       /* kernel path of continuum a in bits 4a..4a+3 (MC_PATH_*): which
                                          pass streamed its rows, i.e. which byte model applies */
  int64_t iters[MC_MAX_CONTINUA];      /* CG iterations of each solve                      */
  double relres[MC_MAX_CONTINUA];      /* final recursive ||r|| / ||b|| (0 when b = 0)     */
  double bnorm[MC_MAX_CONTINUA];       /* ||b||_2 of each solve                            */
  double ms_solve[MC_MAX_CONTINUA];    /* device time of each solve (globaltimer)          */
  double ms;                           /* device time of the whole step kernel             */
} mc_step_report;

/* Create a context for n_continua (1..MC_MAX_CONTINUA) continua. */
mc_status mc_create(mc_ctx** out, int32_t n_continua, const mc_options* opt);

/* Define continuum alpha (0 <= alpha < n_continua).  May be called once per alpha. */
mc_status mc_set_continuum(mc_ctx* ctx, int32_t alpha, const mc_continuum_desc* desc);

/* Add a transfer Q_ab.  All continua must be set first (else MC_ERR_STATE). */
mc_status mc_set_coupling(mc_ctx* ctx, const mc_coupling_desc* desc);

/* CG preconditioner (the paper defers solver comparison,
 * PAPER.md:852).  MC_PRECOND_JACOBI (default): D^{-1} = 1/diag(K) (reading C14).
 * MC_PRECOND_BLOCK: for graph continua with <= 4 connections per cell and uniform T
 * (fracture networks): the cells are renumbered in chain order and M = the tridiagonal
 * part of K on every 64-cell block (cells i, i+1 of a block connected along the network),
 * solved exactly; other continua keep Jacobi.  Same solution, fewer iterations; two
 * reductions per iteration instead of one.  Must precede mc_set_continuum. */
typedef enum { MC_PRECOND_JACOBI = 0, MC_PRECOND_BLOCK = 1 } mc_precond;
mc_status mc_set_preconditioner(mc_ctx* ctx, int32_t kind);

/* Order of the continua by ascending permeability k_1 < k_2 < ...:
 * order[0] is the least permeable.  Required before MC_DECOUPLED_L / MC_DECOUPLED_U. */
mc_status mc_set_permeability_order(mc_ctx* ctx, const int32_t* order);

/* Advance one time layer by `scheme` (any mc_scheme). */
mc_status mc_step(mc_ctx* ctx, int32_t scheme, mc_step_report* rep);

/* Advance one time layer by the D-scheme / the coupled scheme.  Blocks until the step
 * completed; fills *rep (may be NULL).  On MC_ERR_NOCONV / MC_ERR_BREAKDOWN the state is
 * left at p^{n-1}. */
mc_status mc_step_decoupled(mc_ctx* ctx, mc_step_report* rep);
mc_status mc_step_coupled(mc_ctx* ctx, mc_step_report* rep);

/* n_steps steps of `scheme` (the time loop of Eq. ct-mc / si-mc).
 * Coupled, L and U steps, and D steps once the D-scheme's CTA plan is fixed, are enqueued
 * back to back on mc_options.stream: nothing is read back between them (reports, the
 * ping-pong index and the failure flag stay on the device) and the host synchronises once
 * per batch of 256 steps.  The D-scheme's plan (how the CTAs are split between the
 * concurrent solves) follows the previous step's iteration counts until every solve has
 * iterated once, at most the first 3 D steps of a context; those planning steps complete
 * one at a time, exactly as mc_step runs them.  mc_run and a sequence of mc_step calls
 * therefore give bitwise the same states and iteration counts.
 * reps: NULL or n_steps reports.  snapshots: NULL, or n_steps * n_continua pointers
 * (host or device), snapshots[s * n_continua + a] receives p_a after step s
 * (stream-ordered copies; contents undefined from the first failed step on).
 * Stops advancing at the first failed step (later steps are no-ops on the device, their
 * reports say MC_ERR_STATE); the state is the one before the failed step. */
mc_status mc_run(mc_ctx* ctx, int32_t scheme, int32_t n_steps, mc_step_report* reps,
                 double* const* snapshots);

/* Copy the current state p_a (n_a doubles) to / from dst / src (host or device). */
mc_status mc_get_state(mc_ctx* ctx, int32_t alpha, double* dst);
mc_status mc_set_state(mc_ctx* ctx, int32_t alpha, const double* src);

/* Sizes: n_a of continuum alpha (or the total when alpha < 0). */
int64_t mc_size(const mc_ctx* ctx, int32_t alpha);

/* CUDA-event time (ms) of the last step kernel launch, measured on mc_options.stream. */
mc_status mc_last_kernel_ms(mc_ctx* ctx, double* ms_out);

mc_status mc_destroy(mc_ctx* ctx);

/* Last error message of ctx (or of the last failed mc_create when ctx == NULL). */
const char* mc_error_string(const mc_ctx* ctx);

int32_t mc_abi_version(void);

/* ------------------------------------------------------------------------------------
 * NLMC multiscale space (§4.1, :591-729).
 *
 * Coarse cells K_j: the fine grid continua (all MC_GRID2D continua of the context share
 * one nx x ny grid) split into nHx x nHy blocks; K_j^alpha = the cells of continuum
 * alpha in K_j.  A graph continuum's cell belongs to the block of its host grid cell
 * (host[alpha][cell] = iy*nx + ix); every connected piece of a graph continuum inside
 * one block is its own coarse DOF (reading C30).  K_i^+ = K_i plus `oversample` block
 * layers, clipped.
 *
 * For every coarse cell i and every coarse DOF (i, beta) the basis psi^{i,beta} solves
 * Eq. eq:basis: the fine coupled operator D + Q on the cells of K_i^+
 * (zero Dirichlet outside) with the coarse-mean constraints
 * (1/|K_j^alpha|) int psi_alpha = delta_ij delta_alpha beta.  On the
 * GPU: one CTA per K_i^+, banded Cholesky of D + Q in a bandwidth-minimising order, the
 * Schur complement C (D+Q)^{-1} C^T, its dense Cholesky, psi = (D+Q)^{-1} C^T S^{-1} e.
 * Coarse system (Eq. app-nlmc): Abar = Dbar + Qbar + Wbar with Dbar = R D R^T in flux
 * form (reading C32), Qbar, Wbar (well terms), Mbar, Fbar aggregated over K_j^alpha
 * (reading C31); u0bar = measure-weighted means.
 *
 * The fine context must have its continua and couplings set and no step taken yet (the
 * build reads the setup data); it is unchanged by the build.  The build runs on the
 * context's device, is synchronous, and keeps its outputs in the mc_nlmc handle (the
 * bases on the device) until mc_nlmc_destroy.  On failure *out is NULL and
 * mc_error_string(fine) says why.  Graph continua with fixed
 * (Dirichlet) cells are not supported (MC_ERR_ARG).  A K_i^+ whose restricted operator
 * is singular (pure no-flow, K_i^+ = whole domain, no transfer sink) fails with
 * MC_ERR_ARG naming i.
 */
typedef struct mc_nlmc mc_nlmc;

typedef struct {
  int32_t nHx, nHy;                              /* coarse blocks; nx % nHx == ny % nHy == 0 */
  int32_t oversample;                            /* m >= 0 block layers                      */
  const int32_t* host[MC_MAX_CONTINUA];          /* MC_GRAPH continua: host grid cell of each
                                                    cell (host or device); NULL for grids    */
} mc_nlmc_desc;

mc_status mc_nlmc_build(mc_ctx* fine, const mc_nlmc_desc* desc, mc_nlmc** out);

/* Sizes: coarse DOFs per continuum (n_alpha[MC_MAX_CONTINUA], unused = 0), Abar nonzeros,
 * fine DOFs.  Coarse DOFs are numbered continuum-major, then by coarse cell, then piece. */
mc_status mc_nlmc_sizes(const mc_nlmc* nl, int64_t* n_alpha, int64_t* nnz, int64_t* n_fine);

/* Coarse system, host or device output arrays: Abar in CSR (rowptr[n+1], col[nnz],
 * val[nnz], rows sorted by column), Mbar[n], Fbar[n], u0bar[n]; key[3n] = (continuum,
 * coarse cell, piece) of each coarse DOF; fine_dof[n_fine] = coarse DOF of each fine
 * DOF (fine DOFs: the context's continua concatenated in caller numbering).  Any
 * output pointer may be NULL. */
mc_status mc_nlmc_get(const mc_nlmc* nl, int32_t* rowptr, int32_t* col, double* val, double* mass,
                      double* rhs, double* u0, int32_t* key, int32_t* fine_dof);

/* Basis psi^{r} of coarse DOF r as a fine vector (n_fine doubles, zero outside K_i^+). */
mc_status mc_nlmc_basis(const mc_nlmc* nl, int64_t r, double* psi);

/* Device time (ms) of the basis kernel and of the projection kernel of the build. */
mc_status mc_nlmc_times(const mc_nlmc* nl, double* ms_basis, double* ms_project);

/* Cost model of the build: fp64 operations of the basis kernel (banded Cholesky,
 * substitutions and Schur complement of Eq. eq:basis over all K_i^+) and
 * the device bytes that hold the bases (per-region sparse storage + window maps). */
mc_status mc_nlmc_cost(const mc_nlmc* nl, double* flops_basis, double* bytes_bases);

const char* mc_nlmc_error_string(const mc_nlmc* nl);
mc_status mc_nlmc_destroy(mc_nlmc* nl);


#ifdef __cplusplus
}
#endif
#endif /* MC_H */
