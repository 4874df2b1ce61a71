/* flux_pcg.c -- plain Jacobi-preconditioned CG on an operator in flux form.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): called from tests/, smoke()
 * and bench.py's cpu_baseline / --impl reference legs through oracle/fluxcg.py.
 * It shares no code with the CUDA path (paper_2209_01158_b200/csrc).
 *
 * Operator.  Eq. app-md written as a sum over two-point connections, unassembled
 * (reading C15):
 *
 *     (K x)_i = d_i x_i + sum_{e = (i, j)} t_e (x_i - x_j)
 *
 * An undirected edge e = (i, j, t_e) enters row i (neighbour j) and row j
 * (neighbour i).  d holds everything that is not a connection inside the solved
 * system: m/tau, Dirichlet half-cell faces (C3), wells, and in
 * the D-scheme the transfer row sums sum_b Q_ab 1.
 *
 * Solver.  Textbook Jacobi-PCG (the paper's solver is CG; SPEC.md:
 * 184-192 cg_solve), step by step in the order of oracle/cg.py:
 *
 *     r0 = b - K x0,  z0 = D^-1 r0,  p0 = z0,  D = diag(K) = d_i + sum_e t_e
 *     loop k = 1, 2, ...:  q = K p;  a = (r,z)/(p,q);  x += a p;  r -= a q
 *                          stop at the first k with ||r_k||_2 <= rtol ||b||_2  (C13)
 *                          z = D^-1 r;  beta = (r,z)_new/(r,z)_old;  p = z + beta p
 *     b = 0  =>  x = 0 after 0 iterations.
 *
 * Determinism.  Every row sums its connections in edge-input order; every dot
 * product is a sum of fixed 4096-row block partials added in block order, so the
 * result does not depend on the number of OpenMP threads.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORA_BLOCK 4096

typedef struct {
  int64_t n;
  double *d;     /* [n]   non-connection diagonal part                 */
  double *dg;    /* [n]   diag(K) = d_i + sum of the row's t_e          */
  int64_t *ptr;  /* [n+1] row i's connections are ptr[i] .. ptr[i+1]-1 */
  int64_t *col;  /* neighbour of each connection                       */
  double *t;     /* t_e of each connection                             */
} ora_op;

int ora_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

void ora_op_free(void *h) {
  ora_op *op = (ora_op *)h;
  if (!op) return;
  free(op->d);
  free(op->dg);
  free(op->ptr);
  free(op->col);
  free(op->t);
  free(op);
}

/* Build the row adjacency of n rows from ne undirected edges.  Returns NULL on an
 * out-of-range index or allocation failure. */
void *ora_op_create(int64_t n, const double *d, int64_t ne, const int64_t *ei, const int64_t *ej,
                    const double *et) {
  ora_op *op = (ora_op *)calloc(1, sizeof(ora_op));
  if (!op) return NULL;
  op->n = n;
  op->d = (double *)malloc((size_t)(n > 0 ? n : 1) * sizeof(double));
  op->dg = (double *)malloc((size_t)(n > 0 ? n : 1) * sizeof(double));
  op->ptr = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
  op->col = (int64_t *)malloc((size_t)(2 * ne > 0 ? 2 * ne : 1) * sizeof(int64_t));
  op->t = (double *)malloc((size_t)(2 * ne > 0 ? 2 * ne : 1) * sizeof(double));
  if (!op->d || !op->dg || !op->ptr || !op->col || !op->t) {
    ora_op_free(op);
    return NULL;
  }
  memcpy(op->d, d, (size_t)n * sizeof(double));
  for (int64_t e = 0; e < ne; ++e) {
    if (ei[e] < 0 || ei[e] >= n || ej[e] < 0 || ej[e] >= n) {
      ora_op_free(op);
      return NULL;
    }
    op->ptr[ei[e] + 1] += 1;
    op->ptr[ej[e] + 1] += 1;
  }
  for (int64_t i = 0; i < n; ++i) op->ptr[i + 1] += op->ptr[i];
  int64_t *fill = (int64_t *)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
  if (!fill) {
    ora_op_free(op);
    return NULL;
  }
  memcpy(fill, op->ptr, (size_t)n * sizeof(int64_t));
  for (int64_t e = 0; e < ne; ++e) {   /* edge-input order within every row */
    int64_t a = fill[ei[e]]++, b = fill[ej[e]]++;
    op->col[a] = ej[e];
    op->t[a] = et[e];
    op->col[b] = ei[e];
    op->t[b] = et[e];
  }
  free(fill);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    double s = op->d[i];
    for (int64_t k = op->ptr[i]; k < op->ptr[i + 1]; ++k) s += op->t[k];
    op->dg[i] = s;
  }
  return op;
}

/* y = K x */
void ora_op_apply(const void *h, const double *x, double *y) {
  const ora_op *op = (const ora_op *)h;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < op->n; ++i) {
    double s = op->d[i] * x[i];
    for (int64_t k = op->ptr[i]; k < op->ptr[i + 1]; ++k) s += op->t[k] * (x[i] - x[op->col[k]]);
    y[i] = s;
  }
}

void ora_op_diag(const void *h, double *out) {
  const ora_op *op = (const ora_op *)h;
  memcpy(out, op->dg, (size_t)op->n * sizeof(double));
}

/* sum_i u_i v_i  (w == NULL) or sum_i u_i w_i v_i, fixed block order */
static double dot(int64_t n, const double *u, const double *w, const double *v, double *part) {
  const int64_t nb = (n + ORA_BLOCK - 1) / ORA_BLOCK;
#pragma omp parallel for schedule(static)
  for (int64_t b = 0; b < nb; ++b) {
    const int64_t i1 = (b + 1) * ORA_BLOCK < n ? (b + 1) * ORA_BLOCK : n;
    double s = 0.0;
    for (int64_t i = b * ORA_BLOCK; i < i1; ++i) s += w ? u[i] * w[i] * v[i] : u[i] * v[i];
    part[b] = s;
  }
  double s = 0.0;
  for (int64_t b = 0; b < nb; ++b) s += part[b];
  return s;
}

/* Solve K x = b.  x holds x0 on entry, the solution on exit.
 * Returns the iteration count k >= 0; -1: no convergence within maxit; -2: breakdown
 * (p.q <= 0); -3: allocation failure.  *relres = ||r_k|| / ||b||. */
int64_t ora_pcg(const void *h, const double *b, double *x, double rtol, int64_t maxit, double *relres) {
  const ora_op *op = (const ora_op *)h;
  const int64_t n = op->n;
  const int64_t nb = (n + ORA_BLOCK - 1) / ORA_BLOCK;
  double *part = (double *)malloc((size_t)(nb > 0 ? nb : 1) * sizeof(double));
  double *r = (double *)malloc((size_t)(n > 0 ? n : 1) * sizeof(double));
  double *z = (double *)malloc((size_t)(n > 0 ? n : 1) * sizeof(double));
  double *p = (double *)malloc((size_t)(n > 0 ? n : 1) * sizeof(double));
  double *q = (double *)malloc((size_t)(n > 0 ? n : 1) * sizeof(double));
  double *dinv = (double *)malloc((size_t)(n > 0 ? n : 1) * sizeof(double));
  int64_t ret = -3;
  if (!part || !r || !z || !p || !q || !dinv) goto out;
  const double bnorm = sqrt(dot(n, b, NULL, b, part));
  *relres = 0.0;
  if (bnorm == 0.0) {
    memset(x, 0, (size_t)n * sizeof(double));
    ret = 0;
    goto out;
  }
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) dinv[i] = 1.0 / op->dg[i];
  ora_op_apply(op, x, q);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) r[i] = b[i] - q[i];
  double rn = sqrt(dot(n, r, NULL, r, part));
  *relres = rn / bnorm;
  if (rn <= rtol * bnorm) {
    ret = 0;
    goto out;
  }
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    z[i] = dinv[i] * r[i];
    p[i] = z[i];
  }
  double rz = dot(n, r, NULL, z, part);
  for (int64_t k = 1; k <= maxit; ++k) {
    ora_op_apply(op, p, q);
    const double pq = dot(n, p, NULL, q, part);
    if (!(pq > 0.0)) {
      ret = -2;
      goto out;
    }
    const double a = rz / pq;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
      x[i] = x[i] + a * p[i];
      r[i] = r[i] - a * q[i];
    }
    rn = sqrt(dot(n, r, NULL, r, part));
    *relres = rn / bnorm;
    if (rn <= rtol * bnorm) {
      ret = k;
      goto out;
    }
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) z[i] = dinv[i] * r[i];
    const double rz_new = dot(n, r, NULL, z, part);
    const double beta = rz_new / rz;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
    rz = rz_new;
  }
  ret = -1;
out:
  free(part);
  free(r);
  free(z);
  free(p);
  free(q);
  free(dinv);
  return ret;
}
