"""Plain Jacobi-preconditioned conjugate gradient — TEST INFRASTRUCTURE ONLY.

Textbook PCG (SPEC.md:184-192 cg_solve; the paper's solver is CG)
with the Jacobi preconditioner D^{-1} = 1/diag(K), written step by step:

    r0 = b - K x0,  z0 = D^{-1} r0,  p0 = z0
    loop: q = K p;  a = (r,z)/(p,q);  x += a p;  r -= a q
          stop at the first k with ||r_k||_2 <= rtol ||b||_2  (recursive residual, reading C13)
          z = D^{-1} r;  b = (r,z)_new/(r,z)_old;  p = z + b p
If b = 0 the solution is x = 0 after 0 iterations.
"""
from __future__ import annotations

import numpy as np


class CGBreakdown(RuntimeError):
    pass


class CGNoConvergence(RuntimeError):
    pass


def jacobi_pcg(K, b, x0=None, rtol=1e-12, maxit=None):
    """Returns (x, iterations)."""
    b = np.asarray(b, dtype=np.float64)
    n = len(b)
    x = np.zeros(n) if x0 is None else np.array(x0, dtype=np.float64)
    bnorm = np.linalg.norm(b)
    if bnorm == 0.0:
        return np.zeros(n), 0
    if maxit is None:
        maxit = 10 * n
    dinv = 1.0 / K.diagonal()
    r = b - K @ x
    if np.linalg.norm(r) <= rtol * bnorm:
        return x, 0
    z = dinv * r
    p = z.copy()
    rz = r @ z
    for k in range(1, maxit + 1):
        q = K @ p
        pq = p @ q
        if not pq > 0.0:
            raise CGBreakdown(f"p.q = {pq} at iteration {k}")
        a = rz / pq
        x = x + a * p
        r = r - a * q
        if np.linalg.norm(r) <= rtol * bnorm:
            return x, k
        z = dinv * r
        rz_new = r @ z
        p = z + (rz_new / rz) * p
        rz = rz_new
    raise CGNoConvergence(f"no convergence in {maxit} iterations")
