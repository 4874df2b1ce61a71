"""Oracle time stepping: coupled backward Euler and the decoupled D-scheme.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

coupled   Eq. ct-mc:  M (p^n - p^{n-1})/tau + A p^n = F
          =>  (M/tau + A) p^n = M/tau p^{n-1} + F.
D-scheme  Eq. si-mc with the D-split:
          A0 = blockdiag(A_11, ..., A_LL) = diag(D_a + sum_b Q_ab),  A1 = A - A0
          =>  (M/tau + A0) p^n = M/tau p^{n-1} + F - A1 p^{n-1},
          i.e. per continuum  (M_a/tau + D_a + sum_b Q_ab) p_a^n
                              = M_a/tau p_a^{n-1} + F_a + sum_b Q_ab p_b^{n-1}.
F is time-constant (C17).  Solves: SuperLU factorisation once per matrix (tau is
fixed), one back-solve per step; or the plain Jacobi-PCG of oracle.cg.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from .assemble import System
from . import cg as _cg


def split_D(sys: System):
    """A0 = block diagonal of A, A1 = A - A0."""
    A = sp.csr_matrix(sys.A).tocoo()
    blk = np.searchsorted(sys.offsets, A.row, side="right") - 1
    bcol = np.searchsorted(sys.offsets, A.col, side="right") - 1
    same = blk == bcol
    A0 = sp.csr_matrix((A.data[same], (A.row[same], A.col[same])), shape=A.shape)
    A1 = sp.csr_matrix((A.data[~same], (A.row[~same], A.col[~same])), shape=A.shape)
    return A0, A1


class _Solver:
    """x = K^{-1} b via SuperLU ('splu') or Jacobi-PCG ('cg', warm start x0)."""

    def __init__(self, K, method="splu", rtol=1e-13):
        self.K = sp.csc_matrix(K)
        self.method = method
        self.rtol = rtol
        self.iters = []
        if method == "splu":
            self.lu = spla.splu(self.K)
        elif method != "cg":
            raise ValueError(method)

    def solve(self, b, x0):
        if self.method == "splu":
            return self.lu.solve(b)
        x, it = _cg.jacobi_pcg(sp.csr_matrix(self.K), b, x0, rtol=self.rtol, maxit=10 * len(b) + 10)
        self.iters.append(it)
        return x


class Coupled:
    """Coupled backward-Euler stepper on the whole system (Eq. ct-mc)."""

    def __init__(self, sys: System, tau: float, method="splu"):
        self.sys, self.tau = sys, float(tau)
        K = sp.diags(sys.M / self.tau) + sys.A
        self.solver = _Solver(K, method)

    def step(self, u):
        b = self.sys.M / self.tau * u + self.sys.F
        return self.solver.solve(b, u)


class DScheme:
    """Decoupled D-scheme stepper (Eq. si-mc, D-split): L independent solves per step."""

    def __init__(self, sys: System, tau: float, method="splu"):
        self.sys, self.tau = sys, float(tau)
        self.A0, self.A1 = split_D(sys)
        K0 = sp.csr_matrix(sp.diags(sys.M / self.tau) + self.A0)
        self.solvers = []
        for a in range(sys.L):
            s = sys.block(a)
            self.solvers.append(_Solver(K0[s, s], method))

    def rhs(self, u):
        """b = M/tau p^{n-1} + F - A1 p^{n-1}: every coupling term from layer n-1."""
        return self.sys.M / self.tau * u + self.sys.F - self.A1 @ u

    def step(self, u):
        b = self.rhs(u)
        out = np.empty_like(u)
        for a in range(self.sys.L):
            s = self.sys.block(a)
            out[s] = self.solvers[a].solve(b[s], u[s])
        return out


def make_stepper(sys: System, scheme: str, tau: float, method="splu"):
    if scheme == "coupled":
        return Coupled(sys, tau, method)
    if scheme in ("D", "decoupled", "d"):
        return DScheme(sys, tau, method)
    raise ValueError(scheme)


def run(sys: System, scheme: str, tau: float, n_steps: int, method="splu", u0=None):
    """Trajectory [p^1, ..., p^n_steps] (full concatenated vectors)."""
    st = make_stepper(sys, scheme, tau, method)
    u = sys.u0.copy() if u0 is None else np.asarray(u0, dtype=np.float64).copy()
    out = []
    for _ in range(n_steps):
        u = st.step(u)
        out.append(u.copy())
    return out


def rel_error_percent(ref, cand):
    """e_h^n = ||p^n - p~^n|| / ||p^n|| x 100 %, Euclidean norm (C19)."""
    ref = np.asarray(ref)
    return 100.0 * np.linalg.norm(ref - np.asarray(cand)) / np.linalg.norm(ref)
