"""Oracle time stepping: coupled backward Euler and the decoupled D-scheme.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

L, U      the sequential schemes of PAPER.md:541-580 (SeqScheme).
coupled   Eq. ct-mc:  M (p^n - p^{n-1})/tau + A p^n = F
          =>  (M/tau + A) p^n = M/tau p^{n-1} + F.
D-scheme  Eq. si-mc with the D-split:
          A0 = blockdiag(A_11, ..., A_LL) = diag(D_a + sum_b Q_ab),  A1 = A - A0
          =>  (M/tau + A0) p^n = M/tau p^{n-1} + F - A1 p^{n-1},
          i.e. per continuum  (M_a/tau + D_a + sum_b Q_ab) p_a^n
                              = M_a/tau p_a^{n-1} + F_a + sum_b Q_ab p_b^{n-1}.
F is time-constant (C17).  Solves: SuperLU factorisation once per matrix (tau is
fixed), one back-solve per step (the CG steppers for sizes beyond SuperLU are in
oracle/fluxcg.py).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from .assemble import System


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
    """x = K^{-1} b for one solve: SuperLU factorisation of the assembled K, then
    iterative refinement x += K^{-1}(b - K x) with the residual evaluated in long
    double on the unassembled flux form (FluxForm), until the
    correction is below 1e-16 ||x||.  The result is the solution of the exact operator,
    not of its fp64-rounded assembly (reading C15).  (Where a factorisation is out of
    reach, oracle/fluxcg.py steps the same schemes with a plain C Jacobi-PCG.)"""

    def __init__(self, op, method="splu", rtol=1e-13, refine=True):
        if method != "splu":
            raise ValueError(f"{method}: the CG oracle is oracle.fluxcg")
        self.op = op
        self.refine = refine
        self.refinements = []
        self.K = sp.csc_matrix(op.tocsr())
        self.lu = spla.splu(self.K)

    def solve(self, b, x0):
        x = self.lu.solve(b)
        k = 0
        if self.refine and np.any(x):
            bl = np.asarray(b, dtype=np.longdouble)
            for k in range(1, 9):
                r = np.asarray(bl - self.op.apply(x, np.longdouble), dtype=np.float64)
                dx = self.lu.solve(r)
                x = x + dx
                if np.linalg.norm(dx) <= 1e-16 * np.linalg.norm(x):
                    break
        self.refinements.append(k)
        return x


class Coupled:
    """Coupled backward-Euler stepper on the whole system (Eq. ct-mc)."""

    def __init__(self, sys: System, tau: float, method="splu", refine=True):
        self.sys, self.tau = sys, float(tau)
        op = sys.flux.block_op(slice(0, int(sys.offsets[-1])), sys.M / self.tau, "coupled")
        self.solver = _Solver(op, method, refine=refine)

    def step(self, u):
        b = self.sys.M / self.tau * u + self.sys.F
        return self.solver.solve(b, u)


class DScheme:
    """Decoupled D-scheme stepper (Eq. si-mc, D-split): L independent solves per step."""

    def __init__(self, sys: System, tau: float, method="splu", refine=True):
        self.sys, self.tau = sys, float(tau)
        self.A0, self.A1 = split_D(sys)
        self.solvers = []
        for a in range(sys.L):
            op = sys.flux.block_op(sys.block(a), sys.M / self.tau, "D")
            self.solvers.append(_Solver(op, method, refine=refine))

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


class SeqScheme(DScheme):
    """L- / U-scheme: Eq. si-mc with A0 block lower- (L) or upper- (U)
    triangular once the continua are sorted by permeability k_1 < ... < k_L.  Written as
    what the triangular A0 means: the continua are solved one after another — L in
    ascending permeability, U in descending — and each solve takes the transfer from the
    continua already solved in this step at layer n, from the others at layer n-1:

        (M_a/tau + D_a + sum_b Q_ab) p_a^n = M_a/tau p_a^{n-1} + F_a
                                             + sum_{b before a} Q_ab p_b^n + sum_{b after a} Q_ab p_b^{n-1}

    `order_by_k` lists the continuum ids by ascending permeability."""

    def __init__(self, sys: System, tau: float, order_by_k, kind="U", method="splu", refine=True):
        super().__init__(sys, tau, method, refine)
        order = list(order_by_k)
        assert sorted(order) == list(range(sys.L))
        self.order = order if kind == "L" else order[::-1]

    def step(self, u):
        A = sp.csr_matrix(self.sys.A)
        new = u.copy()                      # continua solved so far hold layer n
        for a in self.order:
            s = self.sys.block(a)
            b = self.sys.M[s] / self.tau * u[s] + self.sys.F[s]
            for c in range(self.sys.L):
                if c != a:                  # -A_ac = Q_ac: layer n if c already solved
                    sc = self.sys.block(c)
                    b = b - A[s, sc] @ new[sc]
            new[s] = self.solvers[a].solve(b, u[s])
        return new


def make_stepper(sys: System, scheme: str, tau: float, method="splu", refine=True, order_by_k=None):
    if scheme == "coupled":
        return Coupled(sys, tau, method, refine)
    if scheme in ("D", "decoupled", "d"):
        return DScheme(sys, tau, method, refine)
    if scheme in ("L", "U"):
        if order_by_k is None:
            raise ValueError("L/U schemes need the continua ordered by permeability")
        return SeqScheme(sys, tau, order_by_k, scheme, method, refine)
    raise ValueError(scheme)


def run(sys: System, scheme: str, tau: float, n_steps: int, method="splu", u0=None, refine=True,
        order_by_k=None):
    """Trajectory [p^1, ..., p^n_steps] (full concatenated vectors)."""
    st = make_stepper(sys, scheme, tau, method, refine, order_by_k)
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
