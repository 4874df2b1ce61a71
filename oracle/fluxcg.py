"""Binding of oracle/flux_pcg.c (plain Jacobi-PCG on the flux-form operator, OpenMP)
and the time steppers built on it -- TEST INFRASTRUCTURE ONLY (oracle/__init__.py).

Where a sparse factorisation is out of reach (config 2's coupled system, config 4's
16.6M-row fracture network and 67M-cell matrix: SURVEY.md §8(d) oracle table), the
oracle solves every step's systems with CG to a recursive relative residual of 1e-13
(SURVEY.md §8(c) "Otherwise it uses CG to a recursive relres of 1e-13 with warm start").

Steppers (same equations as oracle/schemes.py, evaluated from the flux form only, so
nothing of size nnz(A) is ever assembled):
  coupled   Eq. ct-mc:  (M/tau + A) p^n = M/tau p^{n-1} + F
  D-scheme  Eq. si-mc, D-split, per continuum
            (M_a/tau + D_a + sum_b Q_ab) p_a^n = M_a/tau p_a^{n-1} + F_a + sum_b Q_ab p_b^{n-1}

The C library is compiled on first use (gcc -O2 -fopenmp -ffp-contract=off) into
oracle/liboracle_pcg.so; `__graft_entry__.build()` compiles it too.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "flux_pcg.c")
LIB = os.path.join(HERE, "liboracle_pcg.so")
CFLAGS = ["-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-std=c11"]

_lib = None


def build(force=False) -> str:
    """Compile flux_pcg.c (stale-checked).  Returns the library path."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        tmp = LIB + f".{os.getpid()}.tmp"
        subprocess.run(["gcc", *CFLAGS, SRC, "-o", tmp, "-lm"], check=True)
        os.replace(tmp, LIB)
    return LIB


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        L.ora_op_create.restype = C.c_void_p
        L.ora_op_create.argtypes = [C.c_int64, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]
        L.ora_op_free.argtypes = [C.c_void_p]
        L.ora_op_apply.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.ora_op_diag.argtypes = [C.c_void_p, C.c_void_p]
        L.ora_pcg.restype = C.c_int64
        L.ora_pcg.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_int64, C.POINTER(C.c_double)]
        L.ora_threads.restype = C.c_int
        _lib = L
    return _lib


def threads() -> int:
    return int(lib().ora_threads())


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p)


class CGBreakdown(RuntimeError):
    pass


class CGNoConvergence(RuntimeError):
    pass


class FluxOp:
    """K x = d x + sum_e t_e (x_i - x_j) on n rows (C library handle)."""

    def __init__(self, n, d, ei, ej, et):
        self.n = int(n)
        self._keep = [np.ascontiguousarray(d, dtype=np.float64)]
        ei = np.ascontiguousarray(ei, dtype=np.int64)
        ej = np.ascontiguousarray(ej, dtype=np.int64)
        et = np.ascontiguousarray(et, dtype=np.float64)
        assert len(self._keep[0]) == self.n and len(ei) == len(ej) == len(et)
        self.h = lib().ora_op_create(self.n, _ptr(self._keep[0]), len(ei), _ptr(ei), _ptr(ej), _ptr(et))
        if not self.h:
            raise ValueError("ora_op_create: index out of range or out of memory")
        self.iters = []

    def apply(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty(self.n)
        lib().ora_op_apply(self.h, _ptr(x), _ptr(y))
        return y

    def diagonal(self):
        out = np.empty(self.n)
        lib().ora_op_diag(self.h, _ptr(out))
        return out

    def solve(self, b, x0, rtol=1e-13, maxit=None):
        """Jacobi-PCG from x0; returns x.  Iteration count appended to self.iters."""
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.array(x0, dtype=np.float64, copy=True)
        if maxit is None:
            maxit = 10 * self.n + 10
        rr = C.c_double(0.0)
        k = lib().ora_pcg(self.h, _ptr(b), _ptr(x), float(rtol), int(maxit), C.byref(rr))
        if k == -2:
            raise CGBreakdown("p.q <= 0")
        if k == -1:
            raise CGNoConvergence(f"no convergence in {maxit} iterations (relres {rr.value:.3e})")
        if k < 0:
            raise MemoryError("ora_pcg")
        self.iters.append(int(k))
        self.relres = rr.value
        return x

    def close(self):
        if self.h:
            lib().ora_op_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def block_op(flux, sl, mtau, scheme) -> FluxOp:
    """FluxOp of one solve: `scheme` 'coupled' (whole system, every connection) or 'D'
    (the A0 block `sl`: its own connections; transfer connections as row sums on the
    diagonal)."""
    n, ei, ej, et, d = flux.block_edges(sl, mtau, scheme)
    return FluxOp(n, d, ei, ej, et)


class CoupledCG:
    """Coupled backward Euler (Eq. ct-mc) with the C Jacobi-PCG."""

    def __init__(self, sys_, tau, rtol=1e-13):
        self.sys, self.tau, self.rtol = sys_, float(tau), rtol
        N = int(sys_.offsets[-1])
        self.op = block_op(sys_.flux, slice(0, N), sys_.M / self.tau, "coupled")

    def step(self, u):
        b = self.sys.M / self.tau * u + self.sys.F
        return self.op.solve(b, u, self.rtol)


class DSchemeCG:
    """D-scheme (Eq. si-mc, D-split) with the C Jacobi-PCG per continuum.  `rtols`:
    one tolerance per continuum (default 1e-13 each)."""

    def __init__(self, sys_, tau, rtols=None):
        self.sys, self.tau = sys_, float(tau)
        self.rtols = list(rtols) if rtols is not None else [1e-13] * sys_.L
        mt = sys_.M / self.tau
        self.ops = [block_op(sys_.flux, sys_.block(a), mt, "D") for a in range(sys_.L)]

    def rhs(self, u):
        """b = M/tau p^{n-1} + F + (transfer from layer n-1)."""
        return self.sys.M / self.tau * u + self.sys.F + self.sys.flux.lagged_transfer(u)

    def step(self, u):
        b = self.rhs(u)
        out = np.empty_like(u)
        for a in range(self.sys.L):
            s = self.sys.block(a)
            out[s] = self.ops[a].solve(b[s], u[s], self.rtols[a])
        return out

    @property
    def iters(self):
        return [op.iters for op in self.ops]


def run(sys_, scheme, tau, n_steps, u0=None, rtols=None, callback=None):
    """Trajectory [p^1, ..., p^n_steps] with the CG steppers ('D' or 'coupled').
    callback(n, u) is called after every step (e.g. to compare and drop states)."""
    st = DSchemeCG(sys_, tau, rtols) if scheme == "D" else CoupledCG(sys_, tau, min(rtols or [1e-13]))
    u = sys_.u0.copy() if u0 is None else np.asarray(u0, dtype=np.float64).copy()
    out = []
    for n in range(n_steps):
        u = st.step(u)
        if callback is None:
            out.append(u.copy())
        else:
            callback(n + 1, u)
    return out, st
