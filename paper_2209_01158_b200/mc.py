"""Thin ctypes binding of libmc (include/mc.h) — argument marshalling only.

Every step of the hot path runs in the sm_100a kernels of ``csrc/``; this module
only mirrors the C structs, loads ``libmc.so`` (failing loudly if it is missing —
there is no CPU fallback) and converts a generator scenario (``inputs/``) into
the ABI's physical-input descriptors.  PyTorch provides device memory and the
CUDA stream.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmc.so")

MC_OK, MC_ERR_ARG, MC_ERR_STATE, MC_ERR_NOMEM, MC_ERR_CUDA, MC_ERR_NOCONV, MC_ERR_BREAKDOWN = range(7)
MC_GRID2D, MC_GRAPH = 0, 1
MC_COUPLED, MC_DECOUPLED_D, MC_DECOUPLED_L, MC_DECOUPLED_U = 0, 1, 2, 3
SCHEMES = {"coupled": MC_COUPLED, "D": MC_DECOUPLED_D, "L": MC_DECOUPLED_L, "U": MC_DECOUPLED_U}
MC_MAX_CONTINUA = 4
STATUS_NAMES = {0: "MC_OK", 1: "MC_ERR_ARG", 2: "MC_ERR_STATE", 3: "MC_ERR_NOMEM", 4: "MC_ERR_CUDA",
                5: "MC_ERR_NOCONV", 6: "MC_ERR_BREAKDOWN"}

_d = C.c_double
_i32 = C.c_int32
_i64 = C.c_int64
_pd = C.POINTER(C.c_double)
_pi = C.POINTER(C.c_int32)


class mc_options(C.Structure):
    _fields_ = [("tau", _d), ("rtol", _d), ("maxit", _i64), ("ctas", _i32), ("device", _i32),
                ("stream", C.c_void_p)]


class mc_continuum_desc(C.Structure):
    _fields_ = [("kind", _i32), ("n", _i64),
                ("c", _pd), ("c_const", _d), ("k", _pd), ("k_const", _d), ("f", _pd), ("u0", _pd),
                ("nx", _i32), ("ny", _i32), ("h", _d), ("bc_left", _i32), ("bc_right", _i32),
                ("g_left", _d), ("g_right", _d),
                ("measure", _pd), ("measure_const", _d), ("n_edges", _i64), ("edge_i", _pi),
                ("edge_j", _pi), ("edge_t", _pd), ("edge_geom", _d), ("dirichlet", _pd), ("rtol", _d),
                ("well_q", _pd), ("well_p", _d), ("diag_extra", _pd), ("signed_edges", _i32)]


class mc_coupling_desc(C.Structure):
    _fields_ = [("a", _i32), ("b", _i32), ("nnz", _i64), ("i_a", _pi), ("j_b", _pi), ("sigma", _pd),
                ("sigma_const", _d), ("scale_by_measure", _i32), ("signed_sigma", _i32)]


class mc_nlmc_desc(C.Structure):
    _fields_ = [("nHx", _i32), ("nHy", _i32), ("oversample", _i32), ("host", C.c_void_p * MC_MAX_CONTINUA)]


class mc_step_report(C.Structure):
    _fields_ = [("step", _i32), ("scheme", _i32), ("nsolves", _i32), ("status", _i32),
                ("failed_solve", _i32), ("paths", _i32), ("iters", _i64 * MC_MAX_CONTINUA),
                ("relres", _d * MC_MAX_CONTINUA), ("bnorm", _d * MC_MAX_CONTINUA),
                ("ms_solve", _d * MC_MAX_CONTINUA), ("ms", _d)]

    def as_dict(self):
        k = self.nsolves
        return dict(step=self.step, scheme=self.scheme, status=self.status, failed_solve=self.failed_solve,
                    iters=list(self.iters[:k]), relres=list(self.relres[:k]), bnorm=list(self.bnorm[:k]),
                    ms_solve=list(self.ms_solve[:k]), ms=self.ms,
                    paths=[(self.paths >> (4 * a)) & 15 for a in range(MC_MAX_CONTINUA)])


EXPORTS = ["mc_create", "mc_set_continuum", "mc_set_coupling", "mc_step_decoupled", "mc_step_coupled",
           "mc_step", "mc_set_permeability_order", "mc_set_preconditioner",
           "mc_run", "mc_get_state", "mc_set_state", "mc_size", "mc_last_kernel_ms", "mc_destroy",
           "mc_error_string", "mc_abi_version", "mc_nlmc_build", "mc_nlmc_sizes", "mc_nlmc_get",
           "mc_nlmc_basis", "mc_nlmc_times", "mc_nlmc_cost", "mc_nlmc_error_string", "mc_nlmc_destroy"]

_lib = None


def load(path: str | None = None):
    """Load libmc.so (or $MC_LIB, a tuning variant); raises (no fallback) when missing."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or os.environ.get("MC_LIB") or LIB_PATH
    if not os.path.exists(path):
        raise RuntimeError(f"libmc.so not found at {path}: build it with "
                           "`python -m paper_2209_01158_b200.build` (there is no CPU fallback)")
    lib = C.CDLL(path)
    P = C.c_void_p
    lib.mc_create.argtypes = [C.POINTER(P), _i32, C.POINTER(mc_options)]
    lib.mc_set_continuum.argtypes = [P, _i32, C.POINTER(mc_continuum_desc)]
    lib.mc_set_coupling.argtypes = [P, C.POINTER(mc_coupling_desc)]
    lib.mc_step_decoupled.argtypes = [P, C.POINTER(mc_step_report)]
    lib.mc_step_coupled.argtypes = [P, C.POINTER(mc_step_report)]
    lib.mc_step.argtypes = [P, _i32, C.POINTER(mc_step_report)]
    lib.mc_set_permeability_order.argtypes = [P, C.c_void_p]
    lib.mc_set_preconditioner.argtypes = [P, _i32]
    lib.mc_run.argtypes = [P, _i32, _i32, C.POINTER(mc_step_report), C.POINTER(C.c_void_p)]
    lib.mc_get_state.argtypes = [P, _i32, C.c_void_p]
    lib.mc_set_state.argtypes = [P, _i32, C.c_void_p]
    lib.mc_size.argtypes = [P, _i32]
    lib.mc_size.restype = _i64
    lib.mc_last_kernel_ms.argtypes = [P, _pd]
    lib.mc_destroy.argtypes = [P]
    lib.mc_error_string.argtypes = [P]
    lib.mc_error_string.restype = C.c_char_p
    lib.mc_abi_version.restype = _i32
    lib.mc_nlmc_build.argtypes = [P, C.POINTER(mc_nlmc_desc), C.POINTER(P)]
    lib.mc_nlmc_sizes.argtypes = [P, C.POINTER(_i64), C.POINTER(_i64), C.POINTER(_i64)]
    lib.mc_nlmc_get.argtypes = [P] + [P] * 8
    lib.mc_nlmc_basis.argtypes = [P, _i64, P]
    lib.mc_nlmc_times.argtypes = [P, _pd, _pd]
    lib.mc_nlmc_cost.argtypes = [P, _pd, _pd]
    lib.mc_nlmc_error_string.argtypes = [P]
    lib.mc_nlmc_error_string.restype = C.c_char_p
    lib.mc_nlmc_destroy.argtypes = [P]
    for name in EXPORTS:
        if name not in ("mc_size", "mc_error_string", "mc_abi_version", "mc_nlmc_error_string"):
            getattr(lib, name).restype = _i32
    _lib = lib
    return lib


class MCError(RuntimeError):
    def __init__(self, status, msg, report=None):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status
        self.report = report


def permeability_order(scn):
    """Continuum ids by ascending permeability: the scenario's k
    (geometric mean of a k field), the fracture's k_f, NLMC k_scale (marshalling of a
    physical description, the order itself is a caller input of the ABI)."""
    if "korder" in scn:
        return list(scn["korder"])
    if scn["kind"] == "fine":
        ks = []
        for c in scn["continua"]:
            k = c["k"]
            ks.append(float(np.exp(np.mean(np.log(k)))) if np.ndim(k) else float(k))
    elif scn["kind"] == "nlmc":
        ks = [float(np.mean(scn["within"][a][2])) for a in range(2)]
    else:
        return None
    return [int(a) for a in np.argsort(ks, kind="stable")]


def _ptr(a, ctype=_pd):
    """Pointer to a torch tensor / numpy array (host or device), or NULL."""
    if a is None:
        return C.cast(None, ctype)
    if hasattr(a, "data_ptr"):
        return C.cast(C.c_void_p(a.data_ptr()), ctype)
    return a.ctypes.data_as(ctype)


class Problem:
    """A libmc context built from a generator scenario (inputs.make / make_fine / make_nlmc).

    The physical inputs are uploaded to device tensors with PyTorch and handed to
    mc_set_continuum / mc_set_coupling; the library derives every operator array on
    its own.
    """

    def __init__(self, scn, tau=None, rtol=1e-12, maxit=0, ctas=0, device=0, stream=None,
                 host_inputs=False, rtols=None, precond="jacobi"):
        """rtols: optional per-continuum CG tolerances (D-scheme), default rtol for all.
        precond: "jacobi" (default, the north star's) or "block" (mc_set_preconditioner)."""
        import torch
        self.lib = load()
        self.torch = torch
        self.scn = scn
        self.tau = float(scn["T"] / scn["NT"] if tau is None else tau)
        self.device = torch.device("cuda", device)
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        self.stream = stream
        self._keep = []
        opt = mc_options(tau=self.tau, rtol=rtol, maxit=maxit, ctas=ctas, device=device,
                         stream=C.c_void_p(stream.cuda_stream))
        self.ctx = C.c_void_p()
        self.host_inputs = host_inputs
        conts, cpls = self._descs(scn)
        self.L = len(conts)
        if rtols is not None:
            for d, t in zip(conts, rtols):
                d.rtol = float(t)
        self._check(self.lib.mc_create(C.byref(self.ctx), self.L, C.byref(opt)), create=True)
        self._check(self.lib.mc_set_preconditioner(self.ctx, {"jacobi": 0, "block": 1}[precond]))
        for a, d in enumerate(conts):
            self._check(self.lib.mc_set_continuum(self.ctx, a, C.byref(d)))
        for d in cpls:
            self._check(self.lib.mc_set_coupling(self.ctx, C.byref(d)))
        self._keep = []
        self.sizes = [int(self.lib.mc_size(self.ctx, a)) for a in range(self.L)]
        self.korder = permeability_order(scn)
        if self.korder is not None:
            arr = np.asarray(self.korder, dtype=np.int32)
            self._check(self.lib.mc_set_permeability_order(self.ctx, arr.ctypes.data_as(C.c_void_p)))

    # ------------------------------------------------------------------ marshalling
    def _arr(self, x, dtype):
        a = np.ascontiguousarray(np.asarray(x), dtype=dtype)
        if self.host_inputs:
            self._keep.append(a)
            return a
        t = self.torch.from_numpy(a).to(self.device)
        self._keep.append(t)
        return t

    def _descs(self, scn):
        conts, cpls = [], []
        if scn["kind"] == "fine":
            n, h = scn["n"], scn["h"]
            fr = scn["fracture"]
            for c in scn["continua"]:
                d = mc_continuum_desc()
                if c["kind"] == "grid":
                    d.kind, d.n, d.nx, d.ny, d.h = MC_GRID2D, n * n, n, n, h
                    if np.ndim(c["k"]) == 0:
                        d.k_const = float(c["k"])
                    else:
                        d.k = _ptr(self._arr(c["k"], np.float64))
                    d.c_const = float(c["c"])
                    if c["dirichlet"] is not None:
                        gL, gR = c["dirichlet"]
                        if gL is not None:
                            d.bc_left, d.g_left = 1, float(gL)
                        if gR is not None:
                            d.bc_right, d.g_right = 1, float(gR)
                else:
                    e = np.asarray(fr["edges"]).reshape(-1, 2)
                    d.kind, d.n = MC_GRAPH, len(fr["cells"])
                    d.c_const, d.k_const = float(c["c"]), float(c["k"])
                    d.measure_const = h                      # |iota| = h (reading C1)
                    d.n_edges = len(e)
                    d.edge_i = _ptr(self._arr(e[:, 0], np.int32), _pi)
                    d.edge_j = _ptr(self._arr(e[:, 1], np.int32), _pi)
                    d.edge_geom = 1.0 / h                    # |E|/d, |E| = 1, d = h (reading C7)
                if "well_q" in c:                            # wells, paper analogue
                    d.well_q = _ptr(self._arr(c["well_q"], np.float64))
                    d.well_p = float(c["well_p"])
                if c.get("u0", 0.0) != 0.0:
                    nn = d.n
                    d.u0 = _ptr(self._arr(np.full(nn, float(c["u0"])), np.float64))
                conts.append(d)
            for cp in scn["couplings"]:
                d = mc_coupling_desc(a=cp["a"], b=cp["b"])
                if cp["type"] == "embedded":
                    d.nnz = len(fr["cells"])
                    d.i_a = _ptr(self._arr(fr["cells"], np.int32), _pi)    # host cell of fracture cell e
                    d.sigma = _ptr(self._arr(cp["sigma"], np.float64))
                else:
                    d.nnz = n * n
                    d.sigma_const = float(cp["sigma"])
                    d.scale_by_measure = 1                   # sigma_12 |cell| (reading C9)
                cpls.append(d)
        elif scn["kind"] == "nlmc":
            nb = scn["nc"] ** 2
            for a in range(2):
                i, j, t = scn["within"][a]
                mask, g = scn["dirichlet"][a]
                d = mc_continuum_desc(kind=MC_GRAPH, n=nb)
                d.c_const = float(scn["c"][a])
                d.measure_const = 1.0                        # unit coarse measure (reading C11)
                d.n_edges = len(i)
                d.edge_i = _ptr(self._arr(i, np.int32), _pi)
                d.edge_j = _ptr(self._arr(j, np.int32), _pi)
                d.edge_t = _ptr(self._arr(t, np.float64))
                d.dirichlet = _ptr(self._arr(np.where(mask, g, np.nan), np.float64))
                conts.append(d)
            bi, bj, bt = scn["between"]
            d = mc_coupling_desc(a=0, b=1, nnz=len(bi))
            d.i_a = _ptr(self._arr(bi, np.int32), _pi)
            d.j_b = _ptr(self._arr(bj, np.int32), _pi)
            d.sigma = _ptr(self._arr(bt, np.float64))
            cpls.append(d)
        elif scn["kind"] == "coarse":
            # an assembled symmetric coarse system (NLMC, NlmcSpace.coarse_scenario): every
            # off-diagonal entry a_ij becomes a signed transmissibility / transfer -a_ij, the
            # row sums go to diag_extra, so the library's diagonal is exactly a_ii (C32)
            for blk in scn["blocks"]:
                d = mc_continuum_desc(kind=MC_GRAPH, n=blk["n"])
                d.c = _ptr(self._arr(blk["mass"], np.float64))
                d.measure_const = 1.0
                d.f = _ptr(self._arr(blk["F"], np.float64))
                d.u0 = _ptr(self._arr(blk["u0"], np.float64))
                d.n_edges = len(blk["ei"])
                d.edge_i = _ptr(self._arr(blk["ei"], np.int32), _pi)
                d.edge_j = _ptr(self._arr(blk["ej"], np.int32), _pi)
                d.edge_t = _ptr(self._arr(blk["et"], np.float64))
                d.signed_edges = 1
                d.diag_extra = _ptr(self._arr(blk["rowsum"], np.float64))
                conts.append(d)
            for cp in scn["couplings"]:
                d = mc_coupling_desc(a=cp["a"], b=cp["b"], nnz=len(cp["i"]))
                d.i_a = _ptr(self._arr(cp["i"], np.int32), _pi)
                d.j_b = _ptr(self._arr(cp["j"], np.int32), _pi)
                d.sigma = _ptr(self._arr(cp["sigma"], np.float64))
                d.signed_sigma = 1
                cpls.append(d)
        else:
            raise ValueError(scn["kind"])
        return conts, cpls

    def nlmc(self, nHx, nHy, oversample):
        """NLMC multiscale space of this (not yet stepped) fine problem: bases and the
        coarse system built by the library on the GPU (mc_nlmc_build)."""
        return NlmcSpace(self, nHx, nHy, oversample)

    # ------------------------------------------------------------------ calls
    def _check(self, st, create=False, report=None):
        if st != MC_OK:
            msg = self.lib.mc_error_string(None if create else self.ctx)
            raise MCError(st, (msg or b"").decode(), report)

    def step(self, scheme="D"):
        rep = mc_step_report()
        st = self.lib.mc_step(self.ctx, SCHEMES[scheme], C.byref(rep))
        self._check(st, report=rep.as_dict())
        return rep.as_dict()

    def run(self, scheme, n_steps, snapshots=None):
        """n_steps steps; snapshots: None or list over steps of lists over continua of tensors."""
        reps = (mc_step_report * max(n_steps, 1))()
        snaps = None
        if snapshots is not None:
            flat = [snapshots[s][a] for s in range(n_steps) for a in range(self.L)]
            snaps = (C.c_void_p * len(flat))(*[C.c_void_p(t.data_ptr()) for t in flat])
        st = self.lib.mc_run(self.ctx, SCHEMES[scheme], n_steps, reps, snaps)
        out = [reps[s].as_dict() for s in range(n_steps)]
        self._check(st, report=out)
        return out

    def get_state(self, alpha, out=None):
        if out is None:
            out = self.torch.empty(self.sizes[alpha], dtype=self.torch.float64, device=self.device)
        self._check(self.lib.mc_get_state(self.ctx, alpha, C.c_void_p(out.data_ptr())))
        return out

    def set_state(self, alpha, src):
        self._check(self.lib.mc_set_state(self.ctx, alpha, C.c_void_p(src.data_ptr())))

    def state(self):
        return [self.get_state(a) for a in range(self.L)]

    def last_kernel_ms(self):
        v = C.c_double()
        self._check(self.lib.mc_last_kernel_ms(self.ctx, C.byref(v)))
        return v.value

    def close(self):
        if self.ctx:
            self.lib.mc_destroy(self.ctx)
            self.ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass



class NlmcSpace:
    """Result of mc_nlmc_build (include/mc.h): coarse system Abar (CSR), Mbar, Fbar, u0bar,
    coarse DOF keys (continuum, coarse cell, piece), fine -> coarse map, bases on demand."""

    def __init__(self, pb: Problem, nHx, nHy, oversample):
        self.lib, self.pb = pb.lib, pb
        scn = pb.scn
        d = mc_nlmc_desc(nHx=nHx, nHy=nHy, oversample=oversample)
        hosts = []
        for a, c in enumerate(scn["continua"]):
            if c["kind"] != "grid":
                h = np.ascontiguousarray(scn["fracture"]["cells"], dtype=np.int32)
                hosts.append(h)
                d.host[a] = h.ctypes.data_as(C.c_void_p)
        self.h = C.c_void_p()
        st = self.lib.mc_nlmc_build(pb.ctx, C.byref(d), C.byref(self.h))
        pb._check(st)
        na = (_i64 * MC_MAX_CONTINUA)()
        nnz, nf = _i64(), _i64()
        self.lib.mc_nlmc_sizes(self.h, na, C.byref(nnz), C.byref(nf))
        self.L = pb.L
        self.sizes = [int(na[a]) for a in range(self.L)]
        n = sum(self.sizes)
        self.n, self.nnz, self.n_fine = n, int(nnz.value), int(nf.value)
        self.rowptr = np.zeros(n + 1, np.int32)
        self.col = np.zeros(self.nnz, np.int32)
        self.val = np.zeros(self.nnz)
        self.mass, self.rhs, self.u0 = np.zeros(n), np.zeros(n), np.zeros(n)
        self.key = np.zeros(3 * n, np.int32)
        self.fine_dof = np.zeros(self.n_fine, np.int32)
        arrs = [self.rowptr, self.col, self.val, self.mass, self.rhs, self.u0, self.key, self.fine_dof]
        st = self.lib.mc_nlmc_get(self.h, *[a.ctypes.data_as(C.c_void_p) for a in arrs])
        if st != MC_OK:
            raise MCError(st, "mc_nlmc_get")
        self.key = self.key.reshape(n, 3)
        tb, tp = C.c_double(), C.c_double()
        self.lib.mc_nlmc_times(self.h, C.byref(tb), C.byref(tp))
        self.ms_basis, self.ms_project = tb.value, tp.value
        fb, bb = C.c_double(), C.c_double()
        self.lib.mc_nlmc_cost(self.h, C.byref(fb), C.byref(bb))
        self.flops_basis, self.bytes_bases = fb.value, bb.value
        self.korder = pb.korder

    def basis(self, r):
        out = np.zeros(self.n_fine)
        st = self.lib.mc_nlmc_basis(self.h, int(r), out.ctypes.data_as(C.c_void_p))
        if st != MC_OK:
            raise MCError(st, "mc_nlmc_basis")
        return out

    def coarse_scenario(self, T, NT):
        """The coarse system as a 'coarse' scenario for Problem (signed ABI-2 descriptors)."""
        return coarse_scenario(self.rowptr, self.col, self.val, self.mass, self.rhs, self.u0, self.sizes,
                               T, NT, self.korder)

    def close(self):
        if self.h:
            self.lib.mc_nlmc_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def coarse_scenario(rowptr, col, val, mass, rhs, u0, sizes, T, NT, korder=None):
    """An assembled symmetric system (CSR, blocks of `sizes` rows) as a 'coarse' scenario:
    within-block off-diagonals -> signed edges, between-block -> signed transfer entries,
    row sums -> diag_extra (marshalling for mc_set_continuum / mc_set_coupling, ABI 2)."""
    n = int(sum(sizes))
    off = np.concatenate([[0], np.cumsum(sizes)])
    rowptr = np.asarray(rowptr, dtype=np.int64)
    rows = np.repeat(np.arange(n), np.diff(rowptr))
    cols, vals = np.asarray(col, dtype=np.int64), np.asarray(val, dtype=np.float64)
    blk = np.searchsorted(off, rows, side="right") - 1
    bcol = np.searchsorted(off, cols, side="right") - 1
    rowsum = np.bincount(rows, weights=vals, minlength=n)
    L = len(sizes)
    blocks, cpls = [], []
    for a in range(L):
        sel = (blk == a) & (bcol == a) & (rows < cols)
        lo, hi = off[a], off[a + 1]
        blocks.append(dict(n=int(hi - lo), mass=np.asarray(mass)[lo:hi], F=np.asarray(rhs)[lo:hi],
                           u0=np.asarray(u0)[lo:hi], ei=rows[sel] - lo, ej=cols[sel] - lo, et=-vals[sel],
                           rowsum=rowsum[lo:hi]))
    for a in range(L):
        for b in range(a + 1, L):
            sel = (blk == a) & (bcol == b)
            if sel.any():
                cpls.append(dict(a=a, b=b, i=rows[sel] - off[a], j=cols[sel] - off[b], sigma=-vals[sel]))
    out = dict(kind="coarse", T=float(T), NT=int(NT), blocks=blocks, couplings=cpls)
    if korder is not None:
        out["korder"] = list(korder)
    return out
