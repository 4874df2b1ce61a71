"""Oracle: the NLMC multiscale space and coarse system (§4.1, :591-729).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Follows the paper step by step:
  * coarse cells K_j (nHx x nHy blocks of the fine grid); K_j^alpha = Omega_alpha cap K_j,
    the fine DOFs of continuum alpha in K_j.  A coarse DOF (j, alpha)
    exists when K_j^alpha is not empty; a fracture continuum contributes one coarse DOF
    per connected piece of the network inside K_j (reading C30).
  * K_i^+ = K_i enlarged by m coarse layers, clipped at the domain.
  * basis psi^{i,beta}: the saddle-point system Eq. eq:basis on the
    fine DOFs of K_i^+ -- the coupled fine operator A = D + Q restricted to K_i^+ (zero
    Dirichlet on the outside), Lagrange multipliers mu imposing
        (1/|K_j^alpha|) int_{K_j^alpha} psi_alpha = delta_ij delta_alpha beta
    for every K_j^alpha in K_i^+ (PAPER.md:600-605, 637).  One sparse direct (SuperLU)
    factorisation of the KKT matrix per i, one solve per beta.
  * R: rows psi^{i,beta};  Abar = R A R^T.
  * Abar = Dbar + Qbar (Eq. app-nlmc): Dbar = R D R^T with D the block
    diagonal diffusion, in flux form (reading C32: off-diagonal
    transmissibilities of R D R^T, diagonal = minus their sum plus the aggregated
    boundary terms, so constants are preserved as in FV); Mbar, Qbar and Fbar by the direct coarse
    formulas, i.e. the fine entries summed over each K_i^alpha
    (aggregation P: P[(i,alpha), c] = 1 for c in K_i^alpha).  Well reaction terms
    q_w|cell| (paper analogue, reading C27) are a source term, not diffusion: they stay
    out of Eq. eq:basis and enter the coarse system like Qbar and Fbar, aggregated
    (reading C31).
  * coarse reference: pbar = measure-weighted mean over K_i^alpha.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla
from scipy.sparse import csgraph

from . import assemble as asm
from .assemble import System


def fine_parts(scn):
    """The fine operator of a 'fine' scenario split as A = D + Q + W:
    D block-diagonal diffusion incl. Dirichlet half-cell faces, Q the transfer in the
    Eq. app-mc layout, W the diagonal well terms; plus M, F (Dirichlet + well sources)."""
    n, h = scn["n"], scn["h"]
    sizes, Ds, Ms, Fs = [], [], [], []
    for cont in scn["continua"]:
        if cont["kind"] == "grid":
            D, M, F = asm.grid_continuum(n, n, h, cont["k"], cont["c"], cont["dirichlet"])
        else:
            fr = scn["fracture"]
            D, M, F = asm.fracture_continuum(n, h, fr["cells"], fr["edges"], cont["k"], cont["c"])
        sizes.append(len(M))
        Ds.append(D)
        Ms.append(M)
        Fs.append(F)
    W = []
    for a, c in enumerate(scn["continua"]):
        w = np.zeros(sizes[a])
        if "well_q" in c:
            w = np.asarray(c["well_q"], dtype=np.float64) * (h * h if c["kind"] == "grid" else h)
            Fs[a] = Fs[a] + w * float(c["well_p"])
        W.append(w)
    zero = [np.zeros(s) for s in sizes]
    # Q alone: block_system with zero diffusion blocks
    qsys = asm.block_system(sizes, [sp.csr_matrix((s, s)) for s in sizes], zero, zero,
                            _transfer(scn, sizes), zero, [""] * len(sizes))
    D = sp.block_diag(Ds, format="csr")
    return sizes, D, sp.csr_matrix(qsys.A), np.concatenate(W), np.concatenate(Ms), np.concatenate(Fs)


def _transfer(scn, sizes):
    h = scn["h"]
    Q = {}
    for cp in scn["couplings"]:
        a, b = cp["a"], cp["b"]
        if cp["type"] == "embedded":
            cells = scn["fracture"]["cells"]
            sig = np.asarray(cp["sigma"], dtype=np.float64)
            Q[(a, b)] = sp.csr_matrix((sig, (cells, np.arange(len(cells)))), shape=(sizes[a], sizes[b]))
        else:
            Q[(a, b)] = sp.diags(np.full(sizes[a], float(cp["sigma"]) * h * h))   # C9
    return Q


def fine_coarse_map(scn, sys_: System, nHx: int, nHy: int):
    """Per fine DOF (global, block order of sys_): continuum, host fine cell, coarse cell,
    measure.  Fracture cells belong to the coarse cell of their host grid cell
    (the coarse cell containing their midpoint)."""
    n, h = scn["n"], scn["h"]
    if n % nHx or n % nHy:
        raise ValueError("fine grid not divisible by the coarse grid")
    bx, by = n // nHx, n // nHy
    cont, host, meas = [], [], []
    for a, c in enumerate(scn["continua"]):
        if c["kind"] == "grid":
            hc = np.arange(n * n, dtype=np.int64)
            ms = np.full(n * n, h * h)
        else:
            hc = np.asarray(scn["fracture"]["cells"], dtype=np.int64)
            ms = np.full(len(hc), h)
        cont.append(np.full(len(hc), a, dtype=np.int64))
        host.append(hc)
        meas.append(ms)
    cont, host, meas = (np.concatenate(v) for v in (cont, host, meas))
    iy, ix = np.divmod(host, n)
    cell = (iy // by) * nHx + ix // bx
    assert len(cont) == sys_.A.shape[0]
    # pieces (C30): connected components of each graph continuum's edges inside one coarse cell
    piece = np.zeros(len(cont), dtype=np.int64)
    off = sys_.offsets
    for a, c in enumerate(scn["continua"]):
        if c["kind"] == "grid":
            continue
        e = np.asarray(scn["fracture"]["edges"], dtype=np.int64).reshape(-1, 2)
        fc = cell[off[a]:off[a + 1]]
        same = fc[e[:, 0]] == fc[e[:, 1]]
        nf = len(fc)
        G = sp.csr_matrix((np.ones(int(same.sum())), (e[same, 0], e[same, 1])), shape=(nf, nf))
        _, lab = csgraph.connected_components(G, directed=False)
        piece[off[a]:off[a + 1]] = lab
    return cont, host, cell, meas, piece


class CoarseSpace:
    """psi^{i,beta} as the rows of R, and the coarse system (Abar, Mbar, Fbar, u0bar).
    Coarse DOF r = (dof_cont[r], dof_cell[r], dof_piece[r]), continuum-major."""

    def __init__(self, L, nHx, nHy, m, keys, fine_dof, R, Abar, Mbar, Fbar, u0bar, kmeas, fine_meas):
        self.L, self.nHx, self.nHy, self.m = L, nHx, nHy, m
        self.keys = keys
        self.dof_cont = np.array([k[0] for k in keys])
        self.dof_cell = np.array([k[1] for k in keys])
        self.dof_piece = np.array([k[2] for k in keys])
        self.fine_dof = fine_dof
        self.R, self.Abar, self.Mbar, self.Fbar, self.u0bar = R, Abar, Mbar, Fbar, u0bar
        self.kmeas, self.fine_meas = kmeas, fine_meas

    @property
    def sizes(self):
        return [int(np.sum(self.dof_cont == a)) for a in range(self.L)]

    def average(self, u_fine):
        """pbar: measure-weighted mean of a fine vector over every K_i^alpha."""
        return np.bincount(self.fine_dof, weights=self.fine_meas * np.asarray(u_fine),
                           minlength=len(self.keys)) / self.kmeas

    def system(self, names=None) -> System:
        """The coarse system Eq. app-nlmc as an oracle System (blocks = continua)."""
        return System(self.sizes, self.Mbar, self.Abar, self.Fbar, self.u0bar,
                      names or [f"c{a}" for a in range(self.L)])


def region(i, nHx, nHy, m):
    """Coarse cells of K_i^+ (m layers, clipped): a set of cell ids."""
    iy, ix = divmod(int(i), nHx)
    return {jy * nHx + jx for jy in range(max(0, iy - m), min(nHy, iy + m + 1))
            for jx in range(max(0, ix - m), min(nHx, ix + m + 1))}


def local_bases(A, cell, meas, kmeas, fine_dof, nHx, nHy, m, i, own):
    """Eq. eq:basis on K_i^+ (PAPER.md:606-637).  own: coarse DOFs of cell i.
    Returns the support S (sorted fine DOFs of K_i^+) and {coarse dof: psi on S}."""
    reg = region(i, nHx, nHy, m)
    S = np.nonzero(np.isin(cell, sorted(reg)))[0]
    cons = sorted(set(int(r) for r in fine_dof[S]))           # K_j^alpha (pieces) in K_i^+
    row_of = {r: k for k, r in enumerate(cons)}
    # constraint rows: (1/|K_j^alpha|) int_{K_j^alpha} psi_alpha dx = delta
    ci = np.array([row_of[int(fine_dof[s])] for s in S])
    cv = meas[S] / kmeas[fine_dof[S]]
    C = sp.csr_matrix((cv, (ci, np.arange(len(S)))), shape=(len(cons), len(S)))
    Aloc = sp.csr_matrix(A)[S][:, S]                 # zero Dirichlet outside K_i^+ 
    K = sp.bmat([[Aloc, C.T], [C, None]], format="csc")
    lu = spla.splu(K)
    out = {}
    for r in own:
        rhs = np.zeros(len(S) + len(cons))
        rhs[len(S) + row_of[r]] = 1.0                 # F^{beta,i}_{alpha,j} = delta_ij delta_ab
        out[r] = lu.solve(rhs)[:len(S)]
    return S, out


def build(scn, sys_: System, nHx: int, nHy: int, m: int) -> CoarseSpace:
    """All bases, R, and the coarse system."""
    cont, host, cell, meas, piece = fine_coarse_map(scn, sys_, nHx, nHy)
    L = sys_.L
    sizes, D, Q, W, M, F = fine_parts(scn)
    Ab = sp.csr_matrix(D + Q)                                             # Eq. eq:basis operator
    keys = sorted({(int(a), int(j), int(p)) for a, j, p in zip(cont, cell, piece)})   # continuum-major
    dof_of = {k: r for r, k in enumerate(keys)}
    nH = len(keys)
    fine_dof = np.array([dof_of[(int(a), int(j), int(p))] for a, j, p in zip(cont, cell, piece)])
    kmeas = np.bincount(fine_dof, weights=meas, minlength=nH)            # |K_j^alpha|
    Mbar = np.bincount(fine_dof, weights=M, minlength=nH)                 # c |K_j^alpha|
    u0bar = np.bincount(fine_dof, weights=meas * sys_.u0, minlength=nH) / kmeas
    own = [[] for _ in range(nHx * nHy)]
    for r, k in enumerate(keys):
        own[k[1]].append(r)
    rows, cols, vals = [], [], []
    for i in range(nHx * nHy):
        if not own[i]:
            continue
        S, psis = local_bases(Ab, cell, meas, kmeas, fine_dof, nHx, nHy, m, i, own[i])
        for r, psi in psis.items():
            rows.append(np.full(len(S), r))
            cols.append(S)
            vals.append(psi)
    R = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                      shape=(nH, len(cont)))
    P = sp.csr_matrix((np.ones(len(cont)), (fine_dof, np.arange(len(cont)))), shape=(nH, len(cont)))
    Dbar = sp.csr_matrix(R @ D @ R.T)
    # flux (finite-volume) form of Dbar (reading C32, "very similar to the
    # traditional finite volume method"): off-diagonal coarse transmissibilities from
    # R D R^T, diagonal such that Dbar 1 = P (D 1) -- the fine row sums aggregated, which
    # are the Dirichlet half-cell faces only (D 1 = 0 under no-flow boundaries)
    off = Dbar - sp.diags(Dbar.diagonal())
    Dbar = sp.csr_matrix(off + sp.diags(P @ (D @ np.ones(D.shape[0])) - off @ np.ones(nH)))
    Qbar = P @ Q @ P.T
    Wbar = P @ sp.diags(W) @ P.T
    Abar = sp.csr_matrix(Dbar + Qbar + Wbar)
    Fbar = P @ F                                                           # f |K_j^alpha|
    return CoarseSpace(L, nHx, nHy, m, keys, fine_dof, R, Abar, Mbar, Fbar, u0bar, kmeas, meas)
