"""Oracle assembly of the multicontinuum block system  M dp/dt + A p = F,  A = D + Q.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Follows PAPER.md §3.1:
  * Eq. app-md: TPFA  sum_j T_ij (p_i - p_j), T = k|E|/d
    (PAPER.md:266-267), storage c|cell|, transfer
    sigma_il (p_m,i - p_f,l).
  * Eq. app-tc: co-located sigma_12,ii.
  * Eq. app-mc: block matrices
        M = diag(M_a),   m_a,ii = c_a,i |cell_i|
        D = diag(D_a),   a_ii = sum_n T_in,  a_ij = -T_ij
        Q: diagonal blocks sum_{b!=a} Q_ab (as the diagonal of row sums),
           off-diagonal blocks -Q_ab,  Q_ba = Q_ab^T
  * NLMC coarse system Eq. app-nlmc with M = c|K|.

Readings:
  C1  |cell| = h^2 (h = 1/n), fracture cell |iota| = h;
  C2  heterogeneous k: T_face = 2 k_i k_j / (k_i + k_j)  (|E|/d = 1); constant k: T = k;
  C3  Dirichlet on the left/right edge: half-cell face T_b = 2 k_i on the diagonal, T_b g in F;
  C6  embedded Q entry (host(l), l) = given per-fracture-cell sigma;
  C7  fracture T_f = k_f / h between consecutive fracture cells;
  C9  co-located Q_ii = sigma_12 h^2;
  C11 NLMC mass m = c (unit coarse measure);
  C12 NLMC Dirichlet DOFs become identity rows (m = 0, F = g, u0 = g), their
      columns eliminated into F of the free rows, free rows keep their diagonal.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp


class System:
    """Assembled block system: sizes per continuum, M (vector), A (CSR), F, u0."""

    def __init__(self, sizes, M, A, F, u0, names):
        self.sizes = list(sizes)
        self.offsets = np.concatenate([[0], np.cumsum(self.sizes)]).astype(np.int64)
        self.M = np.asarray(M, dtype=np.float64)
        self.A = sp.csr_matrix(A)
        self.F = np.asarray(F, dtype=np.float64)
        self.u0 = np.asarray(u0, dtype=np.float64)
        self.names = list(names)
        self._flux = None

    @property
    def flux(self):
        """Flux form of A (set by assemble(); derived from the assembled A otherwise)."""
        if self._flux is None:
            self._flux = flux_from_assembled(self)
        return self._flux

    @flux.setter
    def flux(self, v):
        self._flux = v

    @property
    def L(self):
        return len(self.sizes)

    def block(self, a):
        return slice(int(self.offsets[a]), int(self.offsets[a + 1]))

    def split(self, u):
        return [u[self.block(a)] for a in range(self.L)]


def laplacian_from_edges(n, i, j, t):
    """sum_e t_e (e_i - e_j)(e_i - e_j)^T : a_ii = sum t, a_ij = -t."""
    i = np.asarray(i, dtype=np.int64)
    j = np.asarray(j, dtype=np.int64)
    t = np.asarray(t, dtype=np.float64)
    rows = np.concatenate([i, j, i, j])
    cols = np.concatenate([i, j, j, i])
    vals = np.concatenate([t, t, -t, -t])
    return sp.csr_matrix(sp.coo_matrix((vals, (rows, cols)), shape=(n, n)))


def grid_faces(nx, ny):
    """Interior faces of the nx x ny row-major grid (i = iy*nx + ix): (i, j) pairs."""
    iy, ix = np.divmod(np.arange(nx * ny, dtype=np.int64), nx)
    xm = ix < nx - 1
    ym = iy < ny - 1
    cell = np.arange(nx * ny, dtype=np.int64)
    fi = np.concatenate([cell[xm], cell[ym]])
    fj = np.concatenate([cell[xm] + 1, cell[ym] + nx])
    return fi, fj


def face_transmissibility(k, fi, fj):
    """T = k |E|/d with |E|/d = h/h = 1; harmonic mean for a k field (C2)."""
    if np.isscalar(k) or np.ndim(k) == 0:
        return np.full(len(fi), float(k))
    k = np.asarray(k, dtype=np.float64)
    return 2.0 * k[fi] * k[fj] / (k[fi] + k[fj])


def grid_continuum(nx, ny, h, k, c, dirichlet):
    """One d-dimensional continuum on the nx x ny grid: (D, M, F) per Eq. app-md / app-mc.

    dirichlet = (g_left, g_right) (either may be None = no-flow) or None: all faces
    no-flow, the paper's homogeneous Neumann condition.
    """
    N = nx * ny
    fi, fj = grid_faces(nx, ny)
    D = laplacian_from_edges(N, fi, fj, face_transmissibility(k, fi, fj))
    M = np.full(N, float(c) * h * h)                       # m = c |cell|, |cell| = h^2 (C1)
    F = np.zeros(N)
    if dirichlet is not None:
        gL, gR = dirichlet
        kk = np.full(N, float(k)) if np.ndim(k) == 0 else np.asarray(k, dtype=np.float64)
        ix = np.arange(N) % nx
        bdiag = np.zeros(N)
        for col, g in ((0, gL), (nx - 1, gR)):
            if g is None:
                continue
            cells = np.nonzero(ix == col)[0]
            Tb = kk[cells] * h / (h / 2.0)                 # half-cell face, |E| = h, d = h/2 (C3)
            bdiag[cells] += Tb
            F[cells] += Tb * float(g)
        D = D + sp.diags(bdiag)
    return sp.csr_matrix(D), M, F


def grid_dirichlet_source(nx, ny, h, k, dirichlet):
    """F of a grid continuum: T_b g on the Dirichlet columns (C3), as grid_continuum."""
    N = nx * ny
    F = np.zeros(N)
    if dirichlet is None:
        return F
    kk = np.full(N, float(k)) if np.ndim(k) == 0 else np.asarray(k, dtype=np.float64)
    for col, g in ((0, dirichlet[0]), (nx - 1, dirichlet[1])):
        if g is None:
            continue
        cells = np.arange(col, N, nx)
        F[cells] += kk[cells] * h / (h / 2.0) * float(g)
    return F


def fracture_continuum(n, h, cells, edges, k_f, c_f):
    """1D fracture continuum: T_f = k_f |E|/d with |E| = 1, d = h (C7); m = c_f h (C1)."""
    Nf = len(cells)
    e = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
    D = laplacian_from_edges(Nf, e[:, 0], e[:, 1], np.full(len(e), float(k_f) / h))
    M = np.full(Nf, float(c_f) * h)
    F = np.zeros(Nf)
    return D, M, F


def block_system(sizes, Dblocks, Mblocks, Fblocks, Qpairs, u0blocks, names):
    """A = D + Q with Q laid out as in Eq. app-mc.

    Qpairs: dict (a, b) -> sparse Q_ab (N_a x N_b), a != b, entries sigma >= 0.
    Q_ba := Q_ab^T.  Diagonal block a gets diag(sum_b Q_ab 1).
    """
    L = len(sizes)
    blocks = [[None] * L for _ in range(L)]
    rowsum = [np.zeros(s) for s in sizes]
    for (a, b), Q in Qpairs.items():
        Q = sp.csr_matrix(Q)
        rowsum[a] += np.asarray(Q.sum(axis=1)).ravel()
        rowsum[b] += np.asarray(Q.sum(axis=0)).ravel()      # rows of Q_ba = Q_ab^T
        blocks[a][b] = -Q
        blocks[b][a] = -Q.T
    for a in range(L):
        blocks[a][a] = sp.csr_matrix(Dblocks[a]) + sp.diags(rowsum[a])
        for b in range(L):
            if blocks[a][b] is None:
                blocks[a][b] = sp.csr_matrix((sizes[a], sizes[b]))
    A = sp.bmat(blocks, format="csr")
    return System(sizes, np.concatenate(Mblocks), A, np.concatenate(Fblocks),
                  np.concatenate(u0blocks), names)


def assemble_fine(scn) -> System:
    """Fine-grid FV system of a generator scenario (kind == 'fine')."""
    n, h = scn["n"], scn["h"]
    sizes, Ds, Ms, Fs, names = [], [], [], [], []
    for cont in scn["continua"]:
        if cont["kind"] == "grid":
            D, M, F = grid_continuum(n, n, h, cont["k"], cont["c"], cont["dirichlet"])
        else:
            fr = scn["fracture"]
            D, M, F = fracture_continuum(n, h, fr["cells"], fr["edges"], cont["k"], cont["c"])
        sizes.append(len(M))
        Ds.append(D)
        Ms.append(M)
        Fs.append(F)
        names.append(cont["name"])
    Q = {}
    for cp in scn["couplings"]:
        a, b = cp["a"], cp["b"]
        if cp["type"] == "embedded":
            cells = scn["fracture"]["cells"]
            sig = np.asarray(cp["sigma"], dtype=np.float64)
            Q[(a, b)] = sp.csr_matrix((sig, (cells, np.arange(len(cells)))), shape=(sizes[a], sizes[b]))
        elif cp["type"] == "colocated":
            Q[(a, b)] = sp.diags(np.full(sizes[a], float(cp["sigma"]) * h * h))   # C9
        else:
            raise ValueError(cp["type"])
    u0 = [np.full(s, float(c.get("u0", 0.0))) for s, c in zip(sizes, scn["continua"])]   # C17
    # wells f = q_w (p_w - p) on a continuum (paper analogue; sign per
    # SPEC.md:154): q_w |cell| on the diagonal, q_w p_w |cell| in F
    for a, c in enumerate(scn["continua"]):
        if "well_q" in c:
            meas = h * h if c["kind"] == "grid" else h
            wq = np.asarray(c["well_q"], dtype=np.float64) * meas
            Ds[a] = sp.csr_matrix(Ds[a] + sp.diags(wq))
            Fs[a] = Fs[a] + wq * float(c["well_p"])
    return block_system(sizes, Ds, Ms, Fs, Q, u0, names)


def assemble_nlmc(scn) -> System:
    """NLMC-style coarse system (config 3) with Dirichlet identity rows (C11, C12)."""
    nc = scn["nc"]
    Nb = nc * nc
    sizes = [Nb, Nb]
    Ds = [laplacian_from_edges(Nb, i, j, t) for (i, j, t) in scn["within"]]
    bi, bj, bt = scn["between"]
    Q = {(0, 1): sp.csr_matrix((bt, (bi, bj)), shape=(Nb, Nb))}
    Ms = [np.full(Nb, float(c)) for c in scn["c"]]           # unit coarse measure (C11)
    Fs = [np.zeros(Nb), np.zeros(Nb)]
    u0 = [np.zeros(Nb), np.zeros(Nb)]
    sys = block_system(sizes, Ds, Ms, Fs, Q, u0, ["matrix", "fracture"])
    mask = np.concatenate([scn["dirichlet"][a][0] for a in range(2)])
    g = np.concatenate([scn["dirichlet"][a][1] for a in range(2)])
    return apply_dirichlet_rows(sys, mask, g)


def apply_dirichlet_rows(sys: System, mask, g) -> System:
    """Identity rows for fixed DOFs, columns eliminated symmetrically into F (C12)."""
    mask = np.asarray(mask, dtype=bool)
    g = np.where(mask, np.asarray(g, dtype=np.float64), 0.0)
    A = sp.csr_matrix(sys.A)
    free = ~mask
    F = sys.F - A @ g                                       # move fixed columns to the RHS
    keep = sp.diags(free.astype(np.float64))
    A = keep @ A @ keep + sp.diags(mask.astype(np.float64))  # zero fixed rows/cols, unit diagonal
    F = np.where(mask, g, F)
    M = np.where(mask, 0.0, sys.M)
    u0 = np.where(mask, g, sys.u0)
    return System(sys.sizes, M, A, F, u0, sys.names)


class FluxSystem(System):
    """M, F, u0 and the flux form of a fine-grid scenario WITHOUT the assembled A
    (configs 2 and 4: nnz(A) up to 4e8).  Used by the CG oracle (oracle/fluxcg.py)."""

    def __init__(self, sizes, M, F, u0, names):
        self.sizes = list(sizes)
        self.offsets = np.concatenate([[0], np.cumsum(self.sizes)]).astype(np.int64)
        self.M = np.asarray(M, dtype=np.float64)
        self.F = np.asarray(F, dtype=np.float64)
        self.u0 = np.asarray(u0, dtype=np.float64)
        self.names = list(names)
        self._flux = None

    @property
    def A(self):
        raise AttributeError("FluxSystem has no assembled A (use .flux)")


def assemble_lean(scn) -> FluxSystem:
    """Fine-grid scenario: M, F, u0 per Eq. app-md / app-mc exactly as assemble_fine
    builds them (C1, C3, wells), plus flux_form(); no sparse matrix is built."""
    assert scn["kind"] == "fine"
    n, h = scn["n"], scn["h"]
    sizes, Ms, Fs, names = [], [], [], []
    for cont in scn["continua"]:
        if cont["kind"] == "grid":
            N = n * n
            M = np.full(N, float(cont["c"]) * h * h)                    # C1
            F = grid_dirichlet_source(n, n, h, cont["k"], cont["dirichlet"])
            meas = h * h
        else:
            N = len(scn["fracture"]["cells"])
            M = np.full(N, float(cont["c"]) * h)                        # C1
            F = np.zeros(N)
            meas = h
        if "well_q" in cont:
            F = F + np.asarray(cont["well_q"], dtype=np.float64) * meas * float(cont["well_p"])
        sizes.append(N)
        Ms.append(M)
        Fs.append(F)
        names.append(cont["name"])
    u0 = [np.full(s, float(c.get("u0", 0.0))) for s, c in zip(sizes, scn["continua"])]   # C17
    sys_ = FluxSystem(sizes, np.concatenate(Ms), np.concatenate(Fs), np.concatenate(u0), names)
    sys_.flux = flux_form(scn, sys_)
    return sys_


def assemble(scn) -> System:
    if scn["kind"] == "fine":
        sys_ = assemble_fine(scn)
    elif scn["kind"] == "nlmc":
        sys_ = assemble_nlmc(scn)
    else:
        raise ValueError(scn["kind"])
    sys_.flux = flux_form(scn, sys_)
    return sys_


# --------------------------------------------------------------------------- flux form
class FluxForm:
    """The same operator A written as in Eq. app-md, unassembled:

        (A p)_i = diag_i p_i + sum_{edges e = (i, j)} t_e (p_i - p_j)

    over every two-point connection: TPFA faces and fracture edges (within a
    continuum) and transfer entries sigma_ij (between continua,
    PAPER.md:256, 260, 302), plus non-edge diagonal terms (Dirichlet half-cell faces,
    NLMC fixed-DOF identity rows).  Assembling it gives the assembled A (pinned in
    tests); evaluating it WITHOUT assembly avoids storing a_ii = sum T + sigma, whose
    rounding (eps * T_f ~ 1e-7 for T_f = 1e9) swamps sigma ~ 1e2 in the fracture rows
    (reading C15).  The oracle uses it, in long double, for iterative refinement.
    """

    def __init__(self, N, ei, ej, et, between, diag):
        self.N = int(N)
        self.ei = np.asarray(ei, dtype=np.int64)
        self.ej = np.asarray(ej, dtype=np.int64)
        self.et = np.asarray(et, dtype=np.float64)
        self.between = np.asarray(between, dtype=bool)
        self.diag = np.asarray(diag, dtype=np.float64)

    def block_edges(self, sl, mtau, scheme):
        """(n, ei, ej, et, d) of one solve: coupled (whole system, all edges) or the
        D-scheme block `sl` (A0 block: within-continuum edges, transfer edges as
        diagonal), indices local to the block."""
        lo, hi = sl.start, sl.stop
        if scheme == "coupled":
            keep = np.ones(len(self.ei), dtype=bool)
        else:
            keep = (~self.between) & (self.ei >= lo) & (self.ei < hi)
        d = mtau[lo:hi] + self.diag[lo:hi]
        if scheme != "coupled":               # A0 diagonal: + sum_b Q_ab 1
            for end in (self.ei, self.ej):
                m = self.between & (end >= lo) & (end < hi)
                d = d + np.bincount(end[m] - lo, weights=self.et[m], minlength=hi - lo)
        return hi - lo, self.ei[keep] - lo, self.ej[keep] - lo, self.et[keep], d

    def block_op(self, sl, mtau, scheme):
        """Operator of one solve (see block_edges) as a BlockOp."""
        return BlockOp(*self.block_edges(sl, mtau, scheme))

    def lagged_transfer(self, u):
        """-A1 u = sum_b Q_ab u_b for every row (the transfer connections only,
        PAPER.md:482-484): row i of a transfer edge (i, j, sigma) gets sigma u_j, row j
        gets sigma u_i."""
        m = self.between
        ei, ej, et = self.ei[m], self.ej[m], self.et[m]
        return (np.bincount(ei, weights=et * u[ej], minlength=self.N)
                + np.bincount(ej, weights=et * u[ei], minlength=self.N))


class BlockOp:
    """y = d * x + sum_e t_e (x_i - x_j) on one system (flux form)."""

    def __init__(self, n, ei, ej, et, d):
        self.n, self.d = n, np.asarray(d, dtype=np.float64)
        rows = np.concatenate([ei, ej])
        oth = np.concatenate([ej, ei])
        t = np.concatenate([et, et])
        order = np.argsort(rows, kind="stable")
        self.rows, self.oth, self.t = rows[order], oth[order], t[order]
        self.starts = np.searchsorted(self.rows, np.arange(n))
        self.has = np.diff(np.concatenate([self.starts, [len(self.rows)]])) > 0

    def apply(self, x, dtype=np.float64):
        x = np.asarray(x).astype(dtype)
        y = self.d.astype(dtype) * x
        if len(self.rows):
            c = self.t.astype(dtype) * (x[self.rows] - x[self.oth])
            c = np.append(c, np.zeros(1, dtype=dtype))       # sentinel: every start is a valid index
            s = np.add.reduceat(c, self.starts)
            y[self.has] += s[self.has]
        return y

    def tocsr(self):
        return sp.csr_matrix(laplacian_from_edges(self.n, self.rows[self.rows < self.oth],
                                                  self.oth[self.rows < self.oth],
                                                  self.t[self.rows < self.oth]) + sp.diags(self.d))


def flux_from_assembled(sys_: System) -> FluxForm:
    """Edges t = -a_ij (i < j) and diag = a_ii - sum_j t_ij read back from an assembled A."""
    A = sp.triu(sp.csr_matrix(sys_.A), k=1).tocoo()
    ei, ej, et = A.row.astype(np.int64), A.col.astype(np.int64), -A.data
    blk = lambda v: np.searchsorted(sys_.offsets, v, side="right") - 1
    N = sys_.A.shape[0]
    rs = np.bincount(ei, weights=et, minlength=N) + np.bincount(ej, weights=et, minlength=N)
    return FluxForm(N, ei, ej, et, blk(ei) != blk(ej), sys_.A.diagonal() - rs)


def flux_form(scn, sys_: System) -> FluxForm:
    off = sys_.offsets
    EI, EJ, ET, BT = [], [], [], []
    diag = np.zeros(int(off[-1]))
    if scn["kind"] == "fine":
        n, h = scn["n"], scn["h"]
        for a, cont in enumerate(scn["continua"]):
            if cont["kind"] == "grid":
                fi, fj = grid_faces(n, n)
                EI.append(off[a] + fi)
                EJ.append(off[a] + fj)
                ET.append(face_transmissibility(cont["k"], fi, fj))
                BT.append(np.zeros(len(fi), dtype=bool))
                if "well_q" in cont:                                            # wells
                    diag[off[a]:off[a + 1]] += np.asarray(cont["well_q"], dtype=np.float64) * h * h
                if cont["dirichlet"] is not None:
                    kk = np.full(n * n, float(cont["k"])) if np.ndim(cont["k"]) == 0 else cont["k"]
                    ix = np.arange(n * n) % n
                    for col, g in ((0, cont["dirichlet"][0]), (n - 1, cont["dirichlet"][1])):
                        if g is not None:
                            cells = np.nonzero(ix == col)[0]
                            diag[off[a] + cells] += kk[cells] * h / (h / 2.0)     # C3
            else:
                e = np.asarray(scn["fracture"]["edges"], dtype=np.int64).reshape(-1, 2)
                if "well_q" in cont:                                            # wells
                    diag[off[a]:off[a + 1]] += np.asarray(cont["well_q"], dtype=np.float64) * h
                EI.append(off[a] + e[:, 0])
                EJ.append(off[a] + e[:, 1])
                ET.append(np.full(len(e), float(cont["k"]) / h))                 # C7
                BT.append(np.zeros(len(e), dtype=bool))
        for cp in scn["couplings"]:
            a, b = cp["a"], cp["b"]
            if cp["type"] == "embedded":
                cells = scn["fracture"]["cells"]
                EI.append(off[a] + cells)
                EJ.append(off[b] + np.arange(len(cells)))
                ET.append(np.asarray(cp["sigma"], dtype=np.float64))              # C6
            else:
                m = n * n
                EI.append(off[a] + np.arange(m))
                EJ.append(off[b] + np.arange(m))
                ET.append(np.full(m, float(cp["sigma"]) * h * h))                # C9
            BT.append(np.ones(len(EI[-1]), dtype=bool))
        return FluxForm(off[-1], np.concatenate(EI), np.concatenate(EJ), np.concatenate(ET),
                        np.concatenate(BT), diag)
    # NLMC with fixed-DOF identity rows (C12): edges touching a fixed DOF leave the
    # operator; their t stays on the free endpoint's diagonal (its F got t g).
    Nb = scn["nc"] ** 2
    mask = np.concatenate([scn["dirichlet"][a][0] for a in range(2)])
    for a, (i, j, t) in enumerate(scn["within"]):
        EI.append(a * Nb + i)
        EJ.append(a * Nb + j)
        ET.append(t)
        BT.append(np.zeros(len(i), dtype=bool))
    bi, bj, bt = scn["between"]
    EI.append(bi)
    EJ.append(Nb + bj)
    ET.append(bt)
    BT.append(np.ones(len(bi), dtype=bool))
    ei, ej, et, bw = (np.concatenate(v) for v in (EI, EJ, ET, BT))
    fi, fj = mask[ei], mask[ej]
    for end, other in ((ei, fj), (ej, fi)):
        sel = other & ~mask[end]
        diag += np.bincount(end[sel], weights=et[sel], minlength=2 * Nb)
    diag[mask] = 1.0
    keep = ~fi & ~fj
    return FluxForm(2 * Nb, ei[keep], ej[keep], et[keep], bw[keep], diag)
