"""Seeded generator for the five BASELINE.json workloads (and scaled variants).

Physical inputs only — see ``inputs/__init__.py``.  Every rule below is one of
the conventions fixed in DESIGN.md §3 (readings C1–C12 of SURVEY.md §8(c)); the
docstrings name the reading they implement.

Outputs are plain dicts of Python scalars and NumPy arrays:

fine-grid scenario (``kind == "fine"``)::

    n, h=1/n, T, NT, seed, config_id, conv_version
    continua: list (index = continuum id alpha) of
        {"name", "kind": "grid"|"fracture", "k": float | ndarray[n*n],
         "c": float, "dirichlet": (g_left, g_right) | None}
    fracture: {"cells": int64[Nf] host cell ids (row-major, ascending),
               "edges": int64[E,2] local fracture-cell pairs, i<j, unique}
    couplings: list of
        {"a", "b", "type": "embedded",  "sigma": float64[Nf]}   # Q_ab[host(l), l] = sigma[l]   (C6)
        {"a", "b", "type": "colocated", "sigma": float}         # field coefficient sigma_ab   (C9)

NLMC-style coarse scenario (``kind == "nlmc"``)::

    nc, L=2, c=(c_0, c_1), T, NT, seed
    within:  list over continua of (i, j, t) with i<j local DOF ids, t>0
    between: (i, j, t): DOF i of continuum 0, DOF j of continuum 1, t>0
    dirichlet: list over continua of (mask bool[nc*nc], g float64[nc*nc])

Transmissibilities ``t`` here are the positive magnitudes; the operator
entry is ``-t`` (BASELINE.json config 3: "T_ij = -k_scale*exp(-dist_ij)*U").
"""
from __future__ import annotations

import numpy as np

CONV_VERSION = "mc-conv-1"

# BASELINE.json:7-11 (configs[0..4]) as parameters of the two generators.
CONFIGS = {
    0: dict(kind="fine", n=64, seed=0, T=1.0, NT=50, segments=6, lengths=(10, 40),
            k_m=1.0, k_sigma=None, c_m=1.0, k_f=1e4, c_f=0.01, sigma_f=("const", 10.0),
            natural=None),
    1: dict(kind="fine", n=1024, seed=1, T=1.0, NT=100, segments=400, lengths=(50, 400),
            k_m=None, k_sigma=1.0, c_m=1.0, k_f=1e6, c_f=1e-3, sigma_f=("k_m", 100.0),
            natural=None),
    2: dict(kind="fine", n=2048, seed=2, T=1.0, NT=100, segments=1500, lengths=(100, 800),
            k_m=1.0, k_sigma=None, c_m=1.0, k_f=1e6, c_f=1e-3, sigma_f=("const", 20.0),
            natural=dict(k=1e2, c=0.1, sigma_12=5.0, sigma_2f=50.0)),
    3: dict(kind="nlmc", nc=256, seed=3, T=1.0, NT=100, c=(1.0, 0.01),
            k_scale=(1.0, 1e4), k_between=1.0, radius=2),
    4: dict(kind="fine", n=8192, seed=4, T=1.0, NT=20, segments=20000, lengths=(100, 2000),
            k_m=None, k_sigma=2.0, c_m=1.0, k_f=1e6, c_f=1e-3, sigma_f=("k_m", 100.0),
            natural=None),
}


def fracture_network(n: int, rng: np.random.Generator, segments: int, lengths: tuple[int, int]):
    """Axis-aligned fracture segments on an n x n grid (reading C4, C7, C8).

    Draw order (C4): ``o = rng.integers(0,2,S)`` (0 = horizontal),
    ``ix = rng.integers(0,n,S)``, ``iy = rng.integers(0,n,S)``,
    ``L = rng.integers(a,b+1,S)``.  A segment covers cells ix..ix+L-1 of row iy
    (horizontal) or rows iy..iy+L-1 of column ix (vertical), clipped at the
    domain edge.  Each traversed cell is one fracture cell; cells shared by
    several segments are merged (C8).  Consecutive cells along a segment are
    adjacent; edges are de-duplicated; collinear segments that only abut are
    not connected (C7).

    Returns (cells, edges): host cell ids ascending, local index pairs i<j.
    """
    S = int(segments)
    a, b = lengths
    o = rng.integers(0, 2, S)
    ix = rng.integers(0, n, S)
    iy = rng.integers(0, n, S)
    L = rng.integers(a, b + 1, S)
    start = np.where(o == 0, ix, iy)
    Leff = np.minimum(L, n - start)  # clipped length (>= 1 since start < n)
    total = int(Leff.sum())
    seg = np.repeat(np.arange(S), Leff)
    offs = np.cumsum(Leff) - Leff
    t = np.arange(total, dtype=np.int64) - np.repeat(offs, Leff)
    hor = o[seg] == 0
    cx = np.where(hor, ix[seg] + t, ix[seg]).astype(np.int64)
    cy = np.where(hor, iy[seg], iy[seg] + t).astype(np.int64)
    host = cy * n + cx
    # merged fracture cells (C8): the set of traversed host cells, ascending
    mark = np.zeros(n * n, dtype=bool)
    mark[host] = True
    cells = np.flatnonzero(mark)
    lut = np.full(n * n, -1, dtype=np.int64)
    lut[cells] = np.arange(len(cells))
    # consecutive pairs inside each segment: host id increases by 1 (horizontal) or n (vertical)
    nxt = np.ones(total, dtype=bool)
    nxt[np.cumsum(Leff) - 1] = False  # last cell of each segment has no successor
    idx = np.nonzero(nxt)[0]
    emark = np.zeros(2 * n * n, dtype=bool)  # key = 2*host_lo + (0 horizontal | 1 vertical)
    emark[2 * host[idx] + (~hor[idx]).astype(np.int64)] = True
    key = np.flatnonzero(emark)
    lo_h = key // 2
    hi_h = lo_h + np.where(key % 2 == 0, 1, n)
    edges = np.stack([lut[lo_h], lut[hi_h]], axis=1).astype(np.int64)
    return cells.astype(np.int64), edges


def make_fine(n: int, *, seed: int, T: float, NT: int, segments: int, lengths: tuple[int, int],
              k_m=1.0, k_sigma=None, c_m=1.0, k_f=1e4, c_f=0.01, sigma_f=("const", 10.0),
              natural=None, dirichlet=(1.0, 0.0), config_id=None) -> dict:
    """Fine-grid two/three-continuum scenario (configs 0, 1, 2, 4 and scaled stand-ins).

    Reading C5: a log-normal matrix permeability ``k = exp(k_sigma * Z)`` with
    ``Z = rng.standard_normal(n*n)`` (row-major) is drawn BEFORE the fracture
    draws from the same generator.  ``sigma_f = ("const", s)`` gives every
    fracture cell transfer s; ``("k_m", s)`` gives s * k_m(host cell) (C6).
    ``natural`` adds the co-located dual-porosity continuum of config 2 (C9, C10).
    ``dirichlet`` = (g_left, g_right) on every grid continuum (C3, C10), or None.
    """
    rng = np.random.default_rng(seed)
    if k_sigma is not None:
        Z = rng.standard_normal(n * n)
        k = np.exp(k_sigma * Z)
    else:
        k = float(k_m)
    if segments > 0:
        cells, edges = fracture_network(n, rng, segments, lengths)
    else:
        cells = np.zeros(0, dtype=np.int64)
        edges = np.zeros((0, 2), dtype=np.int64)
    kind_s, val_s = sigma_f
    if kind_s == "const":
        sig = np.full(len(cells), float(val_s))
    elif kind_s == "k_m":
        sig = float(val_s) * (k[cells] if isinstance(k, np.ndarray) else np.full(len(cells), k))
    else:
        raise ValueError(kind_s)
    continua = [dict(name="matrix", kind="grid", k=k, c=float(c_m), dirichlet=dirichlet)]
    couplings = []
    if natural is not None:
        continua.append(dict(name="natural", kind="grid", k=float(natural["k"]), c=float(natural["c"]),
                             dirichlet=dirichlet))
        couplings.append(dict(a=0, b=1, type="colocated", sigma=float(natural["sigma_12"])))
    fid = len(continua)
    if len(cells) > 0:
        continua.append(dict(name="fracture", kind="fracture", k=float(k_f), c=float(c_f), dirichlet=None))
        couplings.append(dict(a=0, b=fid, type="embedded", sigma=sig))
        if natural is not None:
            couplings.append(dict(a=1, b=fid, type="embedded",
                                  sigma=np.full(len(cells), float(natural["sigma_2f"]))))
    return dict(kind="fine", config_id=config_id, conv_version=CONV_VERSION, seed=seed,
                n=int(n), h=1.0 / n, T=float(T), NT=int(NT), continua=continua,
                fracture=dict(cells=cells, edges=edges), couplings=couplings)


# canonical half of the (2r+1)^2 neighbourhood: dy>0, or dy==0 and dx>0, lexicographic (C12)
def _canonical_offsets(r):
    return [(dy, dx) for dy in range(-r, r + 1) for dx in range(-r, r + 1)
            if dy > 0 or (dy == 0 and dx > 0)]


def _all_offsets(r):
    return [(dy, dx) for dy in range(-r, r + 1) for dx in range(-r, r + 1)]


def _pairs(nc, dy, dx):
    """Source cells (iy, ix) whose (iy+dy, ix+dx) neighbour lies inside; returns (src, dst) ids."""
    iy, ix = np.divmod(np.arange(nc * nc, dtype=np.int64), nc)
    ty, tx = iy + dy, ix + dx
    ok = (ty >= 0) & (ty < nc) & (tx >= 0) & (tx < nc)
    return np.nonzero(ok)[0], (ty * nc + tx)[ok], ok


def make_nlmc(nc: int = 256, *, seed: int = 3, T: float = 1.0, NT: int = 100, c=(1.0, 0.01),
              k_scale=(1.0, 1e4), k_between=1.0, radius=2, config_id=None) -> dict:
    """NLMC-style synthetic coarse operator (config 3; reading C11, C12).

    DOF = alpha*nc^2 + iy*nc + ix.  ``rng = default_rng(seed)``.  Within-continuum
    entries: for alpha = 0 then 1, for each canonical offset in lexicographic
    order draw ``U = rng.uniform(0.5, 1.5, nc*nc)`` indexed by the source cell;
    t = k_scale[alpha] * exp(-dist) * U with dist the centre distance in coarse
    cell units.  Between continua: all (2r+1)^2 offsets, same draw shape,
    t = k_between * exp(-dist) * U (dist 0 for the same cell).  Dirichlet: both
    continua, ix == 0 -> g = 1, ix == nc-1 -> g = 0.
    """
    rng = np.random.default_rng(seed)
    within = []
    for a in range(2):
        I, J, V = [], [], []
        for dy, dx in _canonical_offsets(radius):
            U = rng.uniform(0.5, 1.5, nc * nc)
            src, dst, ok = _pairs(nc, dy, dx)
            I.append(src)
            J.append(dst)
            V.append(k_scale[a] * np.exp(-np.hypot(dy, dx)) * U[ok])
        I = np.concatenate(I)
        J = np.concatenate(J)
        V = np.concatenate(V)
        lo, hi = np.minimum(I, J), np.maximum(I, J)
        within.append((lo, hi, V))
    I, J, V = [], [], []
    for dy, dx in _all_offsets(radius):
        U = rng.uniform(0.5, 1.5, nc * nc)
        src, dst, ok = _pairs(nc, dy, dx)
        I.append(src)
        J.append(dst)
        V.append(k_between * np.exp(-np.hypot(dy, dx)) * U[ok])
    between = (np.concatenate(I), np.concatenate(J), np.concatenate(V))
    ix = np.arange(nc * nc) % nc
    mask = (ix == 0) | (ix == nc - 1)
    g = np.where(ix == 0, 1.0, 0.0)
    dirichlet = [(mask.copy(), g.copy()) for _ in range(2)]
    return dict(kind="nlmc", config_id=config_id, conv_version=CONV_VERSION, seed=seed, nc=int(nc),
                L=2, c=tuple(float(x) for x in c), T=float(T), NT=int(NT), within=within,
                between=between, dirichlet=dirichlet)


def make_paper_analogue(kind: str = "2C", n: int = 200, seed: int = 32, segments: int = 25,
                        lengths=(120, 240), T: float = 0.002, NT: int = 50) -> dict:
    """The paper's own test setting with a synthetic network in place
    of the unpublished 25-fracture geometry: unit square, n x n grid,
    25 axis-aligned segments (C4 rules; seed and lengths chosen so the network has 2 667
    cells, the paper's 2 684), homogeneous Neumann boundaries, p_alpha^0 = 1,
    T = 0.002, N_T = 50, wells in the fracture cells whose host cell centre lies in
    [0.1,0.15]^2 or [0.6,0.65]x[0.85,0.9] with q_w = 1e5, p_w = 1.2.
    2C: matrix c=0.1, k=1; fracture c=1, k=1e6.  3C: matrix c=0.05,
    k=1e-3; natural fractures c=0.1, k=1; hydraulic fractures c=1, k=1e6.
    Readings (C26-C28): matrix-fracture transfer sigma = 4 k of the Omega
    continuum (EFM |E|/d with the SPEC.md:68 mean distance h/4); co-located
    sigma_12 = k_1; wells as injection q_w (p_w - p) on the fracture."""
    rng = np.random.default_rng(seed)
    cells, edges = fracture_network(n, rng, segments, lengths)
    h = 1.0 / n
    cy, cx = np.divmod(cells, n)
    xc, yc = (cx + 0.5) * h, (cy + 0.5) * h
    box = ((xc >= 0.1) & (xc <= 0.15) & (yc >= 0.1) & (yc <= 0.15)) | \
          ((xc >= 0.6) & (xc <= 0.65) & (yc >= 0.85) & (yc <= 0.9))
    well_q = np.where(box, 1e5, 0.0)
    if kind == "2C":
        omega = [dict(name="matrix", kind="grid", k=1.0, c=0.1, dirichlet=None, u0=1.0)]
        frac = dict(name="fracture", kind="fracture", k=1e6, c=1.0, dirichlet=None, u0=1.0,
                    well_q=well_q, well_p=1.2)
        couplings = [dict(a=0, b=1, type="embedded", sigma=np.full(len(cells), 4.0 * 1.0))]
    elif kind == "3C":
        omega = [dict(name="matrix", kind="grid", k=1e-3, c=0.05, dirichlet=None, u0=1.0),
                 dict(name="natural", kind="grid", k=1.0, c=0.1, dirichlet=None, u0=1.0)]
        frac = dict(name="fracture", kind="fracture", k=1e6, c=1.0, dirichlet=None, u0=1.0,
                    well_q=well_q, well_p=1.2)
        couplings = [dict(a=0, b=1, type="colocated", sigma=1e-3),
                     dict(a=0, b=2, type="embedded", sigma=np.full(len(cells), 4.0 * 1e-3)),
                     dict(a=1, b=2, type="embedded", sigma=np.full(len(cells), 4.0 * 1.0))]
    else:
        raise ValueError(kind)
    return dict(kind="fine", config_id=None, conv_version=CONV_VERSION, seed=seed, n=int(n), h=h,
                T=float(T), NT=int(NT), continua=omega + [frac],
                fracture=dict(cells=cells, edges=edges), couplings=couplings, paper_analogue=kind)


def crop_fine(scn: dict, m: int) -> dict:
    """The sub-square [0, m)^2 of a fine scenario: same cells (h unchanged), the k field,
    fracture cells hosted inside, fracture edges with both ends inside, their transfer
    coefficients; Dirichlet data on the crop's own left/right edges.  Used as a
    full-parity stand-in for config 4 ('parity unpinned' item (i))."""
    n = scn["n"]
    cells = scn["fracture"]["cells"]
    cy, cx = np.divmod(cells, n)
    keep = (cy < m) & (cx < m)
    new_id = np.full(len(cells), -1, dtype=np.int64)
    new_id[keep] = np.arange(int(keep.sum()))
    e = scn["fracture"]["edges"]
    ek = keep[e[:, 0]] & keep[e[:, 1]]
    edges = np.stack([new_id[e[ek, 0]], new_id[e[ek, 1]]], axis=1)
    continua = []
    for c in scn["continua"]:
        c = dict(c)
        if c["kind"] == "grid" and np.ndim(c["k"]) > 0:
            c["k"] = np.asarray(c["k"]).reshape(n, n)[:m, :m].ravel().copy()
        continua.append(c)
    couplings = []
    for cp in scn["couplings"]:
        cp = dict(cp)
        if cp["type"] == "embedded":
            cp["sigma"] = np.asarray(cp["sigma"])[keep].copy()
        couplings.append(cp)
    if not keep.any():
        continua = [c for c in continua if c["kind"] != "fracture"]
        couplings = [cp for cp in couplings if cp["type"] != "embedded"]
    return dict(scn, n=int(m), continua=continua, couplings=couplings, config_id=None,
                fracture=dict(cells=(cy[keep] * m + cx[keep]).astype(np.int64), edges=edges))


def make(config_id: int) -> dict:
    """The physical inputs of BASELINE.json configs[config_id]."""
    p = dict(CONFIGS[config_id])
    kind = p.pop("kind")
    if kind == "nlmc":
        return make_nlmc(**p, config_id=config_id)
    return make_fine(**p, config_id=config_id)
