"""Pins of the CPU oracle against things other than itself.

SPEC worked examples (tests/golden), closed forms (P2-P4), discrete
conservation (P5), first-order splitting (P6), special cases (P7, P8, P10),
stability (P9), structural invariants (P11), CG unit cases (P12) and brute
force by a literal dense re-assembly on tiny inputs (P1).
"""
import json
import os

import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from inputs import make, make_fine, make_nlmc
from oracle import assemble as asm
from oracle import cg as ocg
from oracle import schemes

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / (nb if nb > 0 else 1.0)


# ---------------------------------------------------------------- SPEC worked examples
def test_spec_tpfa_2x1():
    g = GOLD["tpfa_2x1"]
    D, M, F = asm.grid_continuum(g["nx"], g["ny"], g["h"], g["k"], 1.0, None)
    assert np.array_equal(D.toarray(), np.array(g["D"]))


def test_spec_tpfa_3x3():
    g = GOLD["tpfa_3x3_interior"]
    D, M, F = asm.grid_continuum(g["nx"], g["ny"], g["h"], g["k"], 1.0, None)
    Dd = D.toarray()
    assert Dd[g["interior_cell"], g["interior_cell"]] == pytest.approx(g["interior_diag"], rel=1e-15)
    assert np.allclose(Dd.sum(axis=1), 0.0, atol=1e-14)


def test_spec_tpfa_k0():
    g = GOLD["tpfa_k0"]
    D, M, F = asm.grid_continuum(g["nx"], g["ny"], g["h"], g["k"], 1.0, None)
    assert abs(D).sum() == 0.0


def test_spec_mass():
    g = GOLD["mass_single_cell"]
    D, M, F = asm.grid_continuum(g["nx"], g["ny"], g["h"], 1.0, g["c"], None)
    assert M[0] == pytest.approx(g["m"], rel=1e-15)


def test_spec_cg_cases():                                              # P12
    g = GOLD["cg_2x2"]
    x, it = ocg.jacobi_pcg(sp.csr_matrix(np.array(g["A"])), np.array(g["b"]), rtol=1e-14)
    assert np.allclose(x, g["x"], rtol=1e-14, atol=0)
    g = GOLD["cg_identity"]
    b = np.array(g["b"])
    x, it = ocg.jacobi_pcg(sp.identity(len(b), format="csr"), b, rtol=1e-14)
    assert np.array_equal(x, b) and it <= g["max_iterations"]
    x, it = ocg.jacobi_pcg(sp.identity(GOLD["cg_zero_rhs"]["n"], format="csr"),
                           np.zeros(GOLD["cg_zero_rhs"]["n"]), x0=np.ones(GOLD["cg_zero_rhs"]["n"]))
    assert it == 0 and np.array_equal(x, np.zeros(GOLD["cg_zero_rhs"]["n"]))


def _one_cell_system(c, sigma):
    # one cell per continuum, |cell| = 1, k = 0
    D = [sp.csr_matrix((1, 1)), sp.csr_matrix((1, 1))]
    Q = {(0, 1): sp.csr_matrix(np.array([[sigma]]))}
    return asm.block_system([1, 1], D, [np.array([c[0]]), np.array([c[1]])],
                            [np.zeros(1), np.zeros(1)], Q, [np.zeros(1), np.zeros(1)], ["a", "b"])


def test_spec_one_cell_two_continua():
    g = GOLD["one_cell_two_continua"]
    sys_ = _one_cell_system(g["c"], g["sigma"])
    uc = schemes.run(sys_, "coupled", g["tau"], 1, u0=np.array(g["u0"]))[0]
    ud = schemes.run(sys_, "D", g["tau"], 1, u0=np.array(g["u0"]))[0]
    assert np.allclose(uc, g["coupled"], rtol=1e-15, atol=1e-16)
    assert np.allclose(ud, g["decoupled_D"], rtol=1e-15, atol=1e-16)


def test_d_split_structure():
    sys_ = asm.assemble(make(0))
    A0, A1 = schemes.split_D(sys_)
    assert abs(A0 + A1 - sys_.A).max() == 0
    for a in range(sys_.L):
        s = sys_.block(a)
        assert abs(A1[s, s]).max() == 0 if A1[s, s].nnz else True
        for b in range(sys_.L):
            if a != b:
                assert A0[s, sys_.block(b)].nnz == 0


# ---------------------------------------------------------------- closed forms
def test_P2_linear_steady_state():
    n = 32
    D, M, F = asm.grid_continuum(n, n, 1.0 / n, 3.0, 1.0, (1.0, 0.0))
    u = spla.spsolve(sp.csc_matrix(D), F)
    x = (np.arange(n * n) % n + 0.5) / n
    assert np.max(np.abs(u - (1.0 - x))) <= 1e-12


def test_P3_layered_harmonic():
    n = 16
    rng = np.random.default_rng(7)
    kx = np.exp(rng.standard_normal(n))
    k = np.tile(kx, n)                                 # k depends on ix only
    gL, gR = 1.5, -0.25
    D, M, F = asm.grid_continuum(n, n, 1.0 / n, k, 1.0, (gL, gR))
    u = spla.spsolve(sp.csc_matrix(D), F)
    Tf = 2 * kx[:-1] * kx[1:] / (kx[:-1] + kx[1:])
    q = (gL - gR) / (1 / (2 * kx[0]) + np.sum(1 / Tf) + 1 / (2 * kx[-1]))
    col = np.empty(n)
    col[0] = gL - q / (2 * kx[0])
    for i in range(n - 1):
        col[i + 1] = col[i] - q / Tf[i]
    assert np.max(np.abs(u - np.tile(col, n))) <= 1e-12


@pytest.mark.parametrize("scheme", ["coupled", "D"])
def test_P4_0d_closed_forms(scheme):
    n, c1, c2, sig, tau = 4, 1.0, 0.1, 5.0, 0.05
    scn = make_fine(n, seed=0, T=1, NT=1, segments=0, lengths=(1, 1), c_m=c1,
                    natural=dict(k=1e2, c=c2, sigma_12=sig, sigma_2f=0.0), dirichlet=None)
    sys_ = asm.assemble(scn)
    a, b = 0.7, -0.3
    u = np.concatenate([np.full(n * n, a), np.full(n * n, b)])
    traj = schemes.run(sys_, scheme, tau, 12, u0=u)
    h2 = (1.0 / n) ** 2
    m1, m2, s = c1 * h2, c2 * h2, sig * h2
    G = np.array([[m1 / (m1 + tau * s), tau * s / (m1 + tau * s)],
                  [tau * s / (m2 + tau * s), m2 / (m2 + tau * s)]])
    v = np.array([a, b])
    for k, uk in enumerate(traj, start=1):
        u1, u2 = uk[: n * n], uk[n * n:]
        if scheme == "coupled":
            w = (a - b) / (1 + tau * s * (1 / m1 + 1 / m2)) ** k
            assert np.max(np.abs(u1 - u2 - w)) <= 1e-12
            assert abs(m1 * u1.mean() + m2 * u2.mean() - (m1 * a + m2 * b)) <= 1e-13 * (m1 + m2)
        else:
            v = G @ v
            assert np.max(np.abs(u1 - v[0])) <= 1e-12 and np.max(np.abs(u2 - v[1])) <= 1e-12


# ---------------------------------------------------------------- conservation and order
def _boundary_flux(scn, u_m):
    """tau-free boundary inflow sum_b T_b (g_b - u_b) for the grid continua (C3)."""
    n = scn["n"]
    k = scn["continua"][0]["k"]
    kk = np.full(n * n, float(k)) if np.ndim(k) == 0 else k
    ix = np.arange(n * n) % n
    gL, gR = scn["continua"][0]["dirichlet"]
    L, R = ix == 0, ix == n - 1
    flux = np.sum(2 * kk[L] * (gL - u_m[L])) + np.sum(2 * kk[R] * (gR - u_m[R]))
    gross = np.sum(np.abs(2 * kk[L] * (gL - u_m[L]))) + np.sum(np.abs(2 * kk[R] * (gR - u_m[R])))
    return flux, gross


@pytest.mark.parametrize("scheme", ["coupled", "D"])
def test_P5_mass_balance(scheme):
    scn = make(0)
    sys_ = asm.assemble(scn)
    tau = scn["T"] / scn["NT"]
    n, h = scn["n"], scn["h"]
    m = np.concatenate([np.full(n * n, scn["continua"][0]["c"] * h * h),
                        np.full(len(scn["fracture"]["cells"]), scn["continua"][1]["c"] * h)])
    host = scn["fracture"]["cells"]
    sig = scn["couplings"][0]["sigma"]
    traj = [sys_.u0] + schemes.run(sys_, scheme, tau, 20)
    for k in range(1, len(traj)):
        du = traj[k] - traj[k - 1]
        flux, gross = _boundary_flux(scn, traj[k][: n * n])
        rhs = tau * flux
        if scheme == "D":  # lag defect: -tau sum sigma (du_m(host) + du_f)
            rhs -= tau * np.sum(sig * (du[host] + du[n * n:]))
        assert abs(np.sum(m * du) - rhs) <= 1e-8 * tau * gross


def test_P6_first_order_in_tau():
    base = dict(make(0)["continua"][0])
    errs = []
    for NT in (100, 200, 400, 800):
        scn = make(0)
        T = 0.002                                         # the paper's T
        sys_ = asm.assemble(scn)
        uc = schemes.run(sys_, "coupled", T / NT, NT)[-1]
        ud = schemes.run(sys_, "D", T / NT, NT)[-1]
        errs.append(rel(ud, uc))
    ratios = [errs[i] / errs[i + 1] for i in range(3)]
    assert all(1.7 <= r <= 2.3 for r in ratios), ratios
    assert base["c"] == 1.0


def test_P7_sigma_zero_decouples():
    p = dict(n=64, seed=0, T=1.0, NT=10, segments=6, lengths=(10, 40), k_f=1e4, c_f=0.01,
             sigma_f=("const", 0.0))
    sys_ = asm.assemble(make_fine(**p))
    tc = schemes.run(sys_, "coupled", 0.1, 10)
    td = schemes.run(sys_, "D", 0.1, 10)
    for a, b in zip(tc, td):
        assert rel(b, a) <= 1e-12


@pytest.mark.parametrize("scheme", ["coupled", "D"])
def test_P8_constant_preserved(scheme):
    scn = make_fine(32, seed=3, T=1, NT=5, segments=5, lengths=(4, 12), k_sigma=1.0,
                    dirichlet=(1.0, 1.0))
    sys_ = asm.assemble(scn)
    for u in schemes.run(sys_, scheme, 0.2, 5, u0=np.ones(sum(sys_.sizes))):
        assert np.max(np.abs(u - 1.0)) <= 1e-9   # cond(K) ~ 1e9 here; SPEC.md:270 asks 1e-10 relative-ish


@pytest.mark.parametrize("scheme", ["coupled", "D"])
def test_P9_A_norm_monotone(scheme):
    scn = make_fine(32, seed=9, T=1, NT=30, segments=5, lengths=(4, 12), k_sigma=1.0,
                    dirichlet=(0.0, 0.0), sigma_f=("k_m", 100.0), k_f=1e4)
    sys_ = asm.assemble(scn)
    u0 = np.random.default_rng(2).standard_normal(sum(sys_.sizes))
    norms = [float(u0 @ (sys_.A @ u0))]
    for u in schemes.run(sys_, scheme, 1.0 / 30, 30, u0=u0):
        norms.append(float(u @ (sys_.A @ u)))
    for a, b in zip(norms[:-1], norms[1:]):
        assert b <= a * (1 + 1e-8)


def test_P9_nlmc_A_norm_monotone():
    scn = make_nlmc(8, seed=5)
    sys_ = asm.assemble(scn)
    mask = np.concatenate([d[0] for d in scn["dirichlet"]])
    sysz = asm.System(sys_.sizes, sys_.M, sys_.A, np.zeros_like(sys_.F), sys_.u0, sys_.names)
    u0 = np.random.default_rng(4).standard_normal(sum(sys_.sizes))
    u0[mask] = 0.0
    for scheme in ("coupled", "D"):
        prev = float(u0 @ (sysz.A @ u0))
        for u in schemes.run(sysz, scheme, 0.01, 20, u0=u0):
            cur = float(u @ (sysz.A @ u))
            assert cur <= prev * (1 + 1e-8)
            prev = cur


def test_P10_common_fixed_point():
    """A0 + A1 = A: the steady state A^{-1} F is a fixed point of both schemes."""
    scn = make(0)
    sys_ = asm.assemble(scn)
    steady = spla.spsolve(sp.csc_matrix(sys_.A), sys_.F)
    for scheme in ("coupled", "D"):
        for tau in (0.02, 50.0):
            nxt = schemes.run(sys_, scheme, tau, 1, u0=steady)[0]
            assert rel(nxt, steady) <= 1e-9
    # and the trajectories approach it
    dist = [rel(u, steady) for u in schemes.run(sys_, "D", 5.0, 60)[::10]]
    assert all(b < a for a, b in zip(dist[:-1], dist[1:]))


# ---------------------------------------------------------------- structure
@pytest.mark.parametrize("cid", [0, 3])
def test_P11_assembly_invariants(cid):
    scn = make(cid)
    sys_ = asm.assemble(scn)
    A = sys_.A
    assert abs(A - A.T).max() == 0.0
    if scn["kind"] == "fine":
        n = scn["n"]
        D, M, F = asm.grid_continuum(n, n, 1.0 / n, scn["continua"][0]["k"], 1.0, None)
        assert np.max(np.abs(D @ np.ones(n * n))) == 0.0           # D 1 = 0 before boundary terms
        scn_nb = dict(scn)
        scn_nb["continua"] = [dict(c, dirichlet=None) for c in scn["continua"]]
        A_nb = asm.assemble(scn_nb).A
        assert np.max(np.abs(A_nb @ np.ones(A.shape[0]))) <= 1e-9  # A 1 = 0
        s0, s1 = sys_.block(0), sys_.block(1)
        assert abs(A[s0, s1] - A[s1, s0].T).max() == 0.0            # Q_ba = Q_ab^T
        assert A[s0, s1].min() <= 0 and A[s0, s1].max() == 0        # off-diagonal blocks -Q
    rng = np.random.default_rng(0)
    for _ in range(5):                                              # PSD
        v = rng.standard_normal(A.shape[0])
        assert v @ (A @ v) >= -1e-10 * abs(A).max() * (v @ v)


# ---------------------------------------------------------------- P1 brute force
def dense_fine_bruteforce(scn):
    """Literal dense assembly by loops over cells / faces / fracture cells (Eq. app-md, app-tc)."""
    n, h = scn["n"], scn["h"]
    cont = scn["continua"]
    sizes = [n * n if c["kind"] == "grid" else len(scn["fracture"]["cells"]) for c in cont]
    off = np.concatenate([[0], np.cumsum(sizes)])
    N = off[-1]
    A = np.zeros((N, N))
    M = np.zeros(N)
    F = np.zeros(N)
    for a, c in enumerate(cont):
        if c["kind"] == "grid":
            kf = (lambda i: float(c["k"])) if np.ndim(c["k"]) == 0 else (lambda i: float(c["k"][i]))
            for iy in range(n):
                for ix in range(n):
                    i = iy * n + ix
                    M[off[a] + i] = c["c"] * h * h
                    for jy, jx in ((iy, ix - 1), (iy, ix + 1), (iy - 1, ix), (iy + 1, ix)):
                        if 0 <= jx < n and 0 <= jy < n:
                            j = jy * n + jx
                            if np.ndim(c["k"]) == 0:
                                T = float(c["k"]) * h / h
                            else:
                                T = 2 * kf(i) * kf(j) / (kf(i) + kf(j)) * h / h
                            A[off[a] + i, off[a] + i] += T
                            A[off[a] + i, off[a] + j] -= T
                        elif c["dirichlet"] is not None and jx in (-1, n):
                            g = c["dirichlet"][0] if jx == -1 else c["dirichlet"][1]
                            Tb = kf(i) * h / (h / 2)
                            A[off[a] + i, off[a] + i] += Tb
                            F[off[a] + i] += Tb * g
        else:
            cells = scn["fracture"]["cells"]
            for l in range(len(cells)):
                M[off[a] + l] = c["c"] * h
            for (l, m_) in scn["fracture"]["edges"]:
                T = c["k"] * 1.0 / h
                for (p, q) in ((l, m_), (m_, l)):
                    A[off[a] + p, off[a] + p] += T
                    A[off[a] + p, off[a] + q] -= T
    for cp in scn["couplings"]:
        a, b = cp["a"], cp["b"]
        if cp["type"] == "embedded":
            pairs = [(int(hc), l, cp["sigma"][l]) for l, hc in enumerate(scn["fracture"]["cells"])]
        else:
            pairs = [(i, i, cp["sigma"] * h * h) for i in range(n * n)]
        for i, j, s in pairs:
            A[off[a] + i, off[a] + i] += s
            A[off[b] + j, off[b] + j] += s
            A[off[a] + i, off[b] + j] -= s
            A[off[b] + j, off[a] + i] -= s
    return off, A, M, F


def dense_steps(off, A, M, F, tau, u, steps, scheme):
    out = []
    L = len(off) - 1
    for _ in range(steps):
        if scheme == "coupled":
            u = np.linalg.solve(np.diag(M / tau) + A, M / tau * u + F)
        else:
            new = np.empty_like(u)
            for a in range(L):
                s = slice(off[a], off[a + 1])
                b = M[s] / tau * u[s] + F[s]
                for c in range(L):
                    if c != a:
                        b -= A[s, off[c]:off[c + 1]] @ u[off[c]:off[c + 1]]
                new[s] = np.linalg.solve(np.diag(M[s] / tau) + A[s, s], b)
            u = new
        out.append(u.copy())
    return out


@pytest.mark.parametrize("three", [False, True])
@pytest.mark.parametrize("scheme", ["coupled", "D"])
def test_P1_bruteforce_fine(three, scheme):
    kw = dict(natural=dict(k=1e2, c=0.1, sigma_12=5.0, sigma_2f=50.0)) if three else {}
    scn = make_fine(4, seed=21 if three else 13, T=1, NT=6, segments=2, lengths=(2, 3),
                    k_sigma=1.0, k_f=1e4, c_f=0.01, sigma_f=("k_m", 100.0), **kw)
    off, A, M, F = dense_fine_bruteforce(scn)
    assert off[-1] <= 40
    sys_ = asm.assemble(scn)
    assert np.allclose(sys_.A.toarray(), A, rtol=1e-14, atol=1e-12)
    ref = dense_steps(off, A, M, F, 1.0 / 6, np.zeros(off[-1]), 6, scheme)
    got = schemes.run(sys_, scheme, 1.0 / 6, 6)
    for r, g in zip(ref, got):
        assert rel(g, r) <= 1e-13


def test_P1_bruteforce_nlmc():
    scn = make_nlmc(4, seed=17)
    nb = 16
    A = np.zeros((2 * nb, 2 * nb))
    for a, (i, j, t) in enumerate(scn["within"]):
        for p, q, v in zip(i, j, t):
            for (x, y) in ((p, q), (q, p)):
                A[a * nb + x, a * nb + x] += v
                A[a * nb + x, a * nb + y] -= v
    for p, q, v in zip(*scn["between"]):
        A[p, p] += v
        A[nb + q, nb + q] += v
        A[p, nb + q] -= v
        A[nb + q, p] -= v
    M = np.concatenate([np.full(nb, scn["c"][0]), np.full(nb, scn["c"][1])])
    F = np.zeros(2 * nb)
    u = np.zeros(2 * nb)
    mask = np.concatenate([d[0] for d in scn["dirichlet"]])
    g = np.concatenate([d[1] for d in scn["dirichlet"]])
    for d in np.nonzero(mask)[0]:                     # literal elimination, one column at a time
        for i in range(2 * nb):
            if not mask[i]:
                F[i] -= A[i, d] * g[d]
        A[:, d] = 0.0
        A[d, :] = 0.0
    for d in np.nonzero(mask)[0]:
        A[d, d] = 1.0
        F[d] = g[d]
        M[d] = 0.0
        u[d] = g[d]
    sys_ = asm.assemble(scn)
    assert np.allclose(sys_.A.toarray(), A, rtol=1e-15, atol=1e-15)
    for scheme in ("coupled", "D"):
        ref = dense_steps(np.array([0, nb, 2 * nb]), A, M, F, 0.01, u, 5, scheme)
        got = schemes.run(sys_, scheme, 0.01, 5)
        for r, gg in zip(ref, got):
            assert rel(gg, r) <= 1e-13


# ---------------------------------------------------------------- CG agreement / survey iterations
def test_cg_matches_splu_and_survey_iterations():
    scn = make(0)
    sys_ = asm.assemble(scn)
    tau = scn["T"] / scn["NT"]
    ds = schemes.DScheme(sys_, tau)
    K0 = sp.csr_matrix(sp.diags(sys_.M / tau) + ds.A0)
    u = sys_.u0.copy()
    its = {0: [], 1: []}
    for _ in range(50):
        b = ds.rhs(u)
        ref = ds.step(u)
        new = np.empty_like(u)
        for a in range(2):
            s = sys_.block(a)
            x, it = ocg.jacobi_pcg(K0[s, s], b[s], u[s], rtol=1e-12)
            its[a].append(it)
            nr = np.linalg.norm(ref[s])
            if nr == 0:
                assert np.array_equal(x, np.zeros_like(x))
            else:
                assert np.linalg.norm(x - ref[s]) / nr <= 1e-9
            new[s] = x
        u = new
    want = GOLD["survey_config0_iterations"]
    assert abs(its[0][0] - want["matrix_first"]) <= 2
    assert its[1][0] == want["fracture_first"]
    assert abs(np.mean(its[0]) - want["matrix_mean"]) <= 2
    assert abs(np.mean(its[1]) - want["fracture_mean"]) <= 2


def test_config0_gap_matches_survey():
    scn = make(0)
    sys_ = asm.assemble(scn)
    tau = scn["T"] / scn["NT"]
    tc = schemes.run(sys_, "coupled", tau, 50)
    td = schemes.run(sys_, "D", tau, 50)
    want = GOLD["survey_config0_iterations"]
    for n in (1, 10, 50):
        e = [schemes.rel_error_percent(sys_.split(tc[n - 1])[a], sys_.split(td[n - 1])[a]) for a in range(2)]
        assert abs(e[0] - want["gap_matrix_pct"][str(n)]) <= 1.0
        assert abs(e[1] - want["gap_fracture_pct"][str(n)]) <= 1.0


# ---------------------------------------------------------------- flux form and refinement
@pytest.mark.parametrize("cid", [0, 3])
def test_flux_form_assembles_to_A(cid):
    scn = make(cid)
    sys_ = asm.assemble(scn)
    tau = scn["T"] / scn["NT"]
    N = int(sys_.offsets[-1])
    K = sp.csr_matrix(sp.diags(sys_.M / tau) + sys_.A)
    op = sys_.flux.block_op(slice(0, N), sys_.M / tau, "coupled")
    assert abs(op.tocsr() - K).max() <= 1e-14 * abs(K).max()
    x = np.random.default_rng(1).standard_normal(N)
    assert np.linalg.norm(op.apply(x) - K @ x) <= 1e-13 * np.linalg.norm(K @ x)
    A0, _ = schemes.split_D(sys_)
    K0 = sp.csr_matrix(sp.diags(sys_.M / tau) + A0)
    for a in range(sys_.L):
        s = sys_.block(a)
        opa = sys_.flux.block_op(s, sys_.M / tau, "D")
        assert abs(opa.tocsr() - K0[s, s]).max() <= 1e-14 * abs(K0[s, s]).max()
        assert np.linalg.norm(opa.apply(x[s]) - K0[s, s] @ x[s]) <= 1e-13 * np.linalg.norm(K0[s, s] @ x[s])


def test_refinement_reaches_exact_fracture_plateau():
    """A fracture chain with T_f = k_f/h = 1e9 >> sigma = 1 over host cells held at u_m = 1:
    the D-scheme fracture solve is exactly p_f = sigma / (sigma + m_f/tau) on every cell
    (the flux terms vanish on a constant).  Assembling a_ii = 2 T + sigma + m/tau in fp64
    loses ~eps T / sigma ~ 1e-7 of sigma; the flux-form refinement must not (C15)."""
    n = 64
    scn = make_fine(n, seed=0, T=1, NT=1, segments=0, lengths=(1, 1), dirichlet=None)
    cells = np.arange(5 * n + 3, 5 * n + 53)                    # 50 cells along row 5
    scn["fracture"] = dict(cells=cells, edges=np.stack([np.arange(49), np.arange(1, 50)], 1))
    scn["continua"].append(dict(name="fracture", kind="fracture", k=1e9 / n, c=0.01, dirichlet=None))
    scn["couplings"] = [dict(a=0, b=1, type="embedded", sigma=np.ones(50))]
    sys_ = asm.assemble(scn)
    tau = 0.5
    u = np.concatenate([np.ones(n * n), np.zeros(50)])
    uf = schemes.run(sys_, "D", tau, 1, u0=u)[0][n * n:]
    mt = 0.01 * (1.0 / n) / tau
    assert np.max(np.abs(uf - 1.0 / (1.0 + mt))) <= 1e-15


# ---------------------------------------------------------------- L- and U-schemes
def test_LU_one_cell_worked_example():
    g = GOLD["one_cell_two_continua_LU"]
    base = GOLD["one_cell_two_continua"]
    sys_ = _one_cell_system(base["c"], base["sigma"])
    for k in ("L", "U"):
        u = schemes.run(sys_, k, base["tau"], 1, u0=np.array(base["u0"]), order_by_k=g["order_by_k"])[0]
        assert np.allclose(u, g[k], rtol=1e-15, atol=1e-16)


@pytest.mark.parametrize("kind", ["L", "U"])
def test_LU_0d_closed_form(kind):
    n, c1, c2, sig, tau = 4, 1.0, 0.1, 5.0, 0.05
    scn = make_fine(n, seed=0, T=1, NT=1, segments=0, lengths=(1, 1), c_m=c1,
                    natural=dict(k=1e2, c=c2, sigma_12=sig, sigma_2f=0.0), dirichlet=None)
    sys_ = asm.assemble(scn)
    a, b = 0.7, -0.3
    u = np.concatenate([np.full(n * n, a), np.full(n * n, b)])
    traj = schemes.run(sys_, kind, tau, 10, u0=u, order_by_k=[0, 1])
    h2 = (1.0 / n) ** 2
    m1, m2, s = c1 * h2, c2 * h2, sig * h2
    v1, v2 = a, b
    for uk in traj:
        if kind == "L":                 # continuum 0 first (old v2), then 1 with the new v1
            v1 = (m1 * v1 + tau * s * v2) / (m1 + tau * s)
            v2 = (m2 * v2 + tau * s * v1) / (m2 + tau * s)
        else:                           # continuum 1 first, then 0 with the new v2
            v2 = (m2 * v2 + tau * s * v1) / (m2 + tau * s)
            v1 = (m1 * v1 + tau * s * v2) / (m1 + tau * s)
        assert np.max(np.abs(uk[: n * n] - v1)) <= 1e-12 and np.max(np.abs(uk[n * n:] - v2)) <= 1e-12


def dense_seq_steps(off, A, M, F, tau, u, steps, order):
    """Literal block Gauss-Seidel in `order` on a dense system (brute force for L/U)."""
    out = []
    L = len(off) - 1
    for _ in range(steps):
        new = u.copy()
        for a in order:
            s = slice(off[a], off[a + 1])
            b = M[s] / tau * u[s] + F[s]
            for c in range(L):
                if c != a:
                    b -= A[s, off[c]:off[c + 1]] @ new[off[c]:off[c + 1]]
            new[s] = np.linalg.solve(np.diag(M[s] / tau) + A[s, s], b)
        u = new
        out.append(u.copy())
    return out


@pytest.mark.parametrize("kind", ["L", "U"])
def test_LU_bruteforce_three_continua(kind):
    scn = make_fine(4, seed=21, T=1, NT=6, segments=2, lengths=(2, 3), k_sigma=1.0, k_f=1e4, c_f=0.01,
                    sigma_f=("k_m", 100.0), natural=dict(k=1e2, c=0.1, sigma_12=5.0, sigma_2f=50.0))
    off, A, M, F = dense_fine_bruteforce(scn)
    order = [0, 1, 2]                                   # k: matrix 1 < natural 1e2 < fracture 1e4
    ref = dense_seq_steps(off, A, M, F, 1.0 / 6, np.zeros(off[-1]), 6, order if kind == "L" else order[::-1])
    got = schemes.run(asm.assemble(scn), kind, 1.0 / 6, 6, order_by_k=order)
    for r, g in zip(ref, got):
        assert rel(g, r) <= 1e-13


def test_LU_sigma_zero_equal_coupled():
    p = dict(n=64, seed=0, T=1.0, NT=10, segments=6, lengths=(10, 40), k_f=1e4, c_f=0.01,
             sigma_f=("const", 0.0))
    sys_ = asm.assemble(make_fine(**p))
    tc = schemes.run(sys_, "coupled", 0.1, 5)
    for k in ("L", "U"):
        for a, b in zip(tc, schemes.run(sys_, k, 0.1, 5, order_by_k=[0, 1])):
            assert rel(b, a) <= 1e-12


@pytest.mark.parametrize("kind", ["L", "U"])
def test_LU_A_norm_monotone(kind):                       # Theorem 3 holds for L/U
    scn = make_fine(32, seed=9, T=1, NT=30, segments=5, lengths=(4, 12), k_sigma=1.0,
                    dirichlet=(0.0, 0.0), sigma_f=("k_m", 100.0), k_f=1e4)
    sys_ = asm.assemble(scn)
    u0 = np.random.default_rng(2).standard_normal(sum(sys_.sizes))
    prev = float(u0 @ (sys_.A @ u0))
    for u in schemes.run(sys_, kind, 1.0 / 30, 30, u0=u0, order_by_k=[0, 1]):
        cur = float(u @ (sys_.A @ u))
        assert cur <= prev * (1 + 1e-8)
        prev = cur


@pytest.mark.parametrize("kind", ["L", "U"])
def test_LU_mass_balance(kind):
    """Summing the rows: sum m du = tau [boundary inflow - sum over LAGGED transfer entries of
    sigma * du(of the continuum solved later)] — only the lagged half of Q leaves a defect."""
    scn = make(0)
    sys_ = asm.assemble(scn)
    tau = scn["T"] / scn["NT"]
    n, h = scn["n"], scn["h"]
    m = np.concatenate([np.full(n * n, scn["continua"][0]["c"] * h * h),
                        np.full(len(scn["fracture"]["cells"]), scn["continua"][1]["c"] * h)])
    host = scn["fracture"]["cells"]
    sig = scn["couplings"][0]["sigma"]
    traj = [sys_.u0] + schemes.run(sys_, kind, tau, 20, order_by_k=[0, 1])
    for k in range(1, len(traj)):
        du = traj[k] - traj[k - 1]
        flux, gross = _boundary_flux(scn, traj[k][: n * n])
        # L: matrix (0) first -> its rows lag the fracture: defect sigma * du_fracture
        # U: fracture first -> its rows lag the matrix: defect sigma * du_matrix(host)
        lag = du[n * n:] if kind == "L" else du[host]
        rhs = tau * flux - tau * np.sum(sig * lag)
        assert abs(np.sum(m * du) - rhs) <= 1e-8 * tau * gross


@pytest.mark.parametrize("kind", ["L", "U"])
def test_LU_first_order_in_tau(kind):
    errs = []
    for NT in (100, 200, 400, 800):
        sys_ = asm.assemble(make(0))
        T = 0.002
        uc = schemes.run(sys_, "coupled", T / NT, NT)[-1]
        ud = schemes.run(sys_, kind, T / NT, NT, order_by_k=[0, 1])[-1]
        errs.append(rel(ud, uc))
    ratios = [errs[i] / errs[i + 1] for i in range(3)]
    assert all(1.7 <= r <= 2.3 for r in ratios), ratios


def test_U_more_accurate_than_D_paper_pattern():
    """PAPER.md:956 (and Tables 1-4): the U-scheme is the most accurate decoupled scheme.
    Checked on config-0 inputs at the paper's T = 0.002."""
    sys_ = asm.assemble(make(0))
    T, NT = 0.002, 50
    uc = schemes.run(sys_, "coupled", T / NT, NT)[-1]
    e = {k: rel(schemes.run(sys_, k, T / NT, NT, order_by_k=[0, 1])[-1], uc) for k in ("D", "L", "U")}
    assert e["U"] < e["D"], e


# ---------------------------------------------------------------- wells (paper analogue)
def test_wells_bruteforce_and_mass_balance():
    """Well term f = q_w (p_w - p) on fracture cells (SPEC.md:154 sign): a literal dense
    re-assembly adds q_w |iota| to the diagonal and q_w p_w |iota| to F; the discrete mass
    balance then reads sum m du = tau sum_wells q_w |iota| (p_w - p^n) (coupled, Neumann)."""
    from inputs import make_paper_analogue
    scn = make_paper_analogue("2C", n=8, seed=3, segments=3, lengths=(3, 6), NT=5)
    fr = scn["continua"][1]
    fr["well_q"] = np.zeros(len(scn["fracture"]["cells"]))
    fr["well_q"][:2] = 1e3
    off, A, M, F = dense_fine_bruteforce(dict(scn, continua=[dict(c, dirichlet=None) for c in scn["continua"]]))
    h = scn["h"]
    for l in range(2):
        A[off[1] + l, off[1] + l] += 1e3 * h
        F[off[1] + l] += 1e3 * h * 1.2
    sys_ = asm.assemble(scn)
    assert np.allclose(sys_.A.toarray(), A, rtol=1e-14, atol=1e-10)
    assert np.allclose(sys_.F, F, rtol=1e-15, atol=0)
    tau = scn["T"] / scn["NT"]
    u0 = sys_.u0.copy()
    assert np.all(u0 == 1.0)
    ref = dense_steps(off, A, M, F, tau, u0, 5, "coupled")
    got = schemes.run(sys_, "coupled", tau, 5)
    for r, g in zip(ref, got):   # dense LU in fp64 on a k_f = 1e6 system: cond * eps ~ 1e-12
        assert rel(g, r) <= 1e-10
    prev = u0
    for u in got:
        inflow = np.sum(1e3 * h * (1.2 - u[off[1]:off[1] + 2]))
        assert abs(np.sum(M * (u - prev)) - tau * inflow) <= 1e-9 * tau * abs(inflow)
        prev = u


def test_paper_analogue_table_shape():
    """PAPER.md Tables 1-2 / Fig. 4 pattern on the synthetic paper-analogue 2C problem:
    every decoupled scheme within 1 % of the coupled solution at T, U-scheme the most
    accurate."""
    from inputs import make_paper_analogue
    scn = make_paper_analogue("2C")
    sys_ = asm.assemble(scn)
    tau = scn["T"] / scn["NT"]
    uc = schemes.run(sys_, "coupled", tau, scn["NT"])[-1]
    e = {k: 100 * rel(schemes.run(sys_, k, tau, scn["NT"], order_by_k=[0, 1])[-1], uc) for k in ("L", "D", "U")}
    assert all(v < 1.0 for v in e.values()), e
    assert e["U"] < e["D"] and e["U"] < e["L"], e
