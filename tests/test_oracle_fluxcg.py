"""Pins of the C Jacobi-PCG oracle (oracle/flux_pcg.c via oracle/fluxcg.py) -- the
oracle leg for the sizes SuperLU cannot take (configs 2 and 4).

Pinned against things other than itself: SPEC's CG worked examples (tests/golden),
dense brute-force solves of random flux-form operators, the SuperLU + refinement
oracle (a direct method, pinned by tests/test_oracle_pins.py) on configs 0, 1 and 3,
the survey's independently measured CG iteration counts, and the exact M, F, lagged
transfer of the assembled oracle system.
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from inputs import make
from oracle import assemble as asm
from oracle import fluxcg, schemes

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worst(ref, got, sys_):
    w = 0.0
    for r, g in zip(ref, got):
        for a in range(sys_.L):
            s = sys_.block(a)
            nr = np.linalg.norm(r[s])
            w = max(w, np.linalg.norm(g[s] - r[s]) / nr if nr > 0 else float(np.abs(g[s]).max()))
    return w


def test_spec_cg_cases():
    """SPEC.md:190-192 through the C library.  [[4,1],[1,3]] in flux form: d = (5, 4),
    one connection t = -1 (K_00 = d_0 + t = 4, K_01 = -t = 1)."""
    g = GOLD["cg_2x2"]
    op = fluxcg.FluxOp(2, [5.0, 4.0], [0], [1], [-1.0])
    assert np.allclose(op.diagonal(), np.diag(g["A"]), rtol=0, atol=0)
    x = op.solve(g["b"], [0.0, 0.0], rtol=1e-14)
    assert np.allclose(x, g["x"], rtol=1e-14, atol=0)
    b = np.array(GOLD["cg_identity"]["b"])
    op = fluxcg.FluxOp(len(b), np.ones(len(b)), [], [], [])
    x = op.solve(b, np.zeros(len(b)), rtol=1e-14)
    assert np.array_equal(x, b) and op.iters[-1] <= GOLD["cg_identity"]["max_iterations"]
    n = GOLD["cg_zero_rhs"]["n"]
    op = fluxcg.FluxOp(n, np.ones(n), [0], [1], [2.0])
    x = op.solve(np.zeros(n), np.ones(n))
    assert op.iters[-1] == 0 and np.array_equal(x, np.zeros(n))


@pytest.mark.parametrize("seed", range(4))
def test_bruteforce_random_flux_operators(seed):
    """Random graphs with positive t and d > 0: K is an SPD M-matrix.  Operator entries
    by a literal dense loop; solution by numpy.linalg.solve (forward error bounded by
    cond(K) times the stopping tolerance)."""
    rng = np.random.default_rng(seed)
    n = int(rng.integers(5, 40))
    E = int(rng.integers(n, 3 * n))
    ei = rng.integers(0, n, E)
    ej = rng.integers(0, n, E)
    keep = ei != ej
    ei, ej = ei[keep], ej[keep]
    et = rng.uniform(0.1, 10.0, len(ei)) * 10.0 ** rng.integers(-1, 3, len(ei))
    d = rng.uniform(0.1, 1.0, n)
    K = np.diag(d.astype(float))
    for i, j, t in zip(ei, ej, et):
        K[i, i] += t
        K[j, j] += t
        K[i, j] -= t
        K[j, i] -= t
    op = fluxcg.FluxOp(n, d, ei, ej, et)
    x = rng.standard_normal(n)
    assert np.allclose(op.apply(x), K @ x, rtol=1e-13, atol=1e-13 * np.abs(K).max())
    assert np.allclose(op.diagonal(), np.diag(K), rtol=1e-15, atol=0)
    b = rng.standard_normal(n)
    got = op.solve(b, np.zeros(n), rtol=1e-14)
    ref = np.linalg.solve(K, b)
    assert np.linalg.norm(K @ got - b) <= 1e-13 * np.linalg.norm(b) * 10
    assert np.linalg.norm(got - ref) <= 1e-13 * np.linalg.cond(K) * np.linalg.norm(ref)


def test_breakdown_and_noconv_are_reported():
    op = fluxcg.FluxOp(2, [-1.0, -1.0], [], [], [])              # negative definite
    with pytest.raises(fluxcg.CGBreakdown):
        op.solve([1.0, 1.0], [0.0, 0.0])
    n = 50
    op = fluxcg.FluxOp(n, np.r_[1e-6, np.zeros(n - 1)], np.arange(n - 1), np.arange(1, n), np.ones(n - 1))
    with pytest.raises(fluxcg.CGNoConvergence):
        op.solve(np.ones(n), np.zeros(n), maxit=3)


@pytest.mark.parametrize("cid", [0, 1, 3])
def test_lean_assembly_and_lagged_transfer(cid):
    """assemble_lean gives bitwise the M, F, u0 of the assembled system; the flux form's
    lagged transfer equals -A1 u of the assembled split."""
    scn = make(cid)
    sys_ = asm.assemble(scn)
    if scn["kind"] == "fine":
        lean = asm.assemble_lean(scn)
        assert np.array_equal(lean.M, sys_.M) and np.array_equal(lean.F, sys_.F)
        assert np.array_equal(lean.u0, sys_.u0) and lean.sizes == sys_.sizes
    _, A1 = schemes.split_D(sys_)
    u = np.random.default_rng(cid).standard_normal(len(sys_.M))
    ref = -(A1 @ u)
    assert np.abs(sys_.flux.lagged_transfer(u) - ref).max() <= 1e-14 * max(1.0, np.abs(ref).max())


@pytest.mark.parametrize("scheme", ["D", "coupled"])
def test_matches_splu_config0(scheme):
    """Full 50-step trajectory of config 0 against the SuperLU + refinement oracle."""
    scn = make(0)
    sys_ = asm.assemble(scn)
    tau = scn["T"] / scn["NT"]
    ref = schemes.run(sys_, scheme, tau, 50)
    got, _ = fluxcg.run(asm.assemble_lean(scn), scheme, tau, 50)
    assert _worst(ref, got, sys_) <= 1e-10


def test_matches_splu_config3():
    """NLMC coarse system (identity Dirichlet rows, C12), D-scheme, 3 steps (the coupled
    131k-row SuperLU factorisation alone takes ~100 s; config 0 covers coupled)."""
    scn = make(3)
    sys_ = asm.assemble(scn)
    tau = scn["T"] / scn["NT"]
    ref = schemes.run(sys_, "D", tau, 3)
    got, _ = fluxcg.run(sys_, "D", tau, 3)
    assert _worst(ref, got, sys_) <= 1e-10


@pytest.mark.slow
def test_matches_splu_config1_D():
    """Config 1, D-scheme steps 1-3 (fracture: 0, ~21k, ~19k iterations)."""
    scn = make(1)
    sys_ = asm.assemble(scn)
    tau = scn["T"] / scn["NT"]
    ref = schemes.run(sys_, "D", tau, 3)
    got, st = fluxcg.run(asm.assemble_lean(scn), "D", tau, 3)
    assert _worst(ref, got, sys_) <= 1e-10
    assert st.iters[1][0] == 0 and st.iters[1][1] > 10000


def test_survey_iteration_counts_config0():
    """SURVEY.md App. A item 2 (an independent SciPy Jacobi-PCG on the ASSEMBLED K,
    rtol 1e-12): D-scheme matrix 238 first / 206.5 mean, fracture 0 first / 170.4 mean
    over 50 steps.  The flux form rounds differently (C15), and the fracture systems
    (T_f / sigma ~ 6e4) make the count sensitive to rounding (C16): 5 % band."""
    scn = make(0)
    lean = asm.assemble_lean(scn)
    _, st = fluxcg.run(lean, "D", scn["T"] / scn["NT"], 50, rtols=[1e-12, 1e-12])
    want = GOLD["survey_config0_iterations"]
    its = st.iters
    assert abs(its[0][0] - want["matrix_first"]) <= 2
    assert its[1][0] == want["fracture_first"]
    assert abs(np.mean(its[0]) - want["matrix_mean"]) <= 0.05 * want["matrix_mean"]
    assert abs(np.mean(its[1]) - want["fracture_mean"]) <= 0.05 * want["fracture_mean"]


def test_thread_count_independent():
    """Fixed-order dot products: 1 and 3 OpenMP threads give bitwise the same solution."""
    code = ("import sys; sys.path.insert(0, %r)\n"
            "import numpy as np\nfrom inputs import make\nfrom oracle import assemble as asm, fluxcg\n"
            "scn = make(0)\ngot, _ = fluxcg.run(asm.assemble_lean(scn), 'D', 0.02, 3)\n"
            "sys.stdout.write(got[-1].tobytes().hex())\n") % ROOT
    outs = []
    for t in ("1", "3"):
        env = dict(os.environ, OMP_NUM_THREADS=t)
        outs.append(subprocess.run([sys.executable, "-c", code], env=env, capture_output=True,
                                   text=True, check=True).stdout)
    assert outs[0] == outs[1] and len(outs[0]) > 1000
