"""GPU parity of the optional block-Jacobi preconditioner (mc_set_preconditioner,
SURVEY.md §8(f) rank 4): the same SPD systems are solved to the same recursive
tolerance, so the trajectories must match the oracle exactly as the Jacobi path does
(<= 1e-9 per continuum per step), with fewer CG iterations on the fracture network."""
import numpy as np
import pytest

from inputs import make, make_paper_analogue

pytestmark = pytest.mark.gpu


def _run(scn, scheme, steps, precond, ctas=0):
    from paper_2209_01158_b200 import Problem
    pb = Problem(scn, precond=precond, ctas=ctas)
    out, its = [], []
    for _ in range(steps):
        rep = pb.step(scheme)
        its.append(rep["iters"])
        out.append([t.cpu().numpy() for t in pb.state()])
    pb.close()
    return out, np.array(its)


@pytest.mark.parametrize("case,scheme,steps", [("cfg0", "D", 20), ("cfg1", "D", 3), ("pa2C", "D", 10),
                                               ("pa2C", "U", 10), ("pa3C", "L", 10), ("cfg0", "coupled", 3)])
def test_block_jacobi_parity(case, scheme, steps):
    from oracle import assemble as asm, schemes
    from paper_2209_01158_b200 import permeability_order
    scn = {"cfg0": lambda: make(0), "cfg1": lambda: make(1), "pa2C": lambda: make_paper_analogue("2C"),
           "pa3C": lambda: make_paper_analogue("3C")}[case]()
    sys_ = asm.assemble(scn)
    ref = schemes.run(sys_, scheme, scn["T"] / scn["NT"], steps, order_by_k=permeability_order(scn))
    got, its_b = _run(scn, scheme, steps, "block")
    worst = 0.0
    for n in range(steps):
        for a, r in enumerate(sys_.split(ref[n])):
            nr = np.linalg.norm(r)
            e = np.linalg.norm(got[n][a] - r) / nr if nr > 0 else float(np.abs(got[n][a]).max())
            worst = max(worst, e)
    assert worst <= 1e-9, worst
    if scheme != "coupled":
        _, its_j = _run(scn, scheme, steps, "jacobi")
        frac = len(scn["continua"]) - 1                     # the fracture network is the last continuum
        assert its_b[1:, frac].sum() < its_j[1:, frac].sum(), (its_b[:, frac], its_j[:, frac])


def test_preconditioner_state_and_fallback():
    """mc_set_preconditioner must precede mc_set_continuum; continua it does not apply to
    (grids, CSR graphs with per-edge T) keep Jacobi and give the same trajectory."""
    import ctypes as C
    from paper_2209_01158_b200 import Problem, mc
    scn = make(3)                                         # NLMC CSR graphs: not eligible
    a, _ = _run(scn, "D", 3, "block")
    b, _ = _run(scn, "D", 3, "jacobi")
    for x, y in zip(a, b):
        for u, v in zip(x, y):
            assert np.array_equal(u, v)
    pb = Problem(make(0))
    assert pb.lib.mc_set_preconditioner(pb.ctx, 1) == mc.MC_ERR_STATE
    assert pb.lib.mc_set_preconditioner(pb.ctx, 7) == mc.MC_ERR_ARG
    pb.close()


def test_block_jacobi_run_matches_steps():
    """mc_run (planning steps one at a time, then enqueued back to back: include/mc.h) gives
    bitwise the per-step result."""
    import torch
    from paper_2209_01158_b200 import Problem
    scn = make_paper_analogue("2C")
    a = Problem(scn, precond="block")
    reps = a.run("D", 5)
    ra = [t.cpu().numpy() for t in a.state()]
    b = Problem(scn, precond="block")
    for _ in range(5):
        b.step("D")
    rb = [t.cpu().numpy() for t in b.state()]
    for x, y in zip(ra, rb):
        assert np.array_equal(x, y)
    assert all(r["status"] == 0 for r in reps)
    a.close()
    b.close()


@pytest.mark.parametrize("kind,scheme,ctas", [("2C", "D", 4), ("3C", "U", 4), ("2C", "D", 1)])
def test_block_jacobi_streaming_parity(kind, scheme, ctas):
    """Networks too large to stay resident (here: 4 CTAs for 42 chunks) take the streaming
    block-Jacobi passes (run_group_bjs); same oracle trajectory.  ctas = 1: 8 warps for 42
    chunks, so every warp refills its staging slots (chunk m + 2W lands in slot 0 again and
    flips its mbarrier parity) under the parity check.  Both the block and the Jacobi run
    (the streaming iter_ells pass) are compared with the oracle."""
    from oracle import assemble as asm, schemes
    from paper_2209_01158_b200 import permeability_order
    scn = make_paper_analogue(kind)
    sys_ = asm.assemble(scn)
    steps = 8
    ref = schemes.run(sys_, scheme, scn["T"] / scn["NT"], steps, order_by_k=permeability_order(scn))
    got, its = _run(scn, scheme, steps, "block", ctas=ctas)
    got_j, its_j = _run(scn, scheme, steps, "jacobi", ctas=ctas)
    for g in (got, got_j):
        worst = 0.0
        for n in range(steps):
            for a, r in enumerate(sys_.split(ref[n])):
                worst = max(worst, np.linalg.norm(g[n][a] - r) / np.linalg.norm(r))
        assert worst <= 1e-9, worst
    assert its[1:, -1].sum() < its_j[1:, -1].sum()


def test_block_jacobi_streaming_three_stage_build():
    """The MC_BJS_STAGES=3 build (a third staging slot per warp in the streaming block-Jacobi
    passes: `% kStagesB` slot indexing, mbarrier parity flips on slot reuse) against the
    oracle at 1e-9, one CTA (8 warps for 42 chunks: every slot is refilled).  Runs in a fresh
    process because the library is chosen at load time (MC_LIB)."""
    import os
    import subprocess
    import sys
    from paper_2209_01158_b200 import build
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    lib = os.path.join(root, "paper_2209_01158_b200", "libmc_bjs3.so")
    srcs = [os.path.join(build.CSRC, f) for f in os.listdir(build.CSRC)]
    if not os.path.exists(lib) or any(os.path.getmtime(f) > os.path.getmtime(lib) for f in srcs):
        build.build(force=True, defines=["MC_BJS_STAGES=3"], out=lib)
    code = (
        "import sys, numpy as np\n"
        f"sys.path.insert(0, {root!r})\n"
        "from inputs import make_paper_analogue\n"
        "from oracle import assemble as asm, schemes\n"
        "from paper_2209_01158_b200 import Problem, permeability_order\n"
        "scn = make_paper_analogue('2C')\n"
        "sys_ = asm.assemble(scn)\n"
        "ref = schemes.run(sys_, 'D', scn['T'] / scn['NT'], 6, order_by_k=permeability_order(scn))\n"
        "pb = Problem(scn, precond='block', ctas=1)\n"
        "worst = 0.0\n"
        "for n in range(6):\n"
        "    rep = pb.step('D')\n"
        "    assert rep['paths'][1] == 4, rep['paths']\n"
        "    got = [t.cpu().numpy() for t in pb.state()]\n"
        "    for a, r in enumerate(sys_.split(ref[n])):\n"
        "        worst = max(worst, np.linalg.norm(got[a] - r) / np.linalg.norm(r))\n"
        "print('worst', worst)\n"
        "assert worst <= 1e-9, worst\n")
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, MC_LIB=lib), capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-1500:] + r.stderr[-1500:]
