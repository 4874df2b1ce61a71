"""Checked-build / compute-sanitizer target: a few steps of one case
through the C ABI.
    MC_LIB=paper_2209_01158_b200/libmc_check.so python scripts/sanitize_target.py CASE
    compute-sanitizer --tool memcheck python scripts/sanitize_target.py CASE
With the checked build (-DMC_CHECK=1: device-side bounds asserts, guard bytes behind every
device array) the script ends by calling mc_debug_check and fails on a corrupted guard.
Cases: cfg0 (config 0, D + coupled + U), cfg3 (config 3 NLMC operator, D + coupled),
ell_stream (config-1 recipe at 256^2 with 4 CTAs: the streaming Jacobi ELL pass),
bjs (paper analogue, block-Jacobi, 4 CTAs: the streaming block-Jacobi passes), bj (resident),
run (mc_run batches with snapshots), nlmc (a small NLMC build)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from inputs import CONFIGS, make, make_fine, make_paper_analogue
from paper_2209_01158_b200 import Problem

case = sys.argv[1]
if case == "cfg0":
    pb = Problem(make(0))
    for scheme, n in (("D", 3), ("coupled", 2), ("U", 2)):
        for _ in range(n):
            print(case, scheme, pb.step(scheme)["iters"], flush=True)
elif case == "cfg3":
    pb = Problem(make(3))
    for scheme, n in (("D", 2), ("coupled", 1)):
        for _ in range(n):
            print(case, scheme, pb.step(scheme)["iters"], flush=True)
elif case == "ell_stream":
    p = dict(CONFIGS[1])
    p.pop("kind")
    p.update(n=256, segments=100, lengths=(12, 100))
    pb = Problem(make_fine(**p), ctas=4)
    for _ in range(3):
        rep = pb.step("D")
        print(case, rep["iters"], rep["paths"], flush=True)
    print(case, "coupled", pb.step("coupled")["iters"], flush=True)
elif case in ("bjs", "bj"):
    pb = Problem(make_paper_analogue("2C"), precond="block", ctas=4 if case == "bjs" else 0)
    for _ in range(3):
        rep = pb.step("D")
        print(case, rep["iters"], rep["paths"], flush=True)
elif case == "run":
    pb = Problem(make(0))
    snaps = [[torch.empty(s, dtype=torch.float64, device="cuda") for s in pb.sizes] for _ in range(8)]
    reps = pb.run("D", 8, snapshots=snaps)
    print(case, [r["iters"] for r in reps], flush=True)
elif case == "nlmc":
    pb = Problem(make_paper_analogue("2C", n=40, segments=4, lengths=(10, 25), seed=5))
    sp_ = pb.nlmc(8, 8, 1)
    print(case, sp_.sizes, sp_.nnz, flush=True)
    sp_.close()
else:
    raise SystemExit(f"unknown case {case}")
torch.cuda.synchronize()
if hasattr(pb.lib, "mc_debug_check"):
    bad = pb.lib.mc_debug_check(pb.ctx)
    print(case, "guards corrupted:", bad, flush=True)
    assert bad == 0, bad
pb.close()
print(case, "done", flush=True)
