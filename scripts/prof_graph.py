"""Dev: one continuum of a config alone (random state), capped solves (ncu / A-B target).
    python scripts/prof_graph.py CONFIG MAXIT [fracture|grid] [CTAS]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from inputs import make
from paper_2209_01158_b200 import Problem, MCError

cid, maxit = int(sys.argv[1]), int(sys.argv[2])
kind = sys.argv[3] if len(sys.argv) > 3 else "fracture"
ctas = int(sys.argv[4]) if len(sys.argv) > 4 else 0
scn = make(cid)
scn = dict(scn, continua=[c for c in scn["continua"] if c["kind"] == kind][:1], couplings=[])
pb = Problem(scn, maxit=maxit, ctas=ctas)
g = torch.Generator(device="cuda").manual_seed(0)
pb.set_state(0, torch.rand(pb.sizes[0], dtype=torch.float64, device="cuda", generator=g))
for _ in range(2):
    try:
        rep = pb.step("D")
    except MCError as e:
        rep = e.report
    print(f"cfg{cid} {kind} ctas={ctas or 'all'}", rep["iters"], "ms/iter %.4f" % (rep["ms_solve"][0] / max(1, rep["iters"][0])), flush=True)
