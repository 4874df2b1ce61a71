"""Dev: capped step kernels of a config as an ncu target.
    python scripts/prof_step.py CONFIG SCHEME MAXIT STEPS [PRECOND]
Runs STEPS full steps on one context, then one step capped at MAXIT iterations per
solve on a second context started from that state (the profiled launch)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from inputs import make
from paper_2209_01158_b200 import Problem, MCError

cid, scheme, maxit, steps = int(sys.argv[1]), sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
precond = sys.argv[5] if len(sys.argv) > 5 else "jacobi"
scn = make(cid)
pb = Problem(scn, precond=precond)
for s in range(steps):
    rep = pb.step(scheme)
    print("full", s, rep["iters"], rep["ms_solve"], rep["ms"], flush=True)
state = [t.clone() for t in pb.state()]
pb.close()
pc = Problem(scn, maxit=maxit, precond=precond)
for a, t in enumerate(state):
    pc.set_state(a, t)
try:
    rep = pc.step(scheme)
except MCError as e:
    rep = e.report
print("capped", rep["iters"], rep["ms_solve"], rep["ms"], flush=True)
