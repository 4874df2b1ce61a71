"""Dev: run a few capped step kernels of a config (target for ncu). Usage:
    python scripts/prof_step.py CONFIG SCHEME MAXIT STEPS [segments_override]"""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from inputs import make, CONFIGS, make_fine
from paper_2209_01158_b200 import Problem, MCError

cid, scheme, maxit, steps = int(sys.argv[1]), sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
if len(sys.argv) > 5:
    p = dict(CONFIGS[cid]); p.pop("kind"); p["segments"] = int(sys.argv[5]); scn = make_fine(**p)
else:
    scn = make(cid)
pb = Problem(scn, maxit=maxit)
for s in range(steps):
    t = time.time()
    try:
        rep = pb.step(scheme)
    except MCError as e:
        rep = e.report
    print(s, rep["iters"], rep["ms_solve"], rep["ms"], flush=True)
pb.close()
