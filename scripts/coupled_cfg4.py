"""Config 4's coupled comparator, "timed for comparison" (BASELINE.json configs[4];
SURVEY.md H5): one coupled step capped at MAXIT CG iterations (a full coupled solve
needs ~1e6 Jacobi-PCG iterations at 8192^2), reporting the time per iteration and the
recursive relative residual reached, next to the D-scheme step's per-iteration times.
    python scripts/coupled_cfg4.py [MAXIT] [--out FILE]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from inputs import make
from paper_2209_01158_b200 import Problem, MCError

maxit = int(sys.argv[1]) if len(sys.argv) > 1 and not sys.argv[1].startswith("--") else 400
out = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else None
scn = make(4)
res = {"workload": "config4: 8192^2 2C fine FV, lognormal k", "dof": None}
pb = Problem(scn, maxit=maxit, rtols=[1e-13, 1e-12])
res["dof"] = sum(pb.sizes)
for scheme in ("coupled", "D"):
    try:
        rep = pb.step(scheme)
    except MCError as e:
        rep = e.report
    its = rep["iters"]
    res[scheme] = dict(iters=its, relres=rep["relres"], ms_solve=rep["ms_solve"],
                       ms_per_iteration=[m / max(1, i) for m, i in zip(rep["ms_solve"], its)],
                       status=rep["status"])
    print(scheme, json.dumps(res[scheme]), flush=True)
pb.close()
if out:
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
