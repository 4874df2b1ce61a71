#!/usr/bin/env python
"""Evidence for the tolerance disclosure C25: on config 4's [0,512)^2 crop the
TEXTBOOK Jacobi-PCG of the oracle (oracle/flux_pcg.c: two reductions per iteration, no
recurrence for r.z), stopped at recursive relres 1e-12, is compared with the SuperLU +
long-double-refinement oracle.  If it misses 1e-9 on the matrix continuum as well, the GPU's
need for rtol 1e-13 there is a property of the system (k = exp(2Z)), not of the GPU's
single-reduction recurrence.  CPU only, oracle only.

    python tests/tools/c25_textbook_pcg.py --out profiles/r02_c25_textbook_pcg.json
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from inputs import crop_fine, make          # noqa: E402
from oracle import assemble as asm, fluxcg, schemes   # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--out", default=None)
ap.add_argument("--steps", type=int, default=4)
args = ap.parse_args()
scn = crop_fine(make(4), 512)
tau = scn["T"] / scn["NT"]
sys_ = asm.assemble(scn)
ref = schemes.run(sys_, "D", tau, args.steps)
rows = []
for rt in (1e-12, 1e-13):
    got, st = fluxcg.run(asm.assemble_lean(scn), "D", tau, args.steps, rtols=[rt, 1e-12])
    for n in range(args.steps):
        e = []
        for a in range(sys_.L):
            s = sys_.block(a)
            nr = np.linalg.norm(ref[n][s])
            e.append(float(np.linalg.norm(got[n][s] - ref[n][s]) / nr) if nr > 0 else float(np.abs(got[n][s]).max()))
        rows.append({"matrix_rtol": rt, "step": n + 1, "rel_l2_vs_superlu": e,
                     "iters": [st.iters[a][n] for a in range(sys_.L)]})
        print(json.dumps(rows[-1]), flush=True)
if args.out:
    json.dump({"scenario": "config 4 cropped to [0,512)^2 (h = 1/8192 kept), D-scheme, textbook Jacobi-PCG oracle vs SuperLU oracle",
               "rows": rows}, open(args.out, "w"), indent=1)
