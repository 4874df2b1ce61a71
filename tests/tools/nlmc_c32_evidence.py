#!/usr/bin/env python
"""Evidence for reading C32: the literal coarse operator Dbar = R D R^T
 against its flux (finite-volume) form -- off-diagonals of R D R^T,
diagonal = -(their row sum) + the aggregated boundary terms -- on the paper analogue
(§5: 200^2 fine grid, 2C, wells, T = 0.002, 50 steps, 20 x 20 coarse cells).

CPU only, oracle only (test infrastructure): both variants are stepped by the oracle's
coupled scheme and compared with the averaged fine coupled solution.

    python tests/tools/nlmc_c32_evidence.py --out profiles/r02_nlmc_c32.json
"""
import argparse
import json
import os
import sys

import numpy as np
import scipy.sparse as sp

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from inputs import make_paper_analogue          # noqa: E402
from oracle import assemble as asm, nlmc, schemes   # noqa: E402
from oracle.assemble import System              # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--out", default=None)
ap.add_argument("--coarse", type=int, default=20)
args = ap.parse_args()

scn = make_paper_analogue("2C")
sys_ = asm.assemble(scn)
tau = scn["T"] / scn["NT"]
fine = schemes.run(sys_, "coupled", tau, scn["NT"])
rows = []
for m in (1, 2, 3, args.coarse):                 # m = coarse: full oversampling (K_i^+ = the domain)
    space = nlmc.build(scn, sys_, args.coarse, args.coarse, min(m, args.coarse))
    sizes, D, Q, W, M, F = nlmc.fine_parts(scn)
    R = space.R
    P = sp.csr_matrix((np.ones(len(space.fine_dof)), (space.fine_dof, np.arange(len(space.fine_dof)))),
                      shape=R.shape)
    lit = sp.csr_matrix(R @ D @ R.T)                                   # literal
    Alit = sp.csr_matrix(lit + P @ Q @ P.T + P @ sp.diags(W) @ P.T)
    flux = space.Abar                                                  # reading C32
    one = np.ones(R.shape[0])
    row = {"oversample_layers": int(min(m, args.coarse)), "coarse": args.coarse, "coarse_dofs": int(R.shape[0]),
           "literal_rowsum_max": float(np.abs(lit @ one - P @ (D @ np.ones(D.shape[0]))).max()),
           "literal_offdiag_max": float(np.abs(lit - sp.diags(lit.diagonal())).max()),
           "partition_of_unity_range": [float((R.T @ one).min()), float((R.T @ one).max())]}
    for name, A in (("literal", Alit), ("flux_form_C32", flux)):
        sysc = System(space.sizes, space.Mbar, A, space.Fbar, space.u0bar, [f"c{a}" for a in range(space.L)])
        try:
            cr = schemes.run(sysc, "coupled", tau, scn["NT"])
            e = [100.0 * float(np.linalg.norm(space.average(fine[n]) - cr[n]) / np.linalg.norm(space.average(fine[n])))
                 for n in (9, 29, 49)]
        except Exception as ex:                                        # e.g. an indefinite literal operator
            e = [None, None, None]
            row[name + "_error"] = repr(ex)
        row[name + "_eH_pct_at_steps_10_30_50"] = e
    rows.append(row)
    print(json.dumps(row), flush=True)
if args.out:
    json.dump({"scenario": "paper analogue 2C, 200^2, T = 0.002, 50 coupled steps", "rows": rows},
              open(args.out, "w"), indent=1)
