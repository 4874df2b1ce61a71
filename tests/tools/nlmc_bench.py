"""NLMC space build on the GPU (mc_nlmc_build) for the paper-analogue scenarios, with the
coarse solve of each scheme, and the oracle build timed beside it (one case, CPU).
    python tests/tools/nlmc_bench.py [--oracle] [--out FILE]"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch

from inputs import make_paper_analogue
from paper_2209_01158_b200 import Problem

ap = argparse.ArgumentParser()
ap.add_argument("--oracle", action="store_true")
ap.add_argument("--out", default=None)
args = ap.parse_args()
rows = []
for kind in ("2C", "3C"):
    scn = make_paper_analogue(kind)
    # fine reference: the coupled fine solution (GPU fine path) at t = T, averaged over K_j^alpha
    fp = Problem(scn)
    fp.run("coupled", scn["NT"])
    fine_T = np.concatenate([t.cpu().numpy() for t in fp.state()])
    h = scn["h"]
    meas = np.concatenate([np.full(fp.sizes[a], h * h if c["kind"] == "grid" else h)
                           for a, c in enumerate(scn["continua"])])
    fp.close()
    for nH in (20, 40):
        m = 2
        for _ in range(2):                     # the first build is a warm-up (module load)
            pb = Problem(scn)
            t0 = time.perf_counter()
            sp_ = pb.nlmc(nH, nH, m)
            if _ == 0:
                sp_.close()
                pb.close()
        wall = time.perf_counter() - t0
        row = dict(kind=kind, fine=scn["n"], coarse=nH, oversample=m, coarse_dofs=sp_.sizes,
                   nnz_per_row=sp_.nnz / sp_.n, ms_basis_kernel=sp_.ms_basis, ms_project_kernel=sp_.ms_project,
                   basis_gflop=sp_.flops_basis / 1e9, basis_tflops=sp_.flops_basis / (sp_.ms_basis * 1e-3) / 1e12,
                   bases_MB=sp_.bytes_bases / 1e6, dense_bases_MB_round1=8.0 * sp_.n * sp_.n_fine / 1e6,
                   s_build_wall=wall)
        cs = sp_.coarse_scenario(scn["T"], scn["NT"])
        pbar = np.bincount(sp_.fine_dof, weights=meas * fine_T, minlength=sp_.n) / \
            np.bincount(sp_.fine_dof, weights=meas, minlength=sp_.n)
        for scheme in ("coupled", "L", "D", "U"):
            cp = Problem(cs)
            reps = cp.run(scheme, scn["NT"])
            torch.cuda.synchronize()
            got = np.concatenate([t.cpu().numpy() for t in cp.state()])
            row[f"{scheme}_eH_pct"] = 100.0 * float(np.linalg.norm(got - pbar) / np.linalg.norm(pbar))
            row[f"{scheme}_ms"] = float(sum(r["ms"] for r in reps))
            row[f"{scheme}_iters_per_step"] = [float(np.mean([r["iters"][k] for r in reps]))
                                               for k in range(len(reps[0]["iters"]))]
            cp.close()
        sp_.close()
        pb.close()
        if args.oracle and kind == "2C" and nH == 20:
            from oracle import assemble as asm, nlmc
            sys_ = asm.assemble(scn)
            t0 = time.perf_counter()
            nlmc.build(scn, sys_, nH, nH, m)
            row["oracle_build_s"] = time.perf_counter() - t0
            row["oracle_cores"] = 1
        rows.append(row)
        print(json.dumps(row), flush=True)
if args.out:
    with open(args.out, "w") as f:
        json.dump(rows, f, indent=1)
