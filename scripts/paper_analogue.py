"""Paper-analogue experiment (Tables 1-2, Fig. 4 layout) on the CUDA path.

Runs the synthetic 2C / 3C analogue (inputs.make_paper_analogue: 200x200 matrix grid,
2 667-cell fracture network, Neumann boundaries, wells on the fracture, T = 0.002,
N_T = 50) through libmc for the coupled, L-, D- and U-schemes and prints / writes

    scheme | time_tot | e_h(T) % vs coupled | per continuum: time (mean iterations)

with the same columns as PAPER.md:906-949.  Errors are computed from the GPU's own
coupled trajectory (the oracle parity of every trajectory is covered by
tests/test_gpu_parity.py::test_paper_analogue_full_trajectory).  Timing: each scheme
runs the 50 steps once untimed, the state is reset to u0, and the 50 steps are timed
with CUDA events around one mc_run call on the problem's stream.

    python scripts/paper_analogue.py [--out profiles/r01_paper_analogue]
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def run_kind(kind, torch, Problem, make_paper_analogue, precond="jacobi"):
    scn = make_paper_analogue(kind)
    NT = scn["NT"]
    rows, finals, curves = {}, {}, {}
    for scheme in ("coupled", "L", "D", "U"):
        pb = Problem(scn, precond=precond)
        u0 = [t.clone() for t in pb.state()]
        snaps = [[torch.empty_like(t) for t in u0] for _ in range(NT)]
        pb.run(scheme, NT)                                   # warm-up pass
        for a, t in enumerate(u0):
            pb.set_state(a, t)
        stream = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        reps = pb.run(scheme, NT, snapshots=snaps)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        pb.close()
        ns = reps[0]["nsolves"] if "nsolves" in reps[0] else len(reps[0]["iters"])
        it = np.array([r["iters"] for r in reps], dtype=np.float64)
        msol = np.array([r["ms_solve"] for r in reps], dtype=np.float64)
        rows[scheme] = dict(ms_total=ms, iters_mean=it.mean(axis=0).tolist(),
                            ms_solve_total=msol.sum(axis=0).tolist(), nsolves=ns)
        curves[scheme] = [np.concatenate([s.cpu().numpy() for s in snap]) for snap in snaps]
        finals[scheme] = curves[scheme][-1]
    ref = curves["coupled"]
    for scheme in ("L", "D", "U"):
        e = [100.0 * np.linalg.norm(c - r) / np.linalg.norm(r) for c, r in zip(curves[scheme], ref)]
        rows[scheme]["e_h_final_pct"] = e[-1]
        rows[scheme]["e_h_curve_pct"] = [e[n] for n in (0, 9, 19, 29, 39, 49)]
    sizes = [len(t) for t in Problem(scn).state()]
    return dict(kind=kind, dofs=sizes, dof_total=int(sum(sizes)), NT=NT, rows=rows)


def table(res):
    L = len(res["dofs"])
    out = [f"### {res['kind']}  (DOF_h = {res['dof_total']} = {' + '.join(map(str, res['dofs']))}, N_T = {res['NT']})",
           "",
           "| scheme | time_tot (ms) | e_h(T) (%) | " + " | ".join(f"time_{a + 1} ms (N_it,{a + 1})" for a in range(L)) + " |",
           "|---|---|---|" + "---|" * L]
    for s, r in res["rows"].items():
        e = "-" if s == "coupled" else f"{r['e_h_final_pct']:.3f}"
        if s == "coupled":
            cells = [f"{r['ms_solve_total'][0]:.2f} ({r['iters_mean'][0]:.1f})"] + [""] * (L - 1)
        else:
            cells = [f"{t:.2f} ({n:.1f})" for t, n in zip(r["ms_solve_total"], r["iters_mean"])]
        out.append(f"| {s} | {r['ms_total']:.2f} | {e} | " + " | ".join(cells) + " |")
    return "\n".join(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="profiles/r01_paper_analogue")
    ap.add_argument("--precond", default="jacobi", choices=["jacobi", "block"])
    args = ap.parse_args()
    import torch
    from inputs import make_paper_analogue
    from paper_2209_01158_b200 import Problem
    res = [run_kind(k, torch, Problem, make_paper_analogue, args.precond) for k in ("2C", "3C")]
    md = "\n\n".join(table(r) for r in res)
    print(md)
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    with open(args.out + ".json", "w") as f:
        json.dump(dict(device=torch.cuda.get_device_name(0), results=res), f, indent=1)
    with open(args.out + ".md", "w") as f:
        f.write(f"Paper-analogue experiment on {torch.cuda.get_device_name(0)} "
                "(scripts/paper_analogue.py; columns as PAPER.md:906-949)\n\n" + md + "\n")


if __name__ == "__main__":
    main()
