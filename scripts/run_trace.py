"""Event trace of mc_run against a loop of mc_step (include/mc.h: mc_run enqueues steps back
to back, one host synchronisation per batch).  For each, the span between CUDA events
recorded on the library's stream before and after the n steps is compared with the sum of
the step kernels' own event times: the difference is what the host put between launches.
    python scripts/run_trace.py [--out profiles/r02_run_trace.json]"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from inputs import make
from paper_2209_01158_b200 import Problem

ap = argparse.ArgumentParser()
ap.add_argument("--out", default=None)
ap.add_argument("--config", type=int, default=0)
ap.add_argument("--steps", type=int, default=200)
args = ap.parse_args()
scn = make(args.config)
rows = []
for scheme in ("D", "coupled"):
    for mode in ("mc_step loop", "mc_run"):
        pb = Problem(scn)
        for _ in range(4):                      # planning steps + warm-up (the D plan is frozen after <= 3)
            pb.step(scheme)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0.record()
        if mode == "mc_run":
            reps = pb.run(scheme, args.steps)
        else:
            reps = [pb.step(scheme) for _ in range(args.steps)]
        e1.record()
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        span = e0.elapsed_time(e1)
        kern = sum(r["ms"] for r in reps)
        rows.append({"config": args.config, "scheme": scheme, "mode": mode, "steps": args.steps,
                     "span_ms": span, "sum_kernel_ms": kern, "gap_us_per_step": 1e3 * (span - kern) / args.steps,
                     "host_wall_ms": 1e3 * wall})
        print(json.dumps(rows[-1]), flush=True)
        pb.close()
if args.out:
    json.dump(rows, open(args.out, "w"), indent=1)
