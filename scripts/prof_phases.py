"""Dev: per-phase cycle breakdown of the CG loop (needs a -DMC_PROF=1 build):
    python -m paper_2209_01158_b200.build --variant prof MC_PROF=1
    MC_LIB=paper_2209_01158_b200/libmc_prof.so python scripts/prof_phases.py CONFIG MAXIT [fracture|grid|all]
Phases (thread 0 of each group's first CTA, summed over iterations): pass, CTA reduce +
publish, barrier spin, partial fetch."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from inputs import make
from paper_2209_01158_b200 import Problem, MCError, mc

cid, maxit = int(sys.argv[1]), int(sys.argv[2])
kind = sys.argv[3] if len(sys.argv) > 3 else "fracture"
scn = make(cid)
if kind != "all":
    scn = dict(scn, continua=[c for c in scn["continua"] if c["kind"] == kind][:1], couplings=[])
pb = Problem(scn, maxit=maxit)
lib = mc.load()
buf = np.zeros((4, 8), dtype=np.int64)
g = torch.Generator(device="cuda").manual_seed(0)
for a in range(len(pb.sizes)):
    pb.set_state(a, torch.rand(pb.sizes[a], dtype=torch.float64, device="cuda", generator=g))
for rep_i in range(2):
    lib.mc_prof_read(buf.ctypes.data_as(C.c_void_p), 1)
    try:
        rep = pb.step("D")
    except MCError as e:
        rep = e.report
    torch.cuda.synchronize()
    lib.mc_prof_read(buf.ctypes.data_as(C.c_void_p), 1)
    for gi in range(len(pb.sizes)):
        n = max(1, buf[gi, 4])
        it = rep["iters"][gi]
        ms = rep["ms_solve"][gi]
        print(f"cfg{cid} {kind} group {gi}: iters {it}  {1e3 * ms / max(1, it):.3f} us/iter  cycles/iter: "
              f"pass {buf[gi, 0] / n:.0f}  reduce+publish {buf[gi, 1] / n:.0f}  spin {buf[gi, 2] / n:.0f}  "
              f"fetch {buf[gi, 3] / n:.0f}", flush=True)
