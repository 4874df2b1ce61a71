"""Dev probe: quick parity + timing of a few configs on the GPU (not part of the product)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from inputs import make
from paper_2209_01158_b200 import Problem
from oracle import assemble as asm, schemes

def par(scn, scheme, steps):
    sys_ = asm.assemble(scn); tau = scn["T"]/scn["NT"]
    t=time.time(); ref = schemes.run(sys_, scheme, tau, steps); to=time.time()-t
    pb = Problem(scn); worst=0; ms=0; its=[]
    for n in range(steps):
        rep = pb.step(scheme); ms += rep["ms"]; its.append(rep["iters"])
        for a, r in enumerate(sys_.split(ref[n])):
            g = pb.get_state(a).cpu().numpy(); nr = np.linalg.norm(r)
            e = np.linalg.norm(g-r)/nr if nr>0 else np.abs(g).max()
            worst=max(worst,e)
    print(f"cfg{scn['config_id']} {scheme} steps={steps} worst={worst:.2e} gpu_ms={ms:.1f} oracle_s={to:.1f} iters={its[:3]}...{its[-1]}", flush=True)

cfgs = [int(x) for x in (sys.argv[1:] or ["0","3"])]
for c in cfgs:
    scn = make(c)
    steps = {0:50, 1:5, 3:20, 2:2}.get(c, 2)
    for scheme in ("D","coupled"):
        par(scn, scheme, steps)
