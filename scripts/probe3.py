"""Dev probe: where does the config-1 fracture GPU solution differ from the refined oracle?"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, scipy.sparse as sp
from inputs import make
from paper_2209_01158_b200 import Problem
from oracle import assemble as asm, schemes

def ld_resid(K, x, b):
    K = K.tocsr(); xl = x.astype(np.longdouble)
    prod = K.data.astype(np.longdouble) * xl[K.indices]
    Kx = np.add.reduceat(prod, K.indptr[:-1]); Kx[np.diff(K.indptr) == 0] = 0
    return (b.astype(np.longdouble) - Kx)
def refined_solve(K, lu, b):
    x = lu.solve(b)
    for _ in range(4):
        x = x + lu.solve(np.asarray(ld_resid(K, x, b), dtype=np.float64))
    return x

scn = make(1); sys_ = asm.assemble(scn); tau = 0.01
ds = schemes.DScheme(sys_, tau)
K0 = sp.csr_matrix(sp.diags(sys_.M/tau) + ds.A0)
sl = sys_.block(1); Kf = K0[sl, sl]
out = {}
for ctas in (0, 37):
    for rtol in (1e-12, 1e-15):
        pb = Problem(scn, rtol=rtol, ctas=ctas)
        pb.step("D")
        um1 = np.concatenate([pb.get_state(a).cpu().numpy() for a in range(2)])
        rep = pb.step("D")
        xg = pb.get_state(1).cpu().numpy()
        b = ds.rhs(um1)[sl]
        ref = refined_solve(sp.csc_matrix(Kf), ds.solvers[1].lu, b)
        e = xg - ref
        tr = np.linalg.norm(np.asarray(ld_resid(Kf, xg, b), dtype=np.float64)) / np.linalg.norm(b)
        trr = np.linalg.norm(np.asarray(ld_resid(Kf, ref, b), dtype=np.float64)) / np.linalg.norm(b)
        print(f"ctas={ctas} rtol={rtol:.0e} iters={rep['iters']} relres={rep['relres']} err={np.linalg.norm(e)/np.linalg.norm(ref):.3e} true_res_gpu={tr:.2e} true_res_ref={trr:.2e}", flush=True)
        out[f"x_{ctas}_{rtol:.0e}"] = xg
        out[f"b_{ctas}_{rtol:.0e}"] = b
        out[f"ref_{ctas}_{rtol:.0e}"] = ref
        pb.close()
os.makedirs("gpurun_out", exist_ok=True)
np.savez_compressed("gpurun_out/probe3.npz", **out)
