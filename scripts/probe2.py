"""Dev probe: parity margins at config 1 (per continuum), rtol sweep, oracle refinement."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, scipy.sparse as sp, scipy.sparse.linalg as spla
from inputs import make
from paper_2209_01158_b200 import Problem
from oracle import assemble as asm, schemes

def ld_resid(K, x, b):
    K = K.tocsr(); xl = x.astype(np.longdouble)
    prod = K.data.astype(np.longdouble) * xl[K.indices]
    Kx = np.add.reduceat(prod, K.indptr[:-1]) if K.nnz else np.zeros(len(b), np.longdouble)
    empty = np.diff(K.indptr) == 0; Kx[empty] = 0
    return (b.astype(np.longdouble) - Kx)

def refined_solve(K, lu, b):
    x = lu.solve(b)
    for _ in range(4):
        r = ld_resid(K, x, b)
        x = x + lu.solve(np.asarray(r, dtype=np.float64))
    return x

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 1
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
scn = make(cid); sys_ = asm.assemble(scn); tau = scn["T"]/scn["NT"]
for scheme in ("D", "coupled"):
    st = schemes.make_stepper(sys_, scheme, tau)
    u = sys_.u0.copy(); refs=[]; refs_raw=[]
    for n in range(steps):
        if scheme == "coupled":
            b = sys_.M/tau*u + sys_.F
            xr = st.solver.solve(b, u); xx = refined_solve(st.solver.K, st.solver.lu, b)
        else:
            b = st.rhs(u); xr = np.empty_like(u); xx = np.empty_like(u)
            for a in range(sys_.L):
                s = sys_.block(a); xr[s] = st.solvers[a].solve(b[s], u[s]); xx[s] = refined_solve(st.solvers[a].K, st.solvers[a].lu, b[s])
        for a in range(sys_.L):
            s = sys_.block(a); nr = np.linalg.norm(xx[s])
            print(f"{scheme} step {n+1} cont {a}: splu-vs-refined {np.linalg.norm(xr[s]-xx[s])/max(nr,1e-300):.2e}", flush=True)
        refs.append(xx); u = xx
    for rtol in (1e-12, 1e-13, 1e-14, 1e-15):
        pb = Problem(scn, rtol=rtol)
        for n in range(steps):
            rep = pb.step(scheme)
            errs = []
            for a in range(sys_.L):
                g = pb.get_state(a).cpu().numpy(); r = refs[n][sys_.block(a)]; nr = np.linalg.norm(r)
                errs.append(np.linalg.norm(g-r)/nr if nr > 0 else float(np.abs(g).max()))
            print(f"{scheme} rtol={rtol:.0e} step {n+1}: iters={rep['iters']} relres={['%.1e'%x for x in rep['relres']]} err={['%.2e'%e for e in errs]} ms={rep['ms']:.1f}", flush=True)
        pb.close()
