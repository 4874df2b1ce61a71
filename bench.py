#!/usr/bin/env python
"""Benchmark: fine-grid DOF-steps/s of the decoupled D-scheme (fp64) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--scheme D|coupled]
                    [--impl reference]

One "step" is one time layer of the D-scheme over the whole
workload: the lagged right-hand side of every continuum, one Jacobi-PCG solve per
continuum to rtol 1e-12 and the commit — one launch of libmc's persistent step
kernel.  Default workload: BASELINE.json configs[4], the largest single-GPU fine-grid
configuration (8192^2 matrix + 16,615,213 fracture cells, log-normal k, 83.7M DOF;
DESIGN.md §7) -- the one BASELINE.json's HBM target is stated on; `--config 1` is the
1024^2 case (L2-resident, latency-bound).  The inputs are seeded synthetic (inputs/);
nothing here reads /root/reference.

Timing: W untimed warm-up steps, then exactly K steps, each bracketed by CUDA
events on the stream libmc launches on; L2 is flushed (256 MiB memset) between
timed steps, outside the events.  Multi-GPU: one process per GPU (torchrun), each
rank an independent replica (replicas only), max-over-ranks time.

The CPU oracle (oracle/) runs here only as the `cpu_baseline` leg (rank 0, N=1) and
as `--impl reference`; it is never on the product path.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FALLBACK_HBM_GBS = 6650.0
# CG tolerance per config and continuum (C13, C25): 1e-12 as BASELINE.json
# states; config 4's matrix continuum tightened to 1e-13 because at 1e-12 it misses the
# 1e-9 parity bar (k = exp(2Z)); its fracture solve keeps 1e-12.
CONFIG_RTOL = {0: None, 1: None, 2: None, 3: None, 4: [1e-13, 1e-12]}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--scheme", default="D", choices=["D", "coupled", "L", "U"])
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--precond", default="jacobi", choices=["jacobi", "block"],
                    help="CG preconditioner: jacobi (the north star's, default) or block "
                         "(block-Jacobi on the fracture network, mc_set_preconditioner)")
    return ap.parse_args()


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def ncu_traffic(cid, precond):
    """Mean DRAM bytes (read + write) per step_kernel launch from the committed ncu launch
    list of this bench command (profiles/rNN_launches_config{cid}[_block].csv, newest round
    first; the timed launches = the last `timed` rows of the list named in its .json
    sidecar, else all but the first 3); None when no such capture is committed."""
    import csv
    import glob
    suf = "_block" if precond == "block" else ""
    cands = sorted(glob.glob(os.path.join(ROOT, "profiles", f"r*_launches_config{cid}{suf}.csv")), reverse=True)
    if not cands:
        return None, None
    p = cands[0]
    rows = [r for r in csv.reader(l for l in open(p) if not l.startswith("=="))]
    hdr = rows[0]
    ik, im, iv = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    per = {}
    for r in rows[1:]:
        if "step_kernel" in r[ik] and r[im] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            per.setdefault(r[0], 0.0)
            per[r[0]] += float(r[iv].replace(",", ""))
    skip = 3
    side = p[:-4] + ".json"
    if os.path.exists(side):
        skip = int(json.load(open(side)).get("warmup_launches", 3))
    vals = [per[k] for k in sorted(per, key=int)][skip:]
    if not vals:
        return None, None
    return sum(vals) / len(vals), os.path.relpath(p, ROOT)


def workload_name(cid, scheme):
    return {0: "config0: 64^2 2C fine FV", 1: "config1: 1024^2 2C fine FV, lognormal k",
            2: "config2: 2048^2 3C fine FV", 3: "config3: NLMC 2x256^2 coarse",
            4: "config4: 8192^2 2C fine FV, lognormal k"}[cid] + f", {scheme}-scheme"


# ------------------------------------------------------------------ algorithmic bytes
PATH_NAMES = {0: "stream", 1: "ell-stream", 2: "ell-resident", 3: "bj-resident", 4: "bj-stream"}


def row_bytes(kind, path, nnz_off):
    """Algorithmic HBM bytes per row and CG iteration of the pass that handles a continuum
    (DESIGN.md §5.3 / §6; mc_step_report.paths says which pass ran):
      grid strips          read x, r, q, p, D^-1, Tx, Ty, shift (64) + write x, r, p, q (32) = 96
      streamed ELL chunks  read x, r, q, p, D^-1, shift (48) + 4 int32 codes (16) + write 32 = 96
      CSR rows             read 48 + row pointer 4 + 4 (col) or 12 (col + T) per entry + write 32
      resident ELL         the network's state stays in shared memory: only r, p, q are
                           published for the other warps' gathers, as one 32-byte record per row (32)
      block-Jacobi         resident: z, p published (16); streaming two-pass: 72 + 56 = 128
    Neighbour gathers are cache hits and are not counted."""
    if kind == "grid":
        return 96.0
    return {0: 84.0 + nnz_off, 1: 96.0, 2: 32.0, 3: 16.0, 4: 128.0}[path]


def step_bytes(pb, rep, scheme):
    """Algorithmic HBM bytes of one step kernel: iterations x rows x row_bytes per continuum,
    plus the init pass (~76 B/row)."""
    sizes, kinds, nnz_off = pb.byte_model
    total, per_cont = 0.0, []
    for a, n in enumerate(sizes):
        it = rep["iters"][0] if scheme == "coupled" else rep["iters"][a]
        b = it * row_bytes(kinds[a], rep["paths"][a], nnz_off[a]) * n + 76.0 * n
        per_cont.append(b)
        total += b
    return total, per_cont


def model_for(scn):
    sizes, kinds, off = [], [], []
    if scn["kind"] == "fine":
        n = scn["n"]
        for c in scn["continua"]:
            if c["kind"] == "grid":
                sizes.append(n * n)
                kinds.append("grid")
                off.append(0.0)
            else:
                nf = len(scn["fracture"]["cells"])
                sizes.append(nf)
                kinds.append("graph")
                off.append(4.0 * 2 * len(scn["fracture"]["edges"]) / nf)          # col int32
    else:
        nb = scn["nc"] ** 2
        for a in range(2):
            sizes.append(nb)
            kinds.append("graph")
            off.append(12.0 * 2 * len(scn["within"][a][0]) / nb)                  # col + val
    return sizes, kinds, off


# ------------------------------------------------------------------ clocks
class Clocks:
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        out, _ = self.p.communicate(timeout=10)
        sm, mx, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ distributed
def dist_init(n, backend="nccl"):
    """One process per GPU (torchrun env); replicas only."""
    if n <= 1 or "RANK" not in os.environ:
        return 0, 1, 0
    import torch.distributed as dist
    import torch
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    if backend == "nccl":
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", local))
    else:
        dist.init_process_group(backend, rank=rank, world_size=world)
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def aggregate(world, dof, steps, total_ms):
    """Whole-job DOF-steps/s: every rank a replica of `dof` DOFs, time = max over ranks."""
    return world * dof * steps / (total_ms * 1e-3)


# ------------------------------------------------------------------ oracle legs (CPU)
# Oracle Jacobi-PCG iterations per step and continuum (rtol 1e-13, D-scheme, step 2 of the
# oracle's own trajectory) for the configs whose full oracle step takes minutes to an hour:
# measured by tests/tools/parity_full.py (profiles/r02_parity_config{2,4}_D.json).  Used only to
# scale a bounded sample of oracle iterations to one whole step.
ORACLE_ITERS = {2: [362, 308, 29313], 4: [445, 74151]}


def host_info():
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"os_cpu_count": os.cpu_count(), "affinity": len(os.sched_getaffinity(0)), "cpu_model": model}


def oracle_sample(scn, scheme, steps, budget_s=30.0, warmup=0):
    """Configs 0, 1, 3: time the SuperLU oracle (as it stands, one thread) on `steps` whole
    steps of the workload after `warmup` untimed ones; setup (assembly + factorisation)
    excluded and reported separately.  Returns (dof, steps done, seconds, setup seconds)."""
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    from oracle import assemble as asm, schemes
    t0 = time.perf_counter()
    sys_ = asm.assemble(scn)
    order = list(range(sys_.L))          # continua ascend in permeability in every workload
    st = schemes.make_stepper(sys_, scheme, scn["T"] / scn["NT"], order_by_k=order)
    setup = time.perf_counter() - t0
    u = sys_.u0.copy()
    for _ in range(warmup):
        u = st.step(u)
    done = 0
    t1 = time.perf_counter()
    while done < steps:
        u = st.step(u)
        done += 1
        if time.perf_counter() - t1 > budget_s:
            break
    el = time.perf_counter() - t1
    return sum(sys_.sizes), done, el, setup


class CgOracleSampler:
    """Configs 2 and 4 (no factorisation fits): the C Jacobi-PCG oracle
    (oracle/flux_pcg.c, OpenMP on all host cores) as it stands.  One whole oracle step takes
    minutes (config 2) to an hour (config 4), so a sample is a bounded number of PCG
    iterations of every continuum's D-scheme system from a seeded state; the per-iteration
    times are scaled by the iterations a whole step needs (`iters_per_step`)."""

    def __init__(self, scn, sample_iters):
        import numpy as np
        from oracle import assemble as asm, fluxcg
        self.fluxcg = fluxcg
        t0 = time.perf_counter()
        self.lean = asm.assemble_lean(scn)
        self.st = fluxcg.DSchemeCG(self.lean, scn["T"] / scn["NT"])
        self.setup = time.perf_counter() - t0
        u = np.random.default_rng(0).random(len(self.lean.M))         # a previous layer in (0, 1)
        self.u, self.b = u, self.st.rhs(u)
        self.sample_iters = list(sample_iters)
        self.threads = fluxcg.threads()

    def sample(self):
        """Seconds per PCG iteration of every continuum (one capped solve each)."""
        out = []
        for a, k in enumerate(self.sample_iters):
            s = self.lean.block(a)
            t0 = time.perf_counter()
            try:
                self.st.ops[a].solve(self.b[s], self.u[s], 1e-13, maxit=k)
                k = self.st.ops[a].iters[-1]                          # converged early (small system)
            except self.fluxcg.CGNoConvergence:
                pass
            out.append((time.perf_counter() - t0) / max(k, 1))
        return out


def cg_sample_iters(cid):
    return {2: [20, 20, 200], 4: [20, 100]}[cid]    # ~5-10 s of host work per sample (16 cores)


def run_reference(args):
    rank, world, _ = dist_init(args.gpus)
    if rank != 0:
        return
    from inputs import make
    scn = make(args.config)
    base = {"metric": "fine-grid DOF-steps/s (decoupled, fp64)", "unit": "DOF-steps/s", "n_gpus": args.gpus,
            "warmup": args.warmup, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "impl": "reference"}
    if args.config in (2, 4) and args.scheme == "D":
        smp = CgOracleSampler(scn, cg_sample_iters(args.config))
        dof = sum(smp.lean.sizes)
        need = ORACLE_ITERS[args.config]
        for _ in range(args.warmup):
            smp.sample()
        secs = []
        for _ in range(args.steps):
            per = smp.sample()
            secs.append(sum(t * n for t, n in zip(per, need)))
        el = sum(secs)
        value = dof * args.steps / el
        sample = (f"each step = {smp.sample_iters} Jacobi-PCG iterations per continuum of the C oracle "
                  f"(oracle/flux_pcg.c, {smp.threads} OpenMP threads) on config {args.config}'s D-scheme systems "
                  f"from a seeded state, scaled to the {need} iterations per continuum a whole oracle step "
                  f"needs (profiles/r02_parity_config{args.config}_D.json); setup {smp.setup:.0f}s excluded")
        line = dict(base, value=value, steps=args.steps, ms_per_step=1e3 * el / args.steps,
                    config={"workload": workload_name(args.config, args.scheme), "dof": dof, "scheme": args.scheme},
                    cpu_baseline={"value": value, "unit": "DOF-steps/s", "cores": smp.threads, "kind": "oracle",
                                  "sample": sample, "host": host_info()})
    else:
        dof, done, el, setup = oracle_sample(scn, args.scheme, args.steps, budget_s=240.0, warmup=args.warmup)
        value = dof * done / el
        line = dict(base, value=value, steps=done, ms_per_step=1e3 * el / done,
                    config={"workload": workload_name(args.config, args.scheme), "dof": dof, "scheme": args.scheme},
                    cpu_baseline={"value": value, "unit": "DOF-steps/s", "cores": 1, "kind": "oracle",
                                  "sample": f"{done} full oracle steps (SuperLU back-solves + long-double "
                                            f"flux-form refinement, 1 thread); setup {setup:.1f}s excluded",
                                  "host": host_info()})
    line["e2e"] = {"value": line["value"], "unit": "DOF-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    print(json.dumps(line), flush=True)


def cpu_baseline_leg(args, scn, reps):
    """The oracle timed on this box's host cores on a bounded sample of the workload."""
    if args.config in (2, 4) and args.scheme == "D":
        smp = CgOracleSampler(scn, cg_sample_iters(args.config))
        per = smp.sample()
        need = [sum(r["iters"][a] for r in reps) / len(reps) for a in range(len(per))]
        sec = sum(t * n for t, n in zip(per, need))
        dof = sum(smp.lean.sizes)
        return {"value": dof / sec, "unit": "DOF-steps/s", "cores": smp.threads, "kind": "oracle",
                "sample": (f"config{args.config} D-scheme: {smp.sample_iters} Jacobi-PCG iterations per continuum of "
                           f"the C oracle (oracle/flux_pcg.c, {smp.threads} OpenMP threads) from a seeded state = "
                           f"{['%.4f' % t for t in per]} s per iteration, scaled to the timed steps' mean "
                           f"iteration counts {[round(n, 1) for n in need]}; setup {smp.setup:.0f}s excluded"),
                "host": host_info()}
    d, done, el, setup = oracle_sample(scn, args.scheme, 3 if args.config == 1 else 20, budget_s=25.0)
    return {"value": d * done / el, "unit": "DOF-steps/s", "cores": 1, "kind": "oracle",
            "sample": f"config{args.config} {args.scheme}-scheme, {done} oracle steps (SuperLU back-solves "
                      f"+ long-double flux refinement, 1 thread); assembly+factorisation {setup:.1f}s excluded",
            "host": host_info()}


# ------------------------------------------------------------------ main
def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    rank, world, local = dist_init(args.gpus)
    torch.cuda.set_device(local)
    from inputs import make
    from paper_2209_01158_b200 import Problem, build
    build.build()
    scn = make(args.config)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    pb = Problem(scn, device=local, stream=stream, rtols=CONFIG_RTOL[args.config], precond=args.precond)
    pb.byte_model = model_for(scn)
    dof = sum(pb.sizes)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(args.warmup):
        pb.step(args.scheme)
    saved = [t.clone() for t in pb.state()]          # the e2e leg replays the same K steps from here
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    reps = []
    clocks = Clocks(local)
    barrier(world)
    torch.cuda.synchronize()
    clocks.start()
    for k in range(args.steps):
        flush.zero_()
        ev[k][0].record(stream)
        reps.append(pb.step(args.scheme))
        ev[k][1].record(stream)
    torch.cuda.synchronize()
    barrier(world)
    clk = clocks.stop()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = max_over_ranks(sum(step_ms), world)
    value = aggregate(world, dof, args.steps, total_ms)
    # roofline of the dominant (only) kernel: the step kernel, one launch per step
    sb = [step_bytes(pb, r, args.scheme) for r in reps]
    bytes_per = sum(b for b, _ in sb) / args.steps
    kern_ms = sum(r["ms"] for r in reps) / args.steps
    peak, peak_src = peaks()
    achieved = bytes_per / (kern_ms * 1e-3) / 1e9
    traffic, traffic_src = (ncu_traffic(args.config, args.precond) if args.scheme == "D" else (None, None))
    nsol = len(reps[0]["iters"])
    mean_its = [sum(r["iters"][a] for r in reps) / len(reps) for a in range(nsol)]
    mean_ms = [sum(r["ms_solve"][a] for r in reps) / len(reps) for a in range(nsol)]
    per_solve = []
    if args.scheme != "coupled":
        for a in range(nsol):
            ba = sum(pc[a] for _, pc in sb) / args.steps
            per_solve.append({"rows": pb.sizes[a], "path": PATH_NAMES[reps[-1]["paths"][a]],
                              "us_per_iteration": 1e3 * mean_ms[a] / max(mean_its[a], 1.0),
                              "GBps": ba / max(mean_ms[a], 1e-9) / 1e6})
    # end to end through the C ABI with host buffers (pinned): the SAME K steps replayed from
    # the saved state with the same L2 policy; every step's state goes host -> device before
    # the step and device -> host after it, copies inside the timed region
    e2e = None
    if not args.no_e2e:
        host = [torch.empty(s, dtype=torch.float64, pin_memory=True) for s in pb.sizes]
        for a in range(pb.L):
            host[a].copy_(saved[a])
        torch.cuda.synchronize()
        barrier(world)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        ereps = []
        for _ in range(args.steps):
            flush.zero_()
            for a in range(pb.L):
                pb.set_state(a, host[a])
            ereps.append(pb.step(args.scheme))
            for a in range(pb.L):
                pb.get_state(a, out=host[a])
        e1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = max_over_ranks(e0.elapsed_time(e1), world)
        e2e = {"value": world * dof * args.steps / (e2e_ms * 1e-3), "unit": "DOF-steps/s",
               "h2d_bytes_per_step": 8 * dof, "d2h_bytes_per_step": 8 * dof,
               "same_steps_as_value": [r["iters"] for r in ereps] == [r["iters"] for r in reps],
               "region": "K x (L2 flush + mc_set_state from pinned host + mc_step + mc_get_state to pinned host)"}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_leg(args, scn, reps)
    if rank == 0:
        l2res = all(p["path"] in ("ell-resident", "bj-resident") or p["rows"] * 96 < 120e6 for p in per_solve) \
            if per_solve else False
        line = {
            "metric": "fine-grid DOF-steps/s (decoupled, fp64)" if args.scheme == "D" else
                      f"fine-grid DOF-steps/s ({args.scheme}-scheme, fp64)", "value": value, "unit": "DOF-steps/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_name(args.config, args.scheme), "dof": dof,
                       "sizes": pb.sizes, "scheme": args.scheme, "rtol": CONFIG_RTOL[args.config] or 1e-12,
                       "precond": args.precond,
                       "time_layers": f"{args.warmup + 1}..{args.warmup + args.steps} of the run from u0 "
                                      f"(the config's own N_T is {scn['NT']})",
                       "cg_iters_per_step": mean_its, "ms_per_solve": mean_ms,
                       "l2": "flushed between timed steps (256 MiB memset)",
                       "parallelism": f"replicas x{world}"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                         "peak_source": peak_src, "frac_of_8TBps": achieved / 8000.0,
                         "kernel": "mc::step_kernel", "bytes_per_launch": bytes_per,
                         "ms_per_launch": kern_ms, "per_solve": per_solve,
                         "regime": ("working set L2-resident: latency-bound, frac is not an HBM fraction "
                                    "(see per_solve us_per_iteration; barrier floor profiles/r01_barrier.txt)"
                                    if l2res else "working set >> L2: HBM-bound")},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": args.steps, "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    pb.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
