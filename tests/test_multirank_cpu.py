"""The N>1 path of bench.py on CPU: world_size 2 over gloo (127.0.0.1), replicas only.

Each rank is an independent replica; the job value is world x DOF x steps
divided by the MAX over ranks of the timed span.  No GPU needed."""
import os
import socket
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKER = r"""
import os, sys, json
sys.path.insert(0, os.environ["ROOT"])
import bench
rank, world, local = bench.dist_init(2, backend="gloo")
import torch.distributed as dist
bench.barrier(world)
mine = 10.0 + 5.0 * rank              # rank 1 is the slow one
tmax = bench.max_over_ranks(mine, world)
val = bench.aggregate(world, 1000, 4, tmax)
print(json.dumps({"rank": rank, "world": world, "tmax": tmax, "value": val}), flush=True)
dist.destroy_process_group()
"""


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_rank_replicas_gloo(tmp_path):
    import json
    script = tmp_path / "w.py"
    script.write_text(WORKER)
    port = _free_port()
    procs = []
    for r in range(2):
        env = dict(os.environ, ROOT=ROOT, RANK=str(r), WORLD_SIZE="2", LOCAL_RANK=str(r),
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, str(script)], env=env, stdout=subprocess.PIPE,
                                      stderr=subprocess.PIPE, text=True))
    outs = [p.communicate(timeout=120) for p in procs]
    for p, (o, e) in zip(procs, outs):
        assert p.returncode == 0, e
    res = [json.loads(o.strip().splitlines()[-1]) for o, _ in outs]
    for d in res:
        assert d["world"] == 2
        assert d["tmax"] == 15.0                       # max over ranks, not the local time
        assert abs(d["value"] - 2 * 1000 * 4 / 15e-3) < 1e-6
