"""The checked build of libmc (-DMC_CHECK=1): device-side bounds asserts on every gather
index, staged window and work item, and guard bytes behind every device array -- the
stand-in for compute-sanitizer, which is closed on the B200 pool (SURVEY.md §5,
DESIGN.md §5.5).  Every kernel path runs a few steps under it in a fresh process; a tripped
assert aborts the process, a corrupted guard fails mc_debug_check."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASES = ["cfg0", "cfg3", "ell_stream", "bjs", "bj", "run", "nlmc"]


@pytest.fixture(scope="module")
def check_lib():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2209_01158_b200 import build
    out = os.path.join(ROOT, "paper_2209_01158_b200", "libmc_check.so")
    srcs = [os.path.join(build.CSRC, f) for f in os.listdir(build.CSRC)]
    if not os.path.exists(out) or any(os.path.getmtime(f) > os.path.getmtime(out) for f in srcs):
        build.build(force=True, defines=["MC_CHECK=1"], out=out)
    return out


@pytest.mark.parametrize("case", CASES)
def test_checked_build_runs_clean(check_lib, case):
    env = dict(os.environ, MC_LIB=check_lib)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "sanitize_target.py"), case], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert f"{case} guards corrupted: 0" in r.stdout and f"{case} done" in r.stdout
