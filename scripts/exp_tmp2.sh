python - <<'PY'
import sys; sys.path.insert(0, ".")
from inputs import make
from paper_2209_01158_b200 import Problem
for pc in ("jacobi", "block"):
    pb = Problem(make(1), precond=pc)
    its = [pb.step("D")["iters"] for _ in range(4)]
    print(pc, its, flush=True)
    pb.close()
PY
timeout 400 python -m pytest tests/test_gpu_precond.py -x -q -p no:cacheprovider 2>&1 | tail -2
timeout 300 python bench.py --precond block --no-cpu-baseline 2>&1 | tail -1 | cut -c1-600
