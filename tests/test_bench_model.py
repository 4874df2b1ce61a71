"""Host logic of bench.py that needs no GPU: the byte model per kernel path (DESIGN.md §5.3 /
§6), the ncu launch-list reader, the committed evidence it points at."""
import json
import os

import bench

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_row_bytes_per_path():
    # grid strips and the streamed blocked ELL pass: 64 read + 32 written
    assert bench.row_bytes("grid", 0, 0.0) == 96.0
    assert bench.row_bytes("graph", 1, 12.6) == 96.0
    # CSR rows: 48 + 4 (row pointer) + 32 + bytes of the stored entries
    assert bench.row_bytes("graph", 0, 12.0 * 24.8) == 84.0 + 12.0 * 24.8
    # resident network: one 32-byte record published per row; block-Jacobi: 16 / 72 + 56
    assert bench.row_bytes("graph", 2, 12.6) == 32.0
    assert bench.row_bytes("graph", 3, 12.6) == 16.0
    assert bench.row_bytes("graph", 4, 12.6) == 128.0
    assert set(bench.PATH_NAMES) == {0, 1, 2, 3, 4}


def test_step_bytes_config4_iteration():
    """One CG iteration of config 4's two solves moves 6.44 GB (matrix) and 1.595 GB (fracture)."""
    class PB:
        byte_model = ([67108864, 16615213], ["grid", "graph"], [0.0, 12.56])
    rep = {"iters": [1, 1], "paths": [0, 1, 0, 0]}
    total, per = bench.step_bytes(PB, rep, "D")
    assert abs(per[0] - (96.0 + 76.0) * 67108864) < 1.0
    assert abs((per[1] - 76.0 * 16615213) / 1e9 - 1.595) < 1e-3
    assert total == sum(per)


def test_ncu_launch_list_reader_on_committed_capture():
    traffic, src = bench.ncu_traffic(4, "jacobi")
    assert src == "profiles/r02_launches_config4.csv"
    # two timed launches of the bench command: 127 TB and 58 TB of DRAM traffic
    assert 8.0e13 < traffic < 1.0e14
    assert bench.ncu_traffic(4, "block") == (None, None)


def test_committed_headline_is_consistent():
    d = json.load(open(os.path.join(ROOT, "profiles", "r02_bench_config4.json")))
    assert d["config"]["workload"].startswith("config4") and d["steps"] == 20 and d["warmup"] == 5
    r = d["roofline"]
    assert abs(r["achieved"] - r["bytes_per_launch"] / (r["ms_per_launch"] * 1e-3) / 1e9) < 1e-6 * r["achieved"]
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-12
    assert d["e2e"]["value"] <= d["value"] and d["e2e"]["same_steps_as_value"]
    assert abs(d["value"] - d["config"]["dof"] * d["steps"] / (d["ms_per_step"] * d["steps"] * 1e-3)) < 1e-6 * d["value"]
    for name in ("r02_parity_config4_D", "r02_parity_config2_D", "r02_parity_config2_coupled"):
        p = json.load(open(os.path.join(ROOT, "profiles", name + ".json")))
        assert p["pass"] and all(e <= 1e-9 for row in p["steps"] for e in row["rel_l2"])
