"""The seeded generator (inputs/) against the survey's independently measured sizes."""
import json
import os

import numpy as np
import pytest

from inputs import make, make_fine, make_nlmc

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def _frac_stats(s):
    c = s["fracture"]["cells"]
    e = s["fracture"]["edges"]
    deg = np.bincount(e.ravel(), minlength=len(c))
    return len(c), len(c) + 2 * len(e), np.bincount(deg, minlength=5)[:5].tolist()


@pytest.mark.parametrize("cid", [0, 1, 2])
def test_fracture_sizes_match_survey(cid):
    want = GOLD["survey_sizes"][str(cid)]
    cells, nnz, deg = _frac_stats(make(cid))
    assert cells == want["cells"] and nnz == want["nnz"] and deg == want["deg"]


@pytest.mark.slow
def test_fracture_sizes_config4():
    want = GOLD["survey_sizes"]["4"]
    cells, nnz, deg = _frac_stats(make(4))
    assert cells == want["cells"] and nnz == want["nnz"] and deg == want["deg"]


def test_nlmc_sizes_match_survey():
    s = make(3)
    nb = s["nc"] ** 2
    within = sum(2 * len(w[0]) for w in s["within"])
    total = 2 * nb + within + 2 * len(s["between"][0])
    assert total == GOLD["survey_sizes"]["3"]["nnz_total"]
    assert nb + 2 * len(s["within"][0][0]) == GOLD["survey_sizes"]["3"]["nnz_block"]
    assert len(s["between"][0]) == GOLD["survey_sizes"]["3"]["nnz_block"]


def test_deterministic_and_seeded():
    a, b = make(1), make(1)
    assert np.array_equal(a["continua"][0]["k"], b["continua"][0]["k"])
    assert np.array_equal(a["fracture"]["edges"], b["fracture"]["edges"])
    c = make_fine(64, seed=5, T=1, NT=1, segments=6, lengths=(10, 40))
    assert not np.array_equal(c["fracture"]["cells"], make(0)["fracture"]["cells"])


def test_lognormal_drawn_first():
    # reading C5: Z = standard_normal(n*n) is the first draw of default_rng(seed)
    s = make(1)
    Z = np.random.default_rng(1).standard_normal(1024 * 1024)
    assert np.array_equal(s["continua"][0]["k"], np.exp(1.0 * Z))


def test_fracture_structure():
    s = make(2)
    cells = s["fracture"]["cells"]
    e = s["fracture"]["edges"]
    n = s["n"]
    assert np.all(np.diff(cells) > 0)
    assert np.all(e[:, 0] < e[:, 1])
    d = cells[e[:, 1]] - cells[e[:, 0]]
    assert set(np.unique(d).tolist()) <= {1, n}          # grid neighbours only
    # horizontal edges never wrap around a row
    hz = d == 1
    assert np.all(cells[e[hz, 0]] % n != n - 1)
    # three continua: matrix, natural, fracture; couplings 0-1 colocated, 0-2, 1-2 embedded
    assert [c["name"] for c in s["continua"]] == ["matrix", "natural", "fracture"]
    assert [(c["a"], c["b"], c["type"]) for c in s["couplings"]] == [
        (0, 1, "colocated"), (0, 2, "embedded"), (1, 2, "embedded")]


def test_sigma_km_rule():
    s = make(1)
    k = s["continua"][0]["k"]
    cp = s["couplings"][0]
    assert np.allclose(cp["sigma"], 100.0 * k[s["fracture"]["cells"]], rtol=0, atol=0)


def test_nlmc_small_symmetric_offsets():
    s = make_nlmc(6, seed=11)
    for i, j, t in s["within"]:
        assert np.all(i < j) and np.all(t > 0)
        iy, ix = np.divmod(i, 6)
        jy, jx = np.divmod(j, 6)
        assert np.all(np.maximum(abs(iy - jy), abs(ix - jx)) <= 2)
    bi, bj, bt = s["between"]
    assert np.all(bt > 0) and len(bi) == sum((6 - abs(dy)) * (6 - abs(dx))
                                             for dy in range(-2, 3) for dx in range(-2, 3))
