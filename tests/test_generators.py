"""Input generators (synth/) — recipes of Section 4.1; inputs, not results."""
import json
import os

import numpy as np
import pytest

from synth import generators as G

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_edge_counts_match_paper():
    g = json.load(open(os.path.join(GOLD, "edge_counts.json")))
    assert G.ar1_paper(g["p"]).edges() == g["ar1_edges"]
    assert G.band(g["p"], 4).edges() == g["ar4_edges"]


@pytest.mark.parametrize("fam,p", [("ar1_cov", 40), ("ar1_paper", 300), ("ar4", 300),
                                   ("band3", 300), ("hub", 300), ("er", 300)])
def test_truth_valid_and_sample_covariance(fam, p):
    gt = G.make_truth(fam, p, 3)
    O = gt.dense()
    assert np.array_equal(O, O.T)
    np.linalg.cholesky(O)
    S = np.linalg.inv(O)
    assert np.abs(S @ O - np.eye(p)).max() < 1e-8
    if fam in ("hub", "er"):
        # block-diagonal with 100-node subnetworks
        mask = np.kron(np.eye(p // 100), np.ones((100, 100))) == 0
        assert np.all(O[mask] == 0)
        nz = O[(O != 0) & ~np.eye(p, dtype=bool)]
        assert np.all(np.abs(nz) >= 0.1 - 1e-15)                # magnitude floor
    X = G.sample(gt, 40000, 5)
    assert X.shape == (40000, p) and X.flags["F_CONTIGUOUS"]
    C = X.T @ X / 40000
    scale = np.sqrt(np.outer(np.diag(S), np.diag(S)))
    assert np.abs(C - S).max() / scale.max() < 0.08


def test_ar1_paper_values():
    O = G.ar1_paper(3).dense()
    assert np.array_equal(O, np.array([[1, .48, 0], [.48, 1, .48], [0, .48, 1]]))
    O4 = G.band(8, 4).dense()
    assert O4[0, 2] == pytest.approx(0.36) and O4[0, 5] == 0 and O4[0, 4] == pytest.approx(0.6 ** 4)


def test_hub_degrees():
    gt = G.hub(200, seed=9)
    O = gt.dense()
    deg = ((O != 0).sum(axis=1) - 1)
    for b in range(2):
        d = deg[b * 100:(b + 1) * 100]
        assert np.all((d[:10] >= 14) & (d[:10] <= 17))          # hubs ~15
        assert np.all((d[10:] >= 1) & (d[10:] <= 4))            # non-hubs 1..3 (+1 repair)


def test_determinism():
    a, _, _ = G.make_config(3, p=300)
    b, _, _ = G.make_config(3, p=300)
    assert np.array_equal(a, b)
