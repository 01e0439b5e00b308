"""Pins of the estimation workload's metrics and the scale-free generator."""
import math

import numpy as np

from synth import generators as G
from workloads.estimation import edge_metrics


def test_edge_metrics_hand_example():
    # p = 4: true edges (0,1), (1,2), (2,3); estimated (0,1), (0,3) -> TP 1, FP 1, FN 2, TN 2
    O = np.eye(4)
    for i, j in [(0, 1), (1, 2), (2, 3)]:
        O[i, j] = O[j, i] = 0.3
    H = np.eye(4) * 2
    for i, j in [(0, 1), (0, 3)]:
        H[i, j] = H[j, i] = -0.1
    m = edge_metrics(H, O)
    assert (m["TP"], m["FP"], m["FN"], m["TN"]) == (1, 1, 2, 2)
    assert m["|E|"] == 2
    assert math.isclose(m["SEN"], 100 / 3) and math.isclose(m["SPE"], 100 * 2 / 3)
    assert math.isclose(m["FDR"], 50.0) and math.isclose(m["MISR"], 50.0)
    assert math.isclose(m["MCC"], 100 * (1 * 2 - 1 * 2) / math.sqrt(2 * 3 * 3 * 4))
    assert math.isclose(m["Frob"], np.linalg.norm(H - O))


def test_edge_metrics_perfect_and_empty():
    O = G.make_truth("ar1_paper", 30, 0).dense()
    m = edge_metrics(O, O)
    assert m["SEN"] == 100 and m["FDR"] == 0 and m["MISR"] == 0 and math.isclose(m["MCC"], 100)
    e = edge_metrics(np.eye(30), O)
    assert e["|E|"] == 0 and e["SEN"] == 0 and e["MCC"] == 0


def test_scale_free_generator():
    # P:1031-1036 + subnetworks of 100 nodes: a tree per block -> |E| = 495 at
    # p = 500 (the paper's Table 4 count), heavy-tailed degrees, positive definite, floor 0.1
    gt = G.make_truth("sf", 500, seed=3)
    O = gt.dense()
    iu = np.triu_indices(500, 1)
    assert np.count_nonzero(O[iu]) == 495
    np.linalg.cholesky(O)
    deg = np.count_nonzero(O - np.diag(np.diag(O)), axis=0)
    assert deg.max() >= 6 and np.median(deg) <= 2 and deg.max() <= 8
    nz = O[iu][O[iu] != 0]
    assert np.all(np.abs(nz) >= 0.1 - 1e-12)
