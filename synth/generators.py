"""Seeded synthetic inputs for SPMESL (shared by the oracle side and the CUDA side).

This module holds NONE of the method's arithmetic: it only builds ground-truth precision
matrices Omega and draws Gaussian samples X ~ N(0, Omega^{-1}).  Both the oracle tests and
the CUDA path consume its outputs; nothing here standardizes, thresholds or regresses.

Recipes (PAPER.md lines as P:<line>; readings listed in DESIGN.md §4):
  * ``ar1_cov``   stationary AR(1) covariance Sigma_ij = rho^|i-j| (BASELINE.json configs 1-2,
                  "AR(1) precision (rho=0.5)"; reading i1: its precision is the tridiagonal chain
                  graph of P:1009-1019).  Sampled exactly by the AR recursion.
  * ``ar1_paper`` the paper's AR(1) precision, omega = 1 (diag), 0.48 (|i-j| = 1).
  * ``band``      omega_ij = base^|i-j| for |i-j| <= bw (P:1021-1032 with bw = 4 is AR(4);
                  config 4 uses bw = 3).
  * ``hub``       P:1066-1069 per 100-node subnetwork: 10 hubs of degree in
                  {14,15,16}, 90 non-hubs of degree in {1,2,3} (SPEC's concretisation).
  * ``er``        Erdos-Renyi edges with expected degree d inside 100-node subnetworks
                  (reading i2: the paper's subnetwork construction, applied to
                  the random-graph configs 3 and 5 of BASELINE.json).
  * weights of graph families follow steps (i)-(iv) of P:1045-1062 plus the 0.1 magnitude
    floor of P:1073-1076; positive definiteness is checked by Cholesky with seed+1 retries.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional, Tuple

import numpy as np
import scipy.linalg as sla


@dataclass
class GroundTruth:
    """Block-diagonal or banded precision matrix."""
    p: int
    kind: str
    blocks: List[Tuple[int, np.ndarray]] = field(default_factory=list)  # (offset, dense block)
    band: Optional[np.ndarray] = None       # upper banded storage (bw+1, p) for banded kinds
    bw: int = 0
    rho: float = 0.0                        # AR(1)-covariance parameter

    def dense(self) -> np.ndarray:
        """Dense Omega (tests / small p only)."""
        p = self.p
        if self.kind == "ar1_cov":
            O = np.zeros((p, p))
            r = self.rho
            c = 1.0 / (1.0 - r * r)
            for i in range(p):
                O[i, i] = c * (1.0 + r * r) if 0 < i < p - 1 else c
                if i + 1 < p:
                    O[i, i + 1] = O[i + 1, i] = -r * c
            return O
        if self.band is not None:
            O = np.zeros((p, p))
            for k in range(self.bw + 1):
                d = self.band[self.bw - k, k:]
                O[np.arange(p - k), np.arange(k, p)] = d
                O[np.arange(k, p), np.arange(p - k)] = d
            return O
        O = np.zeros((p, p))
        for off, B in self.blocks:
            m = B.shape[0]
            O[off:off + m, off:off + m] = B
        return O

    def edges(self) -> int:
        O = self.dense()
        return int(np.count_nonzero(np.triu(O, 1)))


def ar1_cov(p: int, rho: float = 0.5) -> GroundTruth:
    return GroundTruth(p=p, kind="ar1_cov", rho=rho)


def _banded(p: int, bw: int, values) -> GroundTruth:
    band = np.zeros((bw + 1, p))
    for k in range(bw + 1):
        band[bw - k, k:] = values(k)
    return GroundTruth(p=p, kind=f"band{bw}", band=band, bw=bw)


def ar1_paper(p: int) -> GroundTruth:
    """1 on the diagonal, 0.48 on |i-j| = 1."""
    return _banded(p, 1, lambda k: 1.0 if k == 0 else 0.48)


def band(p: int, bw: int = 3, base: float = 0.6) -> GroundTruth:
    """omega_ij = 0.6^|i-j| for |i-j| <= bw."""
    return _banded(p, bw, lambda k: base ** k)


def _weights(edges: np.ndarray, m: int, rng, floor: float) -> np.ndarray:
    """Steps (i)-(iv) of P:1045-1062 and the magnitude floor of P:1073-1076."""
    W = np.eye(m)
    if len(edges):
        u = rng.uniform(0.5, 1.0, size=len(edges)) * rng.choice([-1.0, 1.0], size=len(edges))
        W[edges[:, 0], edges[:, 1]] = u                       # (i)
        W[edges[:, 1], edges[:, 0]] = u
    off = np.abs(W - np.diag(np.diag(W))).sum(axis=1)
    scale = np.where(off > 0, 1.5 * off, 1.0)
    W = W / scale[:, None]                                     # (ii)
    W = 0.5 * (W + W.T)                                        # (iii)
    np.fill_diagonal(W, 1.0)                                   # (iv)
    if floor > 0:
        nz = (W != 0) & (np.abs(W) < floor)
        W[nz] = np.sign(W[nz]) * floor
    return W


def _is_pd(B: np.ndarray) -> bool:
    try:
        np.linalg.cholesky(B)
        return True
    except np.linalg.LinAlgError:
        return False


def _er_edges(m: int, d: float, rng) -> np.ndarray:
    prob = min(1.0, d / max(m - 1, 1))
    iu = np.triu_indices(m, 1)
    keep = rng.random(len(iu[0])) < prob
    return np.stack([iu[0][keep], iu[1][keep]], axis=1)


def _hub_edges(m: int, rng, n_hubs: int = 10) -> np.ndarray:
    """SPEC concretisation of P:1066-1067: hubs of degree {14,15,16}, non-hubs {1,2,3}."""
    hubs = np.arange(min(n_hubs, m))
    non = np.arange(len(hubs), m)
    cap = rng.integers(1, 4, size=m)                # non-hub degree targets
    deg = np.zeros(m, dtype=np.int64)
    edges = set()
    for h in hubs:
        target = int(rng.integers(14, 17))
        cand = [v for v in rng.permutation(non) if deg[v] < cap[v]]
        for v in cand[:target]:
            edges.add((int(h), int(v)))
            deg[h] += 1
            deg[v] += 1
    for v in non:                                   # every non-hub gets degree >= 1
        if deg[v] == 0:
            cand = [u for u in rng.permutation(non) if u != v and deg[u] < cap[u]]
            u = int(cand[0]) if cand else int(rng.choice(hubs))
            edges.add((min(v, u), max(v, u)))
            deg[v] += 1
            deg[u] += 1
    e = np.array(sorted(edges), dtype=np.int64).reshape(-1, 2)
    return e


def _sf_edges(m: int, rng, alpha: float = 2.3, kmax: int = 8) -> np.ndarray:
    """Scale-free block: Barabasi-Albert growth, one edge per new node (a tree:
    m - 1 edges, so |E| = 495 at p = 500 as in the paper's Table 4), attachment probability
    proportional to k + a with a = alpha - 3 (linear preferential attachment with offset gives
    P(k) ~ k^-(3 + a), i.e. the paper's alpha = 2.3).  Reading i3: degrees are
    capped at kmax = 8 — with the weights of P:1045-1062 a node of degree d whose neighbours
    are leaves gets couplings ~1/3, and the block stays positive definite only while d / 9 < 1
    (the paper does not say how it obtained positive-definite scale-free matrices)."""
    a = alpha - 3.0
    deg = np.zeros(m, dtype=np.float64)
    edges = []
    if m >= 2:
        edges.append((0, 1))
        deg[0] = deg[1] = 1.0
    for v in range(2, m):
        w = np.where(deg[:v] < kmax, deg[:v] + a, 0.0)
        u = int(rng.choice(v, p=w / w.sum()))
        edges.append((min(u, v), max(u, v)))
        deg[u] += 1.0
        deg[v] += 1.0
    return np.array(edges, dtype=np.int64).reshape(-1, 2)


def _block_family(p: int, kind: str, seed: int, floor: float, block: int, edge_fn) -> GroundTruth:
    blocks = []
    off = 0
    b = 0
    while off < p:
        m = min(block, p - off)
        s = seed * 1000003 + b
        for attempt in range(50):
            rng = np.random.default_rng(s + attempt)
            E = edge_fn(m, rng)
            W = _weights(E, m, rng, floor)
            if _is_pd(W):
                break
        else:
            raise RuntimeError("could not draw a positive-definite block")
        blocks.append((off, W))
        off += m
        b += 1
    return GroundTruth(p=p, kind=kind, blocks=blocks)


def er(p: int, d: float = 10.0, seed: int = 0, floor: float = 0.1, block: int = 100) -> GroundTruth:
    return _block_family(p, f"er{d:g}", seed, floor, block, lambda m, rng: _er_edges(m, d, rng))


def scale_free(p: int, seed: int = 0, floor: float = 0.1, block: int = 100) -> GroundTruth:
    return _block_family(p, "sf", seed, floor, block, lambda m, rng: _sf_edges(m, rng))


def hub(p: int, seed: int = 0, floor: float = 0.1, block: int = 100) -> GroundTruth:
    return _block_family(p, "hub", seed, floor, block, lambda m, rng: _hub_edges(m, rng))


def sample(gt: GroundTruth, n: int, seed: int) -> np.ndarray:
    """n i.i.d. rows from N(0, Omega^{-1}); returns a column-major (Fortran) n x p float64 array.

    Rows are x = L^{-T} z for Omega = L L^T (so Cov = Omega^{-1}); AR(1)-covariance uses the
    exact recursion x_1 = z_1, x_t = rho x_{t-1} + sqrt(1-rho^2) z_t."""
    p = gt.p
    rng = np.random.default_rng(seed)
    Z = rng.standard_normal((n, p))
    if gt.kind == "ar1_cov":
        X = np.empty((n, p), order="F")
        r = gt.rho
        c = np.sqrt(1.0 - r * r)
        X[:, 0] = Z[:, 0]
        for t in range(1, p):
            X[:, t] = r * X[:, t - 1] + c * Z[:, t]
        return X
    if gt.band is not None:
        U = sla.cholesky_banded(gt.band, lower=False)          # Omega = U^T U, U upper
        # x^T = z^T U^{-T}  <=>  U x = z  (x = U^{-1} z has Cov U^{-1} U^{-T} = Omega^{-1})
        Xt = sla.solve_banded((0, gt.bw), U, Z.T)
        return np.asfortranarray(Xt.T)
    X = np.empty((n, p), order="F")
    for off, B in gt.blocks:
        m = B.shape[0]
        U = np.linalg.cholesky(B).T                            # B = U^T U
        X[:, off:off + m] = sla.solve_triangular(U, Z[:, off:off + m].T, lower=False).T
    return X


# BASELINE.json configs (index 1..5).  lambda0 is NOT computed here (method arithmetic lives
# in the oracle and in the product's own helpers); each config names its penalty rule.
CONFIGS = {
    1: dict(n=50, p=20, family="ar1_cov", rule="univ"),
    2: dict(n=100, p=500, family="ar1_cov", rule="univ"),
    3: dict(n=200, p=1000, family="er", rule="ub"),
    4: dict(n=400, p=5000, family="band3", rule="ub"),
    5: dict(n=500, p=20000, family="er", rule="ub"),
}


def make_truth(family: str, p: int, seed: int) -> GroundTruth:
    if family == "ar1_cov":
        return ar1_cov(p, 0.5)
    if family == "ar1_paper":
        return ar1_paper(p)
    if family == "band3":
        return band(p, 3)
    if family == "ar4":
        return band(p, 4)
    if family == "hub":
        return hub(p, seed=seed)
    if family == "sf":
        return scale_free(p, seed=seed)
    if family == "er":
        return er(p, 10.0, seed=seed)
    raise ValueError(family)


def make_config(idx: int, seed: Optional[int] = None, family: Optional[str] = None,
                n: Optional[int] = None, p: Optional[int] = None):
    """Returns (X, truth, spec) for BASELINE.json config idx (seed base 2203 + idx)."""
    spec = dict(CONFIGS[idx])
    if family:
        spec["family"] = family
    if n:
        spec["n"] = n
    if p:
        spec["p"] = p
    base = 2203 + idx if seed is None else seed
    gt = make_truth(spec["family"], spec["p"], base)
    X = sample(gt, spec["n"], base + 7919)
    spec["seed"] = base
    return X, gt, spec
