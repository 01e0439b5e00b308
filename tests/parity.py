"""Parity criteria between the CUDA path and the oracle (BASELINE.json north_star):
  |dTheta_jk| <= 1e-8 |Theta^o_jk| + 1e-12 max_k Theta^o_kk
  |dsigma_k|  <= 1e-10 sigma^o_k
  support identical except where the oracle's threshold margin | |a| - lambda | <= 1e-8
  per-column outer-iteration and sweep counts identical (control flow matches)."""
import numpy as np

THETA_RTOL = 1e-8
THETA_ATOL_FRAC = 1e-12
SIGMA_RTOL = 1e-10
MARGIN = 1e-8


def compare(gpu_theta, gpu_sigma, gpu_iters, gpu_sweeps, ora, cols=None, label=""):
    """ora: oracle FitResult (full).  cols: restrict to these columns (all if None)."""
    Tg = np.asarray(gpu_theta)
    To = ora.Theta
    p = To.shape[0]
    cols = np.arange(p) if cols is None else np.asarray(cols)
    rep = {}
    it_bad = np.nonzero(np.asarray(gpu_iters)[cols] != ora.outer[cols])[0]
    sw_bad = np.nonzero(np.asarray(gpu_sweeps)[cols] != ora.sweeps[cols])[0]
    rep["iters_mismatch"] = cols[it_bad].tolist()
    rep["sweeps_mismatch"] = cols[sw_bad].tolist()
    sg = np.asarray(gpu_sigma)[cols]
    so = ora.sigma[cols]
    rep["sigma_maxrel"] = float(np.max(np.abs(sg - so) / so))
    scale = THETA_ATOL_FRAC * np.max(np.diag(To))
    d = np.abs(Tg[:, cols] - To[:, cols])
    tol = THETA_RTOL * np.abs(To[:, cols]) + scale
    viol = d > tol
    # support mismatches near the threshold are allowed
    sup_diff = (Tg[:, cols] != 0) != (To[:, cols] != 0)
    if ora.margin is not None:
        mg = np.minimum(np.abs(ora.margin[:, cols]), np.abs(ora.margin.T[:, cols]))
        near = mg <= MARGIN
    else:
        near = np.zeros_like(sup_diff)
    rep["support_mismatch"] = int(np.sum(sup_diff))
    rep["support_mismatch_unexplained"] = int(np.sum(sup_diff & ~near))
    rep["theta_violations"] = int(np.sum(viol & ~(sup_diff & near)))
    rel = d / np.maximum(np.abs(To[:, cols]), scale / THETA_RTOL)
    rep["theta_maxrel"] = float(np.max(rel))
    return rep


def assert_parity(rep):
    assert rep["iters_mismatch"] == [], rep
    assert rep["sweeps_mismatch"] == [], rep
    assert rep["sigma_maxrel"] <= SIGMA_RTOL, rep
    assert rep["support_mismatch_unexplained"] == 0, rep
    assert rep["theta_violations"] == 0, rep
