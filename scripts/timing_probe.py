"""Dev probe: per-phase timing of fit_device at a given config."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2203_15031_b200 as S
from synth import generators as G
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
kw = dict(a.split("=") for a in sys.argv[2:])
kw = {k: (v if k in ("family",) else int(v)) for k, v in kw.items() if k != "solver"}
solver = dict(a.split("=") for a in sys.argv[2:]).get("solver", "auto")
X, gt, spec = G.make_config(cfg, **kw)
n, p = X.shape
lam = S.lambda_ub(n, p) if spec["rule"] == "ub" else S.lambda_univ(n, p)
Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda().t()
for it in range(5):
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); e0.record()
    r = S.fit_device(Xd, lam, solver=solver)
    e1.record(); torch.cuda.synchronize(); t1 = time.perf_counter()
    st = r.stats
    print(f"it{it} host {1e3*(t1-t0):.2f} ms  dev {e0.elapsed_time(e1):.2f} ms  std {st['ms_standardize']:.2f} cd {st['ms_cd']:.2f} asm {st['ms_assemble']:.2f} total {st['ms_total']:.2f} sweeps {st["total_sweeps"]} max {st["max_sweeps"]} nnz {st["nnz"]} T {st["tile_cols"]} tail {st["tail_columns"]} cols {st["ms_tail"]:.2f} ms", flush=True)
