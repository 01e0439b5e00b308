"""Dev probe: cost of sweeps of a single small tile (columns [c0, c0+m) of a config)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2203_15031_b200 as S
from synth import generators as G
m = int(sys.argv[1]) if len(sys.argv) > 1 else 8
X, gt, spec = G.make_config(5)
n, p = X.shape
lam = S.lambda_ub(n, p)
Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda().t()
for it in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    r = S.fit_columns_device(Xd, 0, m, lam)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    st = r["stats"]
    sw = int(r["sweeps"].sum())
    print(f"m={m} host {1e3*(t1-t0):.2f} ms cd {st['ms_cd']:.3f} ms sweeps(total) {sw} max {st['max_sweeps']} "
          f"-> {st['ms_cd']/max(st['max_sweeps'],1):.3f} ms per sweep, {1e3*st['ms_cd']/max(st['max_sweeps'],1)/625:.2f} us per block; T {st['tile_cols']} ctas {st['num_ctas']}", flush=True)
