"""Dev: host-side overhead of fit_device (Python + C + launch + sync) vs its device time."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, cProfile, pstats
import paper_2203_15031_b200 as S
from synth import generators as G
X, _, spec = G.make_config(5)
n, p = X.shape
lam = S.lambda_ub(n, p)
Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda().t()
out = dict(theta=torch.empty((p, p), dtype=torch.float64, device="cuda"),
           sigma=torch.empty(p, dtype=torch.float64, device="cuda"),
           iters=torch.empty(p, dtype=torch.int32, device="cuda"),
           sweeps=torch.empty(p, dtype=torch.int32, device="cuda"),
           conv=torch.empty(p, dtype=torch.uint8, device="cuda"))
st = torch.cuda.current_stream()
for _ in range(5):
    r = S.fit_device(Xd, lam, out=out, stream=st)
torch.cuda.synchronize()
N = 50
t0 = time.perf_counter()
for _ in range(N):
    r = S.fit_device(Xd, lam, out=out, stream=st)
t1 = time.perf_counter()
print("host wall per fit %.3f ms, device total %.3f ms, replay %d" % ((t1 - t0) / N * 1e3, r.stats["ms_total"], r.stats["graph_replay"]))
pr = cProfile.Profile()
pr.enable()
for _ in range(N):
    r = S.fit_device(Xd, lam, out=out, stream=st)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
