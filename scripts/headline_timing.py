"""Config 5 (lambda_ub) device time per fit, CUDA-graph replays with an L2 flush before each
(the bench's timed step), for a given build of the library (development aid)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
if len(sys.argv) > 1:
    from paper_2203_15031_b200 import _lib
    _lib.LIB_PATH = sys.argv[1]
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
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream()
for _ in range(4):
    r = S.fit_device(Xd, lam, out=out)
ms = []
for i in range(20):
    flush.fill_(i % 255 + 1)
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(s)
    r = S.fit_device(Xd, lam, out=out)
    b.record(s)
    torch.cuda.synchronize()
    ms.append(a.elapsed_time(b))
print(sys.argv[1:] or ["current"], "median %.4f min %.4f ms" % (np.median(ms), np.min(ms)),
      "screen %.4f ms" % r.stats["ms_screen"], flush=True)
