"""One eager fit of a multi-sweep workload (for ncu on tail_sweep_kernel)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2203_15031_b200 as S
from synth import generators as G
fam = sys.argv[1] if len(sys.argv) > 1 else "band3"
X, _, spec = G.make_config(4, family=fam)
n, p = X.shape
Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda().t()
lam = S.lambda_ub(n, p)
for _ in range(2):
    r = S.fit_device(Xd, lam, eager=True)
print(r.stats)
