"""Small fit of a multi-sweep workload (development: sanitizer target)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2203_15031_b200 as S
from synth import generators as G
X, _, spec = G.make_config(4, family="hub", p=int(sys.argv[1]) if len(sys.argv) > 1 else 600)
n, p = X.shape
Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda().t()
r = S.fit_device(Xd, S.lambda_ub(n, p), eager=True)
print(r.stats["tail_sweeps"], r.stats["tail_passes"])
