"""Dev: device timeline of one fit (torch.profiler / CUPTI activity), gaps between GPU ops."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2203_15031_b200 as S
from synth import generators as G
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
mode = sys.argv[2] if len(sys.argv) > 2 else "per_column"
X, gt, spec = G.make_config(cfg)
n, p = X.shape
lam = S.lambda_ub(n, p) if spec["rule"] == "ub" else S.lambda_univ(n, p)
Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda().t()
out = dict(theta=torch.empty((p, p), dtype=torch.float64, device="cuda"),
           sigma=torch.empty(p, dtype=torch.float64, device="cuda"),
           iters=torch.empty(p, dtype=torch.int32, device="cuda"),
           sweeps=torch.empty(p, dtype=torch.int32, device="cuda"),
           conv=torch.empty(p, dtype=torch.uint8, device="cuda"))
for _ in range(3):
    S.fit_device(Xd, lam, out=out, mode=mode)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for _ in range(2):
        S.fit_device(Xd, lam, out=out, mode=mode)
    torch.cuda.synchronize()
prof.export_chrome_trace("gpurun_out/trace.json")
ev = json.load(open("gpurun_out/trace.json"))["traceEvents"]
gpu = [e for e in ev if e.get("cat") in ("kernel", "gpu_memset", "gpu_memcpy") and "ts" in e]
gpu.sort(key=lambda e: e["ts"])
t0 = gpu[0]["ts"]
prev_end = None
for e in gpu:
    gap = (e["ts"] - prev_end) if prev_end is not None else 0.0
    print(f"{(e['ts']-t0)/1000:8.3f} ms  dur {e.get('dur',0)/1000:7.3f} ms  gap {gap/1000:7.3f}  stream {e.get('args',{}).get('stream','?')}  {e['name'][:60]}")
    prev_end = max(prev_end or 0, e["ts"] + e.get("dur", 0))
