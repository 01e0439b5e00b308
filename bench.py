#!/usr/bin/env python
"""SPMESL hot-path benchmark (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 5]

One step = one whole SPMESL fit of the BASELINE.json workload (config 5: n=500, p=20000,
Erdos-Renyi precision, lambda0 = lambda_ub, tol 1e-4): standardize -> persistent CD over all
p column problems -> CSC export -> Theta assembly + symmetrization (and, for N > 1, the CSC
all-gather).  value = algorithmic coordinate updates (sum_k sweeps_k (p-1)) per second of
device time, whole job.  e2e = the same through the host C-ABI entry point spmesl_fit_ex
with pinned host buffers (H2D of X and D2H of Theta/sigma/iters inside the timed region).
"""
from __future__ import annotations

import argparse
import ctypes
import json
import math
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SPMESL fit time (s) + CD coord-updates/s at p=5k-20k, 1/2/4/8 B200 vs roofline"
UNIT = "coord-updates/s"
TOL = 1e-4
MAX_ITER = 100


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--family", default=None)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--p", type=int, default=None)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-per-config", action="store_true")
    ap.add_argument("--per-config-seeds", type=int, default=3)
    ap.add_argument("--mode", default="per_column", choices=["per_column", "joint"],
                    help="per_column (default; Alg. 1/2 stop) or joint (Algorithm 3, P:938-990)")
    ap.add_argument("--solver", default="auto", choices=["auto", "residual", "gram", "gram16"])
    return ap.parse_args()


def workload(args):
    from synth import generators as G
    over = {k: v for k, v in dict(family=args.family, n=args.n, p=args.p).items() if v}
    X, gt, spec = G.make_config(args.config, **over)
    return X, spec


def lambda0_for(spec, n, p):
    # the product's own penalty helper (rule per config)
    import paper_2203_15031_b200 as S
    return S.lambda_ub(n, p) if spec["rule"] == "ub" else S.lambda_univ(n, p)


def config_dict(spec, world, lam, extra=None):
    d = {"workload": f"BASELINE config {spec.get('idx', '?')}: n={spec['n']}, p={spec['p']}, "
                     f"{spec['family']} precision, lambda0={spec['rule']}",
         "n": spec["n"], "p": spec["p"], "family": spec["family"], "penalty_rule": spec["rule"],
         "lambda0": lam, "tol": TOL, "max_iter": MAX_ITER, "seed": spec["seed"],
         "parallelism": f"column-blocks x{world}",
         "l2": "flushed between timed steps (256 MiB write); Theta (8p^2 B) also exceeds L2"}
    if extra:
        d.update(extra)
    return d


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{os.getpid()}.csv")

    def __enter__(self):
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "10"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.f.close()

    def mark(self):
        """Samples before this call (warm-up) are excluded from the summary."""
        try:
            self.f.flush()
            self.skip = sum(1 for _ in open(self.path))
        except Exception:
            self.skip = 0

    def summary(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        lines = open(self.path).readlines()
        skip = getattr(self, "skip", 0)
        window = "timed steps"
        if len(lines) - skip < 1:          # timed region shorter than one sample interval
            skip, window = max(0, skip - 3), "last warm-up samples + timed steps"
        for line in lines[skip:]:
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": sorted(reasons)}
        load = [x for x in sm if x > 500] or sm
        return {"sm_mhz": statistics.median(load), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "window": window}


# ----------------------------------------------------------------------------- peaks
def fp64_peak():
    """Measured FP64 tensor (DMMA m8n8k4) peak of this pool's B200 (profiles/)."""
    path = os.path.join(ROOT, "profiles", "r01_peaks_microbench.json")
    try:
        d = json.load(open(path))
        keys = [k for k in d if k.startswith("dmma_") and k.endswith("_tflops")]
        return max(d[k] for k in keys), "profiles/r01_peaks_microbench.json (DMMA f64, measured)"
    except Exception:
        return 36.8, "fallback 36.8 TFLOP/s (microbench value)"


def hbm_peak_gbs():
    """Measured HBM copy bandwidth of this pool's B200s (driver-written MEASURED_PEAKS.json)."""
    try:
        d = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(d["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured copy bandwidth)"
    except Exception:
        return 6650.0, "of fallback 6650 GB/s (B200_PROFILING.md)"


def bf16_peak_tflops():
    """Measured dense bf16 tensor throughput (MEASURED_PEAKS.json, burst figure)."""
    try:
        d = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(d["bf16_tflops"]), "MEASURED_PEAKS.json bf16_tflops (cuBLAS, measured)"
    except Exception:
        return 1590.0, "of fallback 1590 TFLOP/s (B200_PROFILING.md)"


def cd_traffic():
    path = os.path.join(ROOT, "profiles", "cd_traffic.json")
    try:
        return json.load(open(path))
    except Exception:
        return None


# ----------------------------------------------------------------------------- oracle baseline
def cpu_baseline(X, lam, seconds, seed=0):
    """The oracle (as it stands) on a bounded random sample of columns of the same workload."""
    from oracle import oracle as O
    n, p = X.shape
    Xs, mu, s = O.standardize(X)
    rng = np.random.default_rng(seed)
    order = rng.permutation(p)
    threads = O.num_threads()
    done, t_tot, sweeps = 0, 0.0, 0
    batch = max(threads * 4, 16)
    while t_tot < seconds and done < p:
        cols = np.sort(order[done:done + batch])
        t0 = time.perf_counter()
        r = O.spmesl_columns(Xs, cols, lam, delta=TOL, max_outer=MAX_ITER, want_margin=False)
        t_tot += time.perf_counter() - t0
        sweeps += int(r.sweeps.sum())
        done += len(cols)
    v = sweeps * (p - 1)
    return {"value": v / t_tot, "unit": UNIT, "cores": threads, "kind": "oracle",
            "sample": f"{done} of {p} columns (each with all p-1 predictors), {t_tot:.1f} s",
            "seconds": t_tot, "columns": done, "sweeps": sweeps, "cols": order[:done]}


# ----------------------------------------------------------------------------- per-config block
PER_CONFIG = [
    # (label, BASELINE config, generator overrides, penalty rule)
    ("config 4: n=400, p=5000, band(3), lambda_ub", 4, {"family": "band3"}, "ub"),
    ("config 4: n=400, p=5000, hub, lambda_ub", 4, {"family": "hub"}, "ub"),
    ("config 5: n=500, p=20000, ER, lambda_univ", 5, {}, "univ"),
]


def dfma_peak():
    """Measured FP64 FMA throughput of this pool's B200 (microbench/peaks.cu, profiles/)."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "r01_peaks_microbench.json")))
        return float(d["dfma_tflops"]), "profiles/r01_peaks_microbench.json dfma_tflops (measured)"
    except Exception:
        return 36.8, "fallback 36.8 TFLOP/s (round-1 microbench)"


def per_config_block(S, dev, stream, flush, seeds=3, fits=5):
    """The rest of the metric's range (p = 5k-20k, BASELINE configs 4 and 5 at the paper's
    recommended lambda_univ): per workload and seed, the device time per fit
    (CUDA-graph replays, L2 flushed before each, CUDA events on the launching stream), the
    algorithmic coordinate updates per second, the sweep counts, and the covariance-update sweep
    kernel's own time from an eager fit with its algorithmic FP64 rate (every coordinate change
    updates all p entries of z: p FMAs) against the measured DFMA peak; the kernel is bound by
    latency, so that fraction is small.
    Mean +- SE over `seeds` datasets (P:1121-1127 reports means over datasets)."""
    import torch
    from synth import generators as G
    fpk, fsrc = dfma_peak()
    hpk, hsrc = hbm_peak_gbs()
    out = []
    for label, cfg, over, rule in PER_CONFIG:
        rows = []
        for k in range(seeds):
            X, _, spec = G.make_config(cfg, seed=2203 + cfg + 1000 * k, **over)
            n, p = X.shape
            lam = S.lambda_ub(n, p) if rule == "ub" else S.lambda_univ(n, p)
            Xd = torch.from_numpy(np.ascontiguousarray(X.T)).to(dev).t()
            ob = dict(theta=torch.empty((p, p), dtype=torch.float64, device=dev),
                      sigma=torch.empty(p, dtype=torch.float64, device=dev),
                      iters=torch.empty(p, dtype=torch.int32, device=dev),
                      sweeps=torch.empty(p, dtype=torch.int32, device=dev),
                      conv=torch.empty(p, dtype=torch.uint8, device=dev))
            eager = S.fit_device(Xd, lam, TOL, MAX_ITER, stream=stream, out=ob, eager=True)
            st = eager.stats
            for _ in range(3):      # (the second call captures the graph)
                S.fit_device(Xd, lam, TOL, MAX_ITER, stream=stream, out=ob)
            e0 = [torch.cuda.Event(enable_timing=True) for _ in range(fits)]
            e1 = [torch.cuda.Event(enable_timing=True) for _ in range(fits)]
            for i in range(fits):
                flush.fill_(i % 255 + 1)
                torch.cuda.synchronize()
                e0[i].record(stream)
                S.fit_device(Xd, lam, TOL, MAX_ITER, stream=stream, out=ob)
                e1[i].record(stream)
                torch.cuda.synchronize()
            ms = float(np.median([a.elapsed_time(b) for a, b in zip(e0, e1)]))
            sweep_ms = float(st.get("ms_tail", 0.0))
            sweep_flops = 2.0 * p * st.get("tail_changes", 0)
            rows.append(dict(ms=ms, ups=st["coord_updates"] / (ms / 1000.0),
                             sweeps=st["total_sweeps"], max_sweeps=st["max_sweeps"],
                             multi=st["tail_columns"], nnz=st["nnz"], sweep_ms=sweep_ms,
                             tf=(sweep_flops / (sweep_ms / 1000.0) / 1e12) if sweep_ms > 0 else None,
                             gbs=(8.0 * p * st.get("tail_changes", 0) / (sweep_ms / 1000.0) / 1e9)
                             if sweep_ms > 0 else None,
                             changes=st.get("tail_changes", 0), passes=st.get("tail_passes", 0),
                             cand=st.get("screen_candidates"),
                             seed=spec["seed"]))
            del ob, Xd
        def ms_se(key):
            v = np.array([r[key] for r in rows], dtype=np.float64)
            return float(v.mean()), float(v.std(ddof=1) / np.sqrt(len(v))) if len(v) > 1 else 0.0
        fit_ms, fit_se = ms_se("ms")
        ups, ups_se = ms_se("ups")
        sw_ms, sw_se = ms_se("sweep_ms")
        out.append({"workload": label, "n": n, "p": p, "lambda0_rule": rule, "seeds": [r["seed"] for r in rows],
                    "fit_ms": fit_ms, "fit_ms_se": fit_se, "value": ups, "value_se": ups_se,
                    "unit": UNIT, "sweeps_total": [r["sweeps"] for r in rows],
                    "max_sweeps": [r["max_sweeps"] for r in rows],
                    "multi_sweep_columns": [r["multi"] for r in rows], "nnz": [r["nnz"] for r in rows],
                    "screen_candidates": [r["cand"] for r in rows],
                    "sweep_kernel": {"kernel": "tail_sweep_kernel", "ms": sw_ms, "ms_se": sw_se,
                                     "bound": "latency", "changes": [r["changes"] for r in rows],
                                     "passes": [r["passes"] for r in rows],
                                     "algorithmic": "p FP64 FMAs per coordinate change (2 p flops)",
                                     "achieved_tflops": [r["tf"] for r in rows],
                                     "frac_of_fp64": [(r["tf"] / fpk) if r["tf"] else None for r in rows],
                                     "peak_tflops": fpk, "peak_source": fsrc,
                                     # the north_star's memory view: a row-at-a-time
                                     # covariance-update CD reads one Gram column (8 p B) per
                                     # coordinate change and S (8 p^2 B) exceeds L2 at these p;
                                     # the multi-sweep passes read each support column once for
                                     # up to 32 sweeps, so the bytes actually moved are well below
                                     # these (ncu: profiles/r02_tail_*_ncu_summary.txt)
                                     "memory_view": {
                                         "algorithmic": "one Gram column (8 p B) per coordinate change",
                                         "achieved_gbs": [r["gbs"] for r in rows],
                                         "peak_gbs": hpk, "peak_source": hsrc,
                                         "frac_of_hbm": [(r["gbs"] / hpk) if r["gbs"] else None
                                                         for r in rows]},
                                     "timing": "eager fit (CUDA events around the kernel)"}})
    return out


# ----------------------------------------------------------------------------- main arms
def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    X, spec = workload(args)
    spec["idx"] = args.config
    n, p = X.shape
    from oracle import oracle as O
    lam = O.lambda_ub(n, p) if spec["rule"] == "ub" else O.lambda_univ(n, p)
    per_step = max(2.0, min(20.0, 120.0 / max(args.steps + args.warmup, 1)))
    for _ in range(args.warmup):
        cpu_baseline(X, lam, per_step / 4, seed=1)
    vals, secs = [], []
    base = None
    for k in range(args.steps):
        b = cpu_baseline(X, lam, per_step, seed=100 + k)
        vals.append(b["value"])
        secs.append(b["seconds"])
        base = b
    v = float(np.mean(vals))
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000 * float(np.mean(secs)), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(spec, 1, lam, {"reference": "CPU oracle (oracle/spmesl_oracle.c), "
                                                  "bounded column sample per step"}),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": base["cores"], "kind": "oracle",
                             "sample": base["sample"]},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # SPMESL_BENCH_SHARE_GPU=1: all ranks on cuda:0 over gloo (functional test of the multi-rank
    # path on a one-GPU box; not a performance configuration)
    share = os.environ.get("SPMESL_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    dist = None
    if world > 1 and args.mode != "per_column":
        raise SystemExit("--mode joint runs on one GPU (its stop is a max over all columns)")
    if world > 1:
        import torch.distributed as dist
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2203_15031_b200 as S
    from paper_2203_15031_b200 import distributed as D
    S.load()
    X, spec = workload(args)
    spec["idx"] = args.config
    n, p = X.shape
    lam = lambda0_for(spec, n, p)
    dev = torch.device("cuda", local)
    Xd = torch.from_numpy(np.ascontiguousarray(X.T)).to(dev).t()   # (n, p) column-major
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def barrier():
        if dist:
            dist.barrier()

    # output buffers allocated once and reused (no allocator traffic inside the timed steps)
    outbuf = dict(theta=torch.empty((p, p), dtype=torch.float64, device=dev),
                  sigma=torch.empty(p, dtype=torch.float64, device=dev),
                  iters=torch.empty(p, dtype=torch.int32, device=dev),
                  sweeps=torch.empty(p, dtype=torch.int32, device=dev),
                  conv=torch.empty(p, dtype=torch.uint8, device=dev)) if world == 1 else None

    def step():
        if world == 1:
            r = S.fit_device(Xd, lam, TOL, MAX_ITER, stream=stream, out=outbuf, mode=args.mode,
                             solver=args.solver)
            return r.stats, r
        r = D.fit_distributed(Xd, lam, TOL, MAX_ITER, stream=stream, solver=args.solver)
        return r["stats"], r

    ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    for e in ev0 + ev1:   # (torch creates CUDA events lazily at the first record: do it here,
        e.record(stream)  # not between a timed step's end and its closing record)
    torch.cuda.synchronize()
    cd_ms, updates, stats_last = [], 0, None
    # the clock sampler starts before the warm-up (its first nvidia-smi queries can stall the
    # GPU briefly) and its summary covers the timed steps
    with ClockSampler(local) as clk:
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        clk.mark()
        for k in range(args.steps):
            flush.fill_(k % 255 + 1)   # (never 0: a zero fill may take a memset path)
            torch.cuda.synchronize()
            barrier()
            torch.cuda.synchronize()
            ev0[k].record(stream)
            st, res = step()
            ev1[k].record(stream)
            torch.cuda.synchronize()
            barrier()
            cd_ms.append(st["ms_cd"])
            updates += st["coord_updates"]
            stats_last = st
    step_ms = [a.elapsed_time(b) for a, b in zip(ev0, ev1)]
    # the replayed steps time only the whole fit and the screening kernel: one eager fit after
    # the timed region gives the other kernels' times (ms_breakdown, the sweep kernel)
    eager_st = None
    if world == 1:
        eager_st = S.fit_device(Xd, lam, TOL, MAX_ITER, stream=stream, out=outbuf, mode=args.mode,
                                solver=args.solver, eager=True).stats
        torch.cuda.synchronize()
    print(f"[rank {rank}] step ms: {[round(x, 3) for x in step_ms]}  cd ms: {[round(x, 3) for x in cd_ms]}",
          file=sys.stderr, flush=True)
    tot_ms = sum(step_ms)
    cd_tot = sum(cd_ms)
    cdev = torch.device("cpu") if share else dev
    if dist:
        t = torch.tensor([tot_ms, cd_tot], dtype=torch.float64, device=cdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms, cd_tot = float(t[0]), float(t[1])
        u = torch.tensor([updates], dtype=torch.int64, device=cdev)
        dist.all_reduce(u)
        updates = int(u[0])
    value = updates / (tot_ms / 1000.0)
    upd_per_step = updates / args.steps
    # roofline of the dominant kernel (DESIGN.md §5/§7)
    peak, peak_src = fp64_peak()
    traffic = cd_traffic()
    step_ms_mean = tot_ms / args.steps
    if stats_last.get("solver") == 3 and world > 1:
        # multi-GPU: this rank's share of the certified screening tiles (no Theta fill in that
        # kernel: each rank zero-fills its own column block in the assembly); the contraction
        # is reported against the f16 tensor peak (bf16 measured; same rate for f16)
        scr_ms = float(stats_last.get("ms_screen") or stats_last["ms_gram"])
        t0, t1 = stats_last.get("screen_tiles", (0, 0))
        n_pad64 = -(-n // 64) * 64
        flops = 2.0 * 128 * 256 * n_pad64 * (t1 - t0)
        tpk, tsrc = bf16_peak_tflops()
        achieved = flops / (scr_ms / 1000.0) / 1e12
        roof = {"kernel": "screen16_tc_kernel", "bound": "tensor", "achieved": achieved,
                "peak": tpk, "unit": "TFLOP/s", "frac": achieved / tpk, "traffic": None,
                "peak_source": tsrc, "dtype": "f16 x f16 -> f32 (tcgen05.mma kind::f16)",
                "kernel_ms": scr_ms, "kernel_share_of_step": scr_ms / step_ms_mean,
                "algorithmic": "2 * 128 * 256 * n_pad flops per 128 x 256 tile of this rank's share",
                "screen_tiles": [t0, t1]}
    elif stats_last.get("solver") == 3 and not stats_last.get("gram_fallback"):
        # default solver: the certified f16 screening kernel (tcgen05) is the longest kernel of
        # the step; it also writes its share of Theta's p^2 zeros, which makes it HBM-bound:
        # algorithmic bytes = its zero-fill bytes + the f16 operand tiles read once
        # (2 p_pad n_pad64) + the p candidate flags
        scr_ms = float(stats_last["ms_screen"])
        p_pad, n_pad64 = -(-p // 128) * 128, -(-n // 64) * 64
        fill = float(stats_last.get("screen_fill_bytes", 8 * p * p))
        nbytes = fill + 2.0 * p_pad * n_pad64 + p
        achieved = nbytes / (scr_ms / 1000.0) / 1e9
        hbm_peak = hbm_peak_gbs()
        flops = float(n_pad64) * p_pad * (p_pad + 128)   # the triangle of 128 x 128 tiles
        roof = {"kernel": "screen16_tc_kernel", "bound": "hbm", "achieved": achieved,
                "peak": hbm_peak[0], "unit": "GB/s", "frac": achieved / hbm_peak[0],
                "traffic": (traffic or {}).get("screen16_dram_bytes_per_launch"),
                "peak_source": hbm_peak[1], "dtype": "f16 x f16 -> f32 (tcgen05.mma kind::f16)",
                "kernel_ms": scr_ms, "kernel_share_of_step": scr_ms / step_ms_mean,
                "algorithmic": "its share of Theta's zero fill (screen_fill_bytes) + 2 p_pad n_pad "
                               "bytes (f16 tiles) + p",
                "screen_fill_bytes": fill,
                "tensor_tflops": flops / (scr_ms / 1000.0) / 1e12,
                "screen_candidates": stats_last.get("screen_candidates"),
                "rest_of_step_ms": step_ms_mean - scr_ms,
                "sweep_kernel_ms": (eager_st or stats_last).get("ms_tail", 0.0),
                "sweep_kernel_timing": "eager fit after the timed steps",
                "sweep_columns": stats_last.get("tail_columns", 0)}
    elif stats_last.get("solver") in (2, 3):
        # Gram solver: the symmetric Gram kernel; algorithmic work n p (p + 1) flops (each of
        # the p (p + 1) / 2 distinct entries of X~^T X~ is a length-n dot product)
        gram_ms = float(stats_last.get("ms_screen") or stats_last["ms_gram"])
        share = 1.0
        if world > 1:      # this rank screened tiles [t0, t1) of the triangle
            nt = S.gram_tile_count(p)
            t0, t1 = D.tile_range(nt, rank, world)
            share = (t1 - t0) / nt
        achieved = n * p * (p + 1) * share / (gram_ms / 1000.0) / 1e12
        roof = {"kernel": "syrk_screen_kernel", "bound": "tensor", "achieved": achieved,
                "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                "traffic": (traffic or {}).get("syrk_dram_bytes_per_launch"),
                "peak_source": peak_src, "dtype": "fp64 (DMMA m8n8k4)",
                "kernel_ms": gram_ms, "kernel_share_of_step": gram_ms / step_ms_mean,
                "algorithmic": "n p (p+1) flops: the distinct entries of X~^T X~ (symmetric)",
                "sweep_kernel_ms": stats_last.get("ms_tail", 0.0),
                "sweep_columns": stats_last.get("tail_columns", 0)}
    else:
        # residual solver: the persistent CD kernel; 2n flops per coordinate update (§8(d))
        cd_updates = (stats_last["total_sweeps"] - stats_last["tail_sweeps"]) * (p - 1)
        achieved = 2.0 * n * cd_updates / (float(np.mean(cd_ms)) / 1000.0) / 1e12
        roof = {"kernel": "cd_sweep_kernel", "bound": "tensor", "achieved": achieved, "peak": peak,
                "unit": "TFLOP/s", "frac": achieved / peak,
                "traffic": (traffic or {}).get("dram_bytes_per_launch"),
                "peak_source": peak_src, "dtype": "fp64 (DMMA m8n8k4)",
                "kernel_share_of_step": float(np.mean(cd_ms)) / step_ms_mean,
                "algorithmic": "2n flops per coordinate update of the CD kernel "
                               "(sweeps done in the tail solver excluded)",
                "tail_solver_ms": stats_last.get("ms_tail", 0.0),
                "tail_columns": stats_last.get("tail_columns", 0)}
    # e2e through the host C-ABI entry point (pinned host buffers)
    e2e = None
    if not args.no_e2e:
        c0, c1 = D.column_range(p, rank, world) if world > 1 else (0, p)
        Xh = torch.from_numpy(np.ascontiguousarray(X.T)).pin_memory()   # col-major X
        if world == 1:
            Th = torch.empty((p, p), dtype=torch.float64).pin_memory()
            sh = torch.empty(p, dtype=torch.float64).pin_memory()
            ih = torch.empty(p, dtype=torch.int32).pin_memory()
            import ctypes
            L = S.load()
            o = S.default_options(mode=S.MODES[args.mode], solver=S.SOLVERS[args.solver])

            def e2e_step():
                rc = L.spmesl_fit_ex(ctypes.c_void_p(Xh.data_ptr()), n, p, lam, TOL, MAX_ITER,
                                     ctypes.byref(o), ctypes.c_void_p(Th.data_ptr()),
                                     ctypes.c_void_p(sh.data_ptr()),
                                     ctypes.c_void_p(ih.data_ptr()), None, None, None)
                assert rc >= 0, L.spmesl_last_error()
            # bytes that cross PCIe per step: X in; Theta's nonzeros (COO: 4+4+8 B each) +
            # diagonal + sigma + iters out (the dense zero-fill of Theta runs on host threads)
            h2d, d2h = 8 * n * p, None
        else:
            m = c1 - c0
            Th = torch.empty((m, p), dtype=torch.float64).pin_memory()
            sh = torch.empty(m, dtype=torch.float64).pin_memory()
            ih = torch.empty(m, dtype=torch.int32).pin_memory()

            def e2e_step():
                Xg = Xh.to(dev, non_blocking=True).t()
                r = D.fit_distributed(Xg, lam, TOL, MAX_ITER, stream=stream)
                Th.copy_(r["theta"].t(), non_blocking=True)
                sh.copy_(r["sigma"], non_blocking=True)
                ih.copy_(r["iters"], non_blocking=True)
                torch.cuda.synchronize()
            h2d, d2h = 8 * n * p, 8 * m * p + 8 * m + 4 * m
        for _ in range(2):
            e2e_step()
        e_ms = []
        for k in range(max(1, min(args.steps, 3))):
            flush.fill_(k % 255 + 1)
            torch.cuda.synchronize()
            barrier()
            t0 = time.perf_counter()
            e2e_step()
            torch.cuda.synchronize()
            e_ms.append(1000 * (time.perf_counter() - t0))
            barrier()
        e_tot = float(np.mean(e_ms))
        if dist:
            t = torch.tensor([e_tot], dtype=torch.float64, device=cdev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_tot = float(t[0])
        if d2h is None:
            nnz_sym = int(np.count_nonzero(Th.numpy())) - p      # off-diagonal nonzeros of Theta
            d2h = 16 * nnz_sym + 8 * p + 8 * p + 4 * p
        e2e = {"value": upd_per_step / (e_tot / 1000.0), "unit": UNIT,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": e_tot,
               "api": "spmesl_fit_ex (host pointers)" if world == 1 else
                      "fit_distributed with host pinned H2D/D2H"}
        if world == 1:
            # the same fit through the host sparse-output entry (Theta as CSC host arrays: no
            # 8 p^2-byte host array to fill); context beside the dense BASELINE signature
            cap = p + 16 * p
            cph = np.empty(p + 1, np.int64)
            rh = np.empty(cap, np.int32)
            vh = np.empty(cap, np.float64)
            sh2 = np.empty(p)
            ih2 = np.empty(p, np.int32)
            L = S.load()
            o2 = S.default_options(mode=S.MODES[args.mode], solver=S.SOLVERS[args.solver])

            def sparse_step():
                nz = ctypes.c_int64(0)
                rc = L.spmesl_fit_sparse(ctypes.c_void_p(Xh.data_ptr()), n, p, lam, TOL, MAX_ITER,
                                         ctypes.byref(o2), ctypes.c_void_p(cph.ctypes.data),
                                         ctypes.c_void_p(rh.ctypes.data),
                                         ctypes.c_void_p(vh.ctypes.data), cap, ctypes.byref(nz),
                                         ctypes.c_void_p(sh2.ctypes.data),
                                         ctypes.c_void_p(ih2.ctypes.data), None, None, None)
                assert rc >= 0, L.spmesl_last_error()
                return nz.value
            for _ in range(2):
                sparse_step()
            s_ms = []
            for k in range(max(1, min(args.steps, 5))):
                flush.fill_(k % 255 + 1)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                nnz_e = sparse_step()
                s_ms.append(1000 * (time.perf_counter() - t0))
            sm_ = float(np.median(s_ms))
            e2e["sparse_output"] = {"value": upd_per_step / (sm_ / 1000.0), "unit": UNIT,
                                    "ms_per_step": sm_, "h2d_bytes_per_step": 8 * n * p,
                                    "d2h_bytes_per_step": 8 * (p + 1) + 12 * int(nnz_e) + 12 * p,
                                    "api": "spmesl_fit_sparse (host pointers, Theta as CSC)"}
    per_config = None
    if world == 1 and not args.no_per_config and args.mode == "per_column" and args.solver == "auto":
        per_config = per_config_block(S, dev, stream, flush, seeds=args.per_config_seeds)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and args.mode == "per_column":
        cpu = cpu_baseline(X, lam, args.cpu_seconds)
        # the GPU's sweep total on the same columns (same algorithmic work, per-column counts
        # are identical to the oracle's: tests/test_gpu_fullsize.py)
        gsw = res.sweeps.cpu().numpy() if world == 1 else None
        if gsw is not None:
            cpu["gpu_sweeps_same_columns"] = int(gsw[cpu["cols"]].sum())
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot_ms / args.steps,
                "fit_time_s": tot_ms / args.steps / 1000.0, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": config_dict(spec, world, lam, {
                    "sweeps_total": stats_last["total_sweeps"],
                    "max_sweeps": stats_last["max_sweeps"], "max_outer": stats_last["max_outer"],
                    "nnz": stats_last["nnz"], "tile_cols": stats_last["tile_cols"],
                    "num_ctas": stats_last["num_ctas"], "mode": args.mode,
                    "solver": {1: "residual", 2: "gram", 3: "gram16"}.get(stats_last.get("solver"), "?")}),
                "roofline": roof, "clocks": clk.summary(), "e2e": e2e,
                "gpu_launches": int(stats_last["kernel_launches"]) * args.steps,
                "ms_breakdown": {k: (v if v is None or v >= 0 else None) for k, v in {
                    "standardize": (eager_st or stats_last)["ms_standardize"],
                    "solve": (eager_st or stats_last)["ms_cd"],
                    "gram": (eager_st or stats_last).get("ms_gram", 0.0),
                    "sweeps": (eager_st or stats_last).get("ms_tail", 0.0),
                    "assemble": (eager_st or stats_last)["ms_assemble"],
                    "screen": stats_last.get("ms_screen"),
                    "total_device": stats_last.get("ms_total")}.items()},
                "ms_breakdown_source": ("phases from one eager fit after the timed steps; screen "
                                        "and total_device from the replayed steps")
                if eager_st else "the last timed step",
                "graph_replay": bool(stats_last.get("graph_replay", 0))}
        if cpu:
            line["cpu_baseline"] = {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")}
            line["cpu_baseline"]["oracle_sweeps"] = cpu["sweeps"]
            line["cpu_baseline"]["gpu_sweeps_same_columns"] = cpu.get("gpu_sweeps_same_columns")
        if per_config is not None:
            line["per_config"] = per_config
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
