"""Column-block sharding of SPMESL over the ranks of a torch.distributed process group
(one process per GPU; BASELINE.json north_star (3) and SURVEY.md §8(e)).

The p column problems are independent, so each rank solves the columns
[c0, c1) of its contiguous block with X replicated and needs no communication during CD.
The only exchange is ONE all-gather of the fitted coefficients in CSC form (counts, rows,
values, sigma) — the nonzeros, not p x p doubles — after which every rank assembles and
symmetrizes its own column block of Theta from the global CSC (the symmetrization of
Eq. (symm), needs b_kj from column j, which may live on another rank).

With the Gram solver (default when it applies) there is one more, tiny exchange before the
fit: every rank screens an equal share of the tiles of S = X~^T X~ / n (the first sweeps of all
columns; by default the certified f16 screening) and the p screening flags are
max-all-reduced, so each rank knows which of its columns may need more than one sweep (their
exact FP64 Gram columns then decide, on the rank that owns the column).

``gather_csc`` / ``allreduce_hits`` are backend-agnostic host logic (gloo on CPU tensors in
the tests, NCCL on CUDA tensors in production); ``fit_distributed`` runs the CUDA path around
them.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def column_range(p: int, rank: int, world: int):
    """Contiguous, balanced block of columns for `rank` (first p % world ranks get one more)."""
    base, rem = divmod(p, world)
    c0 = rank * base + min(rank, rem)
    return c0, c0 + base + (1 if rank < rem else 0)


def tile_range(ntiles: int, rank: int, world: int):
    """Contiguous, balanced share of the Gram tiles for `rank` (same rule as column_range)."""
    return column_range(ntiles, rank, world)


def _comm_device(t: torch.Tensor, group=None) -> torch.device:
    """gloo moves CPU tensors only: stage CUDA tensors through the host for it."""
    if t.is_cuda and dist.get_backend(group) == "gloo":
        return torch.device("cpu")
    return t.device


def _all_gather_padded(t: torch.Tensor, length: int, group=None):
    """All-gather a 1-D tensor whose length differs per rank (padded to `length`)."""
    world = dist.get_world_size(group)
    cdev = _comm_device(t, group)
    buf = torch.zeros(length, dtype=t.dtype, device=cdev)
    buf[: t.numel()] = t.to(cdev)
    out = torch.empty(world * length, dtype=t.dtype, device=cdev)
    dist.all_gather_into_tensor(out, buf, group=group)
    return out.to(t.device).view(world, length)


def gather_csc(p: int, counts: torch.Tensor, rows: torch.Tensor, vals: torch.Tensor,
               sigma_std: torch.Tensor, group=None):
    """Concatenate every rank's column block (in rank = column order) into the global CSC.

    counts[m_r] (int32), rows[nnz_r] (int32), vals[nnz_r] (float64), sigma_std[m_r] (float64)
    -> (col_ptr[p+1] int64, rows[nnz] int32, vals[nnz] float64, sigma_std[p] float64)."""
    world = dist.get_world_size(group)
    dev = counts.device
    m_max = -(-p // world)
    cdev = _comm_device(counts, group)
    meta = torch.tensor([counts.numel(), rows.numel()], dtype=torch.int64, device=cdev)
    metas = torch.empty(world * 2, dtype=torch.int64, device=cdev)
    dist.all_gather_into_tensor(metas, meta, group=group)
    metas = metas.view(world, 2).cpu()
    nnz_max = max(int(metas[:, 1].max()), 1)
    cnt_all = _all_gather_padded(counts, m_max, group)
    sig_all = _all_gather_padded(sigma_std, m_max, group)
    rows_all = _all_gather_padded(rows, nnz_max, group)
    vals_all = _all_gather_padded(vals, nnz_max, group)
    cnt_list, sig_list, row_list, val_list = [], [], [], []
    for r in range(world):
        m_r, z_r = int(metas[r, 0]), int(metas[r, 1])
        cnt_list.append(cnt_all[r, :m_r])
        sig_list.append(sig_all[r, :m_r])
        row_list.append(rows_all[r, :z_r])
        val_list.append(vals_all[r, :z_r])
    cnt = torch.cat(cnt_list).to(torch.int64)
    if cnt.numel() != p:
        raise ValueError("column blocks do not cover p columns")
    col_ptr = torch.zeros(p + 1, dtype=torch.int64, device=dev)
    col_ptr[1:] = torch.cumsum(cnt, 0)
    return col_ptr, torch.cat(row_list), torch.cat(val_list), torch.cat(sig_list)


def allreduce_hits(hit: torch.Tensor, group=None) -> torch.Tensor:
    """Elementwise max (= OR of 0/1 flags) of the uint8 screening flags over all ranks."""
    cdev = _comm_device(hit, group)
    buf = hit.to(cdev)
    dist.all_reduce(buf, op=dist.ReduceOp.MAX, group=group)
    if buf is not hit:
        hit.copy_(buf.to(hit.device))
    return hit


def fit_distributed(X: torch.Tensor, lambda0: float, tol: float = 1e-4, max_iter: int = 100,
                    group=None, stream=None, solver: str = "auto", **options):
    """Fit this rank's column block and return its block of Theta (p x m, column-major view).

    X: (n, p) float64 CUDA tensor, identical on every rank.  solver: "auto" (the Gram solver
    with certified f16 screening when it applies), "gram16", "gram" (FP64 Gram screening) or
    "residual"."""
    from . import (as_colmajor, assemble_device, fit_columns_device, fit_columns_gram_device,
                   gram_screen_device, gram_supported, gram_tile_count)
    if stream is not None:
        # every library call, collective and torch op of this fit on the caller's stream, in
        # order (a collective's result is read by the next library call)
        with torch.cuda.stream(stream):
            return fit_distributed(X, lambda0, tol, max_iter, group=group, stream=None,
                                   solver=solver, **options)
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    n, p = X.shape
    c0, c1 = column_range(p, rank, world)
    mode = options.get("mode", "per_column")
    use_gram = solver in ("gram", "gram16") or (solver == "auto" and mode in ("per_column", 0)
                                                and gram_supported(n, p))
    screen_stats = None
    if use_gram:
        X = as_colmajor(X)
        t0, t1 = tile_range(gram_tile_count(p, solver=solver), rank, world)
        hit = torch.zeros(p, dtype=torch.uint8, device=X.device)
        screen_stats = gram_screen_device(X, lambda0, t0, t1, hit, stream=stream, solver=solver,
                                          **options)
        allreduce_hits(hit, group)
        part = fit_columns_gram_device(X, c0, c1, lambda0, hit, tol, max_iter, stream=stream,
                                       solver=solver, **options)
    else:
        part = fit_columns_device(X, c0, c1, lambda0, tol, max_iter, stream=stream,
                                  solver="residual" if solver == "auto" else solver, **options)
    col_ptr, rows, vals, sig_all = gather_csc(p, part["counts"], part["rows"], part["vals"],
                                              part["sigma_std"], group)
    theta, sigma = assemble_device(p, c0, c1, col_ptr, rows, vals, sig_all, part["scale"],
                                   stream=stream, **options)
    stats = dict(part["stats"])
    stats["kernel_launches"] = stats.get("kernel_launches", 0) + 2   # assemble entries + diag
    if screen_stats is not None:
        stats["ms_gram"] = screen_stats["ms_gram"]
        stats["ms_screen"] = screen_stats.get("ms_screen", 0.0)
        stats["screen_fill_bytes"] = 0
        stats["screen_tiles"] = (t0, t1)
        stats["kernel_launches"] += screen_stats["kernel_launches"]
    return dict(theta=theta, sigma=sigma, iters=part["iters"], sweeps=part["sweeps"],
                converged=part["converged"], col_range=(c0, c1), stats=stats,
                code=part["code"])
