"""Multi-GPU sharding of the DFGT path.

Queries are independent units: each query's error is charged only against its own
lower bound and |R| (engine.cpp:131), so ranks can split the
query set with no exchange during the traversal.  For a CV sweep the only
collective is ONE all-reduce per batch of the per-bandwidth partial sums
(sum_j log LOO_j, clamp count, sum_j LS term_j) -- 3 doubles per bandwidth
(lkcv_from_sums / lscv_from_sums, cv.cpp:61-97).

One process per GPU (`torch.distributed`, NCCL on GPUs, gloo in the CPU tests).
The per-rank sum provider is pluggable so the host logic is testable without a GPU.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Callable, Sequence

import numpy as np


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced query shard [lo, hi) of rank in a world of `world`."""
    if not 0 <= rank < world:
        raise ValueError("rank outside [0, world)")
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def cv_partials(sums: np.ndarray, conv_sums: np.ndarray | None, n_total: int, dim: int,
                h: float, conv_h: float | None) -> np.ndarray:
    """Per-shard partial sums for one bandwidth: [sum log LOO density, clamps, sum LS
    term] over this shard's queries (the full-set scores divide by N, cv.cpp:74, 95)."""
    two_pi = 6.283185307179586476925286766559
    nh = (n_total - 1) * math.pow(two_pi * h * h, 0.5 * dim)
    loo = sums - 1.0
    clamped = loo <= 0.0
    loo = np.where(clamped, np.finfo(np.float64).tiny, loo)
    lk = float(np.sum(np.log(loo / nh)))
    ls = 0.0
    if conv_sums is not None:
        nc = (n_total - 1) * math.pow(two_pi * conv_h * conv_h, 0.5 * dim)
        ls = float(np.sum((conv_sums - 1.0) / nc - 2.0 * ((sums - 1.0) / nh)))
    return np.array([lk, float(np.count_nonzero(clamped)), ls])


@dataclass
class ShardedRow:
    h: float
    lk_score: float
    lk_clamped: int
    ls_score: float


def sharded_sweep(refs: np.ndarray, scales: Sequence[float], base_h: float,
                  sums_for: Callable[[np.ndarray, Sequence[float]], np.ndarray],
                  rank: int, world: int, allreduce: Callable[[np.ndarray], np.ndarray],
                  sqrt2: bool = False, order: np.ndarray | None = None) -> list[ShardedRow]:
    """CV sweep with the queries sharded across ranks.

    sums_for(queries, hs) -> (len(hs), len(queries)) kernel sums against ALL of
    `refs` (on a GPU: DualTreeEngine(refs).compute_batch(queries, hs)).  allreduce
    sums a float64 array over ranks (on GPUs: NCCL all_reduce).  Every rank returns
    the same rows.

    order (optional): a permutation of the points -- e.g. the reference kd-tree's
    `perm` -- whose contiguous ranges become the shards, so every rank's queries are
    a few spatially compact subtrees (a smaller query tree and fewer node pairs than
    a random slice of the input order)."""
    n, d = refs.shape
    lo, hi = shard_range(n, rank, world)
    mine = slice(lo, hi) if order is None else np.asarray(order)[lo:hi]
    hs = [s * base_h for s in scales]
    cs = [(math.sqrt(2.0) if sqrt2 else 2.0) * h for h in hs]
    part = np.zeros((len(hs), 3))
    if hi > lo:
        g = sums_for(refs[mine], list(hs) + list(cs))
        for k, (h, c) in enumerate(zip(hs, cs)):
            part[k] = cv_partials(g[k], g[len(hs) + k], n, d, h, c)
    tot = allreduce(part.ravel()).reshape(part.shape)
    return [ShardedRow(h, tot[k, 0] / n, int(round(tot[k, 1])), tot[k, 2] / n)
            for k, h in enumerate(hs)]


def torch_allreduce(group=None) -> Callable[[np.ndarray], np.ndarray]:
    """Sum over ranks with torch.distributed (NCCL tensors on the current CUDA device
    when the backend is NCCL, CPU tensors for gloo)."""
    import torch
    import torch.distributed as dist

    def f(x: np.ndarray) -> np.ndarray:
        dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
        t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).to(dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        return t.cpu().numpy()

    return f
