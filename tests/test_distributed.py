"""Multi-rank (query-sharded) CV sweep host logic on CPU: world_size 2 over gloo.

Each rank computes kernel sums for its query shard (here with the CPU oracle's
exact naive sums standing in for the GPU engine), reduces three partial sums per
bandwidth with ONE all_reduce, and must reproduce the single-process
lkcv/lscv_from_sums scores (cv.cpp:61-97) to summation-order rounding.
"""
import os
import socket

import numpy as np
import pytest

from paper_1102_2878_b200.distributed import cv_partials, shard_range, sharded_sweep


def test_shard_range_partitions():
    for n in (1, 7, 100, 101):
        for world in (1, 2, 3, 8):
            got = [shard_range(n, r, world) for r in range(world)]
            assert got[0][0] == 0 and got[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(got, got[1:]))
            assert max(h - l for l, h in got) - min(h - l for l, h in got) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def test_partials_sum_to_full_scores(orc):
    g = np.random.default_rng(3)
    refs = g.random((300, 2))
    h = 0.05
    s1, s2 = orc.naive_kde(refs, refs, h), orc.naive_kde(refs, refs, 2 * h)
    p = cv_partials(s1[:120], s2[:120], 300, 2, h, 2 * h) + cv_partials(s1[120:], s2[120:], 300, 2, h, 2 * h)
    lk, cl = orc.lkcv(2, h, s1)
    assert p[0] / 300 == pytest.approx(lk, rel=1e-12) and int(p[1]) == cl
    assert p[2] / 300 == pytest.approx(orc.lscv(2, h, s1, 2 * h, s2), rel=1e-12)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, refs, scales, base_h, out):
    import torch.distributed as dist

    from oracle import load_oracle
    from paper_1102_2878_b200.distributed import sharded_sweep, torch_allreduce
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = load_oracle()

    def sums_for(q, hs):
        return np.stack([orc.naive_kde(q, refs, h) for h in hs])

    rows = sharded_sweep(refs, scales, base_h, sums_for, rank, world, torch_allreduce())
    out[rank] = [(r.h, r.lk_score, r.lk_clamped, r.ls_score) for r in rows]
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_sweep_matches_single_process(orc):
    import torch.multiprocessing as mp
    g = np.random.default_rng(5)
    refs = np.clip(g.random((6, 2))[g.integers(0, 6, 401)] + 0.03 * g.standard_normal((401, 2)), 0, 1)
    scales, base_h = [0.1, 1.0, 10.0], 0.02
    with mp.Manager() as man:
        out = man.dict()
        port = _free_port()
        mp.spawn(_worker, args=(2, port, refs, scales, base_h, out), nprocs=2, join=True)
        res = dict(out)
    assert res[0] == res[1]  # every rank holds the same rows
    for (h, lk, cl, ls), s in zip(res[0], scales):
        hh = s * base_h
        s1, s2 = orc.naive_kde(refs, refs, hh), orc.naive_kde(refs, refs, 2 * hh)
        lk_ref, cl_ref = orc.lkcv(2, hh, s1)
        assert lk == pytest.approx(lk_ref, rel=1e-12) and cl == cl_ref
        assert ls == pytest.approx(orc.lscv(2, hh, s1, 2 * hh, s2), rel=1e-11, abs=1e-14)


def test_single_rank_degenerates_to_plain_sweep(orc):
    refs = np.random.default_rng(9).random((50, 3))
    rows = sharded_sweep(refs, [1.0], 0.2,
                         lambda q, hs: np.stack([orc.naive_kde(q, refs, h) for h in hs]),
                         0, 1, lambda x: x)
    s1, s2 = orc.naive_kde(refs, refs, 0.2), orc.naive_kde(refs, refs, 0.4)
    assert rows[0].lk_score == pytest.approx(orc.lkcv(3, 0.2, s1)[0], rel=1e-12)
    assert rows[0].ls_score == pytest.approx(orc.lscv(3, 0.2, s1, 0.4, s2), rel=1e-12)
