"""Multi-process host logic of the data-parallel path on CPU (gloo, world_size 2):
contiguous batch shards and the single packed allreduce (parallel.py)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2501_11407_b200.parallel import GradPacker, shard_range


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n, k, m, B = 5, 7, 3, 9
    lo, hi = shard_range(B, rank, world)
    # per-sample "gradients" of the global batch; each rank owns its shard only
    rng = np.random.default_rng(0)
    gw_all = rng.standard_normal((B, n, k))
    gwo_all = rng.standard_normal((B, m, n))
    loss_all = rng.random(B)
    corr_all = rng.integers(0, 2, B)
    pk = GradPacker(n, k, m, "cpu")
    acc = torch.zeros((n, k + 3), dtype=torch.float64)        # column-padded accumulator
    acc[:, :k] = torch.from_numpy(gw_all[lo:hi].sum(0))
    pk.pack(acc, torch.from_numpy(gwo_all[lo:hi].sum(0)), torch.from_numpy(loss_all[lo:hi]),
            torch.from_numpy(corr_all[lo:hi]).to(torch.int32))
    gw, gwo, ls, nc = pk.allreduce()
    out_q.put((rank, gw.numpy().copy(), gwo.numpy().copy(), float(ls), float(nc), (lo, hi)))
    dist.destroy_process_group()


def test_shard_range_partitions_batch():
    for B in (1, 7, 256, 1024):
        for world in (1, 2, 3, 8):
            spans = [shard_range(B, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == B
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            sizes = [h - l for l, h in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)


def test_packed_allreduce_two_ranks_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(0)
    B, n, k, m = 9, 5, 7, 3
    gw_all = rng.standard_normal((B, n, k))
    gwo_all = rng.standard_normal((B, m, n))
    loss_all = rng.random(B)
    corr_all = rng.integers(0, 2, B)
    spans = sorted(r[5] for r in res)
    assert spans == [(0, 5), (5, 9)]
    for _, gw, gwo, ls, nc, _ in res:   # every rank holds the global (summed) result
        assert np.allclose(gw, gw_all.sum(0), atol=1e-5)
        assert np.allclose(gwo, gwo_all.sum(0), atol=1e-5)
        assert ls == pytest.approx(loss_all.sum(), rel=1e-6)
        assert nc == corr_all.sum()
