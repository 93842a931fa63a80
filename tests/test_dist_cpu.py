"""Multi-process (gloo, world size 2, CPU) tests of the data-parallel host logic."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2106_06150_b200.dist import make_allreduce, max_over_ranks, rank_batches


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_rank_batches_partition():
    for nb in (0, 1, 7, 1111):
        for w in (1, 2, 4, 8):
            got = sorted(i for r in range(w) for i in rank_batches(nb, r, w))
            assert got == list(range(nb))
    with pytest.raises(ValueError):
        rank_batches(10, 2, 2)


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # per-rank gradient of its own batches; all-reduce + 1/W == the mean
        g = torch.arange(10, dtype=torch.float32) * (rank + 1)
        scale = make_allreduce()(g)
        out[rank] = (g * scale).numpy().tolist()
        out[f"t{rank}"] = max_over_ranks(1.5 + rank)
        # identical cache on every rank: same Philox key -> same keys
        from oracle import philox
        k = philox.key53(0, 3, 0, philox.stream_word(33), 0, np.arange(64))
        ks = torch.tensor(k.astype(np.int64))
        ref = ks.clone()
        dist.broadcast(ref, src=0)
        out[f"c{rank}"] = bool(torch.equal(ks, ref))
    finally:
        dist.destroy_process_group()


def test_gloo_allreduce_mean_and_max_timing():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    expect = (np.arange(10) * 1.5).tolist()
    assert out[0] == expect and out[1] == expect
    assert out["t0"] == 2.5 and out["t1"] == 2.5
    assert out["c0"] and out["c1"]
