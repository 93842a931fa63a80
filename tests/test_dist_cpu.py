"""Multi-process (gloo, world size 2, CPU) tests of the data-parallel host logic."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2106_06150_b200.dist import epoch_schedule, make_allreduce, max_over_ranks, rank_batches, steps_per_epoch


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


def test_rank_batches_padded_equal_steps():
    """Data-parallel schedule: the same number of steps on every rank, every
    batch exactly once, the short ranks padded with None (zero gradient)."""
    for nb in (0, 1, 7, 1110, 1111):
        for w in (1, 2, 3, 4, 8):
            per = [rank_batches(nb, r, w, pad=True) for r in range(w)]
            assert {len(p) for p in per} == {steps_per_epoch(nb, w)}
            got = sorted(i for p in per for i in p if i is not None)
            assert got == list(range(nb))
            for r, p in enumerate(per):      # pool.py:80 striding, pad only at the end
                real = [i for i in p if i is not None]
                assert real == list(range(r, nb, w))
                assert all(i is None for i in p[len(real):])


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


def _schedule_worker(rank, world, port, nb, epochs, period, out):
    """Each rank drives its own epoch schedule with one gloo all-reduce per
    step (the engine's captured gradient all-reduce) and a cache-key
    broadcast check at every refresh point; a rank with fewer steps would
    hang the collective (the test runs under a timeout)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import philox
        sched = epoch_schedule(nb, rank, world, epochs, cache_period=period)
        n_coll, trained, keys_equal, refresh_epochs = 0, [], True, []
        for epoch, index, refresh in sched:
            if refresh:
                refresh_epochs.append(epoch)
                # replicated cache: the same Philox key [seed, 33, epoch] on every rank
                k = torch.tensor(philox.key53(0, epoch, 0, philox.stream_word(33), 0, np.arange(32)).astype(np.int64))
                ref = k.clone()
                dist.broadcast(ref, src=0)
                keys_equal &= bool(torch.equal(k, ref))
            g = torch.ones(4) * (0.0 if index is None else 1.0)   # padded step: zero gradient
            dist.all_reduce(g)
            n_coll += 1
            if index is not None:
                trained.append((epoch, index))
        out[rank] = dict(n_coll=n_coll, trained=trained, keys_equal=keys_equal, refresh=refresh_epochs)
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("nb,period", [(7, 1), (1111, 2), (1, 1)])
def test_gloo_engine_rank_schedule_across_epochs(nb, period):
    world, epochs = 2, 3
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_schedule_worker, args=(world, port, nb, epochs, period, out), nprocs=world, join=True)
    assert out[0]["n_coll"] == out[1]["n_coll"] == epochs * steps_per_epoch(nb, world)
    assert out[0]["refresh"] == out[1]["refresh"] == [e for e in range(epochs) if e == 0 or e % period == 0]
    assert out[0]["keys_equal"] and out[1]["keys_equal"]
    trained = sorted(out[0]["trained"] + out[1]["trained"])
    assert trained == [(e, i) for e in range(epochs) for i in range(nb)]
