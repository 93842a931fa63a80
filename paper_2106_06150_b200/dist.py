"""Data-parallel plumbing.

One process per GPU (torchrun).  Mini-batches shard with no data-path
collective: rank r takes batch indices r, r+W, r+2W, ... of every epoch —
the reference's worker striding (pool.py:80) — and every rank draws the same
cache from the same Philox key (replicated, no collective).  The only
collective is one all-reduce of the flat gradient buffer per step; Adam then
scales by 1/W (mean gradient of the W batches).
"""

from __future__ import annotations

import os

import torch
import torch.distributed as dist


def rank_batches(num_batches: int, rank: int, world_size: int, pad: bool = False) -> list:
    """Batch indices owned by ``rank`` (pool.py:80 striding).

    ``pad=True`` is the data-parallel schedule: every rank gets the same
    number of steps per epoch, ceil(num_batches / W); a rank whose stripe is
    one batch short gets ``None`` for its last step and trains on an empty
    batch there, i.e. contributes a zero gradient to that step's all-reduce
    ("a rank that is one batch short contributes a zero
    gradient").  Every batch of the epoch is still trained exactly once and
    every rank issues the same number of collectives."""
    if world_size < 1 or not (0 <= rank < world_size):
        raise ValueError("need 0 <= rank < world_size")
    own = list(range(rank, num_batches, world_size))
    if pad:
        steps = -(-num_batches // world_size)
        own += [None] * (steps - len(own))
    return own


def steps_per_epoch(num_batches: int, world_size: int) -> int:
    """Training steps (= gradient all-reduces) per epoch on every rank."""
    return -(-num_batches // world_size)


def epoch_schedule(num_batches: int, rank: int, world_size: int, epochs: int, cache_period: int = 1,
                   start_epoch: int = 0):
    """The rank's whole step schedule over ``epochs`` epochs: a list of
    ``(epoch, index_or_None, refresh_cache_before)`` in issue order.  This is
    what ``GraphedTrainer.run_epoch`` executes; the cache is redrawn at the
    first step of every epoch with ``epoch % cache_period == 0``
    (pool.py:133-135) with the key ``[seed, 33, epoch]`` — the same points on
    every rank, so the replicated caches stay identical."""
    out = []
    for e in range(start_epoch, start_epoch + epochs):
        idx = rank_batches(num_batches, rank, world_size, pad=world_size > 1)
        for j, i in enumerate(idx):
            out.append((e, i, j == 0 and (e == start_epoch or e % cache_period == 0)))
    return out


def make_allreduce(group=None, force: bool = False):
    """Sum-all-reduce of the flat gradient; returns the 1/W scale for Adam.
    Stream-ordered and CUDA-graph capturable with NCCL (the engine captures it
    between backward and Adam).  ``force`` issues the collective even at
    W == 1 (exercises the captured-NCCL path on one GPU)."""

    def allreduce(grad: torch.Tensor) -> float:
        w = dist.get_world_size(group)
        if w > 1 or force:
            dist.all_reduce(grad, op=dist.ReduceOp.SUM, group=group)
        return 1.0 / w

    return allreduce


def init_from_env(backend: str = "nccl"):
    """Initialise from torchrun's env (RANK / WORLD_SIZE / LOCAL_RANK / MASTER_*)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    force = os.environ.get("GNS_FORCE_DIST", "0") == "1"
    if (world > 1 or force) and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29531")
        os.environ.setdefault("RANK", str(rank))
        os.environ.setdefault("WORLD_SIZE", str(world))
        # collectives are captured into the step's CUDA graph (torch CUDA
        # graphs + DDP notes: no async error-handling watchdog on them)
        os.environ.setdefault("TORCH_NCCL_ASYNC_ERROR_HANDLING", "0")
        kw = {}
        if backend == "nccl":
            torch.cuda.set_device(local)
            kw["device_id"] = torch.device("cuda", local)
        dist.init_process_group(backend, **kw)
    return rank, world, local


def max_over_ranks(value: float, device=None) -> float:
    """Timing rule: the step time is the max over ranks."""
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
