"""GPU data loader (reference: pool.py).

``SamplerPool(g, config, num_workers=1, queue_capacity=8)`` keeps the
reference's contract (pool.py:1-13, 88-198): batch content is a pure function
of (seed, epoch, index), batches arrive in index order, the cache is rebuilt
at epoch boundaries every ``cache_period`` epochs (stop-the-world swap).

B200 mapping of the reference's process pool: a "worker" is an in-flight
sampling slot — a ``MiniBatchSampler`` with its own HBM buffers — driven on a
dedicated CUDA stream, so batch i+1 is sampled while the consumer trains on
batch i.  ``num_workers`` slots (capped at ``queue_capacity``) are kept in
flight.  Rank striding for data parallelism is ``index ≡ rank (mod world)``
exactly like the reference's worker striding (pool.py:80).

Batch lifetime: a yielded ``BatchItem.minibatch`` is a view of its slot's
buffers and stays valid until the consumer advances the iterator ``depth``
more times (the slot is then re-sampled).  ``copy=True`` yields independent
clones instead — the reference's semantics (every batch its own arrays), at
the cost of one device copy per batch; use it when batches are kept (e.g.
``list(pool.iter_epoch(e))``).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _lib
from . import cache as cache_mod
from .graph import Graph
from .sampling import BatchRng, MiniBatch, MiniBatchSampler, SamplerConfig

_SHUFFLE = 31
_BATCH = 32
_CACHE = 33


@dataclass
class BatchItem:
    """pool.py:36-41; sample_ms is measured with CUDA events on the sampling stream."""

    epoch: int
    index: int
    minibatch: MiniBatch
    _t0: object = None
    _t1: object = None

    @property
    def sample_ms(self) -> float:
        if self._t0 is None:
            return 0.0
        self._t1.synchronize()
        return float(self._t0.elapsed_time(self._t1))


def cache_probs(g: Graph, config: SamplerConfig):
    """pool.py:44-57: "auto" -> degree iff >= 50% of nodes train, else walk."""
    mode = config.cache_mode
    if mode == "auto":
        n_train = g.train_ids().numel()
        mode = "degree" if n_train * 2 >= g.num_nodes else "walk"
    if mode == "degree":
        return cache_mod.degree_probs(g)
    return cache_mod.random_walk_probs(g, g.train_ids(), config.fanouts, config.num_layers)


def exact_tables(g: Graph, config: SamplerConfig, probs, cache_size: int) -> dict:
    """pool.py:140-151: one gns-exact edge-inclusion table per distinct
    (fanout, cache_only) of the layer chain."""
    from .sampling import estimate_edge_inclusion
    tables = {}
    L = config.num_layers
    for layer in range(L, 0, -1):
        k = int(config.fanouts[L - layer])
        co = bool(config.input_layer_cache_only and layer == 1)
        if (k, co) not in tables:
            tables[(k, co)] = estimate_edge_inclusion(g, probs, cache_size, k, co,
                                                      resamples=config.exact_resamples, seed=config.seed)
    return tables


def num_batches(g: Graph, config: SamplerConfig) -> int:
    n = g.train_ids().numel()
    return (n + config.batch_size - 1) // config.batch_size


def epoch_targets_device(g: Graph, config: SamplerConfig, epoch: int, index: int, out: torch.Tensor,
                         stream=None) -> int:
    """Batch ``index`` of pool.py:60-66's partition, written into ``out``."""
    ids = g.train_ids()
    n = ids.numel()
    b = config.batch_size
    begin = index * b
    count = min(b, n - begin)
    _lib.call("gns_epoch_targets", ids.data_ptr(), n, config.seed & 0xFFFFFFFF, epoch & 0xFFFFFFFF,
              begin, count, out.data_ptr(), _lib.stream_ptr(stream))
    return count


def epoch_targets(g: Graph, config: SamplerConfig, epoch: int) -> list:
    """pool.py:60-66: shuffled train-node partition, one device tensor per batch."""
    ids = g.train_ids()
    n = ids.numel()
    out = torch.empty(max(n, 1), dtype=torch.int32, device=g.device)
    _lib.call("gns_epoch_targets", ids.data_ptr(), n, config.seed & 0xFFFFFFFF, epoch & 0xFFFFFFFF, 0, n,
              out.data_ptr(), _lib.stream_ptr())
    return [out[i:i + config.batch_size] for i in range(0, n, config.batch_size)]


class SamplerPool:
    """Produces one epoch of mini-batches at a time (pool.py:88-198)."""

    def __init__(self, g: Graph, config: SamplerConfig, num_workers: int = 1, queue_capacity: int = 8,
                 rank: int = 0, world_size: int = 1, copy: bool = False):
        if num_workers < 1:
            raise ValueError("num_workers must be >= 1")
        if queue_capacity < 1:
            raise ValueError("queue_capacity must be >= 1")
        _lib.require_cuda()
        self.graph = g
        self.config = config
        self.num_workers = num_workers
        self.queue_capacity = queue_capacity
        self.rank = rank
        self.world_size = world_size
        self.copy = bool(copy)
        self.cache = None
        self._probs = None
        self._tables = None
        self.depth = max(1, min(num_workers, queue_capacity, 4))
        self.slots = [MiniBatchSampler(g, config) for _ in range(self.depth)]
        self.stream = torch.cuda.Stream(device=g.device)
        self._released = [None] * self.depth

    def _refresh_cache(self, epoch: int) -> None:
        """pool.py:109-129 (degree/analytic; gns-exact tables are §8(f)3)."""
        if self.config.strategy != "GNS":
            return
        if self._probs is None:
            self._probs = cache_probs(self.graph, self.config)
        cache_size = int(round(self.config.cache_frac * self.graph.num_nodes))
        self.cache = cache_mod.build_cache(self.graph, self._probs, cache_size, epoch=epoch,
                                           rng_seed=[self.config.seed, _CACHE, epoch],
                                           positions=self.config.weight_policy == "gns-exact")
        if self.config.weight_policy == "gns-exact" and self._tables is None:
            self._tables = exact_tables(self.graph, self.config, self._probs, cache_size)

    def indices(self, epoch: int):
        from .dist import rank_batches
        return rank_batches(num_batches(self.graph, self.config), self.rank, self.world_size)

    def _launch(self, slot: int, epoch: int, index: int):
        eng = self.slots[slot]
        with torch.cuda.stream(self.stream):
            if self._released[slot] is not None:
                self.stream.wait_event(self._released[slot])
            t0 = torch.cuda.Event(enable_timing=True)
            t0.record(self.stream)
            n = epoch_targets_device(self.graph, self.config, epoch, index, eng.targets, self.stream)
            ev = eng.sample_async(None, n, BatchRng(self.config.seed, epoch, index), self.cache, self.stream,
                                  exact_tables=self._tables)
            t1 = torch.cuda.Event(enable_timing=True)
            t1.record(self.stream)
        return ev, t0, t1

    def iter_epoch(self, epoch: int):
        """Yield this epoch's BatchItems in batch-index order (this rank's share)."""
        if self.config.strategy == "GNS" and (self.cache is None or epoch % self.config.cache_period == 0):
            # stop-the-world swap: no slot may still read the old cache
            self.stream.synchronize()
            self._refresh_cache(epoch)
            torch.cuda.current_stream().synchronize()
        idx = self.indices(epoch)
        pending = {}
        nxt = 0
        for j in range(min(self.depth, len(idx))):
            pending[j] = self._launch(j % self.depth, epoch, idx[j])
            nxt = j + 1
        for j, index in enumerate(idx):
            slot = j % self.depth
            ev, t0, t1 = pending.pop(j)
            mb = self.slots[slot].collect(ev, policy_gns=self.config.weight_policy)
            torch.cuda.current_stream().wait_event(ev)
            if self.copy:
                mb = mb.clone()
            yield BatchItem(epoch=epoch, index=index, minibatch=mb, _t0=t0, _t1=t1)
            # the consumer is done with this slot once its queued work finishes
            rel = torch.cuda.Event()
            rel.record(torch.cuda.current_stream())
            self._released[slot] = rel
            if nxt < len(idx):
                pending[nxt] = self._launch(nxt % self.depth, epoch, idx[nxt])
                nxt += 1

    def run(self, epochs: int):
        """pool.py:195-198."""
        for epoch in range(epochs):
            yield from self.iter_epoch(epoch)
