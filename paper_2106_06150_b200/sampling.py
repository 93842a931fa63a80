"""Mini-batch construction on B200 (reference: sampling.py).

Drop-in names: ``SamplerConfig``, ``LayerBlock``, ``MiniBatch``,
``sample_neighbors_uniform``, ``sample_neighbors_gns``, ``build_minibatch``,
``gns_weight_paper``, ``isolated_fraction``, ``validate_minibatch``.

The ``rng`` argument is a :class:`BatchRng` — the Philox key (seed, epoch,
batch[, layer]) — instead of a numpy ``Generator``: the B200 kernels draw
their own counter-based keys per (node, layer, phase, position), which is the
SPEC's "deterministic per (seed, epoch, batch_index, layer, dst node id)"
contract.  ``SamplerPool`` derives it from (seed, epoch, index)
exactly where the reference derives ``default_rng([seed, 32, epoch, index])``
(pool.py:70).

``MiniBatchSampler`` is the engine: capacity-sized HBM buffers for every
layer (static bounds from the fanout product) so a whole
batch is sampled with device-side counts and no host synchronisation; the
host reads all counts once per batch (``DeviceMiniBatch.sync``).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import InvariantError
from .cache import CacheState
from .graph import Graph

STRATEGIES = ("NS", "GNS", "LADIES")
WEIGHT_POLICIES = ("uniform", "gns-paper", "gns-exact", "ladies")


@dataclass(frozen=True)
class SamplerConfig:
    """sampling.py:80-126 (same fields, defaults and validation)."""

    strategy: str = "NS"
    fanouts: tuple = (15, 10, 5)
    layer_size: int = 512
    cache_frac: float = 0.01
    cache_period: int = 1
    cache_mode: str = "auto"
    input_layer_cache_only: bool = True
    batch_size: int = 1000
    seed: int = 0
    weight_policy: str = ""
    exact_resamples: int = 64

    def __post_init__(self):
        if self.strategy not in STRATEGIES:
            raise ValueError(f"unknown strategy {self.strategy!r}")
        if len(self.fanouts) < 1 or any(k < 1 for k in self.fanouts):
            raise ValueError("fanouts must be a non-empty tuple of counts >= 1")
        if not (0.0 < self.cache_frac <= 1.0):
            raise ValueError("cache_frac must be in (0, 1]")
        if self.cache_period < 1:
            raise ValueError("cache_period must be >= 1")
        if self.cache_mode not in ("auto", "degree", "walk"):
            raise ValueError(f"unknown cache_mode {self.cache_mode!r}")
        if self.batch_size < 1:
            raise ValueError("batch_size must be >= 1")
        if self.layer_size < 1:
            raise ValueError("layer_size must be >= 1")
        if not self.weight_policy:
            default = {"NS": "uniform", "GNS": "gns-paper", "LADIES": "ladies"}[self.strategy]
            object.__setattr__(self, "weight_policy", default)
        if self.weight_policy not in WEIGHT_POLICIES:
            raise ValueError(f"unknown weight_policy {self.weight_policy!r}")

    @property
    def num_layers(self) -> int:
        return len(self.fanouts)


@dataclass(frozen=True)
class BatchRng:
    """Philox key of one mini-batch: (seed, epoch, batch); ``layer`` is only
    used by the single-layer entry points."""

    seed: int = 0
    epoch: int = 0
    batch: int = 0
    layer: int = 0

    def cstruct(self, layer=None):
        return _lib.GnsRng(self.seed & 0xFFFFFFFF, self.epoch & 0xFFFFFFFF, self.batch & 0xFFFFFFFF,
                           (self.layer if layer is None else layer) & 0xFF)


def _as_rng(rng) -> BatchRng:
    """The reference injects a duck-typed numpy ``rng`` (sampling.py:166,214,
    233).  The device sampler draws counter-based Philox keys, so a numpy
    ``Generator`` (or anything with ``.integers``) seeds one: three 32-bit
    draws become the (seed, epoch, batch) Philox key.  Deterministic in the
    generator's state and it advances the generator, but the keys are not the
    ones numpy's ``random()`` would have produced (PCG64 is not restated on
    the device); pass ``BatchRng`` to name the key directly."""
    if isinstance(rng, BatchRng):
        return rng
    if hasattr(rng, "integers"):
        s, e, b = (int(x) for x in rng.integers(0, 1 << 32, size=3, dtype=np.uint64))
        return BatchRng(s, e, b)
    raise TypeError("the B200 sampler draws counter-based Philox keys: pass "
                    "paper_2106_06150_b200.BatchRng(seed, epoch, batch) or a numpy Generator as rng")


@dataclass(eq=False)
class LayerBlock:
    """sampling.py:32-60, device tensors (ids int32, weights float64)."""

    dst_nodes: torch.Tensor
    src_nodes: torch.Tensor
    edge_src: torch.Tensor
    edge_dst: torch.Tensor
    edge_weight: torch.Tensor
    edge_cached: torch.Tensor
    dst_degree: torch.Tensor
    fanout: int | None
    policy: str
    self_pos: torch.Tensor | None = None
    edge_node: torch.Tensor | None = None
    row_scan: torch.Tensor | None = None
    _c: object = None  # gns_block_t of the engine buffers
    counts: torch.Tensor | None = None  # int32[GNS_CNT_N] device counters of this block

    @property
    def num_edges(self) -> int:
        return int(self.edge_src.shape[0])

    def clone(self) -> "LayerBlock":
        """Independent copy (own device buffers and gns_block_t), no longer
        tied to the sampler slot that produced it."""
        def c(t):
            return None if t is None else t.clone()
        b = LayerBlock(dst_nodes=c(self.dst_nodes), src_nodes=c(self.src_nodes), edge_src=c(self.edge_src),
                       edge_dst=c(self.edge_dst), edge_weight=c(self.edge_weight), edge_cached=c(self.edge_cached),
                       dst_degree=c(self.dst_degree), fanout=self.fanout, policy=self.policy,
                       self_pos=c(self.self_pos), edge_node=c(self.edge_node), row_scan=c(self.row_scan),
                       counts=c(self.counts))
        if self.counts is not None:
            b._c = _lib.GnsBlock(*(0 if t is None else t.data_ptr() for t in (
                b.row_scan, b.dst_degree, b.self_pos, None, b.edge_node, b.edge_src, b.edge_dst,
                b.edge_weight, b.edge_cached, b.src_nodes, b.counts)))
        return b

    def to_numpy(self):
        """Reference dtypes (int64 / float64 / bool) on the host."""
        from types import SimpleNamespace
        return SimpleNamespace(
            dst_nodes=self.dst_nodes.long().cpu().numpy(), src_nodes=self.src_nodes.long().cpu().numpy(),
            edge_src=self.edge_src.long().cpu().numpy(), edge_dst=self.edge_dst.long().cpu().numpy(),
            edge_weight=self.edge_weight.cpu().numpy(), edge_cached=self.edge_cached.bool().cpu().numpy(),
            dst_degree=self.dst_degree.long().cpu().numpy(), fanout=self.fanout, policy=self.policy,
            num_edges=self.num_edges)


@dataclass(eq=False)
class MiniBatch:
    """sampling.py:63-77: blocks input layer first."""

    blocks: tuple
    targets: torch.Tensor
    input_nodes: torch.Tensor

    @property
    def num_layers(self) -> int:
        return len(self.blocks)

    def clone(self) -> "MiniBatch":
        """Independent copy of a batch (the façade's batches are views of a
        sampler slot's buffers that the slot's next batch overwrites)."""
        blocks = tuple(b.clone() for b in self.blocks)
        return MiniBatch(blocks=blocks, targets=blocks[-1].dst_nodes, input_nodes=blocks[0].src_nodes)


# ---------------------------------------------------------------------------
# engine
# ---------------------------------------------------------------------------

@dataclass
class _LayerBuffers:
    k: int
    layer: int
    cache_only: bool
    max_dst: int
    max_edges: int
    max_src: int
    row_scan: torch.Tensor
    dst_degree: torch.Tensor
    self_pos: torch.Tensor
    hub_rows: torch.Tensor
    edge_node: torch.Tensor
    edge_src: torch.Tensor
    edge_dst: torch.Tensor
    edge_weight: torch.Tensor
    edge_cached: torch.Tensor
    src_nodes: torch.Tensor
    counts: torch.Tensor
    cblock: object = None


class MiniBatchSampler:
    """Static-capacity device buffers + the L-layer sampling chain.

    Layer buffers are ordered output layer first (the reference's loop order
    ``layer = L..1``, sampling.py:314).  Capacities: the top layer has at most
    ``batch_size`` dst rows; each layer's edges <= dst * k; src <= min(N, dst +
    edges), which is the next layer's dst bound.
    """

    def __init__(self, g: Graph, config: SamplerConfig, max_targets: int | None = None):
        _lib.require_cuda()
        if config.strategy == "LADIES":
            raise NotImplementedError("LADIES is a baseline outside the GNS hot path (SURVEY.md §2)")
        self.g = g
        self.config = config
        dev = g.device
        self.device = dev
        L = config.num_layers
        self.max_targets = int(max_targets or config.batch_size)
        n = g.num_nodes
        # all per-layer device counters in one tensor -> one D2H per batch
        self.counts = torch.zeros((L, _lib.CNT_N), dtype=torch.int32, device=dev)
        self.counts_host = torch.zeros((L, _lib.CNT_N), dtype=torch.int32).pin_memory()
        self.layers: list[_LayerBuffers] = []
        dst_cap = self.max_targets
        for i, layer in enumerate(range(L, 0, -1)):
            k = int(config.fanouts[L - layer])
            edge_cap = dst_cap * k
            src_cap = min(n, dst_cap + edge_cap)
            lb = _LayerBuffers(
                k=k, layer=layer,
                cache_only=(config.strategy == "GNS" and config.input_layer_cache_only and layer == 1),
                max_dst=dst_cap, max_edges=edge_cap, max_src=src_cap,
                row_scan=torch.empty(dst_cap + 1, dtype=torch.int64, device=dev),
                dst_degree=torch.empty(dst_cap, dtype=torch.int32, device=dev),
                self_pos=torch.empty(dst_cap, dtype=torch.int32, device=dev),
                hub_rows=torch.empty(6 * max(dst_cap, 1), dtype=torch.int32, device=dev),
                edge_node=torch.empty(max(edge_cap, 1), dtype=torch.int32, device=dev),
                edge_src=torch.empty(max(edge_cap, 1), dtype=torch.int32, device=dev),
                edge_dst=torch.empty(max(edge_cap, 1), dtype=torch.int32, device=dev),
                edge_weight=torch.empty(max(edge_cap, 1), dtype=torch.float64, device=dev),
                edge_cached=torch.empty(max(edge_cap, 1), dtype=torch.uint8, device=dev),
                src_nodes=torch.empty(max(src_cap, 1), dtype=torch.int32, device=dev),
                counts=self.counts[i],
            )
            lb.cblock = _lib.GnsBlock(*(t.data_ptr() for t in (
                lb.row_scan, lb.dst_degree, lb.self_pos, lb.hub_rows, lb.edge_node, lb.edge_src,
                lb.edge_dst, lb.edge_weight, lb.edge_cached, lb.src_nodes, lb.counts)))
            self.layers.append(lb)
            dst_cap = src_cap
        lib = _lib.lib()
        self.targets = torch.empty(max(self.max_targets, 1), dtype=torch.int32, device=dev)
        self.seeds0 = torch.empty(max(self.max_targets, 1), dtype=torch.int32, device=dev)
        self.n_seeds0 = torch.zeros(1, dtype=torch.int32, device=dev)
        # dedup bitmaps must start zeroed; every call leaves them zeroed
        self.ws_sample = _lib.workspace(lib.gns_sample_workspace_size(n, max(l.max_dst for l in self.layers)), dev,
                                        zero=True)
        self.ws_relabel = _lib.workspace(lib.gns_relabel_workspace_size(n), dev, zero=True)

    # -- device-side chain -------------------------------------------------------
    def _exact(self, tables, lb):
        if self.config.strategy != "GNS" or self.config.weight_policy != "gns-exact":
            return None
        t = (tables or {}).get((lb.k, bool(lb.cache_only)))
        if t is None:
            raise ValueError(f"missing edge-inclusion table for fanout={lb.k}, cache_only={bool(lb.cache_only)}")
        return t.data_ptr()

    def sample_async(self, targets: torch.Tensor | None, n_targets: int, rng: BatchRng,
                     cache: CacheState | None, stream=None, exact_tables=None):
        """Enqueue the whole L-layer chain on ``stream``; targets (int32 device,
        any order, may repeat) are deduplicated+sorted first (sampling.py:312).
        If ``targets`` is None the caller already wrote ``self.targets``."""
        s = _lib.stream_ptr(stream)
        if targets is not None:
            if targets.numel() > self.max_targets:
                raise ValueError(f"{targets.numel()} targets exceed capacity {self.max_targets}")
            self.targets[:targets.numel()].copy_(targets.to(torch.int32), non_blocking=True)
            n_targets = targets.numel()
        _lib.call("gns_unique_sorted", self.g.num_nodes, self.targets.data_ptr(), None, int(n_targets),
                  self.seeds0.data_ptr(), self.n_seeds0.data_ptr(), self.ws_relabel.data_ptr(),
                  self.ws_relabel.numel(), s)
        gns = self.config.strategy == "GNS"
        if gns and cache is None:
            raise ValueError("GNS sampling needs a CacheState")
        cstruct = cache.cstruct() if gns else None
        seeds, n_dev = self.seeds0, self.n_seeds0
        gc = self.g.cstruct()
        for lb in self.layers:
            _lib.call("gns_sample_layer", gc, cstruct, seeds.data_ptr(), n_dev.data_ptr(), lb.max_dst,
                      lb.k, int(lb.cache_only), self._exact(exact_tables, lb), rng.cstruct(lb.layer), None, lb.cblock,
                      self.ws_sample.data_ptr(), self.ws_sample.numel(), s)
            seeds = lb.src_nodes
            n_dev = lb.counts[_lib.CNT_SRC:_lib.CNT_SRC + 1]
        self.counts_host.copy_(self.counts, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(stream if stream is not None else torch.cuda.current_stream())
        return ev

    def enqueue_device(self, train_ids: torch.Tensor | None, step_dev: torch.Tensor, cache: CacheState | None,
                       stream=None, exact_tables=None, after_layer=None, epoch_perm: torch.Tensor | None = None,
                       step_src: torch.Tensor | None = None):
        """Graph-capturable chain: the batch's targets (pool.py:60-66 slice
        begin/count) and Philox key come from the device gns_step_t
        ``step_dev``; no host synchronisation, fixed kernel arguments.  With
        ``train_ids=None`` the caller already wrote ``targets`` and
        ``n_targets_dev`` (host-provided targets)."""
        s = _lib.stream_ptr(stream)
        if not hasattr(self, "n_targets_dev"):
            self.n_targets_dev = torch.zeros(1, dtype=torch.int32, device=self.device)
        if step_src is not None and (epoch_perm is None or self.max_targets > 1024):
            with torch.cuda.stream(stream or torch.cuda.current_stream()):
                step_dev.copy_(step_src, non_blocking=True)
            step_src = None
        if epoch_perm is not None and self.max_targets <= 1024:
            # slice of the precomputed epoch permutation + np.unique, one CTA
            # step_src (pinned host) -> step_dev inside the kernel when given
            src = step_src if step_src is not None else step_dev
            _lib.call("gns_batch_slice_sorted", epoch_perm.data_ptr(), epoch_perm.numel(), src.data_ptr(),
                      step_dev.data_ptr() if step_src is not None else None, self.max_targets,
                      self.seeds0.data_ptr(), self.n_seeds0.data_ptr(), s)
        elif train_ids is not None and self.max_targets <= 1024:
            # epoch slice + np.unique in one single-CTA kernel
            _lib.call("gns_batch_targets_sorted", train_ids.data_ptr(), train_ids.numel(), step_dev.data_ptr(),
                      self.max_targets, self.seeds0.data_ptr(), self.n_seeds0.data_ptr(), s)
        else:
            if train_ids is not None:
                _lib.call("gns_epoch_targets_dev", train_ids.data_ptr(), train_ids.numel(), step_dev.data_ptr(),
                          self.max_targets, self.targets.data_ptr(), self.n_targets_dev.data_ptr(), s)
            _lib.call("gns_unique_sorted", self.g.num_nodes, self.targets.data_ptr(), self.n_targets_dev.data_ptr(),
                      self.max_targets, self.seeds0.data_ptr(), self.n_seeds0.data_ptr(),
                      self.ws_relabel.data_ptr(), self.ws_relabel.numel(), s)
        gns = self.config.strategy == "GNS"
        if gns and cache is None:
            raise ValueError("GNS sampling needs a CacheState")
        cstruct = cache.cstruct() if gns else None
        seeds, n_dev = self.seeds0, self.n_seeds0
        gc = self.g.cstruct()
        rng = BatchRng()
        for lb in self.layers:
            _lib.call("gns_sample_layer", gc, cstruct, seeds.data_ptr(), n_dev.data_ptr(), lb.max_dst,
                      lb.k, int(lb.cache_only), self._exact(exact_tables, lb), rng.cstruct(lb.layer),
                      step_dev.data_ptr(), lb.cblock,
                      self.ws_sample.data_ptr(), self.ws_sample.numel(), s)
            if after_layer is not None:
                after_layer(lb)
            seeds = lb.src_nodes
            n_dev = lb.counts[_lib.CNT_SRC:_lib.CNT_SRC + 1]

    def collect(self, event=None, policy_ns="uniform", policy_gns="gns-paper") -> MiniBatch:
        """Wait for the counts of the last ``sample_async`` and wrap the buffers
        as a MiniBatch (views sized to the real counts; blocks input first)."""
        if event is not None:
            event.synchronize()
        else:
            torch.cuda.current_stream().synchronize()
        return self._wrap(self.counts_host.tolist(), policy_ns, policy_gns)

    def snapshot(self, policy_ns="uniform", policy_gns="gns-paper") -> MiniBatch:
        """The batch currently held in this slot's buffers, whoever sampled it
        (e.g. a captured engine step): synchronises the device, reads the
        device counts and wraps the buffers (views; raises on error flags)."""
        torch.cuda.synchronize()
        return self._wrap(self.counts.cpu().tolist(), policy_ns, policy_gns)

    def _wrap(self, c, policy_ns, policy_gns) -> MiniBatch:
        err = 0
        blocks = []
        seeds_n = None
        for i, lb in enumerate(self.layers):
            nd, ne, nsrc, e = c[i][_lib.CNT_DST], c[i][_lib.CNT_EDGES], c[i][_lib.CNT_SRC], c[i][_lib.CNT_ERR]
            err |= e
            dst = self.seeds0[:nd] if i == 0 else self.layers[i - 1].src_nodes[:nd]
            blocks.append(LayerBlock(
                dst_nodes=dst, src_nodes=lb.src_nodes[:nsrc], edge_src=lb.edge_src[:ne],
                edge_dst=lb.edge_dst[:ne], edge_weight=lb.edge_weight[:ne],
                edge_cached=lb.edge_cached[:ne], dst_degree=lb.dst_degree[:nd], fanout=lb.k,
                policy=policy_gns if self.config.strategy == "GNS" else policy_ns,
                self_pos=lb.self_pos[:nd], edge_node=lb.edge_node[:ne], row_scan=lb.row_scan[:nd + 1],
                _c=lb.cblock, counts=lb.counts))
            seeds_n = nsrc
        if err & _lib.ERRBIT_ZEROPROB:
            raise ValueError("inclusion probability is zero for a cached draw")
        if err & _lib.ERRBIT_CAPACITY:
            raise InvariantError("neighbour selection did not converge (capacity)")
        if err & _lib.ERRBIT_ZEROQ:
            raise InvariantError("sampled an edge with zero estimated inclusion")
        blocks.reverse()
        return MiniBatch(blocks=tuple(blocks), targets=blocks[-1].dst_nodes,
                         input_nodes=blocks[0].src_nodes)

    def sample(self, targets, rng: BatchRng, cache: CacheState | None = None, exact_tables=None) -> MiniBatch:
        t = torch.as_tensor(targets, device=self.device)
        ev = self.sample_async(t, t.numel(), rng, cache, exact_tables=exact_tables)
        return self.collect(ev, policy_gns=self.config.weight_policy)


_ENGINES: dict = {}


def _engine(g: Graph, config: SamplerConfig, n_targets: int) -> MiniBatchSampler:
    key = (id(g), config, )
    eng = _ENGINES.get(key)
    if eng is None or eng.max_targets < n_targets:
        eng = MiniBatchSampler(g, config, max_targets=max(n_targets, config.batch_size))
        _ENGINES.clear()
        _ENGINES[key] = eng
    return eng


def build_minibatch(g: Graph, cache: CacheState | None, targets, config: SamplerConfig, rng,
                    exact_tables: dict | None = None) -> MiniBatch:
    """sampling.py:299-336.  Returned tensors are views of engine buffers that
    the next call on the same (graph, config) overwrites; clone to keep."""
    rng = _as_rng(rng)
    if config.strategy == "LADIES":
        raise NotImplementedError("LADIES is outside the GNS hot path (SURVEY.md §2)")
    if config.strategy == "GNS" and cache is None:
        raise ValueError("GNS sampling needs a CacheState")
    t = torch.as_tensor(targets, device=g.device)
    eng = _engine(g, config, t.numel())
    return eng.sample(t, rng, cache if config.strategy == "GNS" else None, exact_tables=exact_tables)


def _single_layer(g, cache, seeds, k, cache_only, rng, strategy, policy="", exact=None):
    rng = _as_rng(rng)
    if k < 1:
        raise ValueError("fanout must be >= 1")
    cfg = SamplerConfig(strategy=strategy, fanouts=(int(k),), weight_policy=policy,
                        input_layer_cache_only=bool(cache_only), batch_size=max(1, len(seeds)))
    t = torch.as_tensor(seeds, device=g.device)
    eng = MiniBatchSampler(g, cfg, max_targets=max(1, t.numel()))
    eng.layers[0].layer = rng.layer
    eng.layers[0].cache_only = bool(cache_only) and strategy == "GNS"
    tables = None if exact is None else {(int(k), bool(cache_only) and strategy == "GNS"): exact}
    mb = eng.sample(t, rng, cache, exact_tables=tables)
    return mb.blocks[0]


def sample_neighbors_uniform(g: Graph, seeds, k: int, rng) -> LayerBlock:
    """sampling.py:155-170: min(k, deg) uniform neighbours, weight deg/min(k, deg)."""
    return _single_layer(g, None, seeds, k, False, rng, "NS")


def sample_neighbors_gns(g: Graph, cache: CacheState, seeds, k: int, cache_only: bool, rng,
                         policy: str = "gns-paper", exact_weights=None) -> LayerBlock:
    """sampling.py:189-266 (gns-paper policy)."""
    if k < 1:
        raise ValueError("fanout must be >= 1")
    if policy not in ("gns-paper", "gns-exact"):
        raise ValueError(f"unsupported GNS weight policy {policy!r}")
    if policy == "gns-exact":
        if exact_weights is None:
            raise ValueError("gns-exact policy needs an edge-inclusion table")
        return _single_layer(g, cache, seeds, k, cache_only, rng, "GNS", "gns-exact",
                             torch.as_tensor(exact_weights, device=g.device).to(torch.float64).contiguous())
    return _single_layer(g, cache, seeds, k, cache_only, rng, "GNS")


def estimate_edge_inclusion(g: Graph, probs, cache_size: int, k: int, cache_only: bool, resamples: int = 64,
                            seed=0) -> torch.Tensor:
    """sampling.py:269-296 on the device: CSR-aligned float64 table of per-edge
    inclusion probabilities over ``resamples`` cache draws (Philox key
    (seed, r), stream tag 21 = sampling.py:29 _FILL_STREAM)."""
    from .cache import seed_epoch
    _lib.require_cuda()
    w = probs.normalize().weights
    s32, _ = seed_epoch(seed)
    out = torch.empty(max(g.num_edges, 1), dtype=torch.float64, device=g.device)[:g.num_edges]
    ws = _lib.workspace(_lib.lib().gns_edge_inclusion_workspace_size(g.num_nodes, int(cache_size)), g.device)
    _lib.call("gns_estimate_edge_inclusion", g.cstruct(), w.data_ptr(), int(cache_size), int(k), int(bool(cache_only)),
              int(resamples), s32, out.data_ptr(), ws.data_ptr(), ws.numel(), _lib.stream_ptr())
    return out


def gns_weight_paper(p_v: float, cache_size: int, k: int, n_cached: int) -> float:
    """sampling.py:173-186 (scalar helper; Eq. 9 from the device kernel)."""
    if n_cached < 1 or k < 1:
        raise ValueError("need n_cached >= 1 and k >= 1")
    from .cache import inclusion_prob
    p_c = inclusion_prob(p_v, cache_size)
    if p_c <= 0.0:
        raise ValueError("inclusion probability is zero; cannot weight draw")
    return min(k, n_cached) / (k * p_c)


def isolated_fraction(mb: MiniBatch) -> float:
    """sampling.py:413-425 on the device."""
    block = mb.blocks[0]
    if mb.targets.numel() == 0:
        return 0.0
    indeg = torch.bincount(block.edge_dst.long(), minlength=block.dst_nodes.numel())
    tpos = torch.searchsorted(block.dst_nodes, mb.targets)
    return float((indeg[tpos] == 0).float().mean())


def validate_minibatch(g: Graph, mb: MiniBatch) -> None:
    """sampling.py:428-470 structural invariants, evaluated with device ops."""
    for i, block in enumerate(mb.blocks):
        d, s = block.dst_nodes, block.src_nodes
        if (d[1:] <= d[:-1]).any() or (s[1:] <= s[:-1]).any():
            raise InvariantError(f"block {i}: node arrays must be sorted unique")
        if not torch.isin(d, s).all():
            raise InvariantError(f"block {i}: dst nodes missing from src")
        if block.num_edges:
            if int(block.edge_src.max()) >= s.numel() or int(block.edge_dst.max()) >= d.numel():
                raise InvariantError(f"block {i}: edge index out of range")
            srcs = s[block.edge_src.long()].long()
            dsts = d[block.edge_dst.long()].long()
            # (src, dst) is an edge iff dst is in src's sorted row
            lo = g.indptr[srcs]
            hi = g.indptr[srcs + 1]
            # binary search per edge in its row
            l, h = lo.clone(), hi.clone()
            for _ in range(40):
                mid = (l + h) // 2
                v = g.indices[torch.clamp(mid, max=g.num_edges - 1)].long()
                go = v < dsts
                l = torch.where(go & (l < h), mid + 1, l)
                h = torch.where(~go & (l < h), mid, h)
            ok = (l < hi) & (g.indices[torch.clamp(l, max=g.num_edges - 1)].long() == dsts)
            if not ok.all():
                raise InvariantError(f"block {i}: sampled a non-edge")
            w = block.edge_weight
            if not torch.isfinite(w).all() or (w <= 0).any():
                raise InvariantError(f"block {i}: edge weights must be finite > 0")
            if block.fanout is not None:
                indeg = torch.bincount(block.edge_dst.long(), minlength=d.numel())
                if int(indeg.max()) > block.fanout:
                    raise InvariantError(f"block {i}: fanout bound {block.fanout} exceeded")
        if not torch.equal(block.dst_degree.long(), g.degrees[d.long()].long()):
            raise InvariantError(f"block {i}: stale dst degrees")
        if i + 1 < len(mb.blocks) and not torch.equal(d, mb.blocks[i + 1].src_nodes):
            raise InvariantError(f"block {i}: dst set does not chain into block {i + 1} src")
    if not torch.equal(mb.targets, mb.blocks[-1].dst_nodes):
        raise InvariantError("targets must equal the last block's dst set")
    if not torch.equal(mb.input_nodes, mb.blocks[0].src_nodes):
        raise InvariantError("input_nodes must equal the first block's src set")
