"""Cache engine on B200 (reference: cache.py).

Same API as the reference: ``ProbVector``, ``degree_probs``, ``sample_cache``,
``inclusion_prob``, ``CacheState``, ``build_cache``.  Every array lives in
HBM and every computation is a libgns.so kernel:

* ``degree_probs``  -> gns_degree_probs            (cache.py:53-58)
* ``sample_cache``  -> gns_cache_draw              (cache.py:87-103): Philox
  exponential race + 11-bit radix select + ordered compaction
* ``inclusion_prob``-> gns_inclusion               (cache.py:106-117)
* ``build_cache``   -> draw + inclusion + gns_cached_csr_count/fill
  (cache.py:160-197; the induced CSR is built by filtering the full CSR with
  the cache bitmap, which yields the same ascending rows)

``rng_seed`` follows the reference's call sites: ``[seed, 33, epoch]`` (pool.py:117)
keys Philox with (seed, epoch); a bare int is (seed, 0).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .graph import Graph, NodeSet

_CACHE_TAG = 33


def seed_key(rng_seed) -> tuple[int, int, int]:
    """Map the reference's ``rng_seed`` forms to the Philox key (seed, epoch)
    and stream tag: ``[seed, tag, epoch]`` (pool.py:117 uses tag 33,
    sampling.py:284 tag 21) keeps its tag; other forms use 33."""
    if np.isscalar(rng_seed):
        return int(rng_seed) & 0xFFFFFFFF, 0, _CACHE_TAG
    s = [int(x) for x in np.asarray(rng_seed, dtype=np.int64).ravel()]
    if len(s) == 3:
        return s[0] & 0xFFFFFFFF, s[2] & 0xFFFFFFFF, s[1] & 0xFF
    if len(s) == 2:
        return s[0] & 0xFFFFFFFF, s[1] & 0xFFFFFFFF, _CACHE_TAG
    if len(s) == 1:
        return s[0] & 0xFFFFFFFF, 0, _CACHE_TAG
    h = 0
    for x in s:
        h = (h * 1000003 + x) & 0xFFFFFFFF
    return h, 0, _CACHE_TAG


def seed_epoch(rng_seed) -> tuple[int, int]:
    s, e, _ = seed_key(rng_seed)
    return s, e


@dataclass(frozen=True, eq=False)
class ProbVector:
    """Non-negative per-node weights on the device (cache.py:25-50)."""

    weights: torch.Tensor
    normalized: bool = False

    def __post_init__(self):
        w = self.weights
        if not torch.is_tensor(w):
            w = torch.as_tensor(np.asarray(w, dtype=np.float64), device="cuda")
        w = w.to(torch.float64)
        bad = torch.logical_or(w < 0, ~torch.isfinite(w)).any()
        if bool(bad):
            raise ValueError("probability weights must be finite and >= 0")
        if self.normalized and abs(float(w.sum()) - 1.0) > 1e-9:
            raise ValueError("normalized ProbVector must sum to 1")
        object.__setattr__(self, "weights", w)

    def __len__(self) -> int:
        return int(self.weights.shape[0])

    def normalize(self) -> "ProbVector":
        if self.normalized:
            return self
        total = float(self.weights.sum())
        if total <= 0:
            raise ValueError("cannot normalize an all-zero weight vector")
        return ProbVector(self.weights / total, normalized=True)


def degree_probs(g: Graph) -> ProbVector:
    """cache.py:53-58: p_i = deg(i) / sum deg."""
    _lib.require_cuda()
    if g.num_edges == 0:
        raise ValueError("graph has no edges; degree distribution undefined")
    out = torch.empty(g.num_nodes, dtype=torch.float64, device=g.device)
    _lib.call("gns_degree_probs", g.cstruct(), out.data_ptr(), _lib.stream_ptr())
    return ProbVector(out, normalized=True)


def random_walk_probs(g: Graph, train, fanouts, num_layers: int) -> ProbVector:
    """cache.py:61-84: L-step spread of the training-set indicator
    (p <- d*(A p) + p, d_i = min(fanout, deg_i)/max(deg_i, 1)), normalised.
    ``train`` is a NodeSet or an id tensor/array."""
    _lib.require_cuda()
    if num_layers < 1:
        raise ValueError("num_layers must be >= 1")
    if len(fanouts) < num_layers:
        raise ValueError("need one fanout per layer")
    ids = train.ids if isinstance(train, NodeSet) else torch.as_tensor(train, device=g.device)
    ids = ids.to(device=g.device, dtype=torch.int32).contiguous()
    if ids.numel() == 0:
        raise ValueError("training set is empty")
    out = torch.empty(g.num_nodes, dtype=torch.float64, device=g.device)
    ws = _lib.workspace(_lib.lib().gns_random_walk_workspace_size(g.num_nodes), g.device)
    fan = (ctypes.c_int32 * num_layers)(*[int(f) for f in fanouts[:num_layers]])
    _lib.call("gns_random_walk_probs", g.cstruct(), ids.data_ptr(), ids.numel(), fan, num_layers, out.data_ptr(),
              ws.data_ptr(), ws.numel(), _lib.stream_ptr())
    return ProbVector(out, normalized=True)


class _DrawWorkspace:
    _cache: dict = {}

    @classmethod
    def get(cls, n: int, device) -> torch.Tensor:
        key = (n, str(device))
        ws = cls._cache.get(key)
        if ws is None:
            cls._cache.clear()
            ws = _lib.workspace(_lib.lib().gns_cache_draw_workspace_size(n), device)
            cls._cache[key] = ws
        return ws


def _draw(probs: ProbVector, cache_size: int, seed: int, epoch: int, stream=None, tag: int = _CACHE_TAG,
          out=None):
    w = probs.weights
    n = int(w.shape[0])
    dev = w.device
    cs = max(int(cache_size), 0)
    if out is not None:
        ids, bits, counts = out
    else:
        ids = torch.empty(max(cs, 1), dtype=torch.int32, device=dev)
        bits = torch.empty((n + 31) // 32, dtype=torch.int32, device=dev)
        counts = torch.zeros(2, dtype=torch.int64, device=dev)
    ws = _DrawWorkspace.get(n, dev)
    _lib.call("gns_cache_draw", w.data_ptr(), n, cs, seed, epoch, tag, ids.data_ptr(), bits.data_ptr(),
              counts.data_ptr(), ws.data_ptr(), ws.numel(), _lib.stream_ptr(stream))
    return ids, bits, counts


def sample_cache(probs: ProbVector, cache_size: int, rng_seed) -> NodeSet:
    """cache.py:87-103: min(cache_size, #positive) ids drawn without replacement
    with probability proportional to the weights (exponential race)."""
    _lib.require_cuda()
    seed, epoch, tag = seed_key(rng_seed)
    ids, bits, counts = _draw(probs, cache_size, seed, epoch, tag=tag)
    k = int(counts[0])
    return NodeSet(ids=ids[:k], mask_bits=bits, num_nodes=len(probs))


def inclusion_prob(p, cache_size: int):
    """cache.py:106-117: 1 - (1 - p)^|C| as -expm1(|C| log1p(-min(p, 1-1e-15)))."""
    _lib.require_cuda()
    scalar = np.isscalar(p)
    host = not torch.is_tensor(p)
    t = torch.as_tensor(np.asarray(p, dtype=np.float64) if host else p.to(torch.float64),
                        device="cuda").reshape(-1).contiguous()
    out = torch.empty_like(t)
    _lib.call("gns_inclusion", t.data_ptr(), t.numel(), int(cache_size), None, None,
              out.data_ptr(), _lib.stream_ptr())
    if scalar:
        return float(out[0])
    if host:
        return out.cpu().numpy().reshape(np.shape(p))
    return out.reshape(p.shape)


@dataclass(frozen=True, eq=False)
class CacheState:
    """cache.py:130-157: cache set + what samplers need, all in HBM."""

    nodes: NodeSet
    inclusion: torch.Tensor       # float64[N]
    cached_indptr: torch.Tensor   # int64[N+1]
    cached_indices: torch.Tensor  # int32[nnz]
    epoch: int
    source_probs: ProbVector
    cached_pos: torch.Tensor | None = None  # int32[nnz]: position in the full row (gns-exact)

    def __len__(self) -> int:
        return len(self.nodes)

    def num_cached_neighbors(self, v: int) -> int:
        return int(self.cached_indptr[v + 1] - self.cached_indptr[v])

    def cached_neighbors(self, v: int) -> torch.Tensor:
        return self.cached_indices[int(self.cached_indptr[v]):int(self.cached_indptr[v + 1])]

    def cstruct(self):
        c = getattr(self, "_c", None)
        if c is None:
            # the cached CSR arrays are prefixes of their buffers (_buf_cidx /
            # _buf_cpos): pass the buffer bases, which stay put across
            # in-place refreshes even when the prefix was empty (an empty
            # view's data_ptr is 0 — a graph captured with it would keep 0)
            cidx = getattr(self, "_buf_cidx", self.cached_indices)
            cpos = self.cached_pos if self.cached_pos is None else getattr(self, "_buf_cpos", self.cached_pos)
            c = _lib.GnsCache(self.cached_indptr.data_ptr(), cidx.data_ptr(),
                              self.nodes.mask_bits.data_ptr(), self.inclusion.data_ptr(),
                              None if cpos is None or cpos.numel() == 0 else cpos.data_ptr())
            object.__setattr__(self, "_c", c)
        return c

    def mask_word_rank(self, stream=None) -> torch.Tensor:
        """Per-word popcount rank of the cache bitmap (cache-slot lookup).
        Recomputed into the same buffer after a refresh (captured graphs
        that read it stay valid)."""
        r = getattr(self, "_rank", None)
        if r is None or self.__dict__.get("_rank_stale", False):
            bits = self.nodes.mask_bits
            if r is None:
                r = torch.empty_like(bits)
            ws = getattr(self, "_rank_ws", None)
            if ws is None:
                ws = _lib.workspace(1 << 20, bits.device)
                object.__setattr__(self, "_rank_ws", ws)
            _lib.call("gns_bitmap_rank", bits.data_ptr(), bits.numel(), r.data_ptr(), ws.data_ptr(),
                      ws.numel(), _lib.stream_ptr(stream))
            object.__setattr__(self, "_rank", r)
            object.__setattr__(self, "_rank_stale", False)
        return r


def build_cache(g: Graph, probs: ProbVector, cache_size: int, epoch: int = 0, rng_seed=0,
                inclusion_mode: str = "analytic", resamples: int = 64, positions: bool = True) -> CacheState:
    """cache.py:160-197 (analytic inclusion).  ``positions``: also record each
    cached-CSR entry's position in its full row (``cached_pos``, read only by
    the gns-exact policy); False skips that per-row pass."""
    _lib.require_cuda()
    if inclusion_mode == "empirical":
        raise NotImplementedError("empirical inclusion (cache.py:178-181) is outside the B200 "
                                  "hot path (SURVEY.md §8(f)3)")
    if inclusion_mode != "analytic":
        raise ValueError(f"unknown inclusion_mode {inclusion_mode!r}")
    return _build_cache_into(None, g, probs, cache_size, epoch, rng_seed, positions)


def refresh_cache(state: CacheState, g: Graph, probs: ProbVector, cache_size: int, epoch: int, rng_seed,
                  positions: bool = True) -> bool:
    """build_cache into an existing CacheState of the same graph and cache
    size (the per-epoch refresh of pool.py:133-135), in place: ``state`` is
    the new cache afterwards.  Device addresses stay the same unless the new
    cached CSR outgrows its buffer — then ``state`` gets larger buffers (still
    the same object) and CUDA graphs that captured the old addresses must be
    re-captured.  Returns True when every address was kept."""
    return refresh_finish(refresh_begin(state, g, probs, cache_size, epoch, rng_seed, positions=positions))


def empty_like(state: CacheState, g: Graph) -> CacheState:
    """A second CacheState with buffers of the same sizes (double-buffered
    refresh: the next epoch's cache is drawn into it while this one is in
    use).  Contents are undefined until refresh_begin/refresh_finish."""
    n = g.num_nodes
    dev = state.inclusion.device
    ids = torch.empty_like(state._buf_ids)
    bits = torch.empty_like(state.nodes.mask_bits)
    counts = torch.zeros_like(state._buf_counts)
    k = len(state.nodes)
    st = CacheState(nodes=NodeSet(ids=ids[:k], mask_bits=bits, num_nodes=n),
                    inclusion=torch.empty(n, dtype=torch.float64, device=dev),
                    cached_indptr=torch.empty(n + 1, dtype=torch.int64, device=dev),
                    cached_indices=state._buf_cidx[:0], epoch=-1, source_probs=state.source_probs,
                    cached_pos=state._buf_cpos[:0])
    for name, val in (("_buf_ids", ids), ("_buf_counts", counts),
                      ("_buf_cidx", torch.empty_like(state._buf_cidx)),
                      ("_buf_cpos", torch.empty_like(state._buf_cpos))):
        object.__setattr__(st, name, val)
    object.__setattr__(st, "cached_indices", st._buf_cidx[:0])
    object.__setattr__(st, "cached_pos", st._buf_cpos[:0])
    return st


class PendingRefresh:
    """First half of a cache (re)build: the draw (cache.py:87-103), the
    inclusion vector (cache.py:171-183) and the cached-CSR row counts
    (cache.py:185-197) are enqueued on ``stream`` and (|C|, nnz_C) are copied
    to pinned host memory; nothing waits on the host.  ``ready()`` polls;
    ``refresh_finish`` sizes the cached CSR and enqueues its fill."""

    def __init__(self, state, g, probs, epoch, stream, counts, nnz, host, ev, ws, positions):
        self.state, self.g, self.probs, self.epoch, self.stream = state, g, probs, epoch, stream
        self.counts, self.nnz, self.host, self.ev, self._ws = counts, nnz, host, ev, ws
        self.positions = positions
        self.done = None      # event after the fill (refresh_finish)

    def ready(self) -> bool:
        return self.ev.query()


def refresh_begin(state, g: Graph, probs: ProbVector, cache_size: int, epoch: int, rng_seed,
                  stream=None, positions: bool = True) -> PendingRefresh:
    """Enqueue draw + inclusion + cached-CSR count into ``state``'s buffers
    (``state=None``: fresh buffers) on ``stream`` (default: current)."""
    probs = probs.normalize()
    stream = stream if stream is not None else torch.cuda.current_stream()
    sp = _lib.stream_ptr(stream)
    seed, ep, tag = seed_key(rng_seed)
    n = g.num_nodes
    with torch.cuda.stream(stream):
        if state is not None:
            bufs = (state._buf_ids, state.nodes.mask_bits, state._buf_counts)
            incl, c_indptr = state.inclusion, state.cached_indptr
        else:
            bufs = None
            incl = torch.empty(n, dtype=torch.float64, device=g.device)
            c_indptr = torch.empty(n + 1, dtype=torch.int64, device=g.device)
        ids, bits, counts = _draw(probs, cache_size, seed, ep, stream=stream, tag=tag, out=bufs)
        # |C| and |support| stay on the device (counts[0], counts[1])
        _lib.call("gns_inclusion", probs.weights.data_ptr(), n, 0, counts.data_ptr(),
                  counts[1:].data_ptr(), incl.data_ptr(), sp)
        nnz = torch.zeros(1, dtype=torch.int64, device=g.device)
        # the keep bits of every CSR entry live in the workspace until the fill
        ws = _lib.workspace(_lib.lib().gns_cached_csr_workspace_size(n, g.num_edges), g.device)
        _lib.call("gns_cached_csr_count", g.cstruct(), bits.data_ptr(), c_indptr.data_ptr(),
                  nnz.data_ptr(), ws.data_ptr(), ws.numel(), sp)
        host = torch.empty(2, dtype=torch.int64).pin_memory()
        host[:1].copy_(counts[:1], non_blocking=True)
        host[1:].copy_(nnz, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(stream)
    if state is None:
        state = (ids, bits, counts, incl, c_indptr)
    return PendingRefresh(state, g, probs, epoch, stream, counts, nnz, host, ev, ws, positions)


def refresh_finish(p: PendingRefresh):
    """Second half: read (|C|, nnz_C) (waits for the first half), grow the
    cached-CSR buffers if needed and enqueue the fill on the same stream.
    For a refresh into an existing state returns True when every device
    address was kept (False: captured graphs must be re-captured); for a
    fresh build returns the new CacheState."""
    p.ev.synchronize()
    k, nnz_h = int(p.host[0]), int(p.host[1])
    g, stream = p.g, p.stream
    state = p.state if isinstance(p.state, CacheState) else None
    if state is not None and k != len(state.nodes):
        raise ValueError(f"refresh_cache: cache size changed ({len(state.nodes)} -> {k}); use build_cache")
    with torch.cuda.stream(stream):
        keep = state is not None and state._buf_cidx.numel() >= nnz_h
        if keep:
            c_indices, c_pos = state._buf_cidx, state._buf_cpos
        else:
            cap = max(nnz_h + nnz_h // 4, 1)      # headroom: later draws rarely reallocate
            c_indices = torch.empty(cap, dtype=torch.int32, device=g.device)
            c_pos = torch.empty(cap, dtype=torch.int32, device=g.device)
        if state is not None:
            bits, c_indptr = state.nodes.mask_bits, state.cached_indptr
        else:
            ids, bits, counts, incl, c_indptr = p.state
        _lib.call("gns_cached_csr_fill", g.cstruct(), bits.data_ptr(), c_indptr.data_ptr(),
                  c_indices.data_ptr(), c_pos.data_ptr() if p.positions else None, p._ws.data_ptr(),
                  p._ws.numel(), _lib.stream_ptr(stream))
        p.done = torch.cuda.Event()
        p.done.record(stream)
    if state is not None:
        # frozen dataclass: refresh the fields in place.  The draw, inclusion
        # and cached_indptr were written into the state's own buffers; the
        # cached CSR buffers are the old ones or (grown) new ones
        for name, val in (("cached_indices", c_indices[:nnz_h]), ("cached_pos", c_pos[:nnz_h]),
                          ("epoch", p.epoch), ("source_probs", p.probs), ("_buf_cidx", c_indices),
                          ("_buf_cpos", c_pos)):
            object.__setattr__(state, name, val)
        object.__setattr__(state, "_rank_stale", True)   # bitmap content changed
        state.__dict__.pop("_c", None)         # cstruct: cached_indices may have moved
        return keep
    n = g.num_nodes
    nodes = NodeSet(ids=ids[:k], mask_bits=bits, num_nodes=n)
    st = CacheState(nodes=nodes, inclusion=incl, cached_indptr=c_indptr,
                    cached_indices=c_indices[:nnz_h], epoch=p.epoch, source_probs=p.probs,
                    cached_pos=c_pos[:nnz_h])
    for name, val in (("_buf_ids", ids), ("_buf_counts", counts), ("_buf_cidx", c_indices), ("_buf_cpos", c_pos)):
        object.__setattr__(st, name, val)
    return st


def _build_cache_into(state, g, probs, cache_size, epoch, rng_seed, positions=True):
    r = refresh_finish(refresh_begin(state, g, probs, cache_size, epoch, rng_seed, positions=positions))
    return state if state is not None else r
