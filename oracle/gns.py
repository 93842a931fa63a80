"""numpy restatement of the reference GNS sampling path — TEST INFRASTRUCTURE ONLY.

Every function cites the reference lines it restates (paths relative to
``/root/reference/pkg/src/gnsbench``).  Two key sources can drive it:

* ``NumpyStream(rng)`` — consumes ``rng.random(n)`` exactly like the reference
  (one call per phase per layer, ``sampling.py:166,214,233``).  With
  ``np.random.default_rng([seed, 32, epoch, index])`` (``pool.py:70``) the
  oracle reproduces ``gnsbench.build_minibatch`` bit for bit — this is how
  the restatement itself is pinned (``tests/test_oracle.py``) and how the
  CPU baseline is timed (the reference's own RNG cost).
* ``PhiloxKeys(seed, epoch, batch)`` — the build's counter-based keys
  (``oracle/philox.py``).  The B200 kernels must match this mode bit for bit.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import detmath, philox


class InvariantError(RuntimeError):
    """graph.py:48 restated."""


# ---------------------------------------------------------------------------
# Graph helpers
# ---------------------------------------------------------------------------

@dataclass
class OGraph:
    """Minimal CSR holder mirroring ``graph.py:52-80`` (read-only arrays)."""

    num_nodes: int
    indptr: np.ndarray
    indices: np.ndarray
    features: np.ndarray | None = None
    labels: np.ndarray | None = None
    train_mask: np.ndarray | None = None
    val_mask: np.ndarray | None = None
    test_mask: np.ndarray | None = None
    degrees: np.ndarray = field(init=False)

    def __post_init__(self):
        self.degrees = np.diff(self.indptr)

    @property
    def num_edges(self) -> int:
        return int(self.indices.shape[0])


def as_ograph(g) -> OGraph:
    if isinstance(g, OGraph):
        return g
    return OGraph(num_nodes=int(g.num_nodes), indptr=np.asarray(g.indptr),
                  indices=np.asarray(g.indices),
                  features=getattr(g, "features", None),
                  labels=getattr(g, "labels", None),
                  train_mask=getattr(g, "train_mask", None),
                  val_mask=getattr(g, "val_mask", None),
                  test_mask=getattr(g, "test_mask", None))


def build_csr(edge_list, num_nodes: int) -> OGraph:
    """graph.py:142-169: symmetrize, drop self-loops and duplicates, sort rows."""
    edges = np.asarray(edge_list, dtype=np.int64).reshape(-1, 2)
    if edges.size:
        if ((edges < 0) | (edges >= num_nodes)).any():
            raise ValueError("edge out of range")
        edges = edges[edges[:, 0] != edges[:, 1]]
    if edges.size:
        both = np.concatenate([edges, edges[:, ::-1]])
        keys = np.unique(both[:, 0] * num_nodes + both[:, 1])
        src, dst = keys // num_nodes, keys % num_nodes
    else:
        src = dst = np.empty(0, dtype=np.int64)
    indptr = np.zeros(num_nodes + 1, dtype=np.int64)
    np.cumsum(np.bincount(src, minlength=num_nodes), out=indptr[1:])
    return OGraph(num_nodes=num_nodes, indptr=indptr, indices=dst)


def powerlaw_attach_edges(n: int, attach: int, seed: int) -> np.ndarray:
    """graph.py:172-205 (the preferential-attachment generator) as an
    ``(n - attach) * attach`` x 2 edge list: node s >= attach links to the
    previous node's ``attach`` distinct picks, each pick a uniform draw from
    the endpoint multiset so far (degree-proportional).  Same numpy stream:
    the first ``attach`` draws of a node as one ``integers(k, size=attach)``
    call (a batch consumes the generator exactly as that many scalar calls),
    further draws one at a time while duplicates leave the set short, and
    the picks in Python-set iteration order of the same insertions."""
    if attach < 1:
        raise ValueError("attach must be >= 1")
    if n <= attach:
        raise ValueError(f"need n > attach, got n={n}, attach={attach}")
    rng = np.random.default_rng(seed)
    m = attach
    ends = np.empty(2 * (n - m) * m, dtype=np.int64)
    dst = np.empty((n - m) * m, dtype=np.int64)
    cur = np.arange(m, dtype=np.int64)
    k = 0
    for s in range(m, n):
        dst[(s - m) * m:(s - m + 1) * m] = cur
        ends[k:k + m] = cur
        ends[k + m:k + 2 * m] = s
        k += 2 * m
        picks = set()
        for v in ends[rng.integers(k, size=m)].tolist():
            picks.add(v)
        while len(picks) < m:
            picks.add(int(ends[rng.integers(k)]))
        cur = np.fromiter(picks, dtype=np.int64, count=m)
    return np.stack([np.repeat(np.arange(m, n, dtype=np.int64), m), dst], 1)


def generate_powerlaw(n: int, attach: int, seed: int) -> OGraph:
    """graph.py:172-205: the preferential-attachment graph's CSR."""
    return build_csr(powerlaw_attach_edges(n, attach, seed), n)


def gather_rows(indptr, indices, rows):
    """graph.py:399-415."""
    rows = np.asarray(rows, dtype=np.int64)
    counts = indptr[rows + 1] - indptr[rows]
    total = int(counts.sum())
    if total == 0:
        return (np.empty(0, dtype=indices.dtype), counts,
                np.empty(0, dtype=np.int64))
    block_starts = np.cumsum(counts) - counts
    offsets = np.arange(total, dtype=np.int64) - np.repeat(block_starts, counts)
    positions = np.repeat(indptr[rows], counts) + offsets
    return indices[positions], counts, positions


def train_ids(g) -> np.ndarray:
    """graph.py:418-422 (sorted ids of the train mask, all nodes without one)."""
    if g.train_mask is None:
        return np.arange(g.num_nodes, dtype=np.int64)
    return np.flatnonzero(np.asarray(g.train_mask)).astype(np.int64)


# ---------------------------------------------------------------------------
# Key sources
# ---------------------------------------------------------------------------

class NumpyStream:
    """Sequential ``rng.random(n)`` consumption, as the reference does."""

    def __init__(self, rng):
        self.rng = rng

    def keys(self, layer, phase, row_nodes, pos):
        return self.rng.random(len(pos))


@dataclass
class PhiloxKeys:
    """The build's per-candidate keys (oracle/philox.py layout)."""

    seed: int
    epoch: int
    batch: int
    record: list | None = None

    def keys(self, layer, phase, row_nodes, pos):
        stream = philox.stream_word(philox.TAG_BATCH, layer, phase)
        u = philox.uniform(self.seed, self.epoch, row_nodes, stream, self.batch,
                           pos)
        if self.record is not None:
            self.record.append(u)
        return u


class ReplayRng:
    """Duck-typed ``rng`` for the reference: ``.random(n)`` returns the next
    recorded key array (used to replay the build's keys into gnsbench)."""

    def __init__(self, arrays):
        self.arrays = list(arrays)

    def random(self, n):
        a = self.arrays.pop(0)
        if len(a) != n:
            raise AssertionError(f"replay length mismatch: {len(a)} != {n}")
        return a


# ---------------------------------------------------------------------------
# Cache engine (cache.py)
# ---------------------------------------------------------------------------

def degree_probs(g) -> np.ndarray:
    """cache.py:53-58: p_i = deg(i) / E."""
    total = int(g.indices.shape[0])
    if total == 0:
        raise ValueError("graph has no edges; degree distribution undefined")
    w = np.diff(np.asarray(g.indptr)) / float(total)
    return w


RW_SUM_THREADS = 148 * 256  # fixed strided-sum width of gns_random_walk_probs


def random_walk_probs(g, train, fanouts, num_layers: int, device_order: bool = True):
    """cache.py:61-84.  The iterate uses scipy's CSR matvec (ascending
    neighbour order, exactly the reference); the final normalising sum is
    the build's fixed-order strided reduction (``device_order``) or numpy's
    pairwise ``p.sum()`` (the reference)."""
    import scipy.sparse as sp
    g = as_ograph(g)
    if num_layers < 1:
        raise ValueError("num_layers must be >= 1")
    train = np.asarray(train, dtype=np.int64)
    if len(train) == 0:
        raise ValueError("training set is empty")
    adj = sp.csr_matrix((np.ones(g.num_edges), np.asarray(g.indices), np.asarray(g.indptr)),
                        shape=(g.num_nodes, g.num_nodes))
    deg = g.degrees.astype(np.float64)
    safe_deg = np.maximum(deg, 1.0)
    p = np.zeros(g.num_nodes, dtype=np.float64)
    p[train] = 1.0 / len(train)
    for step in range(num_layers):
        d = np.minimum(float(fanouts[step]), deg) / safe_deg
        p = d * (adj @ p) + p
    if not device_order:
        return p / p.sum()
    T = RW_SUM_THREADS
    m = (len(p) + T - 1) // T
    padded = np.zeros(m * T)
    padded[:len(p)] = p
    rows = padded.reshape(m, T)
    # Neumaier-compensated sums, thread t over x[t], x[t+T], ... then over t
    s_, c_ = np.zeros(T), np.zeros(T)
    for i in range(m):
        x = rows[i]
        t = s_ + x
        big = np.abs(s_) >= np.abs(x)
        c_ = c_ + np.where(big, (s_ - t) + x, (x - t) + s_)
        s_ = t
    partial = s_ + c_
    s1, c1 = 0.0, 0.0
    for x in partial.tolist():
        t = s1 + x
        c1 += ((s1 - t) + x) if abs(s1) >= abs(x) else ((x - t) + s1)
        s1 = t
    return p / (s1 + c1)


def cache_keys_philox(w: np.ndarray, support: np.ndarray, seed: int, epoch: int, tag: int = philox.TAG_CACHE):
    """Exponential-race keys Exp(1)/w over the positive support (cache.py:101),
    with Exp(1) = -log(1 - U), U from Philox at (tag, pos = node id)."""
    stream = philox.stream_word(tag)
    u = philox.uniform(seed, epoch, 0, stream, 0, support)
    e = -detmath.det_log(1.0 - u)
    return e / w[support]


def sample_cache(w: np.ndarray, cache_size: int, seed=0, epoch=0,
                 numpy_seed=None, tag: int = philox.TAG_CACHE) -> np.ndarray:
    """cache.py:87-103 -> sorted unique cached ids.

    ``numpy_seed`` given: the reference's own draw (``default_rng(seed)
    .exponential``, ``argpartition``).  Otherwise Philox keys and the
    (key, id) smallest-|C| rule."""
    n = len(w)
    support = np.flatnonzero(w > 0)
    if cache_size <= 0:
        return np.empty(0, dtype=np.int64)
    if len(support) <= cache_size:
        return support.astype(np.int64)
    if numpy_seed is not None:
        rng = np.random.default_rng(numpy_seed)
        keys = rng.exponential(size=len(support)) / w[support]
        pick = np.argpartition(keys, cache_size)[:cache_size]
        return np.unique(support[pick]).astype(np.int64)
    keys = cache_keys_philox(w, support, seed, epoch, tag)
    order = np.lexsort((support, keys))[:cache_size]
    return np.sort(support[order]).astype(np.int64)


@dataclass
class OCache:
    """cache.py:130-157 restated: ids + mask, inclusion, cached CSR."""

    ids: np.ndarray
    mask: np.ndarray
    inclusion: np.ndarray
    cached_indptr: np.ndarray
    cached_indices: np.ndarray
    epoch: int = 0


def build_cache(g, w: np.ndarray, cache_size: int, epoch: int = 0, seed: int = 0,
                numpy_seed=None, ids=None) -> OCache:
    """cache.py:160-197 (analytic inclusion).  ``ids`` injects a given cache
    set (cache-replay mode)."""
    g = as_ograph(g)
    if ids is None:
        ids = sample_cache(w, cache_size, seed=seed, epoch=epoch,
                           numpy_seed=numpy_seed)
    ids = np.asarray(ids, dtype=np.int64)
    mask = np.zeros(g.num_nodes, dtype=bool)
    mask[ids] = True
    support = w > 0
    incl = detmath.inclusion_prob(w, len(ids))
    if len(ids) >= int(support.sum()):
        incl = np.where(support, 1.0, incl)
    neigh, counts, _ = gather_rows(g.indptr, g.indices, ids)
    owners = np.repeat(ids, counts)
    order = np.lexsort((owners, neigh))
    cached_indices = owners[order]
    cached_indptr = np.zeros(g.num_nodes + 1, dtype=np.int64)
    np.cumsum(np.bincount(neigh, minlength=g.num_nodes), out=cached_indptr[1:])
    return OCache(ids=ids, mask=mask, inclusion=np.asarray(incl, dtype=np.float64),
                  cached_indptr=cached_indptr, cached_indices=cached_indices,
                  epoch=epoch)


FILL_STREAM = 21  # sampling.py:29


def estimate_edge_inclusion(g, w, cache_size, k, cache_only, resamples=64, seed=0, numpy_seed=None):
    """sampling.py:269-296 with the build's Philox resamples (key (seed, r), tag
    21); ``numpy_seed`` = the reference's own draws ``[seed, 21, r]``."""
    g = as_ograph(g)
    n = g.num_nodes
    deg = g.degrees.astype(np.float64)
    rows = np.repeat(np.arange(n), g.degrees)
    q = np.zeros(g.num_edges, dtype=np.float64)
    for r in range(resamples):
        if numpy_seed is not None:
            ids = sample_cache(w, cache_size, numpy_seed=[numpy_seed, FILL_STREAM, r])
        else:
            ids = sample_cache(w, cache_size, seed=seed, epoch=r, tag=FILL_STREAM)
        mask = np.zeros(n, dtype=bool)
        mask[ids] = True
        cflag = mask[g.indices]
        nc = np.bincount(rows, weights=cflag, minlength=n)
        m = np.minimum(k, nc)
        rest = deg - nc
        p_cached = np.divide(m, nc, out=np.zeros(n), where=nc > 0)
        if cache_only:
            p_fill = np.zeros(n)
        else:
            fill = np.minimum(k - m, rest)
            p_fill = np.divide(fill, rest, out=np.zeros(n), where=rest > 0)
        q += np.where(cflag, p_cached[rows], p_fill[rows])
    return q / resamples


def cached_csr_by_filter(g, mask):
    """Equivalent construction used by the build (filter the full CSR by the
    cache mask; rows stay ascending).  Asserted equal to build_cache's."""
    g = as_ograph(g)
    keep = mask[g.indices]
    rows = np.repeat(np.arange(g.num_nodes), g.degrees)
    c_indptr = np.zeros(g.num_nodes + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows[keep], minlength=g.num_nodes), out=c_indptr[1:])
    return c_indptr, g.indices[keep].astype(np.int64)


# ---------------------------------------------------------------------------
# Sampler (sampling.py)
# ---------------------------------------------------------------------------

@dataclass
class OBlock:
    """sampling.py:32-60 LayerBlock restated (int64 / f64 / bool arrays)."""

    dst_nodes: np.ndarray
    src_nodes: np.ndarray
    edge_src: np.ndarray
    edge_dst: np.ndarray
    edge_weight: np.ndarray
    edge_cached: np.ndarray
    dst_degree: np.ndarray
    fanout: int | None
    policy: str

    @property
    def num_edges(self) -> int:
        return int(self.edge_src.shape[0])


@dataclass
class OMiniBatch:
    blocks: tuple
    targets: np.ndarray
    input_nodes: np.ndarray


def select_per_row(counts, take, keys):
    """sampling.py:129-136."""
    total = len(keys)
    row = np.repeat(np.arange(len(counts)), counts)
    order = np.lexsort((keys, row))
    block_starts = np.cumsum(counts) - counts
    rank = np.arange(total, dtype=np.int64) - np.repeat(block_starts, counts)
    return order[rank < np.repeat(take, counts)]


def assemble(g, seeds, dst_rows, srcs, weights, cached, fanout, policy):
    """sampling.py:139-152."""
    src_nodes = np.unique(np.concatenate([seeds, srcs]))
    return OBlock(dst_nodes=seeds, src_nodes=src_nodes,
                  edge_src=np.searchsorted(src_nodes, srcs).astype(np.int64),
                  edge_dst=np.asarray(dst_rows, dtype=np.int64),
                  edge_weight=np.asarray(weights, dtype=np.float64),
                  edge_cached=np.asarray(cached, dtype=bool),
                  dst_degree=g.degrees[seeds].astype(np.int64),
                  fanout=fanout, policy=policy)


def sample_neighbors_uniform(g, seeds, k, keysrc, layer=0) -> OBlock:
    """sampling.py:155-170."""
    if k < 1:
        raise ValueError("fanout must be >= 1")
    g = as_ograph(g)
    seeds = np.unique(np.asarray(seeds, dtype=np.int64))
    cand, counts, positions = gather_rows(g.indptr, g.indices, seeds)
    take = np.minimum(k, counts)
    row_nodes = np.repeat(seeds, counts)
    pos = positions - np.repeat(g.indptr[seeds], counts)
    keys = keysrc.keys(layer, philox.PHASE_UNIFORM, row_nodes, pos)
    sel = select_per_row(counts, take, keys)
    dst_rows = np.repeat(np.arange(len(seeds)), counts)[sel]
    weights = (counts / np.maximum(take, 1))[dst_rows]
    return assemble(g, seeds, dst_rows, cand[sel], weights,
                    np.zeros(len(sel), dtype=bool), k, "uniform")


def sample_neighbors_gns(g, cache: OCache, seeds, k, cache_only, keysrc,
                         layer=0, exact_weights=None) -> OBlock:
    """sampling.py:189-266 (gns-paper policy; gns-exact when exact_weights)."""
    if k < 1:
        raise ValueError("fanout must be >= 1")
    g = as_ograph(g)
    seeds = np.unique(np.asarray(seeds, dtype=np.int64))
    nrows = len(seeds)

    c_cand, c_counts, c_positions = gather_rows(cache.cached_indptr,
                                                cache.cached_indices, seeds)
    m = np.minimum(k, c_counts)
    c_pos = c_positions - np.repeat(cache.cached_indptr[seeds], c_counts)
    c_keys = keysrc.keys(layer, philox.PHASE_CACHED,
                         np.repeat(seeds, c_counts), c_pos)
    c_sel = select_per_row(c_counts, m, c_keys)
    c_dst = np.repeat(np.arange(nrows), c_counts)[c_sel]
    c_src = c_cand[c_sel]

    cand, counts, positions = gather_rows(g.indptr, g.indices, seeds)
    if cache_only:
        u_dst = np.empty(0, dtype=np.int64)
        u_src = np.empty(0, dtype=np.int64)
        fill = np.zeros(nrows, dtype=np.int64)
        rest = counts - c_counts
    else:
        uncached = ~cache.mask[cand]
        rows_all = np.repeat(np.arange(nrows), counts)
        u_cand = cand[uncached]
        u_rows = rows_all[uncached]
        u_positions = positions[uncached]
        rest = np.bincount(u_rows, minlength=nrows).astype(np.int64)
        fill = np.minimum(k - m, rest)
        u_pos = u_positions - g.indptr[seeds][u_rows]
        u_keys = keysrc.keys(layer, philox.PHASE_FILL, seeds[u_rows], u_pos)
        u_sel = select_per_row(rest, fill, u_keys)
        u_dst = u_rows[u_sel]
        u_src = u_cand[u_sel]

    if exact_weights is not None:
        # sampling.py:238-250: CSR positions of the cached picks, then 1/q
        rows_all = np.repeat(np.arange(nrows), counts)
        stride = g.num_nodes + 1
        row_keys = rows_all * stride + cand
        idx = np.searchsorted(row_keys, c_dst * stride + c_src)
        c_gpos = positions[idx]
        u_gpos = u_positions[u_sel] if not cache_only else np.empty(0, dtype=np.int64)
        q = np.concatenate([exact_weights[c_gpos], exact_weights[u_gpos]])
        if np.any(q <= 0):
            raise InvariantError("sampled an edge with zero estimated inclusion")
        weights = 1.0 / q
    else:
        n_cached_of_dst = np.maximum(c_counts, 1)
        coeff = cache.inclusion[c_src] * (k / np.minimum(k, n_cached_of_dst)[c_dst])
        if np.any(coeff <= 0):
            raise ValueError("inclusion probability is zero for a cached draw")
        c_w = 1.0 / coeff
        u_w = (rest / np.maximum(fill, 1))[u_dst]
        weights = np.concatenate([c_w, u_w])
    dst_rows = np.concatenate([c_dst, u_dst])
    srcs = np.concatenate([c_src, u_src])
    cached_flags = np.concatenate([np.ones(len(c_src), dtype=bool),
                                   np.zeros(len(u_src), dtype=bool)])
    return assemble(g, seeds, dst_rows, srcs, weights, cached_flags, k,
                    "gns-exact" if exact_weights is not None else "gns-paper")


def build_minibatch(g, cache, targets, config, keysrc, exact_tables=None) -> OMiniBatch:
    """sampling.py:299-336 (NS / GNS, gns-paper or gns-exact weights)."""
    g = as_ograph(g)
    num_layers = len(config.fanouts)
    seeds = np.unique(np.asarray(targets, dtype=np.int64))
    blocks = []
    for layer in range(num_layers, 0, -1):
        k = config.fanouts[num_layers - layer]
        if config.strategy == "NS":
            block = sample_neighbors_uniform(g, seeds, k, keysrc, layer)
        else:
            if cache is None:
                raise ValueError("GNS sampling needs a CacheState")
            cache_only = bool(config.input_layer_cache_only) and layer == 1
            table = None
            if getattr(config, "weight_policy", "gns-paper") == "gns-exact":
                table = (exact_tables or {}).get((k, cache_only))
                if table is None:
                    raise ValueError(f"missing edge-inclusion table for fanout={k}, cache_only={cache_only}")
            block = sample_neighbors_gns(g, cache, seeds, k, cache_only, keysrc,
                                         layer, exact_weights=table)
        blocks.append(block)
        seeds = block.src_nodes
    blocks.reverse()
    return OMiniBatch(blocks=tuple(blocks), targets=blocks[-1].dst_nodes,
                      input_nodes=blocks[0].src_nodes)


# ---------------------------------------------------------------------------
# Data loader (pool.py)
# ---------------------------------------------------------------------------

def epoch_targets(g, batch_size: int, seed: int, epoch: int, numpy_mode=False):
    """pool.py:60-66.  numpy_mode: the reference's PCG64 permutation; else the
    build's Feistel permutation keyed on (seed, epoch)."""
    ids = train_ids(g)
    if numpy_mode:
        shuffled = np.random.default_rng([seed, philox.TAG_SHUFFLE, epoch]) \
            .permutation(ids)
    else:
        perm = philox.feistel_permute(np.arange(len(ids)), len(ids), seed, epoch)
        shuffled = ids[perm.astype(np.int64)]
    return [shuffled[i:i + batch_size] for i in range(0, len(shuffled), batch_size)]


def cache_size_for(g, cache_frac: float) -> int:
    """pool.py:114."""
    return int(round(cache_frac * g.num_nodes))


def isolated_fraction(mb) -> float:
    """sampling.py:413-425."""
    block = mb.blocks[0]
    if len(mb.targets) == 0:
        return 0.0
    indeg = np.bincount(block.edge_dst, minlength=len(block.dst_nodes))
    tpos = np.searchsorted(block.dst_nodes, mb.targets)
    return float(np.mean(indeg[tpos] == 0))


def validate_minibatch(g, mb) -> None:
    """sampling.py:428-470 restated (structural invariants)."""
    g = as_ograph(g)
    for i, block in enumerate(mb.blocks):
        if np.any(np.diff(block.dst_nodes) <= 0) or np.any(np.diff(block.src_nodes) <= 0):
            raise InvariantError(f"block {i}: node arrays must be sorted unique")
        if not np.all(np.isin(block.dst_nodes, block.src_nodes)):
            raise InvariantError(f"block {i}: dst nodes missing from src")
        if block.num_edges:
            srcs = block.src_nodes[block.edge_src]
            dsts = block.dst_nodes[block.edge_dst]
            rows_g = np.repeat(np.arange(g.num_nodes, dtype=np.int64), g.degrees)
            edge_keys = rows_g * g.num_nodes + g.indices
            query = srcs * g.num_nodes + dsts
            hit = np.searchsorted(edge_keys, query)
            ok = (hit < len(edge_keys)) & \
                (edge_keys[np.minimum(hit, len(edge_keys) - 1)] == query)
            if not ok.all():
                raise InvariantError(f"block {i}: sampled a non-edge")
            if not np.all(np.isfinite(block.edge_weight)) or np.any(block.edge_weight <= 0):
                raise InvariantError(f"block {i}: edge weights must be finite > 0")
            if block.fanout is not None:
                indeg = np.bincount(block.edge_dst, minlength=len(block.dst_nodes))
                if indeg.max() > block.fanout:
                    raise InvariantError(f"block {i}: fanout bound exceeded")
        if not np.array_equal(block.dst_degree, g.degrees[block.dst_nodes]):
            raise InvariantError(f"block {i}: stale dst degrees")
        if i + 1 < len(mb.blocks) and \
                not np.array_equal(block.dst_nodes, mb.blocks[i + 1].src_nodes):
            raise InvariantError(f"block {i}: chain broken")
