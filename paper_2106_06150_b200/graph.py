"""HBM-resident CSR graph and node sets (reference: graph.py:52-139).

``Graph`` mirrors the reference's immutable CSR (``graph.py:52-104``): rows
sorted ascending, symmetric, no self loops.  On B200 it lives in HBM:
``indptr`` int64[N+1], ``indices`` int32[E] (ids < 2^31), features float32
[N, D] row-major (rows padded to a 16-byte multiple for 128-bit gathers),
labels int32, masks bool.  ``NodeSet`` keeps sorted int32 ids plus a packed
membership bitmap (bit v of word v>>5, N/8 bytes — L2-resident at 111M nodes)
instead of the reference's bool[N] mask (``graph.py:107-139``).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import GraphFormatError, InvariantError  # noqa: F401  (re-export)


def _dev(device):
    return torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())


class Graph:
    """Undirected CSR graph resident in HBM (graph.py:52-104)."""

    def __init__(self, num_nodes: int, indptr: torch.Tensor, indices: torch.Tensor,
                 features: torch.Tensor | None = None, labels: torch.Tensor | None = None,
                 train_mask: torch.Tensor | None = None, val_mask: torch.Tensor | None = None,
                 test_mask: torch.Tensor | None = None, feature_dim: int | None = None):
        if indptr.dtype != torch.int64 or indices.dtype != torch.int32:
            raise ValueError("Graph needs indptr int64 and indices int32 device tensors")
        if num_nodes >= 2 ** 31:
            raise ValueError("node ids must fit in int32")
        self.num_nodes = int(num_nodes)
        self.indptr = indptr
        self.indices = indices
        self.features = features              # [N, ld] float32, ld % 4 == 0
        self._feature_dim = feature_dim if feature_dim is not None else (
            0 if features is None else int(features.shape[1]))
        self.labels = labels
        self.train_mask = train_mask
        self.val_mask = val_mask
        self.test_mask = test_mask
        self.degrees = (indptr[1:] - indptr[:-1]).to(torch.int32)
        self._train_ids = None
        self._cstruct = _lib.GnsGraph(self.num_nodes, int(indices.shape[0]), indptr.data_ptr(),
                                      indices.data_ptr())

    # -- reference properties ------------------------------------------------
    @property
    def num_edges(self) -> int:
        """Directed edge entries (graph.py:78-80)."""
        return int(self.indices.shape[0])

    @property
    def feature_dim(self) -> int:
        return self._feature_dim

    @property
    def device(self):
        return self.indptr.device

    def degree(self, v: int) -> int:
        return int(self.degrees[v])

    def neighbors(self, v: int) -> torch.Tensor:
        return self.indices[int(self.indptr[v]):int(self.indptr[v + 1])]

    def cstruct(self):
        return self._cstruct

    def train_ids(self) -> torch.Tensor:
        """graph.py:418-422: sorted train ids (all nodes without a mask), int32."""
        if self._train_ids is None:
            if self.train_mask is None:
                self._train_ids = torch.arange(self.num_nodes, dtype=torch.int32, device=self.device)
            else:
                self._train_ids = torch.nonzero(self.train_mask).flatten().to(torch.int32)
        return self._train_ids

    @property
    def feature_ld(self) -> int:
        return 0 if self.features is None else int(self.features.stride(0))

    # -- construction -----------------------------------------------------------
    @classmethod
    def from_numpy(cls, num_nodes, indptr, indices, features=None, labels=None, train_mask=None,
                   val_mask=None, test_mask=None, device=None) -> "Graph":
        dev = _dev(device)
        ip = torch.as_tensor(np.asarray(indptr, dtype=np.int64)).to(dev)
        ix = torch.as_tensor(np.asarray(indices).astype(np.int32, copy=False)).to(dev)
        feats, fdim = None, None
        if features is not None:
            f = np.asarray(features, dtype=np.float32)
            fdim = f.shape[1]
            ld = (fdim + 3) // 4 * 4
            feats = torch.zeros((f.shape[0], ld), dtype=torch.float32, device=dev)
            feats[:, :fdim] = torch.as_tensor(f).to(dev)
        lab = None if labels is None else torch.as_tensor(np.asarray(labels, dtype=np.int32)).to(dev)

        def m(x):
            return None if x is None else torch.as_tensor(np.asarray(x, dtype=bool)).to(dev)

        return cls(int(num_nodes), ip, ix, feats, lab, m(train_mask), m(val_mask), m(test_mask),
                   feature_dim=fdim)

    @classmethod
    def from_reference(cls, g, device=None) -> "Graph":
        """Upload any reference-shaped graph (gnsbench.Graph, oracle OGraph)."""
        return cls.from_numpy(g.num_nodes, g.indptr, g.indices, getattr(g, "features", None),
                              getattr(g, "labels", None), getattr(g, "train_mask", None),
                              getattr(g, "val_mask", None), getattr(g, "test_mask", None),
                              device=device)

    def to_host(self):
        """numpy copy in the reference's layout (for oracle checks / CPU baseline)."""
        from types import SimpleNamespace
        f = None
        if self.features is not None:
            f = self.features[:, :self.feature_dim].cpu().numpy()
        return SimpleNamespace(
            num_nodes=self.num_nodes, indptr=self.indptr.cpu().numpy(),
            indices=self.indices.cpu().numpy(), features=f,
            labels=None if self.labels is None else self.labels.cpu().numpy(),
            train_mask=None if self.train_mask is None else self.train_mask.cpu().numpy(),
            val_mask=None if self.val_mask is None else self.val_mask.cpu().numpy(),
            test_mask=None if self.test_mask is None else self.test_mask.cpu().numpy())


@dataclass(eq=False)
class NodeSet:
    """Sorted unique ids + packed membership bitmap (graph.py:107-139)."""

    ids: torch.Tensor        # int32 sorted unique
    mask_bits: torch.Tensor  # int32 words (bit v of word v >> 5)
    num_nodes: int

    def __len__(self) -> int:
        return int(self.ids.shape[0])

    @property
    def mask(self) -> torch.Tensor:
        """bool[N] view of the bitmap (materialised on demand)."""
        shifts = torch.arange(32, device=self.mask_bits.device, dtype=torch.int32)
        bits = (self.mask_bits.unsqueeze(1) >> shifts) & 1
        return bits.flatten()[:self.num_nodes].bool()

    def __contains__(self, v) -> bool:
        v = int(v)
        return bool((int(self.mask_bits[v >> 5]) >> (v & 31)) & 1)

    def contains(self, nodes) -> torch.Tensor:
        nodes = torch.as_tensor(nodes, device=self.mask_bits.device).long()
        return ((self.mask_bits[nodes >> 5] >> (nodes & 31).int()) & 1).bool()


# ---------------------------------------------------------------------------
# Synthetic power-law graphs on the device (graph.py:172-205 analogue)
# ---------------------------------------------------------------------------

def generate_powerlaw_device(num_nodes: int, num_pairs: int, alpha: float = 0.6,
                             offset: float = 1000.0, seed: int = 0, feature_dim: int = 0,
                             num_classes: int = 2, train_frac: float = 1.0,
                             feature_noise: float = 3.0, device=None) -> Graph:
    """Symmetric power-law CSR generated on the GPU (gns_gen_powerlaw_*), with
    class-mean + noise features (graph.py:249-253 scheme) and random masks."""
    _lib.require_cuda()
    dev = _dev(device)
    stream = _lib.stream_ptr()
    ws = _lib.workspace(_lib.lib().gns_gen_workspace_size(num_nodes, num_pairs), dev)
    indptr = torch.empty(num_nodes + 1, dtype=torch.int64, device=dev)
    nnz = torch.zeros(1, dtype=torch.int64, device=dev)
    _lib.call("gns_gen_powerlaw_count", num_nodes, num_pairs, float(alpha), float(offset),
              seed & 0xFFFFFFFF, indptr.data_ptr(), nnz.data_ptr(), ws.data_ptr(), ws.numel(), stream)
    e = int(nnz.item())
    indices = torch.empty(max(e, 1), dtype=torch.int32, device=dev)[:e]
    _lib.call("gns_gen_powerlaw_fill", num_nodes, num_pairs, indptr.data_ptr(), indices.data_ptr(),
              ws.data_ptr(), ws.numel(), stream)
    del ws
    return _with_node_data(Graph(num_nodes, indptr, indices), seed, feature_dim, num_classes, train_frac,
                           feature_noise)


def _with_node_data(g: Graph, seed: int, feature_dim: int, num_classes: int, train_frac: float,
                    feature_noise: float) -> Graph:
    """Labels, masks and features as pure functions of (seed, node) on the
    device (gns_gen_node_attrs / gns_gen_features; class mean + noise, the
    graph.py:249-253 scheme), reproducible bit for bit on the host by
    oracle/gen.cc."""
    num_nodes, dev, stream = g.num_nodes, g.device, _lib.stream_ptr()
    indptr, indices = g.indptr, g.indices
    labels = torch.empty(num_nodes, dtype=torch.int32, device=dev)
    train, val, test = (torch.empty(num_nodes, dtype=torch.bool, device=dev) for _ in range(3))
    _lib.call("gns_gen_node_attrs", num_nodes, num_classes, float(train_frac), seed & 0xFFFFFFFF,
              labels.data_ptr(), train.data_ptr(), val.data_ptr(), test.data_ptr(), stream)
    feats = None
    if feature_dim > 0:
        ld = (feature_dim + 3) // 4 * 4
        means = torch.empty((num_classes, ld), dtype=torch.float32, device=dev)
        feats = torch.empty((num_nodes, ld), dtype=torch.float32, device=dev)
        _lib.call("gns_gen_features", num_nodes, feature_dim, ld, num_classes, float(feature_noise),
                  seed & 0xFFFFFFFF, labels.data_ptr(), means.data_ptr(), feats.data_ptr(), stream)
    return Graph(num_nodes, indptr, indices, feats, labels, train, val, test,
                 feature_dim=feature_dim if feature_dim else None)


def generate_powerlaw(num_nodes: int, attach: int, seed: int, feature_dim: int = 0, num_classes: int = 2,
                      train_frac: float = 1.0, feature_noise: float = 3.0, device=None) -> Graph:
    """The reference's preferential-attachment graph (graph.py:172-205) —
    the same graph for the same ``(num_nodes, attach, seed)``: every node
    s >= attach links to ``attach`` distinct endpoints drawn uniformly from
    the list of all edge endpoints so far (degree-proportional).  The draw
    is inherently sequential and defined by numpy's PCG64 stream, so it runs
    on the host (≈3 s at 100K nodes x 10); the CSR is built on the device
    (``build_csr``), and labels / masks / features (``feature_dim > 0``) come
    from the device attribute generator of ``generate_powerlaw_device``."""
    if attach < 1:
        raise ValueError("attach must be >= 1")
    if num_nodes <= attach:
        raise ValueError(f"need n > attach, got n={num_nodes}, attach={attach}")
    from .formats import build_csr
    rng = np.random.default_rng(seed)
    m, n = attach, num_nodes
    pool = np.empty(2 * (n - m) * m, dtype=np.int64)     # every endpoint so far
    heads = np.empty((n - m, m), dtype=np.int64)         # node s's m neighbours
    prev = list(range(m))
    filled = 0
    for s in range(m, n):
        heads[s - m] = prev
        pool[filled:filled + m] = prev
        pool[filled + m:filled + 2 * m] = s
        filled += 2 * m
        # m draws at once consume the stream exactly like m scalar draws; the
        # set needs more only when a draw repeats an earlier pick
        chosen = set()
        for v in pool[rng.integers(filled, size=m)].tolist():
            chosen.add(v)
        while len(chosen) < m:
            chosen.add(int(pool[rng.integers(filled)]))
        prev = list(chosen)          # set iteration order, as np.fromiter(set)
    tails = np.repeat(np.arange(m, n, dtype=np.int64), m)
    g = build_csr(np.stack([tails, heads.reshape(-1)], 1), n, device=device)
    return _with_node_data(g, seed, feature_dim, num_classes, train_frac, feature_noise)
