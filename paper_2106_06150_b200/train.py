"""The reference trainer's module API on B200 (reference: model.py:37-307).

Same names, signatures and dataclass fields as ``gnsbench.model`` so a caller
of the reference's training loop (``init_params``, ``forward``,
``loss_and_grad``, ``backward``, ``adam_step``, ``evaluate``, ``train``) can
switch imports.  Arrays are device tensors instead of numpy arrays; every
numeric step runs in libgns.so through ``GraphSAGE`` (fused gather + weighted
mean SpMM, its transpose, cuBLAS GEMMs for the linear layers, fused softmax
cross-entropy, flat-buffer Adam).  ``init_params`` defaults to float64, the
reference's precision (model.py:7-8: "All model math runs in float64");
``dtype=torch.float32`` is the production mode (TF32 GEMMs unless
``tf32=False``).

Differences a caller can see, all deliberate:

* ``forward``/``backward`` take the feature table as a device tensor (or the
  ``Graph``); logits and gradients come back as device tensors.
* The gradient of the input layer's features is not formed (the reference
  computes and discards it, model.py:223-225).
* ``evaluate`` runs the full-neighbourhood forward as NS blocks with fanout
  = max degree (weights deg/take = 1), so it is meant for graphs
  whose whole L-hop neighbourhood fits on the device (the reference's dense
  evaluation has the same O(N + E) per-layer cost).
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .graph import Graph
from .model import GraphSAGE, TrainConfig, init_params_numpy, micro_f1
from .pool import SamplerPool
from .sampling import LayerBlock, MiniBatch, SamplerConfig


@dataclass(eq=False)
class ModelParams:
    """model.py:37-47: per-layer weights (2*in_dim, out_dim) and biases —
    device views into one flat parameter buffer (the GraphSAGE model that
    owns it is ``model``)."""

    model: GraphSAGE

    @property
    def weights(self) -> list:
        return self.model.weights

    @property
    def biases(self) -> list:
        return self.model.biases

    @property
    def dims(self) -> tuple:
        return self.model.dims

    @property
    def num_layers(self) -> int:
        return self.model.num_layers

    def to_numpy(self):
        """(weights, biases) as float64 numpy arrays (the reference layout)."""
        return self.model.export()


@dataclass(eq=False)
class ParamGrads:
    """model.py:202-205 (device views of the flat gradient buffer)."""

    weights: list
    biases: list


@dataclass(eq=False)
class AdamState:
    """model.py:68-78: first/second moments (flat device buffers, per-tensor
    views in ``m``/``v``) and the step count."""

    m_flat: torch.Tensor
    v_flat: torch.Tensor
    m: list
    v: list
    step: int = 0

    @classmethod
    def zeros_like(cls, params: ModelParams) -> "AdamState":
        mdl = params.model
        mf, vf = torch.zeros_like(mdl.flat), torch.zeros_like(mdl.flat)
        return cls(m_flat=mf, v_flat=vf, m=_views(mdl, mf), v=_views(mdl, vf))


@dataclass
class EpochStats:
    """model.py:81-90."""

    epoch: int
    loss: float
    train_f1: float
    val_f1: float
    test_f1: float
    seconds: float
    mean_input_nodes: float
    mean_cached: float


@dataclass
class TrainReport:
    """model.py:93-110 (same CSV columns and formatting)."""

    rows: list = field(default_factory=list)
    final_train_f1: float = 0.0
    final_val_f1: float = 0.0
    final_test_f1: float = 0.0
    params: ModelParams | None = None

    def write_csv(self, path) -> None:
        import csv
        with open(path, "w", newline="") as f:
            w = csv.writer(f)
            w.writerow(["epoch", "loss", "train_f1", "val_f1", "test_f1", "sec", "mean_input_nodes", "mean_cached"])
            for r in self.rows:
                w.writerow([r.epoch, f"{r.loss:.6f}", f"{r.train_f1:.4f}", f"{r.val_f1:.4f}", f"{r.test_f1:.4f}",
                            f"{r.seconds:.3f}", f"{r.mean_input_nodes:.1f}", f"{r.mean_cached:.1f}"])


def _views(mdl: GraphSAGE, flat: torch.Tensor) -> list:
    """Per-tensor views (weights then biases, model.py:231 order) of a flat
    buffer laid out like the model's parameters."""
    ws, bs = [], []
    off = 0
    for d_in, d_out in zip(mdl.dims[:-1], mdl.dims[1:]):
        nw = 2 * d_in * d_out
        ws.append(flat[off:off + nw].view(2 * d_in, d_out))
        off += nw
        bs.append(flat[off:off + d_out])
        off += d_out
    return ws + bs


def init_params(dims, seed: int = 0, dtype=torch.float64, device=None, tf32: bool = True) -> ModelParams:
    """model.py:113-121: Glorot-uniform weights (limit sqrt(6/(2 d_in + d_out)),
    the reference's own numpy draw, so both start from identical values) and
    zero biases."""
    return ModelParams(GraphSAGE(dims, dtype=dtype, device=device, seed=seed, tf32=tf32))


def _table(features, params: ModelParams) -> torch.Tensor:
    if isinstance(features, Graph):
        features = features.features
    if features is None:
        raise ValueError("graph has no features")
    t = torch.as_tensor(features)
    if t.device != params.model.device:
        t = t.to(params.model.device)
    if t.dtype not in (torch.float32, torch.float64):
        t = t.float()
    return t


def _forward_pass(mb: MiniBatch, features, params: ModelParams, stream=None):
    """model.py:141-159 (returns logits and the saved per-layer tensors)."""
    if len(mb.blocks) != params.num_layers:
        raise ValueError(f"batch has {len(mb.blocks)} layers, model has {params.num_layers}")
    table = _table(features, params)
    d0 = params.dims[0]
    fd = features.feature_dim if isinstance(features, Graph) else table.shape[1]
    if fd not in (d0, (d0 + 3) // 4 * 4) or table.shape[1] < d0:
        raise ValueError(f"feature dim {fd} != model input dim {d0}")
    mdl = params.model
    h = mdl.gather_inputs(mb, None, features=table, stream=stream)
    return mdl.forward(mb, h, stream)


def forward(mb: MiniBatch, features, params: ModelParams) -> torch.Tensor:
    """model.py:162-165: logits for mb.targets (rows follow the sorted target
    order)."""
    logits, _ = _forward_pass(mb, features, params)
    return logits


def loss_and_grad(logits: torch.Tensor, labels):
    """model.py:189-200: mean softmax cross-entropy and its gradient wrt the
    logits (``labels`` = the labels of the logits' rows)."""
    n, c = logits.shape
    lab = torch.as_tensor(labels, device=logits.device).to(torch.int32).contiguous()
    if lab.numel() and (int(lab.min()) < 0 or int(lab.max()) >= c):
        raise ValueError(f"label out of range for {c} classes")
    grad = torch.empty_like(logits)
    loss = torch.zeros(1, dtype=torch.float64, device=logits.device)
    rows = torch.arange(n, dtype=torch.int32, device=logits.device)
    n_dev = torch.tensor([n], dtype=torch.int32, device=logits.device)
    ws = _lib.workspace(8 * max(n, 1024), logits.device)
    _lib.call("gns_softmax_xent", 0 if logits.dtype == torch.float32 else 1, logits.data_ptr(), logits.stride(0),
              n_dev.data_ptr(), n, 0, c, lab.data_ptr(), rows.data_ptr(), grad.data_ptr(), loss.data_ptr(),
              ws.data_ptr(), ws.numel(), _lib.stream_ptr())
    return float(loss), grad


def backward(mb: MiniBatch, features, params: ModelParams, grad_logits: torch.Tensor) -> ParamGrads:
    """model.py:209-226: exact gradients of forward() wrt every weight and
    bias (recomputes the forward, as the reference does)."""
    _, saved = _forward_pass(mb, features, params)
    mdl = params.model
    g = torch.as_tensor(grad_logits, device=mdl.device).to(mdl.dtype)
    mdl.backward(mb, saved, g.contiguous())
    views = _views(mdl, mdl.grad)
    L = params.num_layers
    return ParamGrads(weights=views[:L], biases=views[L:])


def adam_step(params: ModelParams, grads: ParamGrads, state: AdamState, config: TrainConfig) -> None:
    """model.py:229-242: one bias-corrected Adam update, in place (one
    gns_adam launch over the flat buffers)."""
    mdl = params.model
    own = _views(mdl, mdl.grad)
    for dst, src in zip(own, list(grads.weights) + list(grads.biases)):
        if src.data_ptr() != dst.data_ptr():
            dst.copy_(torch.as_tensor(src, device=mdl.device))
    state.step += 1
    _lib.call("gns_adam", 0 if mdl.dtype == torch.float32 else 1, mdl.flat.data_ptr(), mdl.grad.data_ptr(),
              state.m_flat.data_ptr(), state.v_flat.data_ptr(), mdl.numel, config.lr, config.beta1, config.beta2,
              config.eps, state.step, 1.0, _lib.stream_ptr())


def full_block(g: Graph) -> LayerBlock:
    """The whole graph as one block: dst = src = every node, the CSR's edges
    with weight 1 (what an NS draw with fanout >= max degree keeps: weight
    deg/take = 1), dst_degree = degree — the reference's full-neighbourhood
    (A h)/max(deg, 1) aggregation (model.py:168-186).  Built straight from
    the CSR (no sampler: rows of any degree); edge offsets must fit 32 bits."""
    n, E = g.num_nodes, g.num_edges
    if E >= 2 ** 32:
        raise ValueError("full-batch blocks need < 2^32 edges")
    dev = g.device
    ar = torch.arange(n, dtype=torch.int32, device=dev)
    deg = g.degrees
    row = torch.repeat_interleave(ar, deg.long()) if E else torch.empty(0, dtype=torch.int32, device=dev)
    counts = torch.zeros(_lib.CNT_N, dtype=torch.int32, device=dev)
    counts[_lib.CNT_DST] = n
    counts[_lib.CNT_SRC] = n
    counts[_lib.CNT_EDGES] = E
    # row_scan[r] = (cached prefix << 32) | fill prefix: no cached part here
    b = LayerBlock(dst_nodes=ar, src_nodes=ar, edge_src=g.indices, edge_dst=row.to(torch.int32),
                   edge_weight=torch.ones(E, dtype=torch.float64, device=dev),
                   edge_cached=torch.zeros(E, dtype=torch.uint8, device=dev), dst_degree=deg, fanout=None,
                   policy="uniform", self_pos=ar, edge_node=g.indices, row_scan=g.indptr.clone(), counts=counts)
    b._c = _lib.GnsBlock(*(0 if t is None else t.data_ptr() for t in (
        b.row_scan, b.dst_degree, b.self_pos, None, b.edge_node, b.edge_src, b.edge_dst, b.edge_weight,
        b.edge_cached, b.src_nodes, b.counts)))
    return b


def full_batch_forward(g: Graph, params: ModelParams, features=None) -> torch.Tensor:
    """model.py:168-186: full-neighbourhood forward over every node (logits
    for node ids 0..N-1), every layer over the whole-graph block."""
    blk = full_block(g)
    mb = MiniBatch(blocks=(blk,) * params.num_layers, targets=blk.dst_nodes, input_nodes=blk.src_nodes)
    return forward(mb, g if features is None else features, params)


def evaluate(g: Graph, params: ModelParams) -> dict:
    """model.py:245-254: micro-F1 on the masks with full-neighbourhood
    inference."""
    pred = full_batch_forward(g, params).argmax(dim=1)
    out = {}
    for split, mask in (("train", g.train_mask), ("val", g.val_mask), ("test", g.test_mask)):
        out[split] = micro_f1(pred[mask].cpu(), g.labels[mask].cpu()) if mask is not None else 0.0
    return out


def train(g: Graph, sampler_config: SamplerConfig, train_config: TrainConfig, num_workers: int = 1,
          batch_hook=None, dtype=torch.float64, tf32: bool = True) -> TrainReport:
    """model.py:257-307: T epochs over SamplerPool.iter_epoch (cache refreshed
    every P epochs), one Adam step per mini-batch, per-epoch loss / micro-F1 /
    input and cached counts.  ``batch_hook(epoch, index, minibatch, cache,
    sample_ms, train_ms)`` after every step, as in the reference."""
    if g.labels is None or g.train_mask is None:
        raise ValueError("training needs labels and split masks")
    num_classes = int(g.labels.max()) + 1
    L = sampler_config.num_layers
    dims = (g.feature_dim,) + (train_config.hidden_dim,) * (L - 1) + (num_classes,)
    params = init_params(dims, seed=train_config.seed, dtype=dtype, device=g.device, tf32=tf32)
    mdl = params.model
    pool = SamplerPool(g, sampler_config, num_workers=num_workers)
    report = TrainReport()
    for epoch in range(train_config.epochs):
        t_epoch = time.perf_counter()
        losses, input_counts, cached_counts = [], [], []
        for item in pool.iter_epoch(epoch):
            mb = item.minibatch
            t0 = time.perf_counter()
            losses.append(float(mdl.train_step(mb, g, train_config)))
            train_ms = (time.perf_counter() - t0) * 1000.0
            input_counts.append(int(mb.input_nodes.numel()))
            cached = 0
            if pool.cache is not None:
                cached = int(pool.cache.nodes.contains(mb.input_nodes).sum())
            cached_counts.append(cached)
            if batch_hook is not None:
                batch_hook(epoch, item.index, mb, pool.cache, item.sample_ms, train_ms)
        f1 = evaluate(g, params)
        report.rows.append(EpochStats(
            epoch=epoch, loss=float(np.mean(losses)) if losses else 0.0, train_f1=f1["train"], val_f1=f1["val"],
            test_f1=f1["test"], seconds=time.perf_counter() - t_epoch,
            mean_input_nodes=float(np.mean(input_counts)) if input_counts else 0.0,
            mean_cached=float(np.mean(cached_counts)) if cached_counts else 0.0))
    f1 = evaluate(g, params)
    report.final_train_f1, report.final_val_f1, report.final_test_f1 = f1["train"], f1["val"], f1["test"]
    report.params = params
    return report


__all__ = ["AdamState", "EpochStats", "ModelParams", "ParamGrads", "TrainConfig", "TrainReport", "adam_step",
           "backward", "evaluate", "forward", "full_batch_forward", "init_params", "init_params_numpy",
           "loss_and_grad", "micro_f1", "train"]
