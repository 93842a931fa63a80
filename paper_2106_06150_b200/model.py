"""GraphSAGE-mean trainer on B200 (reference: model.py).

The aggregation path is libgns.so: the input-feature gather (model.py:146),
the fused weighted-mean SpMM + self concat (model.py:131-138,153-154), its
transpose (model.py:223-225), softmax cross-entropy (model.py:189-200) and
Adam (model.py:229-242).  The linear layers ``z = cat @ W + b`` and their
weight gradients are cuBLAS GEMMs through torch (north star: "the GraphSAGE
linear layers stay in torch").

Parameters live in ONE flat buffer (W of shape (2*d_in, d_out) then b per
layer, model.py:37-47), gradients in another, so a data-parallel step is one
NCCL all-reduce and one fused Adam launch.

``dtype=torch.float64`` runs the reference-parity mode: fp64 features, the
bit-exact SpMM (scipy CSR summation order, no FMA) and fp64 GEMMs.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .graph import Graph
from .sampling import MiniBatch


@dataclass
class TrainConfig:
    """model.py:50-65."""

    epochs: int = 10
    lr: float = 0.003
    batch_size: int = 100
    hidden_dim: int = 64
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    seed: int = 0

    def __post_init__(self):
        if self.lr <= 0:
            raise ValueError("lr must be positive")
        if self.hidden_dim < 1:
            raise ValueError("hidden_dim must be >= 1")


def init_params_numpy(dims, seed: int = 0):
    """model.py:113-121 Glorot-uniform draw (host RNG, setup only) so the
    device model starts from the reference's exact initial parameters."""
    rng = np.random.default_rng(seed)
    weights, biases = [], []
    for d_in, d_out in zip(dims[:-1], dims[1:]):
        limit = np.sqrt(6.0 / (2 * d_in + d_out))
        weights.append(rng.uniform(-limit, limit, size=(2 * d_in, d_out)))
        biases.append(np.zeros(d_out))
    return weights, biases


def _dt(dtype) -> int:
    return 0 if dtype == torch.float32 else 1


_SPLIT_CHUNK = 2048
_SPLIT_MIN = 8192


def _split_rows(n: int) -> int:
    """Row count padded for the split-K weight gradient (tall-skinny GEMM)."""
    if n < _SPLIT_MIN:
        return n
    return (n + _SPLIT_CHUNK - 1) // _SPLIT_CHUNK * _SPLIT_CHUNK


def _weight_grad(cat: torch.Tensor, dz: torch.Tensor, out: torch.Tensor, part: torch.Tensor | None = None):
    """dW = cat^T dz (model.py:219).  K = rows is ~10^5 while the output is
    only (2 d_in) x d_out, so a single GEMM has too few output tiles to fill
    148 SMs: split K into 2048-row chunks (batched GEMM into ``part``,
    allocated here unless given) and reduce them in a fixed order
    (gns_sum_rows)."""
    n = cat.shape[0]
    if n < _SPLIT_MIN or n % _SPLIT_CHUNK:
        torch.mm(cat.t(), dz, out=out)
        return
    s = n // _SPLIT_CHUNK
    if part is None:
        part = torch.empty((s,) + tuple(out.shape), dtype=out.dtype, device=out.device)
    p = part[:s]
    torch.bmm(cat.view(s, _SPLIT_CHUNK, -1).transpose(1, 2), dz.view(s, _SPLIT_CHUNK, -1), out=p)
    _lib.call("gns_sum_rows", 0 if out.dtype == torch.float32 else 1, p.data_ptr(), s, out.numel(), out.data_ptr(),
              _lib.stream_ptr())


class _TF32:
    """Scoped torch.backends.cuda.matmul.allow_tf32."""

    def __init__(self, on: bool):
        self.on = on

    def __enter__(self):
        self.prev = torch.backends.cuda.matmul.allow_tf32
        torch.backends.cuda.matmul.allow_tf32 = self.on

    def __exit__(self, *exc):
        torch.backends.cuda.matmul.allow_tf32 = self.prev


class GraphSAGE:
    """Flat-buffer GraphSAGE with a manual forward/backward (model.py:141-226)."""

    def __init__(self, dims, dtype=torch.float32, device=None, seed: int = 0, weights=None, biases=None,
                 tf32: bool = True):
        _lib.require_cuda()
        # float32 mode runs the linear layers on tensor cores (TF32, 10-bit
        # mantissa); float64 mode is the reference-parity path
        self.tf32 = bool(tf32) and dtype == torch.float32
        self.dims = tuple(int(d) for d in dims)
        self.dtype = dtype
        self.device = torch.device(device) if device is not None else torch.device("cuda")
        sizes = []
        for d_in, d_out in zip(self.dims[:-1], self.dims[1:]):
            sizes += [2 * d_in * d_out, d_out]
        self.numel = sum(sizes)
        self.flat = torch.zeros(self.numel, dtype=dtype, device=self.device)
        self.grad = torch.zeros_like(self.flat)
        self.m = torch.zeros_like(self.flat)
        self.v = torch.zeros_like(self.flat)
        self.step_count = 0
        self.weights, self.biases, self.gweights, self.gbiases = [], [], [], []
        off = 0
        for d_in, d_out in zip(self.dims[:-1], self.dims[1:]):
            nw = 2 * d_in * d_out
            self.weights.append(self.flat[off:off + nw].view(2 * d_in, d_out))
            self.gweights.append(self.grad[off:off + nw].view(2 * d_in, d_out))
            off += nw
            self.biases.append(self.flat[off:off + d_out])
            self.gbiases.append(self.grad[off:off + d_out])
            off += d_out
        if weights is None:
            weights, biases = init_params_numpy(self.dims, seed)
        self.load(weights, biases)
        self._ws_bwd = None
        self._ws_xent = None
        self._ws_dense = None
        self.loss_dev = torch.zeros(1, dtype=torch.float64, device=self.device)
        self._labels_checked = None

    @property
    def num_layers(self) -> int:
        return len(self.weights)

    def load(self, weights, biases):
        with torch.no_grad():
            for w, src in zip(self.weights, weights):
                w.copy_(torch.as_tensor(np.asarray(src)).to(self.device, self.dtype))
            for b, src in zip(self.biases, biases):
                b.copy_(torch.as_tensor(np.asarray(src)).to(self.device, self.dtype))

    def export(self):
        return ([w.detach().cpu().double().numpy() for w in self.weights],
                [b.detach().cpu().double().numpy() for b in self.biases])

    # -- forward ------------------------------------------------------------------
    def gather_inputs(self, mb: MiniBatch, g: Graph, features=None, stream=None) -> torch.Tensor:
        """features[mb.input_nodes] (model.py:146) through gns_gather_rows."""
        table = g.features if features is None else features
        n = mb.input_nodes.numel()
        d = self.dims[0]
        h = torch.empty((max(n, 1), d), dtype=self.dtype, device=self.device)
        _lib.call("gns_gather_rows", table.data_ptr(), table.stride(0), 0 if table.dtype == torch.float32 else 1,
                  mb.input_nodes.data_ptr(), None, n, d, h.data_ptr(), h.stride(0), _dt(self.dtype),
                  _lib.stream_ptr(stream))
        return h[:n]

    def _tf32(self):
        return _TF32(self.tf32)

    def forward(self, mb: MiniBatch, h: torch.Tensor, stream=None):
        """Layer chain (model.py:141-159); returns logits and saved tensors."""
        with self._tf32():
            return self._forward(mb, h, stream)

    def _forward(self, mb, h, stream):
        s = _lib.stream_ptr(stream)
        saved = []
        L = self.num_layers
        for li, block in enumerate(mb.blocks):
            d_in = self.dims[li]
            nd = block.dst_nodes.numel()
            npad = _split_rows(nd)
            catp = torch.empty((max(npad, 1), 2 * d_in), dtype=self.dtype, device=self.device)
            # layers > 0 read the previous pre-activation and apply relu on load;
            # rows [nd, npad) are zero so the split-K weight gradient can use them
            _lib.call("gns_spmm_fwd", _dt(self.dtype), h.data_ptr(), h.stride(0), d_in, 1 if li > 0 else 0,
                      block._c, nd, npad, catp.data_ptr(), catp.stride(0), s)
            cat = catp[:npad]
            z = torch.addmm(self.biases[li], cat[:nd], self.weights[li])
            saved.append((cat, z))
            h = z
        return h, saved

    def loss_and_grad(self, logits: torch.Tensor, labels: torch.Tensor, mb: MiniBatch, stream=None):
        """model.py:189-200 fused: returns dlogits; mean loss lands in loss_dev."""
        n, c = logits.shape
        key = (labels.data_ptr(), labels.numel(), c)
        if self._labels_checked != key:
            # model.py:192-193 (once per labels tensor: the kernel indexes
            # labels[targets[r]] and would silently use a wrong row otherwise)
            if labels.numel() and (int(labels.min()) < 0 or int(labels.max()) >= c):
                raise ValueError(f"label out of range for {c} classes")
            self._labels_checked = key
        grad = torch.empty_like(logits)
        if self._ws_xent is None or self._ws_xent.numel() < 8 * max(n, 1):
            self._ws_xent = _lib.workspace(8 * max(n, 1024), self.device)
        top = mb.blocks[-1]
        n_dev = top._c.counts + 4 * _lib.CNT_DST
        _lib.call("gns_softmax_xent", _dt(self.dtype), logits.data_ptr(), logits.stride(0), n_dev, n, 0, c,
                  labels.data_ptr(), mb.targets.data_ptr(), grad.data_ptr(), self.loss_dev.data_ptr(),
                  self._ws_xent.data_ptr(), self._ws_xent.numel(), _lib.stream_ptr(stream))
        return grad

    def backward(self, mb: MiniBatch, saved, dlogits: torch.Tensor, stream=None):
        """model.py:209-226 into the flat gradient buffer.  The input layer's
        dh is not formed (features are not trainable; the reference computes
        and discards it)."""
        with self._tf32():
            self._backward(mb, saved, dlogits, stream)

    def _backward(self, mb, saved, dlogits, stream):
        s = _lib.stream_ptr(stream)
        L = self.num_layers
        # output layer: dz = dlogits; db = column sums (model.py:218-220)
        n, d_out = dlogits.shape
        self._ensure_dense_ws(max(n, 1), d_out)
        _lib.call("gns_dense_bwd_bias", _dt(self.dtype), dlogits.data_ptr(), None, dlogits.stride(0), None, n,
                  d_out, None, self.gbiases[L - 1].data_ptr(), self._ws_dense.data_ptr(),
                  self._ws_dense.numel(), s)
        cat, _ = saved[L - 1]
        if cat.shape[0] == n:
            dzp = dlogits
        else:
            dzp = torch.zeros((cat.shape[0], d_out), dtype=self.dtype, device=self.device)
            dzp[:n].copy_(dlogits)
        for li in range(L - 1, -1, -1):
            cat, z = saved[li]
            n = mb.blocks[li].dst_nodes.numel()
            _weight_grad(cat, dzp, self.gweights[li])
            if li == 0:
                break
            dcat = torch.mm(dzp[:n], self.weights[li].t())
            block = mb.blocks[li]
            nsrc = block.src_nodes.numel()
            d_in = self.dims[li]
            need = _lib.lib().gns_spmm_bwd_workspace_size(nsrc, block.num_edges, d_in)
            if self._ws_bwd is None or self._ws_bwd.numel() < need:
                self._ws_bwd = _lib.workspace(int(need * 1.5), self.device)
            # A^T (dagg / norm) + self term (model.py:223-225) fused with the
            # previous layer's relu' mask and bias gradient (model.py:218,220)
            npad_prev = saved[li - 1][0].shape[0]
            z_prev = saved[li - 1][1]
            dzp = torch.empty((max(npad_prev, 1), d_in), dtype=self.dtype, device=self.device)
            _lib.call("gns_spmm_bwd", _dt(self.dtype), dcat.data_ptr(), dcat.stride(0), d_in, block._c,
                      block.dst_nodes.numel(), nsrc, block.num_edges, npad_prev, z_prev.data_ptr(),
                      self.gbiases[li - 1].data_ptr(), dzp.data_ptr(), dzp.stride(0),
                      self._ws_bwd.data_ptr(), self._ws_bwd.numel(), s)
            dzp = dzp[:npad_prev]

    def _ensure_dense_ws(self, n, d):
        need = _lib.lib().gns_dense_bwd_workspace_size(n, d)
        if self._ws_dense is None or self._ws_dense.numel() < need:
            self._ws_dense = _lib.workspace(int(need * 1.5), self.device)

    def adam_step(self, cfg: TrainConfig, grad_scale: float = 1.0, stream=None):
        """model.py:229-242 (bias-corrected), one launch over the flat buffer."""
        self.step_count += 1
        _lib.call("gns_adam", _dt(self.dtype), self.flat.data_ptr(), self.grad.data_ptr(), self.m.data_ptr(),
                  self.v.data_ptr(), self.numel, cfg.lr, cfg.beta1, cfg.beta2, cfg.eps, self.step_count,
                  grad_scale, _lib.stream_ptr(stream))

    def train_step(self, mb: MiniBatch, g: Graph, cfg: TrainConfig, features=None, allreduce=None,
                   stream=None) -> torch.Tensor:
        """model.py:279-285 loop body; returns the device loss (float64[1])."""
        h = self.gather_inputs(mb, g, features, stream)
        logits, saved = self.forward(mb, h, stream)
        dlogits = self.loss_and_grad(logits, g.labels, mb, stream)
        self.backward(mb, saved, dlogits, stream)
        scale = 1.0
        if allreduce is not None:
            scale = allreduce(self.grad)
        self.adam_step(cfg, grad_scale=scale, stream=stream)
        return self.loss_dev

    def logits(self, mb: MiniBatch, g: Graph, features=None) -> torch.Tensor:
        """forward() of the reference (model.py:162-165): logits for sorted targets."""
        h = self.gather_inputs(mb, g, features)
        out, _ = self.forward(mb, h)
        return out


def micro_f1(pred, true) -> float:
    """model.py:124-128."""
    if len(true) == 0:
        return 0.0
    return float((torch.as_tensor(pred) == torch.as_tensor(true)).float().mean())
