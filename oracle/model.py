"""float64 GraphSAGE restatement — TEST INFRASTRUCTURE ONLY.

Restates ``model.py`` of the reference (paths relative to
``/root/reference/pkg/src/gnsbench``): Glorot init (``:113-121``), the
block aggregation matrices (``:131-138``), forward (``:141-165``), softmax
cross-entropy (``:189-200``), the manual backward (``:209-226``) and Adam
(``:229-242``).  scipy's COO->CSR keeps each row's column indices sorted,
which fixes the fp64 summation order the build's exact SpMM mode reproduces.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp


@dataclass
class OParams:
    weights: list
    biases: list
    dims: tuple

    @property
    def num_layers(self):
        return len(self.weights)

    def copy(self):
        return OParams([w.copy() for w in self.weights],
                       [b.copy() for b in self.biases], tuple(self.dims))


def init_params(dims, seed: int = 0) -> OParams:
    """model.py:113-121."""
    rng = np.random.default_rng(seed)
    weights, biases = [], []
    for d_in, d_out in zip(dims[:-1], dims[1:]):
        limit = np.sqrt(6.0 / (2 * d_in + d_out))
        weights.append(rng.uniform(-limit, limit, size=(2 * d_in, d_out)))
        biases.append(np.zeros(d_out))
    return OParams(weights, biases, tuple(dims))


def block_matrices(block):
    """model.py:131-138."""
    nsrc, ndst = len(block.src_nodes), len(block.dst_nodes)
    agg_mat = sp.coo_matrix((block.edge_weight, (block.edge_dst, block.edge_src)),
                            shape=(ndst, nsrc)).tocsr()
    norm = np.maximum(block.dst_degree, 1).astype(np.float64)
    self_pos = np.searchsorted(block.src_nodes, block.dst_nodes)
    return agg_mat, norm, self_pos


def spmm_mean_fwd(block, h):
    """model.py:153: (A_w @ h) / max(deg, 1)."""
    agg_mat, norm, _ = block_matrices(block)
    return (agg_mat @ h) / norm[:, None]


def forward_pass(mb, features, params: OParams):
    """model.py:141-159."""
    h = features[mb.input_nodes].astype(np.float64)
    steps = []
    for li, block in enumerate(mb.blocks):
        agg_mat, norm, self_pos = block_matrices(block)
        agg = (agg_mat @ h) / norm[:, None]
        cat = np.concatenate([h[self_pos], agg], axis=1)
        z = cat @ params.weights[li] + params.biases[li]
        out = np.maximum(z, 0.0) if li + 1 < len(mb.blocks) else z
        steps.append((h, agg_mat, norm, self_pos, cat, z))
        h = out
    return h, steps


def loss_and_grad(logits, labels):
    """model.py:189-200."""
    labels = np.asarray(labels)
    n, c = logits.shape
    shifted = logits - logits.max(axis=1, keepdims=True)
    logp = shifted - np.log(np.exp(shifted).sum(axis=1, keepdims=True))
    loss = float(-logp[np.arange(n), labels].mean())
    grad = np.exp(logp)
    grad[np.arange(n), labels] -= 1.0
    return loss, grad / n


def backward(mb, features, params: OParams, grad_logits, steps=None):
    """model.py:209-226 (``steps`` lets callers reuse the forward's
    intermediates; the reference recomputes them, ``:212``)."""
    if steps is None:
        _, steps = forward_pass(mb, features, params)
    d_w = [None] * params.num_layers
    d_b = [None] * params.num_layers
    dh = np.asarray(grad_logits, dtype=np.float64)
    for li in range(params.num_layers - 1, -1, -1):
        h, agg_mat, norm, self_pos, cat, z = steps[li]
        dz = dh if li == params.num_layers - 1 else dh * (z > 0)
        d_w[li] = cat.T @ dz
        d_b[li] = dz.sum(axis=0)
        dcat = dz @ params.weights[li].T
        d_in = params.dims[li]
        dself, dagg = dcat[:, :d_in], dcat[:, d_in:]
        dh = agg_mat.T @ (dagg / norm[:, None])
        np.add.at(dh, self_pos, dself)
    return d_w, d_b


def spmm_mean_bwd(block, dcat, d_in):
    """model.py:223-225: A_w^T (dagg / norm) then add.at(self_pos, dself)."""
    agg_mat, norm, self_pos = block_matrices(block)
    dself, dagg = dcat[:, :d_in], dcat[:, d_in:]
    dh = agg_mat.T @ (dagg / norm[:, None])
    np.add.at(dh, self_pos, dself)
    return dh


@dataclass
class OAdam:
    m: list
    v: list
    step: int = 0

    @classmethod
    def zeros_like(cls, params: OParams):
        ts = params.weights + params.biases
        return cls([np.zeros_like(t) for t in ts], [np.zeros_like(t) for t in ts])


def adam_step(params: OParams, d_w, d_b, state: OAdam, lr=0.003, beta1=0.9,
              beta2=0.999, eps=1e-8):
    """model.py:229-242."""
    state.step += 1
    t = state.step
    tensors = params.weights + params.biases
    gs = list(d_w) + list(d_b)
    for i, (p, gr) in enumerate(zip(tensors, gs)):
        state.m[i] = beta1 * state.m[i] + (1 - beta1) * gr
        state.v[i] = beta2 * state.v[i] + (1 - beta2) * gr * gr
        m_hat = state.m[i] / (1 - beta1 ** t)
        v_hat = state.v[i] / (1 - beta2 ** t)
        p -= lr * m_hat / (np.sqrt(v_hat) + eps)


def train_step(mb, features, labels, params: OParams, state: OAdam, lr=0.003):
    """model.py:279-285 loop body: forward, loss, backward (which re-runs the
    forward, as the reference does at ``model.py:212``), Adam."""
    logits, _ = forward_pass(mb, features, params)
    loss, grad = loss_and_grad(logits, labels[mb.targets])
    d_w, d_b = backward(mb, features, params, grad)
    adam_step(params, d_w, d_b, state, lr=lr)
    return loss
