"""Synthetic power-law graphs on the host — TEST / BASELINE INFRASTRUCTURE ONLY.

ctypes binding of ``oracle/gen.cc`` (``oracle/libgnsoracle.so``, built by
``__graft_entry__.build()`` through ``oracle/Makefile``): the host restatement
of the device generator ``csrc/gns_gen.cu`` (``gns_gen_powerlaw_*``,
``gns_gen_node_attrs``, ``gns_gen_features``).  bench.py's CPU arm builds its
graph with it, so the reference-side process never loads libgns.so or uses
the GPU; the GPU tests check the device generator against it bit for bit.

The C code is itself pinned here by a numpy restatement of the pair draw and
the node attributes (``gen_pairs_np`` / ``node_attrs_np`` / ``features_np``,
small n) and by ``oracle.gns.build_csr`` (the restatement of the reference's
``graph.py:142-169``) on the same endpoint pairs (tests/test_oracle.py).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from ctypes import c_double, c_float, c_int, c_int32, c_int64, c_uint32, c_void_p

import numpy as np

from . import detmath, philox
from .gns import OGraph

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libgnsoracle.so")
ATTR_KEY = 0x4E4F4445
SQRT3_F = np.float32(float.fromhex("0x1.bb67aep+0"))

_lib = None


def build() -> str:
    r = subprocess.run(["make", "-C", _HERE], capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("oracle/libgnsoracle.so build failed:\n" + r.stdout + r.stderr)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        L.og_gen_powerlaw.restype = c_int64
        L.og_gen_powerlaw.argtypes = [c_int64, c_int64, c_double, c_double, c_uint32, c_void_p, c_void_p, c_int]
        L.og_build_csr.restype = c_int64
        L.og_build_csr.argtypes = [c_int64, c_void_p, c_void_p, c_int64, c_void_p, c_void_p, c_int]
        L.og_gen_pairs.restype = None
        L.og_gen_pairs.argtypes = [c_int64, c_double, c_double, c_uint32, c_int64, c_int64, c_void_p, c_void_p]
        L.og_gen_node_attrs.restype = None
        L.og_gen_node_attrs.argtypes = [c_int64, c_int32, c_double, c_uint32, c_void_p, c_void_p, c_void_p,
                                        c_void_p, c_int]
        L.og_gen_features.restype = None
        L.og_gen_features.argtypes = [c_int64, c_int32, c_int32, c_int32, c_float, c_uint32, c_void_p, c_void_p,
                                      c_int]
        L.og_cached_csr.restype = c_int64
        L.og_cached_csr.argtypes = [c_int64, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int]
        _lib = L
    return _lib


def _threads(threads):
    return int(threads) if threads else len(os.sched_getaffinity(0))


def powerlaw_csr(n, m, alpha, offset, seed=0, threads=None):
    """(indptr int64[n+1], indices int32[nnz]) of the device generator's graph."""
    indptr = np.empty(n + 1, dtype=np.int64)
    raw = np.empty(max(2 * m, 1), dtype=np.int32)
    nnz = lib().og_gen_powerlaw(n, m, float(alpha), float(offset), seed & 0xFFFFFFFF, indptr.ctypes.data,
                                raw.ctypes.data, _threads(threads))
    if nnz < raw.shape[0] // 2:
        raw = raw[:nnz].copy()
    return indptr, raw[:nnz]


def build_csr_pairs(n, u, v, threads=None):
    """graph.py:142-169 on endpoint arrays through the C pipeline."""
    u = np.ascontiguousarray(u, dtype=np.int32)
    v = np.ascontiguousarray(v, dtype=np.int32)
    indptr = np.empty(n + 1, dtype=np.int64)
    raw = np.empty(max(2 * len(u), 1), dtype=np.int32)
    nnz = lib().og_build_csr(n, u.ctypes.data, v.ctypes.data, len(u), indptr.ctypes.data, raw.ctypes.data,
                             _threads(threads))
    return indptr, raw[:nnz].copy()


def gen_pairs(n, alpha, offset, seed, e0, count):
    u = np.empty(count, dtype=np.int32)
    v = np.empty(count, dtype=np.int32)
    lib().og_gen_pairs(n, float(alpha), float(offset), seed & 0xFFFFFFFF, e0, count, u.ctypes.data, v.ctypes.data)
    return u, v


def node_attrs(n, classes, train_frac, seed=0, threads=None):
    labels = np.empty(n, dtype=np.int32)
    masks = [np.empty(n, dtype=np.bool_) for _ in range(3)]
    lib().og_gen_node_attrs(n, classes, float(train_frac), seed & 0xFFFFFFFF, labels.ctypes.data,
                            *(m.ctypes.data for m in masks), _threads(threads))
    return labels, masks[0], masks[1], masks[2]


def features(n, dim, classes, labels, noise=3.0, seed=0, threads=None):
    ld = (dim + 3) // 4 * 4
    out = np.empty((n, ld), dtype=np.float32)
    labels = np.ascontiguousarray(labels, dtype=np.int32)
    lib().og_gen_features(n, dim, ld, classes, float(noise), seed & 0xFFFFFFFF, labels.ctypes.data,
                          out.ctypes.data, _threads(threads))
    return out


def cached_csr(indptr, indices, mask, threads=None):
    """cache.py:185-197 by filtering the CSR with the cache mask (C, OpenMP)."""
    n = len(indptr) - 1
    indptr = np.ascontiguousarray(indptr, dtype=np.int64)
    indices = np.ascontiguousarray(indices, dtype=np.int32)
    mask = np.ascontiguousarray(mask, dtype=np.bool_)
    c_indptr = np.empty(n + 1, dtype=np.int64)
    th = _threads(threads)
    nnz = lib().og_cached_csr(n, indptr.ctypes.data, indices.ctypes.data, mask.ctypes.data, c_indptr.ctypes.data,
                              None, th)
    c_indices = np.empty(max(nnz, 1), dtype=np.int32)
    lib().og_cached_csr(n, indptr.ctypes.data, indices.ctypes.data, mask.ctypes.data, c_indptr.ctypes.data,
                        c_indices.ctypes.data, th)
    return c_indptr, c_indices[:nnz]


def powerlaw_graph(n, m, alpha, offset, seed=0, feature_dim=0, num_classes=2, train_frac=1.0,
                   feature_noise=3.0, threads=None) -> OGraph:
    """The graph ``paper_2106_06150_b200.generate_powerlaw_device`` builds,
    rebuilt on the host (CSR, labels, masks, features: bit-identical)."""
    indptr, indices = powerlaw_csr(n, m, alpha, offset, seed, threads)
    labels, tr, va, te = node_attrs(n, num_classes, train_frac, seed, threads)
    feats = features(n, feature_dim, num_classes, labels, feature_noise, seed, threads) if feature_dim else None
    return OGraph(num_nodes=n, indptr=indptr, indices=indices, features=feats, labels=labels, train_mask=tr,
                  val_mask=va, test_mask=te)


# ---------------------------------------------------------------------------
# numpy restatement (small n) pinning the C code
# ---------------------------------------------------------------------------

def _feistel_ids(x, n, seed):
    h = philox._feistel_bits(n) // 2
    hmask = np.uint64((1 << h) - 1)
    st = philox.stream_word(31)

    def once(y):
        left, right = y >> np.uint64(h), y & hmask
        for r in range(4):
            f = philox.philox4x32_10(right, r, st, 0, seed, 0x47454E)[0] & hmask
            left, right = right, left ^ f
        return (left << np.uint64(h)) | right

    y = once(np.asarray(x, dtype=np.uint64))
    bad = y >= np.uint64(n)
    while bad.any():
        y[bad] = once(y[bad])
        bad = y >= np.uint64(n)
    return y.astype(np.int32)


def gen_pairs_np(n, alpha, offset, seed, e0, count):
    e = np.arange(e0, e0 + count, dtype=np.uint64)
    w = philox.philox4x32_10(e & philox.MASK32, e >> np.uint64(32), philox.stream_word(40), 0, seed, 0x5041)
    u1 = (((w[0] << np.uint64(32)) | w[1]) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    u2 = (((w[2] << np.uint64(32)) | w[3]) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    oma = 1.0 - alpha
    a0 = float(np.power(offset, oma))
    span = float(np.power(float(n) + offset, oma)) - a0

    def rank(u):
        x = detmath.det_pow(a0 + u * span, 1.0 / oma) - offset
        return np.clip(np.trunc(x), 0, n - 1).astype(np.uint64)

    return _feistel_ids(rank(u1), n, seed), _feistel_ids(rank(u2), n, seed)


def _ih4(a, b):
    s = (a & 0xFFFF) + (a >> np.uint64(16)) + (b & 0xFFFF) + (b >> np.uint64(16))
    return ((s.astype(np.float32) * np.float32(2.0 ** -16)) - np.float32(2.0)) * SQRT3_F


def node_attrs_np(n, classes, train_frac, seed=0):
    v = np.arange(n, dtype=np.uint64)
    w = philox.philox4x32_10(v & philox.MASK32, v >> np.uint64(32), philox.stream_word(41), 0, seed, ATTR_KEY)
    labels = ((w[0] * np.uint64(classes)) >> np.uint64(32)).astype(np.int32)
    r = (w[1] >> np.uint64(8)).astype(np.float32) * np.float32(2.0 ** -24)
    t1, t2 = np.float32(train_frac), np.float32(train_frac + (1.0 - train_frac) / 2)
    return labels, r < t1, (r >= t1) & (r < t2), r >= t2


def features_np(n, dim, classes, labels, noise=3.0, seed=0):
    ld = (dim + 3) // 4 * 4
    pairs = ld // 2
    q = np.arange(pairs, dtype=np.uint64)
    c = np.arange(classes, dtype=np.uint64)[:, None]
    wm = philox.philox4x32_10(q[None, :], c, philox.stream_word(42), 0, seed, ATTR_KEY)
    means = np.empty((classes, ld), dtype=np.float32)
    means[:, 0::2] = _ih4(wm[0], wm[1])
    means[:, 1::2] = _ih4(wm[2], wm[3])
    v = np.arange(n, dtype=np.uint64)[:, None]
    w = philox.philox4x32_10(q[None, :], v & philox.MASK32, philox.stream_word(43), v >> np.uint64(32), seed,
                             ATTR_KEY)
    noise = np.float32(noise)
    out = np.empty((n, ld), dtype=np.float32)
    mu = means[np.asarray(labels, dtype=np.int64)]
    out[:, 0::2] = mu[:, 0::2] + noise * _ih4(w[0], w[1])
    out[:, 1::2] = mu[:, 1::2] + noise * _ih4(w[2], w[3])
    out[:, dim:] = 0.0
    return out
