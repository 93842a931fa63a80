"""Graph construction and on-disk formats feeding the device graph
(reference: graph.py:8-28, 142-169, 258-363).

* ``build_csr(edge_list, num_nodes)`` — symmetrise / drop self loops and
  duplicates / sort rows on the device (gns_build_csr_count/fill), the
  graph.py:142-169 contract, including its ValueError on out-of-range ids.
* ``load_binary`` / ``save_binary`` — the GNSG v1 format (little-endian,
  normative field order, graph.py:8-28).  Loading memory-maps the file and
  streams each section to HBM in chunks (indices int64 -> int32 on the way),
  never materialising the whole file in host RAM (graph.py:304-343 reads it
  all); errors name expected vs actual sizes (GraphFormatError).
* ``load_edgelist`` / ``load_feature_csv`` — text formats (graph.py:258-280,
  346-363).
* ``validate_graph`` — graph.py:366-389 invariants, evaluated on the device.
"""

from __future__ import annotations

import os
import struct

import numpy as np
import torch

from . import _lib
from ._lib import GraphFormatError, InvariantError
from .graph import Graph

MAGIC = b"GNSG"
FORMAT_VERSION = 1
_HEADER = struct.Struct("<4sHQQIBB")
_CHUNK = 1 << 26  # elements per host->device chunk


def _dev(device):
    return torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())


def _csr_from_pairs(u: torch.Tensor, v: torch.Tensor, num_nodes: int):
    dev = u.device
    m = int(u.numel())
    ws = _lib.workspace(_lib.lib().gns_gen_workspace_size(num_nodes, m), dev)
    indptr = torch.empty(num_nodes + 1, dtype=torch.int64, device=dev)
    nnz = torch.zeros(1, dtype=torch.int64, device=dev)
    s = _lib.stream_ptr()
    _lib.call("gns_build_csr_count", num_nodes, u.data_ptr(), v.data_ptr(), m, indptr.data_ptr(), nnz.data_ptr(),
              ws.data_ptr(), ws.numel(), s)
    e = int(nnz.item())
    indices = torch.empty(max(e, 1), dtype=torch.int32, device=dev)[:e]
    _lib.call("gns_build_csr_fill", num_nodes, m, indptr.data_ptr(), indices.data_ptr(), ws.data_ptr(), ws.numel(),
              s)
    return indptr, indices


def build_csr(edge_list, num_nodes: int, device=None) -> Graph:
    """graph.py:142-169 on the device."""
    _lib.require_cuda()
    if num_nodes >= 2 ** 31:
        raise ValueError("node ids must fit in int32")
    edges = np.asarray(edge_list, dtype=np.int64).reshape(-1, 2)
    if edges.size:
        bad = (edges < 0) | (edges >= num_nodes)
        if bad.any():
            i = int(np.flatnonzero(bad.any(axis=1))[0])
            a, b = int(edges[i, 0]), int(edges[i, 1])
            raise ValueError(f"edge ({a}, {b}) out of range for num_nodes={num_nodes}")
    dev = _dev(device)
    u = torch.as_tensor(edges[:, 0].astype(np.int32)).to(dev)
    v = torch.as_tensor(edges[:, 1].astype(np.int32)).to(dev)
    indptr, indices = _csr_from_pairs(u, v, num_nodes)
    return Graph(num_nodes, indptr, indices)


def load_edgelist(path, num_nodes: int | None = None, device=None) -> Graph:
    """graph.py:258-280: '#' comments, two non-negative ids per line."""
    edges = []
    with open(path) as f:
        for lineno, line in enumerate(f, start=1):
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            parts = line.split()
            if len(parts) != 2:
                raise GraphFormatError(f"{path}:{lineno}: expected two node ids, got {line!r}")
            try:
                a, b = int(parts[0]), int(parts[1])
            except ValueError:
                raise GraphFormatError(f"{path}:{lineno}: non-integer node id in {line!r}") from None
            if a < 0 or b < 0:
                raise GraphFormatError(f"{path}:{lineno}: negative node id")
            edges.append((a, b))
    if num_nodes is None:
        num_nodes = 1 + max((max(a, b) for a, b in edges), default=-1)
    return build_csr(edges, num_nodes, device=device)


def read_header(path):
    """Parse and size-check a GNSG header (host only)."""
    size = os.path.getsize(path)
    if size < _HEADER.size:
        raise GraphFormatError(f"{path}: truncated header, expected {_HEADER.size} bytes, got {size}")
    with open(path, "rb") as f:
        magic, version, n, e, fdim, has_labels, has_masks = _HEADER.unpack(f.read(_HEADER.size))
    if magic != MAGIC:
        raise GraphFormatError(f"{path}: bad magic {magic!r}, expected {MAGIC!r}")
    if version != FORMAT_VERSION:
        raise GraphFormatError(f"{path}: unsupported version {version}")
    expected = 8 * (n + 1) + 8 * e + 4 * n * fdim + (4 * n if has_labels else 0) + (3 * n if has_masks else 0)
    if size - _HEADER.size != expected:
        raise GraphFormatError(f"{path}: truncated graph data, expected {expected} bytes after header, "
                               f"got {size - _HEADER.size}")
    return dict(num_nodes=int(n), num_edges=int(e), feature_dim=int(fdim), has_labels=bool(has_labels),
                has_masks=bool(has_masks))


def _upload(mm: np.ndarray, out: torch.Tensor, conv=None):
    flat = out.view(-1)
    for s in range(0, mm.shape[0], _CHUNK):
        part = np.array(mm[s:s + _CHUNK])
        t = torch.from_numpy(part).to(out.device, non_blocking=False)
        flat[s:s + part.shape[0]].copy_(t if conv is None else conv(t))


def load_binary(path, device=None) -> Graph:
    """graph.py:302-343: GNSG v1 -> HBM graph (streamed, int64 ids -> int32)."""
    _lib.require_cuda()
    h = read_header(path)
    n, e, fdim = h["num_nodes"], h["num_edges"], h["feature_dim"]
    if n >= 2 ** 31:
        raise GraphFormatError(f"{path}: {n} nodes exceed the int32 id range")
    dev = _dev(device)
    off = _HEADER.size
    indptr_mm = np.memmap(path, dtype="<i8", mode="r", offset=off, shape=(n + 1,))
    off += 8 * (n + 1)
    indices_mm = np.memmap(path, dtype="<i8", mode="r", offset=off, shape=(e,)) if e else np.empty(0, np.int64)
    off += 8 * e
    indptr = torch.empty(n + 1, dtype=torch.int64, device=dev)
    _upload(indptr_mm, indptr)
    indices = torch.empty(max(e, 1), dtype=torch.int32, device=dev)[:e]
    if e:
        _upload(indices_mm, indices, conv=lambda t: t.to(torch.int32))
    feats = None
    if fdim:
        fmm = np.memmap(path, dtype="<f4", mode="r", offset=off, shape=(n, fdim))
        ld = (fdim + 3) // 4 * 4
        feats = torch.zeros((n, ld), dtype=torch.float32, device=dev)
        rows = max(1, _CHUNK // max(fdim, 1))
        for s in range(0, n, rows):
            t = torch.from_numpy(np.array(fmm[s:s + rows])).to(dev)
            feats[s:s + t.shape[0], :fdim].copy_(t)
        off += 4 * n * fdim
    labels = None
    if h["has_labels"]:
        labels = torch.from_numpy(np.array(np.memmap(path, dtype="<i4", mode="r", offset=off, shape=(n,)))).to(dev)
        off += 4 * n
    masks = [None, None, None]
    if h["has_masks"]:
        for i in range(3):
            m = np.array(np.memmap(path, dtype=np.uint8, mode="r", offset=off, shape=(n,))).astype(bool)
            masks[i] = torch.from_numpy(m).to(dev)
            off += n
    return Graph(n, indptr, indices, feats, labels, masks[0], masks[1], masks[2],
                 feature_dim=fdim if fdim else None)


def save_binary(g: Graph, path) -> None:
    """graph.py:283-299: write GNSG v1 (indices widened to int64)."""
    has_masks = g.train_mask is not None
    fdim = g.feature_dim
    header = _HEADER.pack(MAGIC, FORMAT_VERSION, g.num_nodes, g.num_edges, fdim,
                          int(g.labels is not None), int(has_masks))
    with open(path, "wb") as f:
        f.write(header)
        f.write(g.indptr.cpu().numpy().astype("<i8").tobytes())
        for s in range(0, g.num_edges, _CHUNK):
            f.write(g.indices[s:s + _CHUNK].to(torch.int64).cpu().numpy().astype("<i8").tobytes())
        if g.features is not None:
            rows = max(1, _CHUNK // max(fdim, 1))
            for s in range(0, g.num_nodes, rows):
                f.write(g.features[s:s + rows, :fdim].contiguous().cpu().numpy().astype("<f4").tobytes())
        if g.labels is not None:
            f.write(g.labels.cpu().numpy().astype("<i4").tobytes())
        if has_masks:
            for m in (g.train_mask, g.val_mask, g.test_mask):
                f.write(m.cpu().numpy().astype(np.uint8).tobytes())


def load_feature_csv(g: Graph, path) -> Graph:
    """graph.py:346-363: attach features/labels from ``node_id,label,f_0..``."""
    try:
        table = np.loadtxt(path, delimiter=",", ndmin=2)
    except ValueError as exc:
        raise GraphFormatError(f"{path}: {exc}") from None
    if table.shape[1] < 2:
        raise GraphFormatError(f"{path}: need node_id,label,... columns")
    ids = table[:, 0].astype(np.int64)
    if ids.min(initial=0) < 0 or ids.max(initial=0) >= g.num_nodes:
        raise GraphFormatError(f"{path}: node id out of range")
    labels = np.zeros(g.num_nodes, dtype=np.int32)
    labels[ids] = table[:, 1].astype(np.int32)
    feats, fdim = None, None
    if table.shape[1] > 2:
        fdim = table.shape[1] - 2
        f = np.zeros((g.num_nodes, fdim), dtype=np.float32)
        f[ids] = table[:, 2:].astype(np.float32)
        ld = (fdim + 3) // 4 * 4
        feats = torch.zeros((g.num_nodes, ld), dtype=torch.float32, device=g.device)
        feats[:, :fdim] = torch.from_numpy(f).to(g.device)
    return Graph(g.num_nodes, g.indptr, g.indices, feats, torch.from_numpy(labels).to(g.device), g.train_mask,
                 g.val_mask, g.test_mask, feature_dim=fdim)


def validate_graph(g: Graph) -> None:
    """graph.py:366-389 on the device; raises InvariantError on the first failure."""
    n = g.num_nodes
    ip, ix = g.indptr, g.indices
    if ip.shape != (n + 1,) or int(ip[0]) != 0:
        raise InvariantError("indptr must have length n+1 and start at 0")
    if int(ip[-1]) != ix.numel():
        raise InvariantError("indptr[-1] must equal len(indices)")
    deg = ip[1:] - ip[:-1]
    if bool((deg < 0).any()):
        raise InvariantError("indptr must be non-decreasing")
    if ix.numel() and (int(ix.min()) < 0 or int(ix.max()) >= n):
        raise InvariantError("neighbor id out of range")
    rows = torch.repeat_interleave(torch.arange(n, device=ix.device, dtype=torch.int64), deg)
    if bool((rows == ix.long()).any()):
        raise InvariantError("self-loop present")
    same = rows[1:] == rows[:-1]
    if bool((same & (ix[1:].long() - ix[:-1].long() <= 0)).any()):
        raise InvariantError("neighbor lists must be sorted and deduplicated")
    keys = rows * n + ix.long()
    rev = torch.sort(ix.long() * n + rows).values
    if not torch.equal(keys, rev):
        raise InvariantError("adjacency is not symmetric")
