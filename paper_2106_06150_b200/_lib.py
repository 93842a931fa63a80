"""ctypes binding of libgns.so (include/gns.h).

The extension lives in-tree (``paper_2106_06150_b200/libgns.so``), built for
sm_100a by ``build.py``.  There is no fallback: if the library is missing or a
CUDA device is absent, every product entry point raises.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, Structure, c_double, c_int32, c_int64, c_size_t, c_uint32, c_uint64, c_void_p

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# GNS_LIB: load another build of the same ABI (A/B measurements of kernel changes)
LIB_PATH = os.environ.get("GNS_LIB") or os.path.join(_HERE, "libgns.so")

GNS_OK = 0
GNS_EINVAL = 1
GNS_ECAPACITY = 2
GNS_ECUDA = 3
GNS_EZEROPROB = 4

ERRBIT_ZEROPROB = 1
ERRBIT_CAPACITY = 2
ERRBIT_ZEROQ = 4

CNT_DST, CNT_EDGES, CNT_CACHED, CNT_SRC, CNT_HUBS, CNT_ERR, CNT_N = 0, 1, 2, 3, 4, 5, 16
CNT_WARPROWS, CNT_THREADROWS, CNT_STREAMROWS, CNT_TSEGS = 6, 7, 8, 9


class GraphFormatError(ValueError):
    """graph.py:44 GraphFormatError."""


class InvariantError(RuntimeError):
    """graph.py:48 InvariantError."""


class GnsGraph(Structure):
    _fields_ = [("num_nodes", c_int64), ("num_edges", c_int64), ("indptr", c_void_p),
                ("indices", c_void_p)]


class GnsCache(Structure):
    _fields_ = [("cached_indptr", c_void_p), ("cached_indices", c_void_p),
                ("mask_bits", c_void_p), ("inclusion", c_void_p), ("cached_pos", c_void_p)]


class GnsRng(Structure):
    _fields_ = [("seed", c_uint32), ("epoch", c_uint32), ("batch", c_uint32),
                ("layer", c_uint32)]


class GnsStep(Structure):
    _fields_ = [("seed", c_uint32), ("epoch", c_uint32), ("batch", c_uint32), ("pad", c_uint32),
                ("begin", c_int64), ("count", c_int64)]


class GnsBlock(Structure):
    _fields_ = [("row_scan", c_void_p), ("dst_degree", c_void_p), ("self_pos", c_void_p),
                ("hub_rows", c_void_p), ("edge_node", c_void_p), ("edge_src", c_void_p),
                ("edge_dst", c_void_p), ("edge_weight", c_void_p), ("edge_cached", c_void_p),
                ("src_nodes", c_void_p), ("counts", c_void_p)]


_SIGS = {
    "gns_last_error": (ctypes.c_char_p, []),
    "gns_version": (c_int32, []),
    "gns_record_event_external": (c_int32, [c_void_p, c_void_p]),
    "gns_copy_mapped": (c_int32, [c_void_p, c_void_p, c_int64, c_void_p]),
    "gns_errors_accumulate": (c_int32, [c_void_p, c_int32, c_int32, c_void_p, c_void_p]),
    "gns_tune": (c_int32, [ctypes.c_char_p, c_int32]),
    "gns_graph_instantiate": (c_int32, [c_void_p, c_int32, c_void_p]),
    "gns_graph_launch": (c_int32, [c_void_p, c_void_p]),
    "gns_graph_exec_destroy": (c_int32, [c_void_p]),
    "gns_graph_kernel_priorities": (c_int32, [c_void_p, c_void_p, c_int32]),
    "gns_graph_switch_begin": (c_int32, [c_void_p, c_void_p, c_int64, c_int32, c_void_p]),
    "gns_graph_switch_handles": (c_int32, [c_void_p, c_void_p, c_int64, c_int32, c_void_p, c_void_p]),
    "gns_graph_switch_node": (c_int32, [c_void_p, c_uint64, c_int32, c_void_p]),
    "gns_graph_body_capture_begin": (c_int32, [c_void_p, c_void_p]),
    "gns_graph_body_capture_end": (c_int32, [c_void_p]),
    "gns_degree_probs": (c_int32, [POINTER(GnsGraph), c_void_p, c_void_p]),
    "gns_random_walk_workspace_size": (c_size_t, [c_int64]),
    "gns_random_walk_probs": (c_int32, [POINTER(GnsGraph), c_void_p, c_int64, c_void_p, c_int32, c_void_p,
                                        c_void_p, c_size_t, c_void_p]),
    "gns_cache_draw_workspace_size": (c_size_t, [c_int64]),
    "gns_cache_draw": (c_int32, [c_void_p, c_int64, c_int64, c_uint32, c_uint32, c_uint32, c_void_p,
                                 c_void_p, c_void_p, c_void_p, c_size_t, c_void_p]),
    "gns_edge_inclusion_workspace_size": (c_size_t, [c_int64, c_int64]),
    "gns_estimate_edge_inclusion": (c_int32, [POINTER(GnsGraph), c_void_p, c_int64, c_int32, c_int32, c_int32,
                                              c_uint32, c_void_p, c_void_p, c_size_t, c_void_p]),
    "gns_inclusion": (c_int32, [c_void_p, c_int64, c_int64, c_void_p, c_void_p, c_void_p,
                                c_void_p]),
    "gns_cached_csr_workspace_size": (c_size_t, [c_int64, c_int64]),
    "gns_cached_csr_count": (c_int32, [POINTER(GnsGraph), c_void_p, c_void_p, c_void_p,
                                       c_void_p, c_size_t, c_void_p]),
    "gns_cached_csr_fill": (c_int32, [POINTER(GnsGraph), c_void_p, c_void_p, c_void_p,
                                      c_void_p, c_void_p, c_size_t, c_void_p]),
    "gns_sample_workspace_size": (c_size_t, [c_int64, c_int64]),
    "gns_sample_layer": (c_int32, [POINTER(GnsGraph), POINTER(GnsCache), c_void_p, c_void_p,
                                   c_int64, c_int32, c_int32, c_void_p, POINTER(GnsRng), c_void_p,
                                   POINTER(GnsBlock), c_void_p, c_size_t, c_void_p]),
    "gns_relabel_workspace_size": (c_size_t, [c_int64]),
    "gns_relabel": (c_int32, [c_int64, c_void_p, c_void_p, c_int64, POINTER(GnsBlock), c_int64,
                              c_void_p, c_size_t, c_void_p]),
    "gns_unique_sorted": (c_int32, [c_int64, c_void_p, c_void_p, c_int64, c_void_p, c_void_p,
                                    c_void_p, c_size_t, c_void_p]),
    "gns_epoch_targets": (c_int32, [c_void_p, c_int64, c_uint32, c_uint32, c_int64, c_int64,
                                    c_void_p, c_void_p]),
    "gns_epoch_targets_dev": (c_int32, [c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_void_p,
                                        c_void_p]),
    "gns_batch_targets_sorted": (c_int32, [c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_void_p, c_void_p]),
    "gns_batch_slice_sorted": (c_int32, [c_void_p, c_int64, c_void_p, c_void_p, c_int64, c_void_p, c_void_p,
                                         c_void_p]),
    "gns_gather_rows": (c_int32, [c_void_p, c_int64, c_int32, c_void_p, c_void_p, c_int64,
                                  c_int32, c_void_p, c_int64, c_int32, c_void_p]),
    "gns_gather_rows_mixed": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p, c_int64,
                                        c_void_p, c_void_p, c_int64, c_int32, c_void_p,
                                        c_int64, c_void_p]),
    "gns_cache_refresh_rows": (c_int32, [c_void_p, c_int64, c_void_p, c_void_p, c_int64,
                                         c_int32, c_void_p, c_void_p]),
    "gns_bitmap_rank": (c_int32, [c_void_p, c_int64, c_void_p, c_void_p, c_size_t, c_void_p]),
    "gns_spmm_fwd": (c_int32, [c_int32, c_void_p, c_int64, c_int32, c_int32, POINTER(GnsBlock),
                               c_int64, c_int64, c_void_p, c_int64, c_void_p]),
    "gns_spmm_fwd_gather": (c_int32, [c_void_p, c_int64, c_int32, POINTER(GnsBlock), c_void_p, c_int64, c_int64,
                                      c_int64, c_int32, c_void_p, c_int64, c_void_p]),
    "gns_sum_rows": (c_int32, [c_int32, c_void_p, c_int64, c_int64, c_void_p, c_void_p]),
    "gns_spmm_bwd_workspace_size": (c_size_t, [c_int64, c_int64, c_int32]),
    "gns_spmm_bwd": (c_int32, [c_int32, c_void_p, c_int64, c_int32, POINTER(GnsBlock), c_int64,
                               c_int64, c_int64, c_int64, c_void_p, c_void_p, c_void_p, c_int64,
                               c_void_p, c_size_t, c_void_p]),
    "gns_block_transpose": (c_int32, [POINTER(GnsBlock), c_int64, c_int64, c_int64, c_int32, c_void_p, c_size_t,
                                      c_void_p]),
    "gns_spmm_bwd_transposed": (c_int32, [c_int32, c_void_p, c_int64, c_int32, POINTER(GnsBlock), c_int64,
                                          c_int64, c_int64, c_int64, c_void_p, c_void_p, c_void_p, c_int64,
                                          c_void_p, c_size_t, c_void_p]),
    "gns_relu_bits_size": (c_size_t, [c_int64, c_int32]),
    "gns_spmm_fwd_bits": (c_int32, [c_void_p, c_int64, c_int32, POINTER(GnsBlock), c_int64, c_int64, c_void_p,
                                    c_int64, c_void_p, c_void_p]),
    "gns_spmm_bwd_transposed_bits": (c_int32, [c_void_p, c_int64, c_int32, POINTER(GnsBlock), c_int64, c_int64,
                                               c_int64, c_int64, c_void_p, c_void_p, c_void_p, c_int64, c_void_p,
                                               c_size_t, c_void_p]),
    "gns_adam_dev": (c_int32, [c_int32, c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_double,
                               c_double, c_double, c_double, c_void_p, c_double, c_void_p]),
    "gns_dense_bwd_workspace_size": (c_size_t, [c_int64, c_int32]),
    "gns_dense_bwd_bias": (c_int32, [c_int32, c_void_p, c_void_p, c_int64, c_void_p, c_int64, c_int32,
                                     c_void_p, c_void_p, c_void_p, c_size_t, c_void_p]),
    "gns_softmax_xent": (c_int32, [c_int32, c_void_p, c_int64, c_void_p, c_int64, c_int64, c_int32,
                                   c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_size_t,
                                   c_void_p]),
    "gns_softmax_xent_bias_workspace_size": (c_size_t, [c_int64, c_int64, c_int32]),
    "gns_softmax_xent_bias": (c_int32, [c_int32, c_void_p, c_int64, c_void_p, c_int64, c_int64, c_int32,
                                        c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_size_t,
                                        c_void_p]),
    "gns_adam": (c_int32, [c_int32, c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_double,
                           c_double, c_double, c_double, c_int64, c_double, c_void_p]),
    "gns_gen_workspace_size": (c_size_t, [c_int64, c_int64]),
    "gns_build_csr_count": (c_int32, [c_int64, c_void_p, c_void_p, c_int64, c_void_p, c_void_p, c_void_p,
                                      c_size_t, c_void_p]),
    "gns_build_csr_fill": (c_int32, [c_int64, c_int64, c_void_p, c_void_p, c_void_p, c_size_t, c_void_p]),
    "gns_gen_powerlaw_count": (c_int32, [c_int64, c_int64, c_double, c_double, c_uint32,
                                         c_void_p, c_void_p, c_void_p, c_size_t, c_void_p]),
    "gns_gen_powerlaw_fill": (c_int32, [c_int64, c_int64, c_void_p, c_void_p, c_void_p,
                                        c_size_t, c_void_p]),
    "gns_gen_node_attrs": (c_int32, [c_int64, c_int32, c_double, c_uint32, c_void_p, c_void_p, c_void_p,
                                     c_void_p, c_void_p]),
    "gns_gen_features": (c_int32, [c_int64, c_int32, c_int32, c_int32, ctypes.c_float, c_uint32, c_void_p,
                                   c_void_p, c_void_p, c_void_p]),
}

EXPORTED = tuple(_SIGS)

_lib = None


def load(path: str = LIB_PATH):
    """Load libgns.so and declare every C-ABI signature (no CUDA needed)."""
    global _lib
    if _lib is not None and path == LIB_PATH:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(
            f"libgns.so not found at {path}; build it with "
            "`python -m paper_2106_06150_b200.build` (nvcc, sm_100a)")
    lib = ctypes.CDLL(path)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path == LIB_PATH:
        _lib = lib
    # developer A/B knobs: GNS_TUNE="spmm_narrow=0,stream_len=16" (gns_tune)
    for kv in filter(None, os.environ.get("GNS_TUNE", "").split(",")):
        k, v = kv.split("=")
        if lib.gns_tune(k.strip().encode(), int(v)) != GNS_OK:
            raise ValueError(f"GNS_TUNE: {lib.gns_last_error().decode()}")
    return lib


def lib():
    return _lib if _lib is not None else load()


def require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2106_06150_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")


def check(rc: int, what: str = ""):
    if rc == GNS_OK:
        return
    msg = lib().gns_last_error().decode(errors="replace")
    if rc in (GNS_EINVAL, GNS_EZEROPROB):
        raise ValueError(f"{what}: {msg}" if what else msg)
    if rc == GNS_ECAPACITY:
        raise InvariantError(f"{what}: {msg}" if what else msg)
    raise RuntimeError(f"{what}: {msg}" if what else msg)


# device kernels each entry point launches (memsets excluded) — used to report
# how many of OUR kernels ran inside a timed region
KERNELS_PER_CALL = {
    "gns_degree_probs": 1, "gns_random_walk_probs": 9, "gns_cache_draw": 15, "gns_inclusion": 1, "gns_cached_csr_count": 3,
    "gns_cached_csr_fill": 1, "gns_estimate_edge_inclusion": 0, "gns_sample_layer": 7, "gns_relabel": 4, "gns_unique_sorted": 3,
    "gns_epoch_targets": 1, "gns_epoch_targets_dev": 1, "gns_batch_targets_sorted": 1, "gns_batch_slice_sorted": 1, "gns_copy_mapped": 1, "gns_errors_accumulate": 1, "gns_gather_rows": 1, "gns_gather_rows_mixed": 1,
    "gns_cache_refresh_rows": 1, "gns_bitmap_rank": 1, "gns_spmm_fwd": 1, "gns_spmm_fwd_gather": 1, "gns_sum_rows": 1, "gns_graph_switch_begin": 1, "gns_graph_switch_handles": 1, "gns_graph_switch_node": 0, "gns_spmm_bwd": 7, "gns_block_transpose": 5, "gns_spmm_bwd_transposed": 2, "gns_spmm_fwd_bits": 1, "gns_spmm_bwd_transposed_bits": 2,
    "gns_adam_dev": 1,
    "gns_softmax_xent": 2, "gns_softmax_xent_bias": 1, "gns_adam": 1, "gns_dense_bwd_bias": 2, "gns_gen_powerlaw_count": 6, "gns_gen_powerlaw_fill": 1, "gns_build_csr_count": 6, "gns_build_csr_fill": 1,
    "gns_gen_node_attrs": 1, "gns_gen_features": 2,
}
launch_counter = [0]


SMALL_UNIQUE = 4096  # gns_unique_sorted: one single-CTA kernel up to this many ids


def call(name: str, *args):
    check(getattr(lib(), name)(*args), name)
    if name == "gns_unique_sorted" and args[3] <= SMALL_UNIQUE:
        launch_counter[0] += 1
    else:
        launch_counter[0] += KERNELS_PER_CALL.get(name, 0)


def ptr(t) -> int | None:
    """Device pointer of a tensor (None for None)."""
    if t is None:
        return None
    return t.data_ptr()


def stream_ptr(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def workspace(nbytes: int, device, zero: bool = False) -> torch.Tensor:
    nbytes = max(int(nbytes), 256)
    if zero:
        return torch.zeros(nbytes, dtype=torch.uint8, device=device)
    return torch.empty(nbytes, dtype=torch.uint8, device=device)
