"""Whole-step CUDA-graph training engine (the B200 answer to pool.py + model.py:257-307).

One replay of a captured graph = one training step (``steps_per_graph`` > 1:
several): on a high-priority side branch it samples the NEXT mini-batch into
one sampler slot (epoch-permutation slice, L x (sample, dedup, relabel), the
backward's block transposes — all device-count driven), while the main branch
runs the fused feature gather + aggregation -> L x (SpMM + GEMM) -> softmax-CE
-> backward -> [NCCL all-reduce] -> Adam on the CURRENT batch held in the
other slot.  Two graphs alternate the slot roles, so the host issues one
graph launch per step.

Per-batch values (Philox key, the batch's slice of the epoch permutation)
live in a device ``gns_step_t`` that the step's first sampler kernel reads
from pinned host memory (written by the host before the launch).  Dense tensors are allocated at the static
capacity bounds; kernels zero-fill rows past the device counts, so GEMMs
over padded rows contribute exact zeros, and the input layer's two
capacity-sized GEMMs are SWITCH conditional nodes that run over
ceil(n / chunk) * chunk rows of the batch's device count.

The cache (cache.py) is redrawn at epoch boundaries every ``cache_period``
epochs (pool.py:133-135) with the key ``[seed, 33, epoch]``.  It is
double-buffered: two cache buffer sets (plus, for the mixed placement, two
HBM feature tables) with step graphs captured once per set.  While epoch e
trains on one set, the cache of the next refresh epoch is drawn into the
other on a low-priority stream (draw + inclusion + cached-CSR count, then —
polled from the host loop without blocking — the cached-CSR fill and the
pinned-host -> HBM feature-row refresh), and the epoch boundary only flips
the active set.  Graphs are re-captured only if a cached-CSR buffer grows.

Data parallel: every rank runs ceil(num_batches / W) steps per epoch
(dist.rank_batches(pad=True)); a rank whose stripe is short trains its last
step on an empty batch (zero gradient), so all ranks issue the same
collectives and refresh their (identical, replicated) caches at the same
steps.  Device error flags of every sampled batch are OR-ed into a sticky
word (gns_errors_accumulate) that ``run_epoch`` / ``run_host`` check once per
call and raise as the reference does (sampling.py:248-249,255-256).
"""

from __future__ import annotations

import ctypes
import os

import torch

from . import _lib
from . import cache as cache_mod
from .graph import Graph
from .model import GraphSAGE, TrainConfig, _split_rows, _weight_grad
from .dist import rank_batches, steps_per_epoch
from .pool import cache_probs, exact_tables, num_batches
from .sampling import MiniBatchSampler, SamplerConfig

_CACHE = 33


class GraphedTrainer:
    """CUDA-graph GNS trainer.  One replay = S training steps on the main
    branch (gather -> forward -> backward -> [all-reduce] -> Adam, each on
    the batch held in its sampler slot) while S side branches sample the next
    S batches into the other S slots; the sampler is a chain of short,
    latency-bound kernels, so S independent chains overlap each other and the
    training kernels.  2S slots alternate roles between the two graphs."""

    def __init__(self, g: Graph, config: SamplerConfig, dims, train_config: TrainConfig | None = None,
                 rank: int = 0, world_size: int = 1, allreduce=None, seed: int = 0, host_targets: bool = False,
                 feature_placement: str = "device", host_features: torch.Tensor | None = None,
                 steps_per_graph: int | None = None, switch_chunk: int | None = None, tf32: bool = True):
        _lib.require_cuda()
        if g.features is None or g.labels is None:
            raise ValueError("training needs features and labels")
        self.g, self.cfg = g, config
        self.tc = train_config or TrainConfig()
        self.rank, self.world = rank, world_size
        self.allreduce = allreduce
        self.dev = g.device
        # float32 storage; tf32=True runs the linear layers' GEMMs on the
        # tensor cores in TF32 (10-bit mantissa inputs, fp32 accumulate),
        # tf32=False in full fp32 (the SpMMs, gather, loss and Adam are fp32
        # either way)
        self.model = GraphSAGE(dims, dtype=torch.float32, device=self.dev, seed=seed, tf32=tf32)
        self.dims = self.model.dims
        lab = g.labels
        if lab.numel() and (int(lab.min()) < 0 or int(lab.max()) >= self.dims[-1]):
            # model.py:192-193 (checked once here: the labels are fixed)
            raise ValueError(f"label out of range for {self.dims[-1]} classes")
        self.L = config.num_layers
        # two steps per replay by default: half the graph launches and host
        # round trips (papers100M e2e 1645 vs 1614 mb/s, OAG/products/cfg1
        # +2-3%; the device-timed papers100M step is unchanged)
        S = steps_per_graph if steps_per_graph is not None else int(os.environ.get("GNS_STEPS_PER_GRAPH", "2"))
        if S < 1:
            raise ValueError("steps_per_graph must be >= 1")
        self.S = S
        self.slots = [MiniBatchSampler(g, config) for _ in range(2 * S)]
        for sl in self.slots:
            sl.n_targets_dev = torch.zeros(1, dtype=torch.int32, device=self.dev)
        self.train_ids = g.train_ids()
        # the epoch's whole target permutation, computed once per epoch
        # (gns_epoch_targets) so a step's first sampler kernel only slices it
        self.epoch_perm = (torch.empty_like(self.train_ids)
                           if os.environ.get("GNS_EPOCH_PERM", "1") == "1" and self.train_ids.numel() else None)
        self._perm_epoch = None
        self.step_host = [torch.zeros(4, dtype=torch.int64).pin_memory() for _ in range(2 * S)]
        self.step_dev = [torch.zeros(4, dtype=torch.int64, device=self.dev) for _ in range(2 * S)]
        self.done = [None] * (2 * S)
        # host-provided targets (the end-to-end API): pinned buffers read by a
        # copy kernel inside the graph (gns_copy_mapped)
        self.host_targets = host_targets
        B = config.batch_size
        self.tgt_host = [torch.zeros(B, dtype=torch.int32).pin_memory() for _ in range(2 * S)]
        self.ntgt_host = [torch.zeros(1, dtype=torch.int32).pin_memory() for _ in range(2 * S)]
        # per-step losses of the replays of graph p (host_targets: written by
        # the graph itself, read by run_host after the replay's event)
        self.loss_host = [torch.zeros(S, dtype=torch.float64).pin_memory() for _ in range(2)]
        # Adam's step count lives on the device (gns_adam_dev), per-step losses
        # are kept for the host to read after a replay
        self.adam_t = torch.zeros(2, dtype=torch.int64, device=self.dev)   # [step count, gns_adam_dev ticket]
        self.step_loss = torch.zeros(S, dtype=torch.float64, device=self.dev)
        self._cur_j = 0
        # feature placement: "device" (whole table in HBM) or "mixed" (paper
        # §3.1: table in pinned host memory, the cached rows in an HBM table
        # refreshed with the cache; uncached rows are read over the host link)
        if feature_placement not in ("device", "mixed"):
            raise ValueError(f"unknown feature_placement {feature_placement!r}")
        self.placement = feature_placement
        # device placement: the input layer's SpMM reads the feature table
        # directly (gns_spmm_fwd_gather) instead of a gathered copy
        self.fused_gather = feature_placement == "device" and os.environ.get("GNS_FUSED_GATHER", "1") == "1"
        self.host_features = None
        self.tables = [None, None]
        if feature_placement == "mixed":
            if config.strategy != "GNS":
                raise ValueError("mixed placement needs the GNS cache")
            hf = host_features if host_features is not None else g.features.cpu().pin_memory()
            if not hf.is_pinned():
                hf = hf.pin_memory()
            self.host_features = hf
            cs = int(round(config.cache_frac * g.num_nodes))
            self.tables[0] = torch.empty((max(cs, 1), hf.shape[1]), dtype=torch.float32, device=g.device)
        # double-buffered cache: csets[cur] is the active CacheState; the
        # other set receives the next refresh epoch's cache (prefetch)
        # (epoch, batch indices, slot group, cache set) the last replay of the
        # previous run_epoch call sampled ahead, and the first group's parity
        # of the latest call (slot_of)
        self._ready = None
        self._q0 = 0
        self.prologues = 0         # eager first-group samplings (run_epoch calls that could not continue)
        self._adam_mark = None     # model.step_count the device step count (adam_t[0]) matches after the queued replays
        self.csets = [None, None]
        self._adopted = None       # a caller's CacheState set through `cache` (never written)
        self.cur = 0
        self._pf = None
        self.prefetch = os.environ.get("GNS_CACHE_PREFETCH", "1") == "1"
        self.refresh_log = []      # (epoch, how) of every cache refresh, for tests / bench
        # sticky device error word (gns_errors_accumulate after every sampled batch)
        self.err_dev = torch.zeros(1, dtype=torch.int32, device=self.dev)
        self._probs = None
        self._tables = None
        self._prof_events = None
        # stream priorities (captured into the kernel nodes and honoured by
        # gns_graph_instantiate): which branch of a step the block scheduler
        # serves first when both have CTAs waiting.  Default "main": the
        # training branch is the step's critical path and the sampler (whose
        # result is only needed by the next replay) fills the SM slots it
        # leaves (measured: 0.599 vs 0.646 ms/step with "side", 0.628 "none")
        self.prio_mode = os.environ.get("GNS_STEP_PRIORITY", "main")
        if self.prio_mode not in ("none", "side", "main"):
            raise ValueError(f"GNS_STEP_PRIORITY must be none|side|main, not {self.prio_mode!r}")
        lo, hi = torch.cuda.Stream.priority_range()
        self.sides = [torch.cuda.Stream(device=self.dev, priority=hi if self.prio_mode == "side" else lo)
                      for _ in range(S)]
        self.side = self.sides[0]
        self.main = torch.cuda.Stream(device=self.dev, priority=hi if self.prio_mode == "main" else lo)
        self.refresh_stream = torch.cuda.Stream(device=self.dev, priority=lo)
        self.taux = [torch.cuda.Stream(device=self.dev, priority=hi if self.prio_mode == "side" else lo)
                     for _ in range(2 * S)]
        # size-switched input-layer dense ops: the capacity-sized GEMMs run
        # over the first ceil(n / chunk) * chunk rows (SWITCH graph node on
        # the device row count); bodies are recorded on aux_dense
        self.switch_chunk = switch_chunk if switch_chunk is not None else \
            int(os.environ.get("GNS_SWITCH_CHUNK", "8192"))
        self.aux_dense = torch.cuda.Stream(device=self.dev, priority=hi if self.prio_mode == "main" else lo)
        self._execs = {}
        self._warmed = False
        self._per_replay = 0
        self._alloc()

    @property
    def cache(self):
        """The active CacheState (the one the current epoch samples with)."""
        return self.csets[self.cur]

    @cache.setter
    def cache(self, state):
        """Adopt an externally built cache as the active set.  The caller's
        CacheState is never written: later refreshes draw into buffers of the
        engine's own (_own_set)."""
        self._adopted = state
        self._ready = None
        self.csets[self.cur] = state
        self._free_execs(self.cur)
        if self.placement == "mixed" and state is not None:
            self._fill_table(self.cur, torch.cuda.current_stream())

    @property
    def cache_table(self):
        return self.tables[self.cur]

    # -- static buffers -----------------------------------------------------------
    def _alloc(self):
        sl = self.slots[0]
        L, dims, dev = self.L, self.dims, self.dev
        # model layer li (input first) <-> sampler layer L-1-li
        self.cap_dst = [sl.layers[L - 1 - li].max_dst for li in range(L)]
        self.cap_src = [sl.layers[L - 1 - li].max_src for li in range(L)]
        self.cap_edges = [sl.layers[L - 1 - li].max_edges for li in range(L)]
        self.npad = [_split_rows(c) for c in self.cap_dst]
        f32 = torch.float32
        self.h0 = torch.empty((1 if self.fused_gather else max(self.cap_src[0], 1), dims[0]), dtype=f32, device=dev)
        self.cat = [torch.empty((max(self.npad[li], 1), 2 * dims[li]), dtype=f32, device=dev) for li in range(L)]
        self.z = [torch.empty((max(self.cap_dst[li], 1), dims[li + 1]), dtype=f32, device=dev) for li in range(L)]
        self.dz = [torch.zeros((max(self.npad[li], 1), dims[li + 1]), dtype=f32, device=dev) for li in range(L)]
        self.dcat = [torch.empty((max(self.cap_dst[li], 1), 2 * dims[li]), dtype=f32, device=dev) for li in range(L)]
        lib = _lib.lib()
        self.ws_dense = _lib.workspace(max(lib.gns_dense_bwd_workspace_size(max(p, 1), d)
                                           for p, d in zip(self.npad, dims[1:])), dev)
        # per slot and model layer li >= 1: the block transpose for the
        # backward SpMM, built on the sampling branch (gns_block_transpose);
        # zeroed so an unsampled slot reads as empty
        self.tws = [[None] + [_lib.workspace(lib.gns_spmm_bwd_workspace_size(self.cap_src[li], self.cap_edges[li],
                                                                            dims[li]), dev, zero=True)
                              for li in range(1, L)] for _ in self.slots]
        # the output layer's fused loss + dlogits + bias gradient (one launch;
        # its ticket counter starts at zero and every launch leaves it there)
        self.ws_xent = _lib.workspace(max(lib.gns_softmax_xent_bias_workspace_size(self.cap_dst[L - 1],
                                                                                    self.npad[L - 1], dims[L]),
                                          8 * max(self.cap_dst[L - 1], 1024)), dev, zero=True)
        self.use_switch = self.switch_chunk > 0 and self.switch_chunk % 2048 == 0 and \
            self.cap_dst[0] >= 2 * self.switch_chunk
        # split-K partial products of the input layer's weight gradient
        self.part0 = torch.empty((max(self.npad[0] // 2048, 1), 2 * dims[0], dims[1]), dtype=f32, device=dev)
        # relu' bits of z[li-1] written by layer li's forward, read by its
        # backward (gns_spmm_fwd_bits / gns_spmm_bwd_transposed_bits)
        self.relu_bits = [None] + [
            _lib.workspace(lib.gns_relu_bits_size(max(self.cap_src[li], self.npad[li - 1]), dims[li]), dev)
            for li in range(1, L)]
        self.loss = self.model.loss_dev

    # -- one training step on a slot (captured) ------------------------------------
    def _train_body(self, slot: int, with_adam: bool):
        self._gather(slot)
        self._train_rest(slot, with_adam)

    def _gather(self, slot: int):
        """features[input_nodes] -> h0 (model.py:146); fused into the input
        layer's SpMM (no-op here) when ``fused_gather``."""
        if self.fused_gather:
            return
        sl, L, s = self.slots[slot], self.L, _lib.stream_ptr()
        b0 = sl.layers[L - 1]
        n_in_dev = b0.counts[_lib.CNT_SRC:_lib.CNT_SRC + 1]
        ev = self._prof_events
        if ev is not None:
            _lib.call("gns_record_event_external", ev[0].cuda_event, s)
        if self.placement == "mixed":
            hf, c = self.host_features, self.cache
            _lib.call("gns_gather_rows_mixed", hf.data_ptr(), self.tables[self.cur].data_ptr(),
                      c.nodes.mask_bits.data_ptr(), c.mask_word_rank().data_ptr(), hf.stride(0),
                      b0.src_nodes.data_ptr(), n_in_dev.data_ptr(), self.cap_src[0], self.dims[0],
                      self.h0.data_ptr(), self.h0.stride(0), s)
        else:
            tab = self.g.features
            _lib.call("gns_gather_rows", tab.data_ptr(), tab.stride(0), 0, b0.src_nodes.data_ptr(),
                      n_in_dev.data_ptr(), self.cap_src[0], self.dims[0], self.h0.data_ptr(), self.h0.stride(0), 0,
                      s)
        if ev is not None:
            _lib.call("gns_record_event_external", ev[1].cuda_event, s)

    def _train_rest(self, slot: int, with_adam: bool, loss_out: torch.Tensor | None = None):
        """The training step after the gather; the mean loss goes to
        ``loss_out`` (a float64 device scalar; default model.loss_dev)."""
        m, sl, L, s = self.model, self.slots[slot], self.L, _lib.stream_ptr()
        blocks = [sl.layers[L - 1 - li] for li in range(L)]
        h = self.h0
        with m._tf32():
            # the input layer's two size-switched dense ops (forward GEMM,
            # weight gradient) share one selector kernel
            n0 = blocks[0].counts[_lib.CNT_DST:_lib.CNT_DST + 1]
            hs = self._switch_handles(n0, [self.cap_dst[0], self.npad[0]]) if self.use_switch else None
            h_fwd, h_wg = (hs if hs is not None else (None, None))
            for li in range(L):
                d_in = self.dims[li]
                ev = self._prof_events if li == 0 else None
                if ev is not None:
                    _lib.call("gns_record_event_external", ev[2].cuda_event, s)
                if li == 0 and self.fused_gather:
                    tab = self.g.features
                    dst_ids = sl.layers[L - 2].src_nodes if L > 1 else sl.seeds0
                    _lib.call("gns_spmm_fwd_gather", tab.data_ptr(), tab.stride(0), d_in, blocks[0].cblock,
                              dst_ids.data_ptr(), self.cap_dst[0], self.npad[0],
                              self.switch_chunk if self.use_switch else 0, blocks[0].k, self.cat[0].data_ptr(),
                              self.cat[0].stride(0), s)
                elif li > 0:
                    _lib.call("gns_spmm_fwd_bits", h.data_ptr(), h.stride(0), d_in, blocks[li].cblock,
                              self.cap_dst[li], self.npad[li], self.cat[li].data_ptr(), self.cat[li].stride(0),
                              self.relu_bits[li].data_ptr(), s)
                else:
                    _lib.call("gns_spmm_fwd", 0, h.data_ptr(), h.stride(0), d_in, 0, blocks[li].cblock,
                              self.cap_dst[li], self.npad[li], self.cat[li].data_ptr(), self.cat[li].stride(0), s)
                if ev is not None:
                    _lib.call("gns_record_event_external", ev[3].cuda_event, s)
                if li == 0 and self.use_switch:
                    self._switched(n0, self.cap_dst[0],
                                   lambda R: torch.addmm(m.biases[0], self.cat[0][:R], m.weights[0],
                                                         out=self.z[0][:R]), handle=h_fwd)
                else:
                    torch.addmm(m.biases[li], self.cat[li][:self.cap_dst[li]], m.weights[li], out=self.z[li])
                h = self.z[li]
            top = blocks[L - 1]
            logits = self.z[L - 1]
            # dlogits straight into the output layer's dz (rows >= n zero), the
            # mean loss and the output bias gradient, in one launch
            n_top = top.counts[_lib.CNT_DST:_lib.CNT_DST + 1]
            loss_ptr = (self.loss if loss_out is None else loss_out).data_ptr()
            if self.dims[L] <= 256 and os.environ.get("GNS_FUSED_XENT", "1") == "1":
                _lib.call("gns_softmax_xent_bias", 0, logits.data_ptr(), logits.stride(0), n_top.data_ptr(),
                          self.cap_dst[L - 1], self.npad[L - 1], logits.shape[1], self.g.labels.data_ptr(),
                          sl.seeds0.data_ptr(), self.dz[L - 1].data_ptr(), loss_ptr,
                          m.gbiases[L - 1].data_ptr(), self.ws_xent.data_ptr(), self.ws_xent.numel(), s)
            else:
                _lib.call("gns_softmax_xent", 0, logits.data_ptr(), logits.stride(0), n_top.data_ptr(),
                          self.cap_dst[L - 1], self.npad[L - 1], logits.shape[1], self.g.labels.data_ptr(),
                          sl.seeds0.data_ptr(), self.dz[L - 1].data_ptr(), loss_ptr,
                          self.ws_xent.data_ptr(), self.ws_xent.numel(), s)
                d_last = self.dims[L]
                _lib.call("gns_dense_bwd_bias", 0, self.dz[L - 1].data_ptr(), None, d_last, None,
                          self.cap_dst[L - 1], d_last, None, m.gbiases[L - 1].data_ptr(), self.ws_dense.data_ptr(),
                          self.ws_dense.numel(), s)
            for li in range(L - 1, -1, -1):
                if li == 0 and self.use_switch:
                    self._switched(n0, self.npad[0],
                                   lambda R: _weight_grad(self.cat[0][:R], self.dz[0][:R], m.gweights[0], self.part0),
                                   empty=lambda: m.gweights[0].zero_(), handle=h_wg)
                else:
                    _weight_grad(self.cat[li][:self.npad[li]], self.dz[li][:self.npad[li]], m.gweights[li])
                if li == 0:
                    break
                torch.mm(self.dz[li][:self.cap_dst[li]], m.weights[li].t(), out=self.dcat[li])
                # transpose SpMM fused with the previous layer's relu' and bias grad
                # transpose SpMM fused with the previous layer's relu' (from the
                # forward's bits) and bias grad.  dz rows past the count are not
                # zeroed: the weight gradient multiplies them by cat's zero rows
                ws = self.tws[slot][li]
                evb = self._prof_events if li == 1 else None
                if evb is not None:
                    _lib.call("gns_record_event_external", evb[4].cuda_event, s)
                _lib.call("gns_spmm_bwd_transposed_bits", self.dcat[li].data_ptr(), self.dcat[li].stride(0),
                          self.dims[li], blocks[li].cblock, self.cap_dst[li], self.cap_src[li], self.cap_edges[li],
                          0, self.relu_bits[li].data_ptr(), m.gbiases[li - 1].data_ptr(),
                          self.dz[li - 1].data_ptr(), self.dz[li - 1].stride(0), ws.data_ptr(), ws.numel(), s)
                if evb is not None:
                    _lib.call("gns_record_event_external", evb[5].cuda_event, s)
        if with_adam:
            self._adam_dev()

    def _switch_handles(self, n_dev: torch.Tensor, limits):
        """One selector kernel for all SWITCH nodes over the same device row
        count (gns_graph_switch_handles); returns the handles, or None when
        not capturing."""
        if not torch.cuda.is_current_stream_capturing():
            return None
        C = self.switch_chunk
        nb = (ctypes.c_int32 * len(limits))(*[-(-lim // C) + 1 for lim in limits])
        hs = (ctypes.c_uint64 * len(limits))()
        _lib.call("gns_graph_switch_handles", _lib.stream_ptr(), n_dev.data_ptr(), C, len(limits), nb, hs)
        return list(hs)

    def _switched(self, n_dev: torch.Tensor, limit: int, fn, empty=None, handle=None):
        """fn(R) over the first R = min(k * chunk, limit) rows, k = ceil(n /
        chunk) from the device count: a SWITCH graph node with one recorded
        body per k when capturing (gns_graph_switch_begin), fn(limit) eagerly.
        Bodies must not allocate (they are recorded outside torch's graph
        memory pool): out= ops and preallocated buffers only."""
        if not torch.cuda.is_current_stream_capturing():
            fn(limit)
            return
        C = self.switch_chunk
        K = -(-limit // C) + 1
        bodies = (ctypes.c_void_p * K)()
        if handle is not None:   # selector already appended (_switch_handles)
            _lib.call("gns_graph_switch_node", _lib.stream_ptr(), handle, K, bodies)
        else:
            _lib.call("gns_graph_switch_begin", _lib.stream_ptr(), n_dev.data_ptr(), C, K, bodies)
        aux = self.aux_dense
        c0 = _lib.launch_counter[0]
        per_body = 0
        for k in range(K):
            _lib.call("gns_graph_body_capture_begin", _lib.stream_ptr(aux), bodies[k])
            before = _lib.launch_counter[0]
            with torch.cuda.stream(aux):
                if k:
                    fn(min(k * C, limit))
                elif empty is not None:
                    empty()
            per_body = max(per_body, _lib.launch_counter[0] - before)
            _lib.call("gns_graph_body_capture_end", _lib.stream_ptr(aux))
        # one body runs per replay: count its launches once
        _lib.launch_counter[0] = c0 + per_body

    def _adam_dev(self):
        """[all-reduce of the flat gradient] + Adam with the device step count
        (captured: t advances on the device at every replay)."""
        m = self.model
        scale = 1.0
        if self.allreduce is not None:
            scale = self.allreduce(m.grad)
        _lib.call("gns_adam_dev", 0, m.flat.data_ptr(), m.grad.data_ptr(), m.m.data_ptr(), m.v.data_ptr(), m.numel,
                  self.tc.lr, self.tc.beta1, self.tc.beta2, self.tc.eps, self.adam_t.data_ptr(), scale,
                  _lib.stream_ptr())

    def _sample_body(self, slot: int):
        sl = self.slots[slot]
        # with the epoch permutation the first sampler kernel fetches the
        # step struct from pinned host memory itself
        fetch = self.epoch_perm is not None and not self.host_targets
        s = _lib.stream_ptr()
        if not fetch:
            _lib.call("gns_copy_mapped", self.step_dev[slot].data_ptr(), self.step_host[slot].data_ptr(), 32, s)
        if self.host_targets:
            # the host's target ids, read from pinned memory by a kernel
            B = self.cfg.batch_size
            _lib.call("gns_copy_mapped", sl.n_targets_dev.data_ptr(), self.ntgt_host[slot].data_ptr(), 4, s)
            _lib.call("gns_copy_mapped", sl.targets.data_ptr(), self.tgt_host[slot].data_ptr(), 4 * B, s)
        # the backward's block transposes depend only on a finished layer:
        # each is forked onto the slot's aux stream as soon as its layer is
        # sampled and overlaps the sampling of the next (larger) layer
        L, cur, aux = self.L, torch.cuda.current_stream(), self.taux[slot]
        joins = []

        def transpose(lb):
            li = L - 1 - sl.layers.index(lb)
            if li < 1:
                return
            ev = torch.cuda.Event()
            ev.record(cur)
            aux.wait_event(ev)
            ws = self.tws[slot][li]
            _lib.call("gns_block_transpose", lb.cblock, self.cap_dst[li], self.cap_src[li], self.cap_edges[li],
                      self.dims[li], ws.data_ptr(), ws.numel(), _lib.stream_ptr(aux))
            done = torch.cuda.Event()
            done.record(aux)
            joins.append(done)
        sl.enqueue_device(None if self.host_targets else self.train_ids, self.step_dev[slot],
                          self.cache if self.cfg.strategy == "GNS" else None, exact_tables=self._tables,
                          after_layer=transpose, epoch_perm=self.epoch_perm if fetch else None,
                          step_src=self.step_host[slot] if fetch else None)
        _lib.call("gns_errors_accumulate", sl.counts.data_ptr(), self.L, _lib.CNT_N, self.err_dev.data_ptr(), s)
        for ev in joins:
            cur.wait_event(ev)

    # -- cache + capture ------------------------------------------------------------
    @property
    def _positions(self) -> bool:
        """Cached-CSR row positions are read only by the gns-exact policy."""
        return self.cfg.weight_policy == "gns-exact"

    def _cache_size(self) -> int:
        return int(round(self.cfg.cache_frac * self.g.num_nodes))     # pool.py:114

    def _needs_refresh(self, epoch: int) -> bool:
        """pool.py:133-135: redraw when there is no cache or epoch % P == 0."""
        if self.cfg.strategy != "GNS":
            return False
        c = self.cache
        return c is None or (epoch % self.cfg.cache_period == 0 and c.epoch != epoch)

    def _fill_table(self, cs: int, stream):
        """Mixed placement, feature refresh (paper §3.1): the cached rows of
        cache set ``cs``, pinned host -> its HBM table, read through UVA by
        gns_cache_refresh_rows on ``stream``; plus the bitmap word ranks the
        mixed gather uses to find a row's slot."""
        st = self.csets[cs]
        hf, ids = self.host_features, st.nodes.ids
        if self.tables[cs] is None:
            self.tables[cs] = torch.empty_like(self.tables[1 - cs])
        with torch.cuda.stream(stream):
            _lib.call("gns_cache_refresh_rows", hf.data_ptr(), hf.stride(0), ids.data_ptr(),
                      st._buf_counts.data_ptr(), ids.numel(), self.dims[0], self.tables[cs].data_ptr(),
                      _lib.stream_ptr(stream))
            st.mask_word_rank(stream)

    def _refresh_cache(self, epoch: int):
        """pool.py:109-135 at an epoch boundary: activate the prefetched
        cache of this epoch if there is one, else draw it now (stop-the-world,
        into the idle set).  Re-captures only the graphs of a set whose
        buffers moved."""
        if self.cfg.strategy != "GNS":
            return
        self._ready = None      # batches sampled ahead used the previous cache
        if self._probs is None:
            self._probs = cache_probs(self.g, self.cfg)
        cs = self._cache_size()
        seed = [self.cfg.seed, _CACHE, epoch]
        pf = self._pf
        if pf is not None and pf[1].epoch == epoch:
            t, p, stage = pf
            if stage == 1:
                self._prefetch_finish()
            self._pf = None
            torch.cuda.synchronize()
            self.cur = t
            self.refresh_log.append((epoch, "prefetched"))
        else:
            self._pf = None
            t = self.cur if self.cache is None else 1 - self.cur
            self._own_set(t)
            if self.csets[t] is None:
                if self.csets[1 - t] is None:
                    self.csets[t] = cache_mod.build_cache(self.g, self._probs, cs, epoch=epoch, rng_seed=seed,
                                                          positions=self._positions)
                else:
                    self.csets[t] = cache_mod.empty_like(self.csets[1 - t], self.g)
                    cache_mod.refresh_cache(self.csets[t], self.g, self._probs, cs, epoch, seed,
                                            positions=self._positions)
                self._free_execs(t)
            elif not cache_mod.refresh_cache(self.csets[t], self.g, self._probs, cs, epoch, seed,
                                             positions=self._positions):
                self._free_execs(t)
            if self.placement == "mixed":
                self._fill_table(t, torch.cuda.current_stream())
            torch.cuda.synchronize()
            self.cur = t
            self.refresh_log.append((epoch, "sync"))
        if self.cfg.weight_policy == "gns-exact" and self._tables is None:
            self._tables = exact_tables(self.g, self.cfg, self._probs, cs)

    def _own_set(self, t: int):
        """Cache set ``t`` as a refresh target: replaced by fresh buffers if it
        is an adopted (caller-owned) CacheState."""
        if self.csets[t] is not None and self.csets[t] is self._adopted:
            self.csets[t] = cache_mod.empty_like(self.csets[t], self.g)
            self._free_execs(t)

    def _prefetch_begin(self, epoch: int):
        """Start drawing the cache of ``epoch`` into the idle set on the
        low-priority refresh stream (no host wait)."""
        if self.cfg.strategy != "GNS" or self.cache is None:
            return
        if self._pf is not None and self._pf[1].epoch == epoch:
            return
        if self._probs is None:       # the active cache was adopted (cache setter)
            self._probs = cache_probs(self.g, self.cfg)
        t = 1 - self.cur
        self._own_set(t)
        if self.csets[t] is None:
            self.csets[t] = cache_mod.empty_like(self.cache, self.g)
            self._free_execs(t)
        rs = self.refresh_stream
        rs.wait_stream(torch.cuda.current_stream())
        # the refresh stream writes the idle set's buffers: tell the caching
        # allocator, so memory freed with this engine (or a replaced set) is
        # not handed out again before the refresh stream is done with it
        st = self.csets[t]
        for buf in (st._buf_ids, st.nodes.mask_bits, st._buf_counts, st.inclusion, st.cached_indptr, st._buf_cidx,
                    st._buf_cpos):
            buf.record_stream(rs)
        if self.placement == "mixed" and self.tables[t] is not None:
            self.tables[t].record_stream(rs)
        p = cache_mod.refresh_begin(st, self.g, self._probs, self._cache_size(), epoch,
                                    [self.cfg.seed, _CACHE, epoch], stream=rs, positions=self._positions)
        self._pf = (t, p, 1)

    def _prefetch_poll(self, block: bool = False):
        if self._pf is not None and self._pf[2] == 1 and (block or self._pf[1].ready()):
            self._prefetch_finish()

    def _prefetch_finish(self):
        t, p, _ = self._pf
        if not cache_mod.refresh_finish(p):
            self._free_execs(t)
        if self.placement == "mixed":
            self._fill_table(t, self.refresh_stream)
        self._pf = (t, p, 2)

    def _set_step(self, slot: int, epoch: int, index: int | None):
        b = self.cfg.batch_size
        h = self.step_host[slot]
        if self.done[slot] is not None:
            self.done[slot].synchronize()
        if index is None:  # nothing to sample next (epoch/cache boundary)
            h[0], h[1], h[2], h[3] = 0, 0, 0, 0
            return
        h[0] = (self.cfg.seed & 0xFFFFFFFF) | ((epoch & 0xFFFFFFFF) << 32)
        h[1] = index & 0xFFFFFFFF
        h[2] = index * b
        h[3] = b

    def capture_profiled(self):
        """Re-capture with timing events around the input-feature gather
        (gns_gather_rows), the input-layer SpMM and layer 1's transposed
        SpMM of every step of each replay, so their durations can be read
        after a replay (bench.py's rooflines; not the headline)."""
        # one event set per step of a replay (the first step runs beside both
        # sampling branches, the later ones mostly alone): the readers average
        self._prof_steps = [[torch.cuda.Event(enable_timing=True) for _ in range(6)] for _ in range(self.S)]
        for evs in self._prof_steps:     # materialise the driver events
            for e in evs:
                e.record(self.main)
        self._prof_events = self._prof_steps[0]
        torch.cuda.synchronize()
        self._free_execs()

    def _prof_mean(self, a: int, b: int) -> float:
        """Mean event interval (a -> b) over the steps of the last replay."""
        steps = getattr(self, "_prof_steps", None) or [self._prof_events]
        vals = []
        for e in steps:
            e[b].synchronize()
            vals.append(float(e[a].elapsed_time(e[b])))
        return sum(vals) / len(vals)

    def gather_ms(self) -> float:
        return self._prof_mean(0, 1)

    def spmm0_ms(self) -> float:
        """Duration of the input-layer aggregation SpMM in the last replay
        (mean over its steps)."""
        return self._prof_mean(2, 3)

    def bwd1_ms(self) -> float:
        """Duration of model layer 1's transposed SpMM (backward) in the last
        replay (0 for a one-layer model)."""
        if self.L < 2:
            return 0.0
        return self._prof_mean(4, 5)

    # -- capture / replay ---------------------------------------------------------------
    def _group(self, p: int):
        return [p * self.S + j for j in range(self.S)]

    def slot_of(self, k: int) -> int:
        """Sampler slot holding the k-th batch of the latest run_epoch call."""
        return ((k // self.S + self._q0) % 2) * self.S + k % self.S

    def _warm(self):
        # outside capture: cuBLAS handles / workspaces, NCCL communicator
        ev, self._prof_events = self._prof_events, None
        with torch.cuda.stream(self.main):
            self._train_body(0, with_adam=False)
            if self.allreduce is not None:
                self.allreduce(self.model.grad)
        if self.use_switch:   # cuBLAS / cuBLASLt handles and workspaces of aux_dense
            m, C = self.model, self.switch_chunk
            with torch.cuda.stream(self.aux_dense), m._tf32():
                torch.addmm(m.biases[0], self.cat[0][:C], m.weights[0], out=self.z[0][:C])
                _weight_grad(self.cat[0][:C], self.dz[0][:C], m.gweights[0], self.part0)
                m.gweights[0].zero_()
        self._prof_events = ev
        self._warmed = True
        torch.cuda.synchronize()

    def _capture(self, p: int, r: int):
        """Graph (p, r): train the first r slots of group p (r <= S) and
        sample the next S batches into group 1-p."""
        torch.cuda.synchronize()
        c0 = _lib.launch_counter[0]
        gph = torch.cuda.CUDAGraph(keep_graph=True)
        train, nxt = self._group(p)[:r], self._group(1 - p)
        with torch.cuda.graph(gph, stream=self.main):
            # the HBM-bound gather of the first step runs alone; the
            # (latency-bound) sampler branches then overlap the rest
            self._gather(train[0])
            fork = torch.cuda.Event()
            fork.record(self.main)
            joins = []
            for j, sl in enumerate(nxt):
                side = self.sides[j]
                side.wait_event(fork)
                with torch.cuda.stream(side):
                    self._sample_body(sl)
                    ev = torch.cuda.Event()
                    ev.record(side)
                joins.append(ev)
            ev_prof, self._prof_events = self._prof_events, None
            ev_steps = getattr(self, "_prof_steps", None) if ev_prof is not None else None
            for j, sl in enumerate(train):
                self._prof_events = (ev_steps[j] if ev_steps else ev_prof) if ev_prof is not None and \
                    (ev_steps or j == 0) else None
                if j > 0:
                    self._gather(sl)
                # the step's loss straight into its step_loss slot
                self._train_rest(sl, with_adam=True, loss_out=self.step_loss[j:j + 1])
            if self.host_targets:   # every step's loss straight into pinned host memory
                _lib.call("gns_copy_mapped", self.loss_host[p].data_ptr(), self.step_loss.data_ptr(), 8 * r,
                          _lib.stream_ptr())
            self._prof_events = ev_prof
            for ev in joins:
                self.main.wait_event(ev)
        if p == 0 and r == self.S:
            self._per_replay = _lib.launch_counter[0] - c0
        # captured launches are not executions: remove them from the counter
        _lib.launch_counter[0] = c0
        ex = ctypes.c_void_p()
        _lib.call("gns_graph_instantiate", gph.raw_cuda_graph(), 0 if self.prio_mode == "none" else 1,
                  ctypes.byref(ex))
        self._execs[(p, r, self.cur)] = (gph, ex)
        torch.cuda.synchronize()

    def _free_execs(self, cset: int | None = None):
        """Destroy the step graphs (of one cache set, or all)."""
        for key in [k for k in self._execs if cset is None or k[2] == cset]:
            _lib.call("gns_graph_exec_destroy", self._execs.pop(key)[1])

    def __del__(self):
        try:
            self.refresh_stream.synchronize()   # a prefetch may still write the idle cache set
            self._free_execs()
        except Exception:
            pass

    def _replay(self, p: int, r: int | None = None):
        r = self.S if r is None else r
        if (p, r, self.cur) not in self._execs:
            if not self._warmed:
                self._warm()
            self._capture(p, r)
        _lib.call("gns_graph_launch", self._execs[(p, r, self.cur)][1], _lib.stream_ptr(self.main))

    def prepare(self, steps: int):
        """Capture every step graph a run of ``steps`` steps replays, so no
        capture happens inside a timed region: both graphs (p = 0, 1) for
        every replay size the run can use (S; shorter groups at an epoch's
        end), for the active cache set and — when the run may cross a cache
        refresh — for the idle set it will switch to (allocated here)."""
        if not self._warmed:
            self._warm()
        sizes = set(range(1, self.S + 1)) if steps >= self.S else {steps % self.S}
        sets = [self.cur]
        # (the mixed placement's idle set gets its graphs at its first use:
        # its HBM feature table and bitmap ranks are filled with the cache)
        if self.cfg.strategy == "GNS" and self.cache is not None and self.placement != "mixed":
            if steps >= len(self.batches(0)) or self.prefetch:
                t = 1 - self.cur
                if self.csets[t] is None:
                    self.csets[t] = cache_mod.empty_like(self.cache, self.g)
                sets.append(t)
        cur = self.cur
        try:
            for cs in sets:
                self.cur = cs
                for r in sorted(sizes - {0}):
                    for p in (0, 1):
                        if (p, r, cs) not in self._execs:
                            self._capture(p, r)
        finally:
            self.cur = cur

    @property
    def graphs(self):
        """Captured step graphs of the current cache (torch CUDAGraph objects)."""
        return [self._execs[k][0] for k in sorted(self._execs)]

    def kernel_priorities(self, p: int = 0):
        """Histogram of |priority| over the kernel nodes of step graph (p, S)."""
        if (p, self.S, self.cur) not in self._execs:
            self._capture(p, self.S)
        hist = (ctypes.c_int32 * 8)()
        _lib.call("gns_graph_kernel_priorities", self._execs[(p, self.S, self.cur)][0].raw_cuda_graph(), hist, 8)
        return list(hist)

    def loss_value(self) -> float:
        """Loss of the step reported by the last on_step/on_loss callback
        (synchronises the engine stream)."""
        self.main.synchronize()
        return float(self.step_loss[self._cur_j])

    def kernels_per_step(self) -> float:
        """libgns kernels inside the captured step graph, per training step."""
        if not self._per_replay and (0, self.S, self.cur) not in self._execs:
            self._capture(0, self.S)
        return self._per_replay / self.S

    # -- driving ----------------------------------------------------------------------
    def batches(self, epoch: int):
        """This rank's step schedule of ``epoch``: batch indices (pool.py:80
        striding); data parallel (W > 1): padded to ceil(nb / W) steps with
        None = an empty batch (zero gradient), the same count on every rank."""
        return rank_batches(num_batches(self.g, self.cfg), self.rank, self.world, pad=self.world > 1)

    def run(self, steps: int, epoch: int = 0, first: int = 0, on_step=None):
        """Run ``steps`` training steps starting at batch ``first`` of
        ``epoch`` (crossing epochs as needed); returns the (epoch, first)
        position to continue from."""
        while steps > 0:
            n = self.run_epoch(epoch, first=first, max_steps=steps, on_step=on_step)
            steps -= n
            if first + n >= len(self.batches(epoch)):
                epoch, first = epoch + 1, 0
            else:
                first += n
        return epoch, first

    def _begin(self, epoch: int):
        # fast path for a call continuing the previous one (same epoch, no
        # refresh, Adam's device step count already the host's): nothing to
        # synchronise or enqueue before the first replay
        if (self.model.step_count == self._adam_mark and not self._needs_refresh(epoch)
                and (self.epoch_perm is None or self._perm_epoch == epoch)):
            # (work the caller queued on its current stream still precedes the
            # replays, without blocking the host)
            self.main.wait_stream(torch.cuda.current_stream())
            return
        torch.cuda.synchronize()
        if self._needs_refresh(epoch):
            self._refresh_cache(epoch)
        self.adam_t[0].fill_(self.model.step_count)
        self._adam_mark = self.model.step_count
        if self.epoch_perm is not None and self._perm_epoch != epoch:
            n = self.train_ids.numel()
            _lib.call("gns_epoch_targets", self.train_ids.data_ptr(), n, self.cfg.seed & 0xFFFFFFFF,
                      epoch & 0xFFFFFFFF, 0, n, self.epoch_perm.data_ptr(), _lib.stream_ptr())
            torch.cuda.synchronize()
            self._perm_epoch = epoch

    def _next_refresh_epoch(self, epoch: int):
        """The epoch after ``epoch`` if it redraws the cache (pool.py:133-135)."""
        e = epoch + 1
        return e if self.cfg.strategy == "GNS" and e % self.cfg.cache_period == 0 else None

    def run_epoch(self, epoch: int, first: int = 0, max_steps: int | None = None, on_step=None) -> int:
        """Steps ``first``, ``first+1``, ... of this rank's schedule of
        ``epoch`` (at most ``max_steps``); returns the number of steps run.
        ``on_step(epoch, index, k)`` (index None = padded empty step) runs
        after each step is enqueued."""
        idx = self.batches(epoch)[first:]
        if max_steps is not None:
            idx = idx[:max_steps]
        if not idx:
            return 0
        self._begin(epoch)
        nre = self._next_refresh_epoch(epoch) if self.prefetch else None
        S = self.S
        groups = [idx[i:i + S] for i in range(0, len(idx), S)]
        full = self.batches(epoch)
        end = first + len(idx)
        rd, self._ready = self._ready, None
        if rd is not None and rd == (epoch, tuple(groups[0]), rd[2], self.cur) and len(groups[0]) == S:
            # the previous call's last replay already sampled this call's
            # first group (same epoch and cache set): no eager prologue
            q0 = rd[2]
        else:
            # prologue: sample the first group into group-0 slots
            q0 = 0
            self.prologues += 1
            for j, sl in enumerate(self._group(0)):
                self._set_step(sl, epoch, groups[0][j] if j < len(groups[0]) else None)
            with torch.cuda.stream(self.main):
                for sl in self._group(0):
                    self._sample_body(sl)
        self._q0 = q0
        k = 0
        for gi, grp in enumerate(groups):
            p = (gi + q0) % 2
            if gi + 1 < len(groups):
                nxt = groups[gi + 1]
            else:
                # the batches after this call's last one (same epoch): sampled
                # by the last replay so a continuing call starts without a
                # prologue
                nxt = full[end:end + S] if len(full[end:end + S]) == S else []
                if nxt:
                    self._ready = (epoch, tuple(nxt), 1 - p, self.cur)
            for j, sl in enumerate(self._group(1 - p)):
                self._set_step(sl, epoch, nxt[j] if j < len(nxt) else None)
            with torch.cuda.stream(self.main):
                self._replay(p, len(grp))
                ev = torch.cuda.Event()
                ev.record(self.main)
                for sl in self._group(1 - p):
                    self.done[sl] = ev
            if nre is not None:
                # the next refresh epoch's cache is drawn into the idle set on
                # the low-priority refresh stream, behind the first replay
                if gi == 0:
                    self._prefetch_begin(nre)
                else:
                    self._prefetch_poll()
            self.model.step_count += len(grp)
            self._adam_mark = self.model.step_count
            for j, index in enumerate(grp):
                self._cur_j = j
                if on_step is not None:
                    on_step(epoch, index, k)
                k += 1
        self.check_errors()
        return len(idx)

    def run_host(self, batches, epoch: int = 0, on_loss=None, base: int = 0, lookahead=None):
        """End-to-end API with host buffers: ``batches`` are host int arrays of
        target ids; every step reads them from pinned memory (a copy kernel in
        the graph) and writes every step's loss into pinned memory (another
        copy kernel at the end of the replay), read by the host one replay
        late.  Requires ``host_targets=True``.

        Batch ``batches[i]`` draws Philox batch key ``base + i``.  A continuous
        loop over host batches passes the next call's first S arrays as
        ``lookahead`` (with ``len(batches) % S == 0``): the last replay samples
        them, and the next call — ``base`` advanced by ``len(batches)``, its
        first S arrays those same objects — starts without the eager
        prologue, as consecutive replays do within a call."""
        if not self.host_targets:
            raise ValueError("construct with host_targets=True")
        if not batches:
            return []
        nref = len(self.refresh_log)
        rd, self._ready = self._ready, None
        self._begin(epoch)
        if len(self.refresh_log) != nref:
            rd = None           # sampled ahead with the previous cache
        S = self.S
        n = len(batches)
        ahead = list(lookahead)[:S] if lookahead is not None and n % S == 0 else []
        losses = []
        # double-buffered loss read-back: replay g+1 is queued before the host
        # waits for replay g's losses, so the GPU never idles on the host
        lh = self.loss_host   # written by graph p at the end of its replay
        pending = []

        def drain():
            ev, buf, first, r = pending.pop(0)
            ev.synchronize()
            for j in range(r):
                losses.append(float(buf[j]))
                if on_loss is not None:
                    on_loss(first + j, losses[-1])

        def put(slot, k):
            if self.done[slot] is not None:
                self.done[slot].synchronize()
            arr = batches[k] if k < n else (ahead[k - n] if k - n < len(ahead) else None)
            if arr is None:
                self.ntgt_host[slot][0] = 0
                return
            t = torch.as_tensor(arr, dtype=torch.int32)
            self.tgt_host[slot][:t.numel()].copy_(t)
            self.ntgt_host[slot][0] = t.numel()
            h = self.step_host[slot]
            h[0] = (self.cfg.seed & 0xFFFFFFFF) | ((epoch & 0xFFFFFFFF) << 32)
            h[1] = (base + k) & 0xFFFFFFFF
        # (the arrays themselves are kept in _ready and compared by identity:
        # holding them keeps their ids from being reused by new arrays)
        same = (rd is not None and n >= S and rd[:3] == ("host", epoch, base) and rd[4] == self.cur
                and len(rd[3]) == S and all(a is b for a, b in zip(rd[3], batches[:S])))
        if same:
            q0 = rd[5]      # sampled ahead by the previous call's last replay
        else:
            q0 = 0
            self.prologues += 1
            for j, sl in enumerate(self._group(0)):
                put(sl, j)
            with torch.cuda.stream(self.main):
                for sl in self._group(0):
                    self._sample_body(sl)
        self._q0 = q0
        for gi, b0 in enumerate(range(0, n, S)):
            p = (gi + q0) % 2
            r = min(S, n - b0)
            for j, sl in enumerate(self._group(1 - p)):
                put(sl, b0 + S + j)
            if b0 + S >= n and len(ahead) == S:
                self._ready = ("host", epoch, base + n, tuple(ahead), self.cur, 1 - p)
            with torch.cuda.stream(self.main):
                self._replay(p, r)
                ev = torch.cuda.Event()
                ev.record(self.main)
                for sl in self._group(1 - p):
                    self.done[sl] = ev
            self.model.step_count += r
            self._adam_mark = self.model.step_count
            pending.append((ev, lh[p], b0, r))
            if len(pending) > 1:
                drain()
        while pending:
            drain()
        self.check_errors()
        return losses

    def check_errors(self):
        """Raise the reference's exception for any device error flag of a
        batch sampled since the last check (sticky word; one sync)."""
        torch.cuda.synchronize()
        err = int(self.err_dev.item())
        if not err:
            return
        self.err_dev.zero_()
        if err & _lib.ERRBIT_ZEROPROB:
            raise ValueError("inclusion probability is zero for a cached draw")   # sampling.py:255-256
        if err & _lib.ERRBIT_CAPACITY:
            raise _lib.InvariantError("neighbour selection did not converge (capacity)")
        if err & _lib.ERRBIT_ZEROQ:
            raise _lib.InvariantError("sampled an edge with zero estimated inclusion")   # sampling.py:248-249
