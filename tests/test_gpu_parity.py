"""GPU parity: libgns.so kernels vs the reference's golden outputs and the oracle.

Bit-exact for ids, offsets, relabel maps, float64 weights, cached CSR and the
float64 SpMM; statistical tests for the draws; tolerance-stated for training.
"""

import os

import numpy as np
import pytest
import torch

from oracle import detmath, philox
from oracle import gns as O
from oracle import model as OM

pytestmark = pytest.mark.gpu

FIELDS = ("dst_nodes", "src_nodes", "edge_src", "edge_dst", "edge_weight", "edge_cached", "dst_degree")


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2106_06150_b200 as P
    return P


def _golden_graph(P, gold):
    n = len(gold["indptr"]) - 1
    og = O.OGraph(num_nodes=n, indptr=gold["indptr"], indices=gold["indices"])
    return og, P.Graph.from_numpy(n, gold["indptr"], gold["indices"])


def assert_mb_equal(mb_gpu, mb_ref, tag=""):
    assert len(mb_gpu.blocks) == len(mb_ref.blocks), tag
    for i, (bg, br) in enumerate(zip(mb_gpu.blocks, mb_ref.blocks)):
        h = bg.to_numpy()
        for f in FIELDS:
            a, b = getattr(h, f), np.asarray(getattr(br, f))
            assert a.shape == b.shape, (tag, i, f, a.shape, b.shape)
            assert np.array_equal(a, b), (tag, i, f)
        # relabel map: self_pos = searchsorted(src_nodes, dst_nodes) (model.py:137)
        sp = np.searchsorted(h.src_nodes, h.dst_nodes)
        assert np.array_equal(bg.self_pos.cpu().numpy(), sp), (tag, i, "self_pos")
        assert np.array_equal(bg.edge_node.cpu().numpy(), h.src_nodes[h.edge_src]), (tag, i, "edge_node")


# ---- cache engine -----------------------------------------------------------------

def test_degree_probs_bit_exact(P, golden):
    gold = golden["sampler"]
    og, g = _golden_graph(P, gold)
    probs = P.degree_probs(g)
    assert np.array_equal(probs.weights.cpu().numpy(), O.degree_probs(og))
    assert np.array_equal(probs.weights.cpu().numpy(), gold["probs"])


def test_cache_draw_matches_oracle(P, golden):
    gold = golden["sampler"]
    og, g = _golden_graph(P, gold)
    probs = P.degree_probs(g)
    ns = P.sample_cache(probs, 40, [0, 33, 0])
    assert np.array_equal(ns.ids.cpu().numpy(), gold["philox_cache_ids"])
    mask = ns.mask.cpu().numpy()
    assert np.array_equal(np.flatnonzero(mask), gold["philox_cache_ids"])
    w = O.degree_probs(og)
    for cs, (seed, epoch) in [(1, (3, 0)), (7, (0, 9)), (500, (1, 1)), (1999, (2, 2))]:
        got = P.sample_cache(probs, cs, [seed, 33, epoch]).ids.cpu().numpy()
        assert np.array_equal(got, O.sample_cache(w, cs, seed=seed, epoch=epoch)), cs


def test_cache_draw_edge_cases(P):
    # empty draw, saturation returns exactly the positive support
    w = torch.tensor([0.0, 0.5, 0.25, 0.0, 0.25], dtype=torch.float64, device="cuda")
    pv = P.ProbVector(w, normalized=True)
    assert P.sample_cache(pv, 0, 0).ids.numel() == 0
    assert P.sample_cache(pv, 3, 0).ids.tolist() == [1, 2, 4]
    assert P.sample_cache(pv, 10, 0).ids.tolist() == [1, 2, 4]
    # ties: uniform weights -> identical p; (key, id) order decides
    n = 100_003
    wu = np.full(n, 1.0 / n)
    pu = P.ProbVector(torch.as_tensor(wu, device="cuda"), normalized=True)
    got = P.sample_cache(pu, 12_345, [5, 33, 2]).ids.cpu().numpy()
    assert np.array_equal(got, O.sample_cache(wu, 12_345, seed=5, epoch=2))


def test_inclusion_bit_exact(P, golden):
    kat = golden["kat"]
    rng = np.random.default_rng(3)
    p = np.concatenate([10.0 ** -rng.uniform(0, 12, 20000), [0.0, 1.0, 0.5, 0.999999999999999]])
    for cs in (0, 1, 100, 111_000, 1_110_000):
        got = P.inclusion_prob(p, cs)
        assert np.array_equal(got, detmath.inclusion_prob(p, cs)), cs
    assert abs(P.inclusion_prob(0.01, 100) - 0.63397) < 1e-5
    for cs in (1, 100, 111000):
        ref = kat[f"incl_ref_{cs}"]
        got = P.inclusion_prob(kat["incl_p"], cs)
        assert np.max(np.abs(got - ref) / np.spacing(np.maximum(np.abs(ref), 1e-300))) <= 4


def test_build_cache_matches_reference(P, golden):
    gold = golden["sampler"]
    og, g = _golden_graph(P, gold)
    cache = P.build_cache(g, P.degree_probs(g), 40, epoch=0, rng_seed=[0, 33, 0])
    assert np.array_equal(cache.nodes.ids.cpu().numpy(), gold["philox_cache_ids"])
    assert np.array_equal(cache.cached_indptr.cpu().numpy(), gold["cached_indptr"])
    assert np.array_equal(cache.cached_indices.cpu().numpy(), gold["cached_indices"])
    oc = O.build_cache(og, O.degree_probs(og), 40, ids=gold["philox_cache_ids"])
    assert np.array_equal(cache.inclusion.cpu().numpy(), oc.inclusion)
    ref = gold["cache_inclusion_ref"]
    inc = cache.inclusion.cpu().numpy()
    assert np.max(np.abs(inc - ref) / np.spacing(np.maximum(np.abs(ref), 1e-300))) <= 4


def test_build_cache_full_and_empty(P):
    # C = V -> cached CSR equals the full CSR; C = {} -> empty rows
    og = O.build_csr(np.random.default_rng(0).integers(0, 300, size=(1500, 2)), 300)
    g = P.Graph.from_numpy(300, og.indptr, og.indices)
    probs = P.degree_probs(g)
    full = P.build_cache(g, probs, 300)
    support = np.flatnonzero(np.diff(og.indptr) > 0)
    assert np.array_equal(full.nodes.ids.cpu().numpy(), support)
    assert np.array_equal(full.cached_indptr.cpu().numpy(), og.indptr)
    assert np.array_equal(full.cached_indices.cpu().numpy(), og.indices)
    inc = full.inclusion.cpu().numpy()
    assert np.all(inc[support] == 1.0)
    empty = P.build_cache(g, probs, 0)
    assert len(empty) == 0 and int(empty.cached_indptr[-1]) == 0


# ---- sampler --------------------------------------------------------------------

CASES = {"gns": dict(strategy="GNS", fanouts=(15, 10, 5), input_layer_cache_only=True, seed=0),
         "gnsfill": dict(strategy="GNS", fanouts=(6, 4), input_layer_cache_only=False, seed=3),
         "ns": dict(strategy="NS", fanouts=(15, 10, 5), input_layer_cache_only=True, seed=0)}


def test_minibatch_bit_exact_vs_reference_golden(P, golden):
    """The reference's own outputs (Philox keys replayed into gnsbench)."""
    gold = golden["sampler"]
    og, g = _golden_graph(P, gold)
    cache = P.build_cache(g, P.degree_probs(g), 40, epoch=0, rng_seed=[0, 33, 0])
    for name, kw in CASES.items():
        cfg = P.SamplerConfig(batch_size=64, cache_mode="degree", **kw)
        for epoch, index in ((0, 0), (2, 5)):
            mb = P.build_minibatch(g, cache if cfg.strategy == "GNS" else None,
                                   gold[f"{name}_targets"], cfg, P.BatchRng(cfg.seed, epoch, index))
            pre = f"{name}_e{epoch}_i{index}"

            class R:
                pass
            ref = R()
            ref.blocks = []
            for i in range(int(gold[f"{pre}_nblocks"])):
                b = R()
                for f in FIELDS:
                    setattr(b, f, gold[f"{pre}_b{i}_{f}"])
                ref.blocks.append(b)
            assert_mb_equal(mb, ref, pre)
            P.validate_minibatch(g, mb)


def _hub_graph(n=6000, seed=0):
    """Power-law-ish graph with hub rows > 2048 (exercises the CTA-per-row path)."""
    rng = np.random.default_rng(seed)
    hubs = np.arange(8)
    e1 = np.stack([rng.choice(hubs, 30000), rng.integers(0, n, 30000)], 1)
    e2 = rng.integers(0, n, size=(40000, 2))
    return O.build_csr(np.concatenate([e1, e2]), n)


@pytest.mark.parametrize("strategy,cache_only,frac", [("GNS", True, 0.02), ("GNS", False, 0.02),
                                                      ("GNS", False, 0.3), ("NS", False, 0.0)])
def test_minibatch_bit_exact_vs_oracle_hubs(P, strategy, cache_only, frac):
    og = _hub_graph()
    assert np.diff(og.indptr).max() > 2048
    g = P.Graph.from_numpy(og.num_nodes, og.indptr, og.indices)
    cfg = P.SamplerConfig(strategy=strategy, fanouts=(15, 10, 5), batch_size=500,
                          input_layer_cache_only=cache_only, cache_mode="degree",
                          cache_frac=max(frac, 0.01), seed=11)
    cache = oc = None
    if strategy == "GNS":
        cs = O.cache_size_for(og, frac)
        cache = P.build_cache(g, P.degree_probs(g), cs, rng_seed=[11, 33, 1])
        oc = O.build_cache(og, O.degree_probs(og), cs, seed=11, epoch=1)
        assert np.array_equal(cache.nodes.ids.cpu().numpy(), oc.ids)
        assert np.array_equal(cache.cached_indptr.cpu().numpy(), oc.cached_indptr)
        assert np.array_equal(cache.cached_indices.cpu().numpy(), oc.cached_indices)
        assert np.array_equal(cache.inclusion.cpu().numpy(), oc.inclusion)
    targets = np.concatenate([np.arange(8), np.random.default_rng(1).choice(og.num_nodes, 480, replace=False)])
    for index in range(3):
        mb = P.build_minibatch(g, cache, targets, cfg, P.BatchRng(11, 1, index))
        ref = O.build_minibatch(og, oc, targets, cfg, O.PhiloxKeys(11, 1, index))
        assert_mb_equal(mb, ref, f"{strategy}-{cache_only}-{index}")


def _mid_hub_graph(n=5000, seed=17):
    """_hub_graph plus 150 rows of degree ~130-1900 (long warp-tier rows)."""
    rng = np.random.default_rng(seed)
    base = _hub_graph(n, seed)
    src = np.repeat(np.arange(8, 8 + 150), rng.integers(65, 950, 150))
    e3 = np.stack([src, rng.integers(0, n, src.size)], 1)
    rows = np.repeat(np.arange(n), np.diff(base.indptr))
    return O.build_csr(np.concatenate([np.stack([rows, base.indices], 1), e3]), n)


@pytest.mark.parametrize("tune", [{"thread_len": 16, "stream_len": 0}, {"thread_len": 16, "stream_len": 32},
                                  {"thread_len": 0, "stream_len": 64}, {"sampler_ctas": 1},
                                  {"warp_sort": 0}, {"stream_len": 0, "count_items": 1},
                                  {"count_items": 2, "stream_minb": 4}, {"stream_k5": 0}])
def test_minibatch_selection_tiers_all_exact(P, tune):
    """Every routing of (row, phase) items over the selection tiers (sorting
    network, streaming top-k, warp, CTA) gives the reference's blocks."""
    from paper_2106_06150_b200 import _lib
    og = _mid_hub_graph(5000, 17)
    g = P.Graph.from_numpy(og.num_nodes, og.indptr, og.indices)
    cfg = P.SamplerConfig(strategy="GNS", fanouts=(15, 10, 5), batch_size=400, input_layer_cache_only=False,
                          cache_mode="degree", cache_frac=0.05, seed=3)
    cs = O.cache_size_for(og, cfg.cache_frac)
    cache = P.build_cache(g, P.degree_probs(g), cs, rng_seed=[3, 33, 0])
    oc = O.build_cache(og, O.degree_probs(og), cs, seed=3, epoch=0)
    targets = np.random.default_rng(2).choice(og.num_nodes, 400, replace=False)
    defaults = {"thread_len": 0, "stream_len": 32, "sampler_ctas": 0, "warp_sort": 1, "count_items": 4,
                "stream_minb": 1, "stream_k5": 1}
    try:
        for k, v in tune.items():
            _lib.call("gns_tune", k.encode(), v)
        for index in range(2):
            mb = P.build_minibatch(g, cache, targets, cfg, P.BatchRng(3, 0, index))
            ref = O.build_minibatch(og, oc, targets, cfg, O.PhiloxKeys(3, 0, index))
            assert_mb_equal(mb, ref, f"{tune}-{index}")
    finally:
        for k, v in defaults.items():
            _lib.call("gns_tune", k.encode(), v)


def test_minibatch_layers_with_large_capacities(P):
    """Layers whose capacities differ by > 32K rows share one sampler
    workspace: consecutive batches through the same MiniBatchSampler stay
    bit-exact (regression: the count pass's tile sums once overlapped the
    dedup bitmap of a smaller layer's layout)."""
    n = 60_000
    rng = np.random.default_rng(11)
    og = O.build_csr(rng.integers(0, n, size=(600_000, 2)), n)
    g = P.Graph.from_numpy(n, og.indptr, og.indices)
    cfg = P.SamplerConfig(strategy="GNS", fanouts=(15, 10, 5), batch_size=1000, cache_mode="degree",
                          cache_frac=0.01, seed=6)
    cs = O.cache_size_for(og, cfg.cache_frac)
    cache = P.build_cache(g, P.degree_probs(g), cs, rng_seed=[6, 33, 0])
    oc = O.build_cache(og, O.degree_probs(og), cs, seed=6, epoch=0)
    from paper_2106_06150_b200.sampling import MiniBatchSampler
    eng = MiniBatchSampler(g, cfg)
    assert eng.layers[-1].max_dst > 32 * 1024
    for b in range(3):
        targets = rng.choice(n, 1000, replace=False)
        mb = eng.sample(targets, P.BatchRng(6, 0, b), cache)
        ref = O.build_minibatch(og, oc, targets, cfg, O.PhiloxKeys(6, 0, b))
        assert_mb_equal(mb, ref, f"batch {b}")


def test_single_layer_entry_points(P):
    og = _hub_graph(2000, 3)
    g = P.Graph.from_numpy(og.num_nodes, og.indptr, og.indices)
    seeds = np.array([5, 3, 3, 1999, 0, 7, 100])
    b = P.sample_neighbors_uniform(g, seeds, 4, P.BatchRng(1, 2, 3, layer=2))
    r = O.sample_neighbors_uniform(og, seeds, 4, O.PhiloxKeys(1, 2, 3), layer=2)
    for f in FIELDS:
        assert np.array_equal(getattr(b.to_numpy(), f), getattr(r, f)), f
    cache = P.build_cache(g, P.degree_probs(g), 50, rng_seed=[1, 33, 0])
    oc = O.build_cache(og, O.degree_probs(og), 50, seed=1, epoch=0)
    for co in (True, False):
        b = P.sample_neighbors_gns(g, cache, seeds, 6, co, P.BatchRng(1, 2, 3, layer=1))
        r = O.sample_neighbors_gns(og, oc, seeds, 6, co, O.PhiloxKeys(1, 2, 3), layer=1)
        for f in FIELDS:
            assert np.array_equal(getattr(b.to_numpy(), f), getattr(r, f)), (co, f)
    with pytest.raises(ValueError):
        P.sample_neighbors_uniform(g, seeds, 0, P.BatchRng())
    with pytest.raises(TypeError):       # no .integers: not an rng
        P.sample_neighbors_uniform(g, seeds, 3, object())


def test_zero_degree_and_repeated_targets(P):
    # d = 0 -> no sampled edges, src contains only the seed
    og = O.build_csr([(0, 1), (1, 2)], 6)
    g = P.Graph.from_numpy(6, og.indptr, og.indices)
    cfg = P.SamplerConfig(strategy="NS", fanouts=(3, 2), batch_size=8)
    mb = P.build_minibatch(g, None, [5, 4, 4, 0, 5], cfg, P.BatchRng(0, 0, 0))
    ref = O.build_minibatch(og, None, [5, 4, 4, 0, 5], cfg, O.PhiloxKeys(0, 0, 0))
    assert_mb_equal(mb, ref, "zero-degree")
    assert mb.targets.tolist() == [0, 4, 5]


@pytest.mark.parametrize("n", [0, 1, 7, 1000, 4096, 4097, 50000])
def test_unique_sorted_both_paths(P, n):
    """np.unique (sampling.py:208,312): the single-CTA sort path (n <= 4096)
    and the bitmap path, with repeats and ids up to N-1."""
    from paper_2106_06150_b200 import _lib
    N = 200_000
    rng = np.random.default_rng(n)
    ids = rng.integers(0, N, n).astype(np.int32)
    if n > 2:
        ids[: n // 3] = ids[n // 3: 2 * (n // 3)]   # repeats
        ids[-1] = N - 1
    d_ids = torch.as_tensor(ids, device="cuda") if n else torch.zeros(1, dtype=torch.int32, device="cuda")
    out = torch.full((max(n, 1),), -1, dtype=torch.int32, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
    ws = _lib.workspace(_lib.lib().gns_relabel_workspace_size(N), "cuda", zero=True)
    for n_dev in (None, torch.tensor([n], dtype=torch.int32, device="cuda")):
        _lib.call("gns_unique_sorted", N, d_ids.data_ptr(), None if n_dev is None else n_dev.data_ptr(), n,
                  out.data_ptr(), cnt.data_ptr(), ws.data_ptr(), ws.numel(), _lib.stream_ptr())
        u = np.unique(ids)
        assert int(cnt) == len(u)
        assert np.array_equal(out[:len(u)].cpu().numpy(), u)
    # both bitmap levels are left zeroed (dedup_ws layout: bits, then summary)
    r256 = lambda b: (b + 255) // 256 * 256  # noqa: E731
    nw = (N + 31) // 32
    nbytes = r256((nw + 1) * 4) + r256(((nw + 31) // 32 + 1) * 4)
    assert int(ws[:nbytes].count_nonzero()) == 0


@pytest.mark.parametrize("tma", [2, 0])
@pytest.mark.parametrize("dim,rows", [(4, 1), (64, 33), (100, 1001), (128, 4099), (256, 4098), (768, 517)])
def test_gather_rows_shapes(P, dim, rows, tma):
    """gns_gather_rows over tile tails and row widths (16-B chunks per row
    from 1 to 192), device row count, output stride > dim and == dim; tma=2
    takes the TMA gather4 path for every float32 D <= 256, tma=0 the register
    kernel."""
    from paper_2106_06150_b200 import _lib
    N = 5000
    tab = torch.randn(N, dim, device="cuda")
    idx = torch.sort(torch.randint(0, N, (rows,), device="cuda", dtype=torch.int32)).values
    n_dev = torch.tensor([rows], dtype=torch.int32, device="cuda")
    try:
        _lib.call("gns_tune", b"gather_tma", tma)
        for pad in (4, 0):
            out = torch.full((rows + 3, dim + pad), 7.0, device="cuda")
            _lib.call("gns_gather_rows", tab.data_ptr(), tab.stride(0), 0, idx.data_ptr(), n_dev.data_ptr(),
                      rows + 3, dim, out.data_ptr(), out.stride(0), 0, _lib.stream_ptr())
            assert torch.equal(out[:rows, :dim], tab[idx.long()]), pad
            assert bool((out[rows:] == 7.0).all()) and bool((out[:, dim:] == 7.0).all()), pad
        # rows read from a strided table view (row pitch > dim)
        wide = torch.randn(N, dim + 8, device="cuda")
        out = torch.full((rows, dim), 7.0, device="cuda")
        _lib.call("gns_gather_rows", wide.data_ptr(), wide.stride(0), 0, idx.data_ptr(), n_dev.data_ptr(), rows,
                  dim, out.data_ptr(), out.stride(0), 0, _lib.stream_ptr())
        assert torch.equal(out, wide[idx.long(), :dim])
    finally:
        _lib.call("gns_tune", b"gather_tma", 1)


def test_epoch_targets_feistel(P):
    og = O.build_csr(np.random.default_rng(0).integers(0, 5000, size=(20000, 2)), 5000)
    mask = np.random.default_rng(1).random(5000) < 0.3
    g = P.Graph.from_numpy(5000, og.indptr, og.indices, train_mask=mask)
    og.train_mask = mask
    cfg = P.SamplerConfig(strategy="NS", batch_size=97, seed=4)
    got = [t.cpu().numpy() for t in P.epoch_targets(g, cfg, 3)]
    ref = O.epoch_targets(og, 97, 4, 3)
    assert len(got) == len(ref)
    for a, b in zip(got, ref):
        assert np.array_equal(a, b)
    allv = np.concatenate(got)
    assert np.array_equal(np.sort(allv), np.flatnonzero(mask))


@pytest.mark.parametrize("nbytes", [4, 32, 4000, 4 * 1000 + 3, 1 << 20])
def test_copy_mapped_host_device(P, nbytes):
    """gns_copy_mapped moves bytes pinned host -> device and device -> pinned
    host (UVA), including a ragged tail and multi-CTA sizes, and re-reads
    the host source on every launch (the step graph's per-replay inputs)."""
    from paper_2106_06150_b200 import _lib
    src = torch.randint(0, 256, (nbytes,), dtype=torch.uint8).pin_memory()
    dev = torch.zeros(nbytes + 4, dtype=torch.uint8, device="cuda")
    _lib.call("gns_copy_mapped", dev.data_ptr(), src.data_ptr(), nbytes, _lib.stream_ptr())
    torch.cuda.synchronize()
    assert torch.equal(dev[:nbytes].cpu(), src) and int(dev[nbytes:].sum()) == 0
    src.fill_(7)   # host rewrites between launches
    _lib.call("gns_copy_mapped", dev.data_ptr(), src.data_ptr(), nbytes, _lib.stream_ptr())
    back = torch.zeros(nbytes, dtype=torch.uint8).pin_memory()
    _lib.call("gns_copy_mapped", back.data_ptr(), dev.data_ptr(), nbytes, _lib.stream_ptr())
    torch.cuda.synchronize()
    assert bool((back == 7).all())


@pytest.mark.parametrize("batch", [97, 1000, 1024])
def test_batch_targets_sorted_matches_epoch_slice(P, batch):
    """gns_batch_targets_sorted (Feistel epoch slice + np.unique in one CTA)
    = np.unique of the reference's epoch batch (pool.py:60-66), every batch of
    an epoch including the short last one."""
    from paper_2106_06150_b200 import _lib
    n = 7000
    og = O.build_csr(np.random.default_rng(0).integers(0, n, size=(20000, 2)), n)
    mask = np.random.default_rng(2).random(n) < 0.4
    og.train_mask = mask
    g = P.Graph.from_numpy(n, og.indptr, og.indices, train_mask=mask)
    seed, epoch = 6, 2
    ref = O.epoch_targets(og, batch, seed, epoch)
    tid = g.train_ids()
    out = torch.empty(batch, dtype=torch.int32, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
    for k, r in enumerate(ref):
        step = torch.tensor([(seed & 0xFFFFFFFF) | (epoch << 32), k, k * batch, batch], dtype=torch.int64,
                            device="cuda")
        _lib.call("gns_batch_targets_sorted", tid.data_ptr(), tid.numel(), step.data_ptr(), batch, out.data_ptr(),
                  cnt.data_ptr(), _lib.stream_ptr())
        m = int(cnt)
        assert np.array_equal(out[:m].cpu().numpy(), np.unique(r)), k
    # the engine's variant: slice of the epoch permutation computed up front
    perm = torch.empty_like(tid)
    _lib.call("gns_epoch_targets", tid.data_ptr(), tid.numel(), seed, epoch, 0, tid.numel(), perm.data_ptr(),
              _lib.stream_ptr())
    for k, r in enumerate(ref):
        step = torch.tensor([(seed & 0xFFFFFFFF) | (epoch << 32), k, k * batch, batch], dtype=torch.int64,
                            device="cuda")
        out.fill_(-1)
        _lib.call("gns_batch_slice_sorted", perm.data_ptr(), perm.numel(), step.data_ptr(), None, batch,
                  out.data_ptr(), cnt.data_ptr(), _lib.stream_ptr())
        m = int(cnt)
        assert np.array_equal(out[:m].cpu().numpy(), np.unique(r)), k
        # step struct fetched from pinned host memory and published on the device
        hstep, dstep = step.cpu().pin_memory(), torch.zeros_like(step)
        out.fill_(-1)
        _lib.call("gns_batch_slice_sorted", perm.data_ptr(), perm.numel(), hstep.data_ptr(), dstep.data_ptr(),
                  batch, out.data_ptr(), cnt.data_ptr(), _lib.stream_ptr())
        assert torch.equal(dstep, step)
        assert np.array_equal(out[:int(cnt)].cpu().numpy(), np.unique(r)), k


def test_pool_deterministic_and_complete(P):
    og = _hub_graph(3000, 5)
    mask = np.random.default_rng(2).random(3000) < 0.5
    g = P.Graph.from_numpy(3000, og.indptr, og.indices, train_mask=mask)
    cfg = P.SamplerConfig(strategy="GNS", fanouts=(10, 5), batch_size=128, cache_mode="degree", seed=2,
                          cache_frac=0.05)

    def run(workers):
        pool = P.SamplerPool(g, cfg, num_workers=workers)
        out = []
        for epoch in range(2):
            for it in pool.iter_epoch(epoch):
                out.append((it.epoch, it.index, [b.to_numpy() for b in it.minibatch.blocks],
                            it.minibatch.targets.cpu().numpy().copy()))
                assert it.sample_ms >= 0
        return out

    a, b = run(1), run(3)
    assert [x[:2] for x in a] == [x[:2] for x in b]
    for x, y in zip(a, b):
        for bx, by in zip(x[2], y[2]):
            for f in FIELDS:
                assert np.array_equal(getattr(bx, f), getattr(by, f))
    targets = np.concatenate([x[3] for x in a if x[0] == 0])
    assert np.array_equal(np.sort(targets), np.flatnonzero(mask))


# ---- gather / SpMM ---------------------------------------------------------------

def _mb_and_features(P, dim=24, strategy="GNS"):
    og = _hub_graph(4000, 9)
    feats = np.random.default_rng(0).normal(size=(og.num_nodes, dim)).astype(np.float32)
    g = P.Graph.from_numpy(og.num_nodes, og.indptr, og.indices, features=feats)
    cfg = P.SamplerConfig(strategy=strategy, fanouts=(8, 5, 3), batch_size=300, cache_mode="degree",
                          input_layer_cache_only=False, seed=1)
    cache = P.build_cache(g, P.degree_probs(g), 200, rng_seed=[1, 33, 0]) if strategy == "GNS" else None
    oc = O.build_cache(og, O.degree_probs(og), 200, seed=1, epoch=0) if strategy == "GNS" else None
    targets = np.random.default_rng(4).choice(og.num_nodes, 300, replace=False)
    mb = P.build_minibatch(g, cache, targets, cfg, P.BatchRng(1, 0, 0))
    ref = O.build_minibatch(og, oc, targets, cfg, O.PhiloxKeys(1, 0, 0))
    return og, g, feats, mb, ref


def test_gather_rows_exact(P):
    og, g, feats, mb, ref = _mb_and_features(P, dim=24)
    model = P.GraphSAGE((24, 8, 3))
    h = model.gather_inputs(mb, g)
    assert torch.equal(h.cpu(), torch.as_tensor(feats[ref.input_nodes]))
    m64 = P.GraphSAGE((24, 8, 3), dtype=torch.float64)
    h64 = m64.gather_inputs(mb, g)
    assert np.array_equal(h64.cpu().numpy(), feats[ref.input_nodes].astype(np.float64))


@pytest.mark.parametrize("dim", [2, 6, 64, 130])
def test_spmm_fwd_f64_bit_exact(P, dim):
    from paper_2106_06150_b200 import _lib
    og, g, feats, mb, ref = _mb_and_features(P, dim=16)
    for li, (bg, br) in enumerate(zip(mb.blocks, ref.blocks)):
        nsrc, ndst = len(br.src_nodes), len(br.dst_nodes)
        h = np.random.default_rng(li).normal(size=(nsrc, dim))
        ht = torch.as_tensor(h, device="cuda")
        cat = torch.full((ndst + 3, 2 * dim), 7.0, dtype=torch.float64, device="cuda")
        _lib.call("gns_spmm_fwd", 1, ht.data_ptr(), dim, dim, 0, bg._c, ndst, ndst + 3, cat.data_ptr(),
                  2 * dim, _lib.stream_ptr())
        agg = OM.spmm_mean_fwd(br, h)
        self_pos = np.searchsorted(br.src_nodes, br.dst_nodes)
        c = cat.cpu().numpy()
        assert np.all(c[ndst:] == 0)        # static-capacity zero padding
        c = c[:ndst]
        assert np.array_equal(c[:, :dim], h[self_pos])
        assert np.array_equal(c[:, dim:], agg), li
        # float32 production path: same order, FMA; tolerance 1e-5 relative-to-scale
        h32 = torch.as_tensor(h.astype(np.float32), device="cuda")
        if dim % 4 == 0:
            cat32 = torch.empty((ndst, 2 * dim), dtype=torch.float32, device="cuda")
            _lib.call("gns_spmm_fwd", 0, h32.data_ptr(), dim, dim, 0, bg._c, ndst, 0, cat32.data_ptr(), 2 * dim,
                      _lib.stream_ptr())
            np.testing.assert_allclose(cat32.cpu().numpy()[:, dim:], agg, rtol=1e-5, atol=1e-5)
            # relu-on-load variant == spmm of relu(h)
            _lib.call("gns_spmm_fwd", 1, ht.data_ptr(), dim, dim, 1, bg._c, ndst, 0, cat.data_ptr(), 2 * dim,
                      _lib.stream_ptr())
            hr = np.maximum(h, 0.0)
            c = cat.cpu().numpy()[:ndst]
            assert np.array_equal(c[:, :dim], hr[self_pos])
            assert np.array_equal(c[:, dim:], OM.spmm_mean_fwd(br, hr))


@pytest.mark.parametrize("dim", [200, 768])
def test_spmm_fwd_gather_wide_rows_long_lists(P, dim):
    """Wide-row input layer (column-split warp tasks) with rows of > 32 edges
    (ranked window by window): bit-identical to gather then aggregate."""
    from paper_2106_06150_b200 import _lib
    og = _hub_graph(4000, 29)
    g = P.Graph.from_numpy(og.num_nodes, og.indptr, og.indices)
    cfg = P.SamplerConfig(strategy="NS", fanouts=(70, 3), batch_size=200, seed=8)
    targets = np.random.default_rng(8).choice(og.num_nodes, 200, replace=False)
    mb = P.build_minibatch(g, None, targets, cfg, P.BatchRng(8, 0, 0))
    feats = torch.randn(og.num_nodes, dim, device="cuda")
    for bg in mb.blocks:
        nd = bg.dst_nodes.numel()
        h = feats[bg.src_nodes.long()].contiguous()
        a = torch.full((nd + 3, 2 * dim), 7.0, device="cuda")
        b = torch.full((nd + 3, 2 * dim), 9.0, device="cuda")
        _lib.call("gns_spmm_fwd", 0, h.data_ptr(), dim, dim, 0, bg._c, nd, nd + 3, a.data_ptr(), 2 * dim,
                  _lib.stream_ptr())
        dst = bg.dst_nodes.int().contiguous()
        _lib.call("gns_spmm_fwd_gather", feats.data_ptr(), dim, dim, bg._c, dst.data_ptr(), nd, nd + 3, 0, 0,
                  b.data_ptr(), 2 * dim, _lib.stream_ptr())
        assert torch.equal(a, b)


@pytest.mark.parametrize("dim", [4, 64, 128, 200, 768, 1024])
def test_spmm_fwd_gather_equals_gather_then_spmm(P, dim):
    """The fused input-layer kernel (feature table addressed by node id) is
    bit-identical to features[input_nodes] (model.py:146) followed by the
    aggregation (model.py:153)."""
    from paper_2106_06150_b200 import _lib
    og, g, _, mb, ref = _mb_and_features(P, dim=16)
    feats = torch.randn(og.num_nodes, dim, device="cuda")
    for li, (bg, br) in enumerate(zip(mb.blocks, ref.blocks)):
        nsrc, ndst = len(br.src_nodes), len(br.dst_nodes)
        h = feats[torch.as_tensor(br.src_nodes, device="cuda").long()].contiguous()
        a = torch.full((ndst + 5, 2 * dim), 7.0, device="cuda")
        b = torch.full((ndst + 5, 2 * dim), 9.0, device="cuda")
        _lib.call("gns_spmm_fwd", 0, h.data_ptr(), dim, dim, 0, bg._c, ndst, ndst + 5, a.data_ptr(), 2 * dim,
                  _lib.stream_ptr())
        dst = torch.as_tensor(br.dst_nodes.astype(np.int32), device="cuda")
        _lib.call("gns_spmm_fwd_gather", feats.data_ptr(), dim, dim, bg._c, dst.data_ptr(), ndst, ndst + 5, 0, 0,
                  b.data_ptr(), 2 * dim, _lib.stream_ptr())
        assert torch.equal(a, b), li
        # chunk-bounded zero padding: rows [n, ceil(n/8)*8) zeroed, the rest untouched
        c = torch.full((ndst + 40, 2 * dim), 9.0, device="cuda")
        _lib.call("gns_spmm_fwd_gather", feats.data_ptr(), dim, dim, bg._c, dst.data_ptr(), ndst, ndst + 40, 8, 0,
                  c.data_ptr(), 2 * dim, _lib.stream_ptr())
        end = min(-(-ndst // 8) * 8, ndst + 40)
        assert torch.equal(c[:ndst], a[:ndst])
        assert bool((c[ndst:end] == 0).all()) and bool((c[end:] == 9.0).all())
        # the fanout hint does not change the result
        if dim == 128 and bg.fanout <= 5:
            d = torch.full((ndst + 40, 2 * dim), 9.0, device="cuda")
            _lib.call("gns_spmm_fwd_gather", feats.data_ptr(), dim, dim, bg._c, dst.data_ptr(), ndst, ndst + 40, 8,
                      bg.fanout, d.data_ptr(), 2 * dim, _lib.stream_ptr())
            assert torch.equal(c, d), li


@pytest.mark.parametrize("dim", [16, 64, 128])
@pytest.mark.parametrize("fanouts", [(5, 3), (40, 3)])
def test_spmm_fwd_gather_chunk_kernel_variants(P, dim, fanouts):
    """The chunk-staged input-layer kernel (32 rows' metadata and edges staged
    in shared memory, per-row register sort, all feature rows in flight; its
    per-row fallback for rows with > 6 edges and overflowing chunks, forced
    here by a fanout hint of 5 on blocks with up to 40 edges per row) is
    bit-identical to the per-row narrow kernel and the generic kernel, every
    variant, padding included."""
    from paper_2106_06150_b200 import _lib
    og = _hub_graph(4000, 19)
    g = P.Graph.from_numpy(og.num_nodes, og.indptr, og.indices)
    cfg = P.SamplerConfig(strategy="NS", fanouts=fanouts, batch_size=300, seed=2)
    targets = np.random.default_rng(2).choice(og.num_nodes, 300, replace=False)
    mb = P.build_minibatch(g, None, targets, cfg, P.BatchRng(2, 0, 0))
    feats = torch.randn(og.num_nodes, dim, device="cuda")
    try:
        for bg in mb.blocks:
            nd = bg.dst_nodes.numel()
            dst = bg.dst_nodes.to(torch.int32).contiguous()
            outs = []
            for v in (0, 1, 2, 3, 4, 5):
                _lib.call("gns_tune", b"spmm_narrow", v)
                o = torch.full((nd + 37, 2 * dim), 5.0, device="cuda")
                _lib.call("gns_spmm_fwd_gather", feats.data_ptr(), dim, dim, bg._c, dst.data_ptr(), nd, nd + 37, 8, 5,
                          o.data_ptr(), 2 * dim, _lib.stream_ptr())
                outs.append(o)
            for v in range(1, len(outs)):
                assert torch.equal(outs[0], outs[v]), v
    finally:
        _lib.call("gns_tune", b"spmm_narrow", 2)


@pytest.mark.parametrize("dim", [132, 256, 512])
def test_spmm_fwd_wide_equals_generic(P, dim):
    """Hidden-layer forward with relu' bits: the wide kernel (lane-held edges,
    shuffle ranks; rows with > 32 edges ranked window by window) equals the
    generic kernel bit for bit, cat and bits."""
    from paper_2106_06150_b200 import _lib
    og = _hub_graph(4000, 29)
    g = P.Graph.from_numpy(og.num_nodes, og.indptr, og.indices)
    cfg = P.SamplerConfig(strategy="NS", fanouts=(70, 3), batch_size=200, seed=8)
    targets = np.random.default_rng(8).choice(og.num_nodes, 200, replace=False)
    mb = P.build_minibatch(g, None, targets, cfg, P.BatchRng(8, 0, 0))
    lib = _lib.lib()
    try:
        for bg in mb.blocks:
            ns, nd = bg.src_nodes.numel(), bg.dst_nodes.numel()
            h = torch.randn(ns, dim, device="cuda")
            res = []
            for v, sg in ((0, 4), (1, 4), (2, 4), (2, 8), (2, 12), (2, 16)):
                _lib.call("gns_tune", b"spmm_wide", v)
                _lib.call("gns_tune", b"split_g", sg)
                o = torch.full((nd + 3, 2 * dim), 5.0, device="cuda")
                bits = torch.zeros(lib.gns_relu_bits_size(ns, dim) // 4, dtype=torch.int32, device="cuda")
                _lib.call("gns_spmm_fwd_bits", h.data_ptr(), dim, dim, bg._c, nd, nd + 3, o.data_ptr(), 2 * dim,
                          bits.data_ptr(), _lib.stream_ptr())
                res.append((o, bits))
            for v in range(1, len(res)):
                assert torch.equal(res[0][0], res[v][0]), v
                assert torch.equal(res[0][1], res[v][1]), v
    finally:
        _lib.call("gns_tune", b"spmm_wide", 2)
        _lib.call("gns_tune", b"split_g", 4)


@pytest.mark.parametrize("dim", [16, 64, 128])
def test_spmm_fwd_narrow_equals_generic(P, dim):
    """The narrow-row kernel (shuffle sort, <= 32 edges per row; > 32 edges
    take its fallback) is bit-identical to the generic SpMM, with and without
    relu-on-load, fused gather or not."""
    from paper_2106_06150_b200 import _lib
    og = _hub_graph(4000, 21)
    g = P.Graph.from_numpy(og.num_nodes, og.indptr, og.indices)
    cfg = P.SamplerConfig(strategy="NS", fanouts=(40, 3), batch_size=200, seed=5)
    targets = np.random.default_rng(5).choice(og.num_nodes, 200, replace=False)
    mb = P.build_minibatch(g, None, targets, cfg, P.BatchRng(5, 0, 0))
    feats = torch.randn(og.num_nodes, dim, device="cuda")
    try:
        for bg in mb.blocks:
            ns, nd = bg.src_nodes.numel(), bg.dst_nodes.numel()
            h = torch.randn(ns, dim, device="cuda")
            dst = bg.dst_nodes.to(torch.int32).contiguous()
            outs = {}
            for v in (0, 1):
                _lib.call("gns_tune", b"spmm_narrow", v)
                for relu in (0, 1):
                    o = torch.full((nd + 3, 2 * dim), 5.0, device="cuda")
                    _lib.call("gns_spmm_fwd", 0, h.data_ptr(), dim, dim, relu, bg._c, nd, nd + 3, o.data_ptr(),
                              2 * dim, _lib.stream_ptr())
                    outs[(v, relu)] = o
                o = torch.full((nd + 3, 2 * dim), 5.0, device="cuda")
                _lib.call("gns_spmm_fwd_gather", feats.data_ptr(), dim, dim, bg._c, dst.data_ptr(), nd, nd + 3, 0, 0,
                          o.data_ptr(), 2 * dim, _lib.stream_ptr())
                outs[(v, "g")] = o
            for key in ((0, 1), "g"):
                k0 = (0, key) if key == "g" else (0, key[1])
                k1 = (1, key) if key == "g" else (1, key[1])
                assert torch.equal(outs[k0], outs[k1]), key
            assert torch.equal(outs[(0, 0)], outs[(1, 0)])
    finally:
        _lib.call("gns_tune", b"spmm_narrow", 2)


@pytest.mark.parametrize("dim", [2, 8, 64])
def test_spmm_bwd_f64_bit_exact(P, dim):
    from paper_2106_06150_b200 import _lib
    og, g, feats, mb, ref = _mb_and_features(P, dim=16)
    ws = _lib.workspace(1 << 24, "cuda")
    # the transpose's per-row sort paths are all covered: rows of <= 8
    # entries (per lane), 9..32 (warp ranks) and > 32 (warp bitonic)
    tlen = np.concatenate([np.bincount(br.edge_src, minlength=len(br.src_nodes)) for br in ref.blocks])
    assert tlen.max() > 32 and np.any((tlen > 8) & (tlen <= 32)) and np.any((tlen > 0) & (tlen <= 8))
    for li, (bg, br) in enumerate(zip(mb.blocks, ref.blocks)):
        nsrc, ndst = len(br.src_nodes), len(br.dst_nodes)
        dcat = np.random.default_rng(10 + li).normal(size=(ndst, 2 * dim))
        dt = torch.as_tensor(dcat, device="cuda")
        dh = torch.empty((nsrc, dim), dtype=torch.float64, device="cuda")
        dh2 = torch.full((nsrc + 5, dim), 3.0, dtype=torch.float64, device="cuda")
        _lib.call("gns_spmm_bwd", 1, dt.data_ptr(), 2 * dim, dim, bg._c, ndst, nsrc, br.num_edges, 0, None,
                  None, dh.data_ptr(), dim, ws.data_ptr(), ws.numel(), _lib.stream_ptr())
        expect = OM.spmm_mean_bwd(br, dcat, dim)
        assert np.array_equal(dh.cpu().numpy(), expect), li
        # fused epilogue: relu' mask of the previous layer + bias-gradient column sums
        zprev = np.random.default_rng(20 + li).normal(size=(nsrc, dim))
        zt = torch.as_tensor(zprev, device="cuda")
        db = torch.empty(dim, dtype=torch.float64, device="cuda")
        _lib.call("gns_spmm_bwd", 1, dt.data_ptr(), 2 * dim, dim, bg._c, ndst, nsrc, br.num_edges, nsrc + 5,
                  zt.data_ptr(), db.data_ptr(), dh2.data_ptr(), dim, ws.data_ptr(), ws.numel(), _lib.stream_ptr())
        dz = expect * (zprev > 0)
        assert np.array_equal(dh2.cpu().numpy()[:nsrc], dz)
        assert np.all(dh2.cpu().numpy()[nsrc:] == 0)
        np.testing.assert_allclose(db.cpu().numpy(), dz.sum(0), rtol=1e-12, atol=1e-12)
        if dim % 4 == 0:
            dt32 = torch.as_tensor(dcat.astype(np.float32), device="cuda")
            dh32 = torch.empty((nsrc, dim), dtype=torch.float32, device="cuda")
            _lib.call("gns_spmm_bwd", 0, dt32.data_ptr(), 2 * dim, dim, bg._c, ndst, nsrc, br.num_edges, 0, None,
                      None, dh32.data_ptr(), dim, ws.data_ptr(), ws.numel(), _lib.stream_ptr())
            np.testing.assert_allclose(dh32.cpu().numpy(), expect, rtol=1e-5, atol=1e-5)


@pytest.mark.parametrize("dim", [16, 100, 256])
def test_relu_bits_pair_equals_zmask_path(P, dim):
    """gns_spmm_fwd_bits == gns_spmm_fwd(relu) and gns_spmm_bwd_transposed_bits
    (mask from the forward's bits) == gns_spmm_bwd (mask from z), bit for bit
    (dz; the bias gradient within float32 rounding), for every variant."""
    from paper_2106_06150_b200 import _lib
    og, g, feats, mb, ref = _mb_and_features(P, dim=16)
    lib = _lib.lib()
    ws = _lib.workspace(1 << 24, "cuda")
    for li, (bg, br) in enumerate(zip(mb.blocks, ref.blocks)):
        nsrc, ndst = len(br.src_nodes), len(br.dst_nodes)
        gen = torch.Generator(device="cuda").manual_seed(30 + li)
        z = torch.randn((nsrc, dim), device="cuda", generator=gen)
        a = torch.empty((ndst + 2, 2 * dim), device="cuda")
        b = torch.empty((ndst + 2, 2 * dim), device="cuda")
        bits = torch.zeros(lib.gns_relu_bits_size(nsrc, dim) // 4, dtype=torch.int32, device="cuda")
        _lib.call("gns_spmm_fwd", 0, z.data_ptr(), dim, dim, 1, bg._c, ndst, ndst + 2, a.data_ptr(), 2 * dim,
                  _lib.stream_ptr())
        _lib.call("gns_spmm_fwd_bits", z.data_ptr(), dim, dim, bg._c, ndst, ndst + 2, b.data_ptr(), 2 * dim,
                  bits.data_ptr(), _lib.stream_ptr())
        assert torch.equal(a, b), li
        dcat = torch.randn((ndst, 2 * dim), device="cuda", generator=gen)
        d1 = torch.empty((nsrc, dim), device="cuda")
        d2 = torch.empty((nsrc, dim), device="cuda")
        db1 = torch.empty(dim, device="cuda")
        db2 = torch.empty(dim, device="cuda")
        _lib.call("gns_spmm_bwd", 0, dcat.data_ptr(), 2 * dim, dim, bg._c, ndst, nsrc, br.num_edges, 0,
                  z.data_ptr(), db1.data_ptr(), d1.data_ptr(), dim, ws.data_ptr(), ws.numel(), _lib.stream_ptr())
        # every transposed-SpMM variant (0 = per-row; 1-5 lane-staged with
        # 2-8 rows in flight): the same per-row FMA order, so dz is
        # bit-identical; the bias gradient's partial sums are grouped per
        # warp, so it is compared within float32 rounding of the fp64 sum
        try:
            for knob in range(6):
                _lib.call("gns_tune", b"spmm_bwd", knob)
                d2.fill_(float("nan"))
                _lib.call("gns_spmm_bwd_transposed_bits", dcat.data_ptr(), 2 * dim, dim, bg._c, ndst, nsrc,
                          br.num_edges, 0, bits.data_ptr(), db2.data_ptr(), d2.data_ptr(), dim, ws.data_ptr(),
                          ws.numel(), _lib.stream_ptr())
                assert torch.equal(d1, d2), (li, knob)
                ref64 = d1.double().sum(0)
                tol = 1e-5 * d1.double().abs().sum(0) + 1e-6
                assert torch.all((db2.double() - ref64).abs() <= tol), (li, knob)
                assert torch.all((db1.double() - ref64).abs() <= tol), (li, knob)
        finally:
            _lib.call("gns_tune", b"spmm_bwd", 4)


def test_full_batch_equivalence(P):
    """with k >= max degree the sampled forward equals the
    full-neighbourhood forward (NS keeps every neighbour, weight 1)."""
    og = O.build_csr(np.random.default_rng(0).integers(0, 200, size=(600, 2)), 200)
    feats = np.random.default_rng(1).normal(size=(200, 8)).astype(np.float32)
    g = P.Graph.from_numpy(200, og.indptr, og.indices, features=feats)
    kmax = int(np.diff(og.indptr).max())
    cfg = P.SamplerConfig(strategy="NS", fanouts=(kmax, kmax), batch_size=200)
    mb = P.build_minibatch(g, None, np.arange(200), cfg, P.BatchRng())
    model = P.GraphSAGE((8, 16, 4), dtype=torch.float64)
    logits = model.logits(mb, g).cpu().numpy()
    w, b = model.export()
    h = feats.astype(np.float64)
    norm = np.maximum(np.diff(og.indptr), 1).astype(np.float64)
    import scipy.sparse as sp
    adj = sp.csr_matrix((np.ones(og.num_edges), og.indices, og.indptr), shape=(200, 200))
    for li in range(2):
        agg = (adj @ h) / norm[:, None]
        z = np.concatenate([h, agg], 1) @ w[li] + b[li]
        h = np.maximum(z, 0) if li == 0 else z
    np.testing.assert_allclose(logits, h, rtol=1e-10, atol=1e-10)


# ---- training parity ------------------------------------------------------------

def test_training_loss_matches_reference_fp64(P, golden):
    """6 reference steps (golden, fp64 numpy) vs the B200 fp64 mode; tolerance
    1e-9 relative on every loss (GEMM summation order differs from BLAS)."""
    gold = golden["model"]
    n = len(gold["indptr"]) - 1
    g = P.Graph.from_numpy(n, gold["indptr"], gold["indices"], features=gold["features"],
                           labels=gold["labels"], train_mask=gold["train_mask"])
    og = O.OGraph(num_nodes=n, indptr=gold["indptr"], indices=gold["indices"], train_mask=gold["train_mask"])
    cfg = P.SamplerConfig(strategy="GNS", fanouts=(5, 3), batch_size=50, cache_frac=0.1, cache_mode="degree",
                          seed=0)
    cache = P.build_cache(g, P.degree_probs(g), 40, rng_seed=[0, 33, 0])
    assert np.array_equal(cache.nodes.ids.cpu().numpy(), gold["cache_ids"])
    model = P.GraphSAGE((16, 32, 4), dtype=torch.float64, seed=0)
    tc = P.TrainConfig(lr=0.003)
    batches = O.epoch_targets(og, 50, 0, 0)
    losses = []
    for index, targets in enumerate(batches[:6]):
        mb = P.build_minibatch(g, cache, targets, cfg, P.BatchRng(0, 0, index))
        losses.append(float(model.train_step(mb, g, tc)))
    np.testing.assert_allclose(losses, gold["losses"], rtol=1e-9)
    w, b = model.export()
    for i in range(2):
        np.testing.assert_allclose(w[i], gold[f"final_w{i}"], rtol=1e-7, atol=1e-10)
        np.testing.assert_allclose(b[i], gold[f"final_b{i}"], rtol=1e-7, atol=1e-10)


def test_training_fp32_tracks_fp64(P, golden):
    gold = golden["model"]
    n = len(gold["indptr"]) - 1
    g = P.Graph.from_numpy(n, gold["indptr"], gold["indices"], features=gold["features"],
                           labels=gold["labels"], train_mask=gold["train_mask"])
    cfg = P.SamplerConfig(strategy="GNS", fanouts=(5, 3), batch_size=50, cache_frac=0.1, cache_mode="degree",
                          seed=0)
    pool = P.SamplerPool(g, cfg, num_workers=2)
    model = P.GraphSAGE((16, 32, 4), dtype=torch.float32, seed=0)
    tc = P.TrainConfig(lr=0.003)
    losses = [float(model.train_step(it.minibatch, g, tc)) for it in pool.iter_epoch(0)]
    np.testing.assert_allclose(losses[:6], gold["losses"], rtol=1e-3)


# ---- statistics -------------------------------------------------------------------

def test_neighbor_draw_inclusion_frequencies(P):
    """Per-edge inclusion frequency vs the exact probabilities min(k,nc)/nc
    (cached) and fill/rest (uncached) — sampling.py:287-295 — over T
    independent Philox batches; per-edge |z| < 4.5 (Bonferroni)."""
    og = O.build_csr(np.random.default_rng(5).integers(0, 60, size=(300, 2)), 60)
    g = P.Graph.from_numpy(60, og.indptr, og.indices)
    cache = P.build_cache(g, P.degree_probs(g), 12, rng_seed=[0, 33, 0])
    mask = cache.nodes.mask.cpu().numpy()
    seeds = np.arange(60)
    T = 3000
    k = 4
    for cache_only in (False, True):
        cfg = P.SamplerConfig(strategy="GNS", fanouts=(k,), batch_size=60, input_layer_cache_only=cache_only,
                              cache_mode="degree")
        counts = {}
        for t in range(T):
            mb = P.build_minibatch(g, cache, seeds, cfg, P.BatchRng(0, 0, t))
            b = mb.blocks[0]
            d = b.dst_nodes.cpu().numpy()[b.edge_dst.cpu().numpy()]
            s = b.edge_node.cpu().numpy()
            key = d.astype(np.int64) * 60 + s
            for x in key:
                counts[x] = counts.get(x, 0) + 1
        zmax = 0.0
        for v in range(60):
            nb = og.indices[og.indptr[v]:og.indptr[v + 1]]
            c_nb = nb[mask[nb]]
            u_nb = nb[~mask[nb]]
            m = min(k, len(c_nb))
            fill = 0 if cache_only else min(k - m, len(u_nb))
            for u in nb:
                p = (m / len(c_nb)) if mask[u] else (fill / len(u_nb) if len(u_nb) else 0.0)
                f = counts.get(v * 60 + u, 0)
                if p in (0.0, 1.0):
                    assert f == p * T, (v, u, p, f)
                    continue
                z = (f - T * p) / np.sqrt(T * p * (1 - p))
                zmax = max(zmax, abs(z))
        assert zmax < 4.5, zmax


def test_cache_draw_distribution(P):
    """|C| = 1: the draw is exactly p-proportional; chi-square over R epochs."""
    og = O.build_csr(np.random.default_rng(7).integers(0, 40, size=(150, 2)), 40)
    g = P.Graph.from_numpy(40, og.indptr, og.indices)
    probs = P.degree_probs(g)
    p = probs.weights.cpu().numpy()
    R = 6000
    hits = np.zeros(40)
    for e in range(R):
        hits[P.sample_cache(probs, 1, [0, 33, e]).ids.cpu().numpy()] += 1
    sup = p > 0
    exp = R * p[sup]
    chi2 = float(((hits[sup] - exp) ** 2 / exp).sum())
    dof = int(sup.sum()) - 1
    from scipy.stats import chi2 as C
    assert C.sf(chi2, dof) > 1e-3, (chi2, dof)
    # |C| > 1: Spearman(frequency, degree) high
    freq = np.zeros(40)
    for e in range(1500):
        freq[P.sample_cache(probs, 8, [1, 33, e]).ids.cpu().numpy()] += 1
    from scipy.stats import spearmanr
    assert spearmanr(freq[sup], p[sup]).correlation > 0.9


# ---- device generator (graph.py:142-169 contract) ---------------------------------

def test_device_generator_contract(P):
    g = P.generate_powerlaw_device(20000, 150000, alpha=0.6, offset=50.0, seed=3, feature_dim=12,
                                   num_classes=5, train_frac=0.5)
    ip = g.indptr.cpu().numpy()
    ix = g.indices.cpu().numpy().astype(np.int64)
    n = g.num_nodes
    assert ip[0] == 0 and ip[-1] == len(ix) and np.all(np.diff(ip) >= 0)
    rows = np.repeat(np.arange(n), np.diff(ip))
    assert not np.any(rows == ix), "self loop"
    same = rows[1:] == rows[:-1]
    assert not np.any(same & (np.diff(ix) <= 0)), "rows must be sorted + dedup"
    keys = rows * n + ix
    assert np.array_equal(keys, np.sort(ix * n + rows)), "symmetric"
    deg = np.diff(ip)
    assert deg.max() > 10 * max(deg.mean(), 1), "power-law tail"
    assert g.features.shape == (n, 12) and g.feature_dim == 12
    # determinism
    g2 = P.generate_powerlaw_device(20000, 150000, alpha=0.6, offset=50.0, seed=3)
    assert torch.equal(g.indices, g2.indices)


@pytest.mark.parametrize("n,m,alpha,offset,seed", [(20000, 150000, 0.6, 50.0, 3), (100000, 1000000, 0.6, 10.0, 0),
                                                    (5000, 60000, 0.3, 2.0, 11)])
def test_device_generator_equals_host_restatement(P, n, m, alpha, offset, seed):
    """The device generator (gns_gen_powerlaw_*, gns_gen_node_attrs,
    gns_gen_features) and its host restatement oracle/gen.cc build the same
    graph bit for bit: CSR, labels, masks, features (the CPU reference arm of
    bench.py builds its graph on the host with the latter)."""
    from oracle import gen
    g = P.generate_powerlaw_device(n, m, alpha=alpha, offset=offset, seed=seed, feature_dim=30, num_classes=7,
                                   train_frac=0.2)
    og = gen.powerlaw_graph(n, m, alpha, offset, seed, feature_dim=30, num_classes=7, train_frac=0.2)
    assert np.array_equal(g.indptr.cpu().numpy(), og.indptr)
    assert np.array_equal(g.indices.cpu().numpy(), og.indices)
    assert np.array_equal(g.labels.cpu().numpy(), og.labels)
    for a, b in ((g.train_mask, og.train_mask), (g.val_mask, og.val_mask), (g.test_mask, og.test_mask)):
        assert np.array_equal(a.cpu().numpy(), b)
    f = g.features.cpu().numpy()          # row stride padded to 16 B, zero columns
    assert f.shape == (n, 32) and g.feature_dim == 30
    assert np.array_equal(f.view(np.uint32), og.features.view(np.uint32))


# ---- CUDA-graph engine ---------------------------------------------------------------

@pytest.mark.parametrize("S", [1, 2])
def test_graphed_trainer_matches_eager(P, S):
    """The captured whole-step engine (sample || train, static capacities,
    device-side batch parameters; S steps per graph replay) trains on exactly
    the pool's batches and tracks the eager path's losses."""
    og = _hub_graph(5000, 13)
    rng = np.random.default_rng(0)
    feats = rng.normal(size=(og.num_nodes, 16)).astype(np.float32)
    labels = rng.integers(0, 5, og.num_nodes).astype(np.int32)
    mask = rng.random(og.num_nodes) < 0.6
    g = P.Graph.from_numpy(og.num_nodes, og.indptr, og.indices, features=feats, labels=labels, train_mask=mask)
    cfg = P.SamplerConfig(strategy="GNS", fanouts=(10, 5), batch_size=256, cache_frac=0.05, cache_mode="degree",
                          seed=3)
    tc = P.TrainConfig(lr=0.003)
    eager = P.GraphSAGE((16, 32, 5), seed=0)
    pool = P.SamplerPool(g, cfg, num_workers=1)
    ref_losses = []
    for it in pool.iter_epoch(0):
        ref_losses.append(float(eager.train_step(it.minibatch, g, tc)))
    from paper_2106_06150_b200.engine import GraphedTrainer
    tr = GraphedTrainer(g, cfg, (16, 32, 5), tc, seed=0, steps_per_graph=S)
    losses = []
    tr.run_epoch(0, on_step=lambda e, i, k: losses.append(tr.loss_value()))
    tr.check_errors()
    assert len(losses) == len(ref_losses)
    np.testing.assert_allclose(losses, ref_losses, rtol=2e-3)
    we, be = eager.export()
    wg, bg_ = tr.model.export()
    for a, b in zip(we + be, wg + bg_):
        np.testing.assert_allclose(a, b, rtol=1e-2, atol=1e-4)
    # epochs 1 and 2 re-draw the cache (double-buffered: epoch 1's cache is
    # prefetched into the second set during epoch 0, epoch 2's back into the
    # first) and keep tracking the eager pool (which builds a new cache);
    # epoch 2 replays the first set's graphs without re-capturing
    for epoch in (1, 2):
        ref2 = [float(eager.train_step(it.minibatch, g, tc)) for it in pool.iter_epoch(epoch)]
        execs = {k: v[1].value for k, v in tr._execs.items()}
        losses2 = []
        n2 = tr.run_epoch(epoch, on_step=lambda e, i, k: losses2.append(tr.loss_value()))
        assert n2 == len(losses)
        assert tr.refresh_log[-1] == (epoch, "prefetched")
        if epoch == 2:
            assert {k: v[1].value for k, v in tr._execs.items()} == execs
        assert tr.cache.epoch == epoch and pool.cache.epoch == epoch
        assert torch.equal(tr.cache.nodes.ids, pool.cache.nodes.ids)
        assert torch.equal(tr.cache.cached_indices, pool.cache.cached_indices)
        np.testing.assert_allclose(losses2, ref2, rtol=2e-3)


def _engine_graph(P, og, dim=16, classes=5, train=0.6, seed=0):
    rng = np.random.default_rng(seed)
    feats = rng.normal(size=(og.num_nodes, dim)).astype(np.float32)
    labels = rng.integers(0, classes, og.num_nodes).astype(np.int32)
    mask = rng.random(og.num_nodes) < train
    og2 = O.OGraph(num_nodes=og.num_nodes, indptr=og.indptr, indices=og.indices, features=feats, labels=labels,
                   train_mask=mask)
    return og2, P.Graph.from_numpy(og.num_nodes, og.indptr, og.indices, features=feats, labels=labels,
                                   train_mask=mask)


@pytest.mark.parametrize("S,period", [(1, 1), (2, 1), (2, 2)])
def test_engine_epoch_slots_bit_exact_vs_oracle(P, S, period):
    """Every batch the captured engine trains on — read back from its sampler
    slot buffers — is bit-identical to the oracle restatement of
    sampling.py:299-336 on the same (seed, epoch, index) Philox key, the
    Feistel epoch partition (pool.py:60-66) and the epoch's cache
    (pool.py:133-135, double-buffered / prefetched), over 3 epochs."""
    from paper_2106_06150_b200.engine import GraphedTrainer
    og, g = _engine_graph(P, _hub_graph(5000, 29), train=0.5)
    cfg = P.SamplerConfig(strategy="GNS", fanouts=(15, 10, 5), batch_size=400, cache_frac=0.03,
                          cache_mode="degree", cache_period=period, seed=5)
    tr = GraphedTrainer(g, cfg, (16, 32, 32, 5), P.TrainConfig(), seed=0, steps_per_graph=S)
    cs = O.cache_size_for(og, cfg.cache_frac)
    w = O.degree_probs(og)
    seen = []
    for epoch in range(3):
        ce = epoch - epoch % period
        oc = O.build_cache(og, w, cs, seed=cfg.seed, epoch=ce)
        batches = O.epoch_targets(og, cfg.batch_size, cfg.seed, epoch)

        def check(e, index, k):
            mb = tr.slots[tr.slot_of(k)].snapshot()
            ref = O.build_minibatch(og, oc, batches[index], cfg, O.PhiloxKeys(cfg.seed, e, index))
            assert_mb_equal(mb, ref, f"S{S} e{e} i{index}")
            seen.append((e, index))
        n = tr.run_epoch(epoch, on_step=check)
        assert n == len(batches)
        assert tr.cache.epoch == ce
        assert np.array_equal(tr.cache.nodes.ids.cpu().numpy(), oc.ids)
    assert seen == [(e, i) for e in range(3) for i in range(len(batches))]


@pytest.mark.parametrize("S", [1, 2])
def test_engine_continuing_runs_sample_ahead(P, S):
    """run() calls that continue an epoch (bench: warm-up, then the timed
    window) reuse the batches the previous call's last replay sampled ahead —
    one eager prologue in all — and every trained batch, read from the slot
    slot_of() names, stays bit-identical to the oracle."""
    from paper_2106_06150_b200.engine import GraphedTrainer
    og, g = _engine_graph(P, _hub_graph(5000, 47), train=0.6)
    cfg = P.SamplerConfig(strategy="GNS", fanouts=(10, 5), batch_size=200, cache_frac=0.03, cache_mode="degree",
                          seed=6)
    tr = GraphedTrainer(g, cfg, (16, 32, 5), P.TrainConfig(), seed=0, steps_per_graph=S)
    nb = len(tr.batches(0))
    assert nb >= 12
    oc = O.build_cache(og, O.degree_probs(og), O.cache_size_for(og, cfg.cache_frac), seed=cfg.seed, epoch=0)
    batches = O.epoch_targets(og, cfg.batch_size, cfg.seed, 0)
    seen = []

    def check(e, index, k):
        mb = tr.slots[tr.slot_of(k)].snapshot()
        ref = O.build_minibatch(og, oc, batches[index], cfg, O.PhiloxKeys(cfg.seed, e, index))
        assert_mb_equal(mb, ref, f"S{S} i{index}")
        seen.append(index)

    pos = (0, 0)
    for n in (5, 3, 4):
        pos = tr.run(n, epoch=pos[0], first=pos[1], on_step=check)
    assert seen == list(range(12))
    assert tr.prologues == 1


@pytest.mark.parametrize("n,pairs", [(4000, 0), (3000, 1024 * 7), (20000, 100000)])
def test_cached_csr_flat_passes_equal_per_row(P, n, pairs):
    """The cached CSR from the flat (entry-parallel) passes — keep bits per
    CSR entry, tile counts, scanned tile offsets, c_indptr from popcounts,
    flat compaction — equals the per-row path (positions=True) and the oracle's
    filter of the full CSR (cache.py:185-197), for edge counts on and off the
    1024-entry tile boundary."""
    rng = np.random.default_rng(n + pairs)
    if pairs == 0:
        og = _hub_graph(n, 3)
    else:
        og = O.build_csr(rng.integers(0, n, size=(pairs, 2)), n)
    g = P.Graph.from_numpy(og.num_nodes, og.indptr, og.indices)
    probs = P.degree_probs(g)
    cs = max(1, og.num_nodes // 20)
    a = P.build_cache(g, probs, cs, rng_seed=[0, 33, 4], positions=True)
    b = P.build_cache(g, probs, cs, rng_seed=[0, 33, 4], positions=False)
    assert torch.equal(a.cached_indptr, b.cached_indptr)
    assert torch.equal(a.cached_indices, b.cached_indices)
    ci, cx = O.cached_csr_by_filter(og, a.nodes.mask.cpu().numpy())
    assert np.array_equal(b.cached_indptr.cpu().numpy(), ci)
    assert np.array_equal(b.cached_indices.cpu().numpy(), cx)


def test_refresh_cache_grows_cached_csr_in_place(P):
    """a refresh whose cached CSR outgrows the buffer gets larger
    buffers on the SAME CacheState (no stale pointers) and reports it."""
    og = _hub_graph(4000, 31)
    g = P.Graph.from_numpy(og.num_nodes, og.indptr, og.indices)
    probs = P.degree_probs(g)
    st = P.build_cache(g, probs, 60, rng_seed=[0, 33, 0])
    object.__setattr__(st, "_buf_cidx", st._buf_cidx[:3])     # force growth
    object.__setattr__(st, "_buf_cpos", st._buf_cpos[:3])
    from paper_2106_06150_b200 import cache as C
    kept = C.refresh_cache(st, g, probs, 60, 1, [0, 33, 1])
    assert kept is False and st.epoch == 1
    fresh = P.build_cache(g, probs, 60, rng_seed=[0, 33, 1])
    for f in ("cached_indptr", "cached_indices", "inclusion"):
        assert torch.equal(getattr(st, f), getattr(fresh, f)), f
    assert torch.equal(st.nodes.ids, fresh.nodes.ids)
    c = st.cstruct()
    assert c.cached_indices == st.cached_indices.data_ptr()
    # and in place when it fits
    before = st.cached_indices.data_ptr()
    assert C.refresh_cache(st, g, probs, 60, 2, [0, 33, 2]) in (True, False)
    fresh2 = P.build_cache(g, probs, 60, rng_seed=[0, 33, 2])
    assert torch.equal(st.cached_indices, fresh2.cached_indices)
    if st.cached_indices.data_ptr() == before:
        assert st.cstruct().cached_indices == before


@pytest.mark.parametrize("placement", ["device", "mixed"])
def test_engine_never_writes_an_adopted_cache(P, placement):
    """A CacheState handed to the engine (``tr.cache = state``) is the
    caller's: runs that cross several refresh epochs (prefetched into the
    engine's own idle set, the timed-run graphs of both sets captured up
    front by prepare) leave its contents untouched — regression: the second
    refresh drew into the adopted buffers."""
    og, g = _engine_graph(P, _hub_graph(3000, 43), train=0.5)
    cfg = P.SamplerConfig(strategy="GNS", fanouts=(10, 5), batch_size=300, cache_frac=0.05, cache_mode="degree",
                          seed=3)
    st = P.build_cache(g, P.degree_probs(g), O.cache_size_for(og, 0.05), rng_seed=[3, 33, 0])
    before = {f: getattr(st, f).clone() for f in ("cached_indptr", "cached_indices", "inclusion")}
    ids = st.nodes.ids.clone()
    tr = GraphedTrainerCls(P)(g, cfg, (16, 16, 5), P.TrainConfig(), seed=0, feature_placement=placement)
    tr.cache = st
    nb = len(tr.batches(0))
    tr.prepare(3 * nb)
    tr.run(3 * nb + 1)
    torch.cuda.synchronize()
    assert tr.refresh_log and all(e > 0 for e, _ in tr.refresh_log)
    assert torch.equal(st.nodes.ids, ids)
    for f, v in before.items():
        assert torch.equal(getattr(st, f), v), f
    assert tr.cache is not st and tr.cache.epoch == 3


def GraphedTrainerCls(P):
    from paper_2106_06150_b200.engine import GraphedTrainer
    return GraphedTrainer


def test_engine_device_errors_are_sticky(P):
    """A zero-inclusion cached draw in an engine step raises the reference's
    ValueError (sampling.py:255-256) at the end of the run, even though the
    failing batch's slot has been re-sampled since."""
    from paper_2106_06150_b200.engine import GraphedTrainer
    og, g = _engine_graph(P, _hub_graph(3000, 37))
    cfg = P.SamplerConfig(strategy="GNS", fanouts=(10, 5), batch_size=200, cache_frac=0.05, cache_mode="degree",
                          seed=1)
    tr = GraphedTrainer(g, cfg, (16, 32, 5), P.TrainConfig(), seed=0)
    tr.run_epoch(0, max_steps=2)
    tr.cache.inclusion.zero_()        # same buffer the captured steps read
    with pytest.raises(ValueError, match="inclusion probability is zero"):
        tr.run_epoch(0, first=2, max_steps=4)
    tr.check_errors()                 # cleared once raised


def test_engine_rejects_out_of_range_labels(P):
    from paper_2106_06150_b200.engine import GraphedTrainer
    og, g = _engine_graph(P, _hub_graph(2000, 3), classes=7)
    cfg = P.SamplerConfig(strategy="GNS", fanouts=(5,), batch_size=100, cache_mode="degree")
    with pytest.raises(ValueError, match="label out of range"):
        GraphedTrainer(g, cfg, (16, 5), P.TrainConfig())
    m = P.GraphSAGE((16, 5))
    mb = P.build_minibatch(g, P.build_cache(g, P.degree_probs(g), 20), np.arange(50), cfg, P.BatchRng())
    with pytest.raises(ValueError, match="label out of range"):
        m.train_step(mb, g, P.TrainConfig())


def test_engine_padded_data_parallel_schedule(P):
    """World size 2, rank 1 with an odd batch count: ceil(nb/2) steps, the
    last one on an empty batch (zero loss, zero gradient)."""
    from paper_2106_06150_b200.engine import GraphedTrainer
    og, g = _engine_graph(P, _hub_graph(3000, 41), train=0.5)
    cfg = P.SamplerConfig(strategy="GNS", fanouts=(10, 5), batch_size=300, cache_frac=0.05, cache_mode="degree",
                          seed=2)
    nb = -(-int(og.train_mask.sum()) // 300)
    assert nb % 2 == 1
    tr = GraphedTrainer(g, cfg, (16, 32, 5), P.TrainConfig(), rank=1, world_size=2, seed=0, steps_per_graph=1)
    sched = tr.batches(0)
    assert len(sched) == (nb + 1) // 2 and sched[-1] is None and sched[:-1] == list(range(1, nb, 2))
    got = []

    def on(e, i, k):
        got.append((i, tr.loss_value(), float(tr.model.grad.abs().sum())))
    assert tr.run_epoch(0, on_step=on) == len(sched)
    assert [i for i, _, _ in got] == sched
    assert got[-1][1] == 0.0 and got[-1][2] == 0.0
    assert all(l > 0 and gs > 0 for _, l, gs in got[:-1])


def test_pool_copy_batches_are_independent(P):
    og, g = _engine_graph(P, _hub_graph(3000, 43))
    cfg = P.SamplerConfig(strategy="GNS", fanouts=(10, 5), batch_size=200, cache_frac=0.05, cache_mode="degree")
    kept = [it.minibatch for it in P.SamplerPool(g, cfg, num_workers=2, copy=True).iter_epoch(0)]
    views = [it.minibatch.clone() for it in P.SamplerPool(g, cfg, num_workers=2).iter_epoch(0)]
    assert len(kept) == len(views) > 2
    for a, b in zip(kept, views):
        for ba, bb in zip(a.blocks, b.blocks):
            assert torch.equal(ba.edge_src, bb.edge_src) and torch.equal(ba.src_nodes, bb.src_nodes)
    # a cloned batch trains like the slot view it was copied from
    m1, m2 = P.GraphSAGE((16, 32, 5), seed=0), P.GraphSAGE((16, 32, 5), seed=0)
    l1 = float(m1.train_step(kept[0], g, P.TrainConfig()))
    l2 = float(m2.train_step(views[0], g, P.TrainConfig()))
    assert l1 == l2


def test_engine_captured_nccl_allreduce_world1(P, tmp_path):
    """GNS_FORCE_DIST path: the NCCL all-reduce captured in the step graph
    at world size 1 trains exactly like the engine without it."""
    import os
    import socket
    import torch.distributed as dist
    from paper_2106_06150_b200 import dist as gdist
    from paper_2106_06150_b200.engine import GraphedTrainer
    og, g = _engine_graph(P, _hub_graph(3000, 47))
    cfg = P.SamplerConfig(strategy="GNS", fanouts=(10, 5), batch_size=200, cache_frac=0.05, cache_mode="degree",
                          seed=6)
    tc = P.TrainConfig()
    base = GraphedTrainer(g, cfg, (16, 32, 5), tc, seed=0)
    ref = []
    base.run(12, on_step=lambda e, i, k: ref.append(base.loss_value()))
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0", WORLD_SIZE="1")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        tr = GraphedTrainer(g, cfg, (16, 32, 5), tc, seed=0, allreduce=gdist.make_allreduce(force=True))
        got = []
        tr.run(12, on_step=lambda e, i, k: got.append(tr.loss_value()))
        assert got == ref
        assert torch.equal(tr.model.flat, base.model.flat)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("chunk", [0, 4096])
def test_graphed_trainer_size_switched_dense_ops(P, chunk):
    """Input-layer GEMMs as SWITCH graph nodes over the device row count
    (bodies over ceil(n / chunk) * chunk rows) train exactly like the
    capacity-sized ones and the eager model."""
    n = 30_000
    rng = np.random.default_rng(5)
    og = O.build_csr(rng.integers(0, n, size=(150_000, 2)), n)
    feats = rng.normal(size=(n, 16)).astype(np.float32)
    labels = rng.integers(0, 5, n).astype(np.int32)
    mask = rng.random(n) < 0.3
    g = P.Graph.from_numpy(n, og.indptr, og.indices, features=feats, labels=labels, train_mask=mask)
    cfg = P.SamplerConfig(strategy="GNS", fanouts=(10, 5), batch_size=1500, cache_frac=0.02, cache_mode="degree",
                          seed=9)
    tc = P.TrainConfig(lr=0.003)
    from paper_2106_06150_b200.engine import GraphedTrainer
    tr = GraphedTrainer(g, cfg, (16, 32, 5), tc, seed=0, switch_chunk=chunk)
    assert tr.use_switch == (chunk > 0) and tr.cap_dst[0] >= 2 * 4096
    losses = []
    tr.run_epoch(0, max_steps=5, on_step=lambda e, i, k: losses.append(tr.loss_value()))
    eager = P.GraphSAGE((16, 32, 5), seed=0)
    pool = P.SamplerPool(g, cfg, num_workers=1)
    ref = [float(eager.train_step(it.minibatch, g, tc)) for _, it in zip(range(5), pool.iter_epoch(0))]
    np.testing.assert_allclose(losses, ref, rtol=2e-3)
    we, be = eager.export()
    wg, bg_ = tr.model.export()
    for a, b in zip(we + be, wg + bg_):
        np.testing.assert_allclose(a, b, rtol=1e-2, atol=1e-4)


@pytest.mark.parametrize("S", [1, 2])
def test_graphed_trainer_run_host_matches_eager(P, S):
    """The end-to-end API (host target arrays copied into the step graph,
    every step's loss read back, one replay kept in flight) trains exactly
    the given batches: losses track the eager model on the same batches."""
    og = _hub_graph(4000, 23)
    rng = np.random.default_rng(1)
    feats = rng.normal(size=(og.num_nodes, 16)).astype(np.float32)
    labels = rng.integers(0, 5, og.num_nodes).astype(np.int32)
    g = P.Graph.from_numpy(og.num_nodes, og.indptr, og.indices, features=feats, labels=labels)
    cfg = P.SamplerConfig(strategy="GNS", fanouts=(10, 5), batch_size=200, cache_frac=0.05, cache_mode="degree",
                          seed=4)
    tc = P.TrainConfig(lr=0.003)
    batches = [rng.choice(og.num_nodes, 200, replace=False) for _ in range(7)]
    from paper_2106_06150_b200.engine import GraphedTrainer
    tr = GraphedTrainer(g, cfg, (16, 32, 5), tc, seed=0, host_targets=True, steps_per_graph=S)
    got = tr.run_host(batches, epoch=0)
    eager = P.GraphSAGE((16, 32, 5), seed=0)
    ref = [float(eager.train_step(P.build_minibatch(g, tr.cache, b, cfg, P.BatchRng(4, 0, k)), g, tc))
           for k, b in enumerate(batches)]
    assert len(got) == len(batches)
    np.testing.assert_allclose(got, ref, rtol=2e-3)


@pytest.mark.parametrize("S", [1, 2])
def test_run_host_lookahead_equals_one_call(P, S):
    """run_host split into calls that sample the next call's first batches
    ahead (``lookahead``, ``base``) trains exactly what one continuous call
    trains: identical losses, one eager prologue, and the last trained batch
    bit-identical to the oracle on Philox key base + position."""
    og = _hub_graph(4000, 53)
    rng = np.random.default_rng(2)
    feats = rng.normal(size=(og.num_nodes, 16)).astype(np.float32)
    labels = rng.integers(0, 5, og.num_nodes).astype(np.int32)
    g = P.Graph.from_numpy(og.num_nodes, og.indptr, og.indices, features=feats, labels=labels)
    cfg = P.SamplerConfig(strategy="GNS", fanouts=(10, 5), batch_size=200, cache_frac=0.05, cache_mode="degree",
                          seed=7)
    tc = P.TrainConfig(lr=0.003)
    batches = [rng.choice(og.num_nodes, 200, replace=False) for _ in range(12)]
    from paper_2106_06150_b200.engine import GraphedTrainer
    one = GraphedTrainer(g, cfg, (16, 32, 5), tc, seed=0, host_targets=True, steps_per_graph=S)
    ref = one.run_host(batches, epoch=0)
    tr = GraphedTrainer(g, cfg, (16, 32, 5), tc, seed=0, host_targets=True, steps_per_graph=S)
    got = tr.run_host(batches[:4], epoch=0, lookahead=batches[4:4 + S])
    got += tr.run_host(batches[4:10], epoch=0, base=4, lookahead=batches[10:10 + S])
    got += tr.run_host(batches[10:], epoch=0, base=10)
    assert tr.prologues == 1 and one.prologues == 1
    assert got == ref
    ids = tr.cache.nodes.ids.cpu().numpy().astype(np.int64)
    mask = np.zeros(og.num_nodes, dtype=bool)
    mask[ids] = True
    oc = O.OCache(ids=ids, mask=mask, inclusion=tr.cache.inclusion.cpu().numpy(),
                  cached_indptr=tr.cache.cached_indptr.cpu().numpy(),
                  cached_indices=tr.cache.cached_indices.cpu().numpy(), epoch=0)
    k = len(batches[10:]) - 1
    mb = tr.slots[tr.slot_of(k)].snapshot()
    want = O.build_minibatch(og, oc, batches[10 + k], cfg, O.PhiloxKeys(cfg.seed, 0, 10 + k))
    assert_mb_equal(mb, want, f"S{S}")


# ---- random-walk cache distribution -----------------------------

def test_random_walk_probs(P, golden):
    gold = golden["sampler"]
    og, g = _golden_graph(P, gold)
    tid = gold["walk_train_ids"]
    for L, fan, key in ((3, (15, 10, 5), "walk_probs_L3"), (1, (4,), "walk_probs_L1")):
        pv = P.random_walk_probs(g, torch.as_tensor(tid, dtype=torch.int32, device="cuda"), fan, L)
        got = pv.weights.cpu().numpy()
        assert np.array_equal(got, O.random_walk_probs(og, tid, fan, L))          # bit-exact vs oracle
        ref = gold[key]
        nz = np.maximum(np.abs(ref), 1e-300)
        assert np.max(np.abs(got - ref) / np.spacing(nz)) <= 4                   # vs reference
    # pool "auto" mode picks the walk distribution when < 50% of nodes train
    mask = np.zeros(og.num_nodes, dtype=bool)
    mask[tid] = True
    g2 = P.Graph.from_numpy(og.num_nodes, og.indptr, og.indices, train_mask=mask)
    from paper_2106_06150_b200.pool import cache_probs
    cfg = P.SamplerConfig(strategy="GNS", cache_mode="auto")
    pv = cache_probs(g2, cfg)
    assert np.array_equal(pv.weights.cpu().numpy(), O.random_walk_probs(og, tid, (15, 10, 5), 3))


# ---- graph formats ----------------------------------------------

def test_build_csr_matches_reference_contract(P):
    rng = np.random.default_rng(3)
    edges = rng.integers(0, 500, size=(4000, 2))
    edges = np.concatenate([edges, edges[:50], [[7, 7], [9, 9]]])      # duplicates + self loops
    g = P.build_csr(edges, 500)
    ref = O.build_csr(edges, 500)                                      # graph.py:142-169 restated
    assert np.array_equal(g.indptr.cpu().numpy(), ref.indptr)
    assert np.array_equal(g.indices.cpu().numpy(), ref.indices)
    P.validate_graph(g)
    g1 = P.build_csr([(0, 1)], 2)
    assert g1.indptr.tolist() == [0, 1, 2] and g1.indices.tolist() == [1, 0]
    with pytest.raises(ValueError, match=r"edge \(3, 5\) out of range"):
        P.build_csr([(0, 1), (3, 5)], 4)


def test_gnsg_round_trip(P, tmp_path, golden):
    gold = golden["model"]
    n = len(gold["indptr"]) - 1
    g = P.Graph.from_numpy(n, gold["indptr"], gold["indices"], features=gold["features"], labels=gold["labels"],
                           train_mask=gold["train_mask"], val_mask=~gold["train_mask"],
                           test_mask=np.zeros(n, dtype=bool))
    p = tmp_path / "g.gnsg"
    P.save_binary(g, p)
    g2 = P.load_binary(p)
    assert torch.equal(g.indptr, g2.indptr) and torch.equal(g.indices, g2.indices)
    assert torch.equal(g.features, g2.features) and torch.equal(g.labels, g2.labels)
    assert torch.equal(g.train_mask, g2.train_mask) and torch.equal(g.val_mask, g2.val_mask)
    # byte layout: int64 indptr/indices after the 28-byte header (graph.py:8-28)
    raw = p.read_bytes()
    assert raw[:4] == b"GNSG"
    assert np.array_equal(np.frombuffer(raw, dtype="<i8", count=n + 1, offset=28), gold["indptr"])
    P.validate_graph(g2)


def test_edgelist(P, tmp_path):
    p = tmp_path / "e.txt"
    p.write_text("# comment\n0 1\n1 2\n\n2 0\n")
    g = P.load_edgelist(p)
    assert g.num_nodes == 3 and g.indices.tolist() == [1, 2, 0, 2, 0, 1]
    p.write_text("0 x\n")
    with pytest.raises(P.GraphFormatError, match="non-integer"):
        P.load_edgelist(p)


def test_load_reference_written_gnsg(P):
    import os
    from conftest import GOLDEN
    path = os.path.join(GOLDEN, "golden_sbm60.gnsg")
    g = P.load_binary(path)
    raw = open(path, "rb").read()
    n, e = 60, g.num_edges
    off = 28
    ip = np.frombuffer(raw, dtype="<i8", count=n + 1, offset=off); off += 8 * (n + 1)
    ix = np.frombuffer(raw, dtype="<i8", count=e, offset=off); off += 8 * e
    f = np.frombuffer(raw, dtype="<f4", count=n * 5, offset=off).reshape(n, 5); off += 20 * n
    lab = np.frombuffer(raw, dtype="<i4", count=n, offset=off)
    assert np.array_equal(g.indptr.cpu().numpy(), ip) and np.array_equal(g.indices.cpu().numpy(), ix)
    assert np.array_equal(g.features[:, :5].cpu().numpy(), f) and np.array_equal(g.labels.cpu().numpy(), lab)
    P.validate_graph(g)


# ---- device metrics ------------------------------------------------

def test_metrics_match_reference_definitions(P):
    """count_input_nodes / copy_cost / isolated_fraction / CSV, vs the oracle's
    restatement of metrics.py:75-97 and sampling.py:413-425 on the same blocks."""
    from paper_2106_06150_b200 import metrics as M
    og = _hub_graph(3000, 21)
    g = P.Graph.from_numpy(og.num_nodes, og.indptr, og.indices)
    cache = P.build_cache(g, P.degree_probs(g), 60, rng_seed=[0, 33, 0])
    oc = O.build_cache(og, O.degree_probs(og), 60, seed=0, epoch=0)
    cfg = P.SamplerConfig(strategy="GNS", fanouts=(6, 3), batch_size=100, cache_mode="degree")
    targets = np.arange(0, 3000, 30)
    mb = P.build_minibatch(g, cache, targets, cfg, P.BatchRng(0, 0, 0))
    ref_mb = O.build_minibatch(og, oc, targets, cfg, O.PhiloxKeys(0, 0, 0))
    total, cached = len(ref_mb.input_nodes), int(oc.mask[ref_mb.input_nodes].sum())
    assert M.count_input_nodes(mb, cache) == (total, cached)
    assert M.copy_cost(mb, cache, 64) == (total - cached) * 64 * 4
    assert abs(P.isolated_fraction(mb) - O.isolated_fraction(ref_mb)) < 1e-12
    s = M.batch_stats(mb, cache, 64, epoch=1, batch=2, sample_ms=1.4, train_ms=2.6)
    rep = M.MetricsReport(run_id="00_gns", strategy="GNS", config=cfg, seed=0, stats=[s])
    import tempfile, os
    with tempfile.TemporaryDirectory() as d:
        rep.write_csv(os.path.join(d, "a.csv"))
        lines = open(os.path.join(d, "a.csv")).read().splitlines()
    assert lines[0].split(",") == ["run_id", "epoch", "batch", "strategy", "num_input", "num_cached", "copy_bytes",
                                   "isolated_frac", "sample_ms", "train_ms"]
    assert lines[1].startswith("00_gns,1,2,GNS,%d,%d,%d," % (total, cached, (total - cached) * 256))


# ---- mixed CPU-GPU feature placement (paper §3.1) ------------------------------------

def test_mixed_placement_gather_and_training(P):
    from paper_2106_06150_b200 import _lib
    from paper_2106_06150_b200.engine import GraphedTrainer
    og = _hub_graph(4000, 31)
    rng = np.random.default_rng(1)
    feats = rng.normal(size=(og.num_nodes, 16)).astype(np.float32)
    labels = rng.integers(0, 4, og.num_nodes).astype(np.int32)
    g = P.Graph.from_numpy(og.num_nodes, og.indptr, og.indices, features=feats, labels=labels,
                           train_mask=rng.random(og.num_nodes) < 0.5)
    cfg = P.SamplerConfig(strategy="GNS", fanouts=(8, 4), batch_size=200, cache_frac=0.05, cache_mode="degree",
                          seed=5)
    # gather: cached rows from the HBM cache table, the rest from pinned host
    cache = P.build_cache(g, P.degree_probs(g), 200, rng_seed=[5, 33, 0])
    host = torch.as_tensor(feats).pin_memory()
    ids = cache.nodes.ids
    table = torch.empty((ids.numel(), 16), device="cuda")
    n_dev = torch.tensor([ids.numel()], dtype=torch.int64, device="cuda")
    _lib.call("gns_cache_refresh_rows", host.data_ptr(), 16, ids.data_ptr(), n_dev.data_ptr(), ids.numel(), 16,
              table.data_ptr(), _lib.stream_ptr())
    assert torch.equal(table.cpu(), host[ids.long().cpu()])
    rows = torch.as_tensor(np.sort(rng.choice(og.num_nodes, 900, replace=False)).astype(np.int32), device="cuda")
    nr = torch.tensor([900], dtype=torch.int32, device="cuda")
    out = torch.empty((900, 16), device="cuda")
    _lib.call("gns_gather_rows_mixed", host.data_ptr(), table.data_ptr(), cache.nodes.mask_bits.data_ptr(),
              cache.mask_word_rank().data_ptr(), 16, rows.data_ptr(), nr.data_ptr(), 900, 16, out.data_ptr(), 16,
              _lib.stream_ptr())
    assert torch.equal(out.cpu(), host[rows.long().cpu()])
    # the whole engine: identical losses in both placements
    tc = P.TrainConfig(lr=0.003)
    res = {}
    for placement in ("device", "mixed"):
        tr = GraphedTrainer(g, cfg, (16, 32, 4), tc, seed=0, feature_placement=placement)
        losses = []
        tr.run_epoch(0, on_step=lambda e, i, k: losses.append(tr.loss_value()))
        res[placement] = losses
    assert res["device"] == res["mixed"]


# ---- gns-exact weights ----------------------------------------------

def test_gns_exact_table_and_blocks(P):
    og = _hub_graph(3000, 41)
    g = P.Graph.from_numpy(og.num_nodes, og.indptr, og.indices)
    probs = P.degree_probs(g)
    w = O.degree_probs(og)
    tables_g, tables_o = {}, {}
    for k, co in ((10, False), (5, True)):
        t = P.estimate_edge_inclusion(g, probs, 1500, k, co, resamples=64, seed=7)
        to = O.estimate_edge_inclusion(og, w, 1500, k, co, resamples=64, seed=7)
        assert np.array_equal(t.cpu().numpy(), to)
        tables_g[(k, co)], tables_o[(k, co)] = t, to
    cfg = P.SamplerConfig(strategy="GNS", fanouts=(10, 5), batch_size=300, cache_mode="degree", cache_frac=0.5,
                          weight_policy="gns-exact", seed=2)
    cache = P.build_cache(g, probs, 1500, rng_seed=[2, 33, 0])
    oc = O.build_cache(og, w, 1500, seed=2, epoch=0)
    targets = np.random.default_rng(3).choice(og.num_nodes, 300, replace=False)
    mb = P.build_minibatch(g, cache, targets, cfg, P.BatchRng(2, 0, 4), exact_tables=tables_g)
    ref = O.build_minibatch(og, oc, targets, cfg, O.PhiloxKeys(2, 0, 4), exact_tables=tables_o)
    assert_mb_equal(mb, ref, "gns-exact")
    assert mb.blocks[0].policy == "gns-exact"
    with pytest.raises(ValueError, match="missing edge-inclusion table"):
        P.build_minibatch(g, cache, targets, cfg, P.BatchRng(2, 0, 4), exact_tables={})
    # the pool builds the tables once and trains through them
    pool = P.SamplerPool(g, cfg)
    n = sum(1 for _ in pool.iter_epoch(0))
    assert n > 0 and set(pool._tables) == {(10, False), (5, True)}


# ---- training parity on the SPEC convergence task (golden_train.npz) --------------
# SBM(2000, 4 blocks, 0.02, 0.002), 16-d, GNS cache 10% P=1, fanouts (15,10,5),
# batch 100, hidden 64, 10 epochs (model.py:257-307)

@pytest.fixture(scope="module")
def sbm(P):
    import os
    from conftest import GOLDEN
    z = dict(np.load(os.path.join(GOLDEN, "golden_train.npz")))
    n = len(z["indptr"]) - 1
    g = P.Graph.from_numpy(n, z["indptr"], z["indices"], features=z["features"].astype(np.float32),
                           labels=z["labels"], train_mask=z["train_mask"], val_mask=z["val_mask"],
                           test_mask=z["test_mask"])
    cfg = P.SamplerConfig(strategy="GNS", fanouts=(15, 10, 5), batch_size=100, cache_frac=0.1, cache_period=1,
                          cache_mode="degree", seed=0)
    return z, g, cfg


def test_train_api_fp64_matches_reference_on_replayed_keys(P, sbm):
    """The reference's loop body (model.py:279-285) through the drop-in
    module API — init_params / forward / loss_and_grad / backward / adam_step
    in float64 — on the same Philox batches the golden reference run used
    (cache, epoch permutation and per-batch keys replayed): the first 20 step
    losses within 1e-9 relative, every epoch's mean loss within 1e-7, and the
    micro-F1 of every epoch (full-neighbourhood evaluate) within 1 point."""
    z, g, cfg = sbm
    tc = P.TrainConfig(epochs=10, seed=0, hidden_dim=64, lr=0.003)
    params = P.init_params((16, 64, 64, 4), seed=0)
    state = P.AdamState.zeros_like(params)
    pool = P.SamplerPool(g, cfg, num_workers=2)
    losses, epoch_loss, f1 = [], [], []
    for epoch in range(10):
        el = []
        for it in pool.iter_epoch(epoch):
            mb = it.minibatch
            logits = P.forward(mb, g, params)
            loss, grad = P.loss_and_grad(logits, g.labels[mb.targets.long()])
            grads = P.backward(mb, g, params, grad)
            P.adam_step(params, grads, state, tc)
            el.append(loss)
        losses += el
        epoch_loss.append(np.mean(el))
        f = P.evaluate(g, params)
        f1.append([f["train"], f["val"], f["test"]])
    assert len(losses) == len(z["losses"])
    np.testing.assert_allclose(losses[:20], z["losses"][:20], rtol=1e-9)
    np.testing.assert_allclose(epoch_loss, z["epoch_loss"], rtol=1e-7)
    np.testing.assert_allclose(np.array(f1), z["f1"], atol=0.01)


@pytest.mark.parametrize("tf32", [True, False])
def test_engine_fp32_tf32_training_tracks_reference(P, sbm, tf32):
    """The production engine (CUDA-graph steps, float32 storage, GEMMs in TF32
    or full fp32) on the same replayed batches.  Stated tolerances vs the
    float64 reference: the first 5 step losses within 1e-5 relative (fp32) /
    2e-3 (TF32: 10-bit mantissa GEMM inputs); the first 20 within 2e-3 / 1e-2
    (discrete events — a ReLU pre-activation or an Adam update near zero
    flipping sign — appear from step 6 on: measured 6.5e-4 fp32, 3.5e-3
    TF32); every epoch's mean loss within 1e-2; final test micro-F1 within
    1 point."""
    from paper_2106_06150_b200.engine import GraphedTrainer
    z, g, cfg = sbm
    tc = P.TrainConfig(epochs=10, seed=0, hidden_dim=64, lr=0.003)
    tr = GraphedTrainer(g, cfg, (16, 64, 64, 4), tc, seed=0, tf32=tf32)
    losses, epoch_loss = [], []
    for epoch in range(10):
        el = []
        tr.run_epoch(epoch, on_step=lambda e, i, k: el.append(tr.loss_value()))
        losses += el
        epoch_loss.append(np.mean(el))
    f = P.evaluate(g, P.ModelParams(tr.model))
    np.testing.assert_allclose(losses[:5], z["losses"][:5], rtol=2e-3 if tf32 else 1e-5)
    np.testing.assert_allclose(losses[:20], z["losses"][:20], rtol=1e-2 if tf32 else 2e-3)
    np.testing.assert_allclose(epoch_loss, z["epoch_loss"], rtol=1e-2)
    assert abs(f["test"] - z["f1"][-1][2]) <= 0.01, (f, z["f1"][-1])


@pytest.mark.parametrize("strategy", ["GNS", "NS"])
def test_train_free_running_f1_within_two_points(P, sbm, strategy):
    """free-running Philox training (P.train, the
    reference's train() loop, float32 production precision) reaches a test
    micro-F1 within 2 points of the reference's own PCG64 run, and >= 0.90."""
    z, g, cfg = sbm
    if strategy == "NS":
        cfg = P.SamplerConfig(strategy="NS", fanouts=(15, 10, 5), batch_size=100, seed=0)
    rep = P.train(g, cfg, P.TrainConfig(epochs=10, seed=0, hidden_dim=64, lr=0.003), dtype=torch.float32)
    ref = float(z[f"free_{strategy.lower()}_test_f1"])
    assert len(rep.rows) == 10 and rep.rows[-1].mean_input_nodes > 0
    assert abs(rep.final_test_f1 - ref) <= 0.02, (rep.final_test_f1, ref)
    assert rep.final_test_f1 >= 0.90


def test_engine_precisions_at_bench_dims(P):
    """Bench dims (128, 256, 256, 172): the engine in TF32 and fp32 against the
    float64 façade on the same Philox batches of one epoch — per-step loss
    within 1e-3 relative (fp32) / 5e-3 (TF32), epoch mean within 1e-3."""
    from paper_2106_06150_b200.engine import GraphedTrainer
    g = P.generate_powerlaw_device(60_000, 600_000, alpha=0.6, offset=10.0, seed=5, feature_dim=128,
                                   num_classes=172, train_frac=0.2)
    cfg = P.SamplerConfig(strategy="GNS", fanouts=(15, 10, 5), batch_size=1000, cache_frac=0.01,
                          cache_mode="degree", seed=0)
    dims = (128, 256, 256, 172)
    tc = P.TrainConfig(lr=0.003, hidden_dim=256)
    params = P.init_params(dims, seed=0)
    state = P.AdamState.zeros_like(params)
    ref = []
    for it in P.SamplerPool(g, cfg).iter_epoch(0):
        mb = it.minibatch
        loss, grad = P.loss_and_grad(P.forward(mb, g, params), g.labels[mb.targets.long()])
        P.adam_step(params, P.backward(mb, g, params, grad), state, tc)
        ref.append(loss)
    for tf32, tol in ((False, 1e-3), (True, 5e-3)):
        tr = GraphedTrainer(g, cfg, dims, tc, seed=0, tf32=tf32)
        got = []
        tr.run_epoch(0, on_step=lambda e, i, k: got.append(tr.loss_value()))
        assert len(got) == len(ref) >= 10
        np.testing.assert_allclose(got, ref, rtol=tol)
        assert abs(np.mean(got) / np.mean(ref) - 1) < 1e-3


# ---- SPEC statistical properties ------------------------------------------------------

def test_cache_draw_two_sample_vs_reference(P):
    """|C| > 1: per-node inclusion frequencies of the device
    draw (Philox exponential race) vs the reference's own numpy draw
    (golden_stat.npz, 2e4 draws each): two-sample z per node, Bonferroni
    |z| < 4.5."""
    import os
    from conftest import GOLDEN
    z = np.load(os.path.join(GOLDEN, "golden_stat.npz"))
    n = len(z["indptr"]) - 1
    g = P.Graph.from_numpy(n, z["indptr"], z["indices"])
    probs = P.degree_probs(g)
    R, cs = int(z["draws"]), int(z["cache_size"])
    hits = torch.zeros(n, dtype=torch.int64, device="cuda")
    for e in range(R):
        hits[P.sample_cache(probs, cs, [1, 33, e]).ids.long()] += 1
    a, b = hits.cpu().numpy() / R, z["ref_counts"] / R
    pooled = (a + b) / 2
    se = np.sqrt(np.maximum(pooled * (1 - pooled), 1e-12) * 2 / R)
    zs = np.abs(a - b) / se
    assert zs.max() < 4.5, (zs.max(), int(zs.argmax()))


def test_gns_full_cache_marginals_equal_ns(P):
    """GNS with C = V and cache_only = false draws each seed's
    neighbours with NS's marginals (uniform without replacement: min(k,d)/d
    per edge); chi-square over T Philox batches, p > 0.01, on a 30-node
    graph."""
    from scipy.stats import chi2
    og = O.build_csr(np.random.default_rng(11).integers(0, 30, size=(120, 2)), 30)
    g = P.Graph.from_numpy(30, og.indptr, og.indices)
    cache = P.build_cache(g, P.degree_probs(g), 30, rng_seed=[0, 33, 0])
    assert int(cache.nodes.mask.sum()) == int((np.diff(og.indptr) > 0).sum())
    k, T = 3, 4000
    seeds = np.arange(30)
    out = {}
    for strat in ("GNS", "NS"):
        cfg = P.SamplerConfig(strategy=strat, fanouts=(k,), batch_size=30, input_layer_cache_only=False,
                              cache_mode="degree", cache_frac=1.0)
        cnt = np.zeros((30, 30))
        for t in range(T):
            mb = P.build_minibatch(g, cache if strat == "GNS" else None, seeds, cfg, P.BatchRng(0, 0, t))
            b = mb.blocks[0]
            np.add.at(cnt, (b.dst_nodes.cpu().numpy()[b.edge_dst.cpu().numpy()], b.edge_node.cpu().numpy()), 1)
        out[strat] = cnt
    deg = np.diff(og.indptr)
    for strat, cnt in out.items():
        stat, dof = 0.0, 0
        for v in range(30):
            d = deg[v]
            if d <= k:       # every neighbour, every time
                nb = og.indices[og.indptr[v]:og.indptr[v + 1]]
                assert np.all(cnt[v, nb] == T), (strat, v)
                continue
            nb = og.indices[og.indptr[v]:og.indptr[v + 1]]
            e = T * k / d
            stat += float(((cnt[v, nb] - e) ** 2 / e).sum())
            dof += d - 1
        assert chi2.sf(stat, max(dof, 1)) > 0.01, (strat, stat, dof)


def test_ns_weighted_sum_unbiased(P):
    """E[sum over sampled u of w_u h_u] = sum over N(v) of h_u
    for NS weights deg/min(k,deg) (50-node graph; 100 disjoint copies per
    batch x 1000 batches = 1e5 trials per node), relative error < 2%."""
    rng = np.random.default_rng(3)
    base = rng.integers(0, 50, size=(200, 2))
    copies = 100
    edges = np.concatenate([base + 50 * c for c in range(copies)])
    n = 50 * copies
    og = O.build_csr(edges, n)
    g = P.Graph.from_numpy(n, og.indptr, og.indices)
    h = rng.uniform(0.5, 1.5, size=50)
    hh = np.tile(h, copies)
    k = 3
    cfg = P.SamplerConfig(strategy="NS", fanouts=(k,), batch_size=n)
    est = np.zeros(50)
    B = 1000
    for t in range(B):
        b = P.build_minibatch(g, None, np.arange(n), cfg, P.BatchRng(7, 0, t)).blocks[0]
        dst = b.dst_nodes.cpu().numpy()[b.edge_dst.cpu().numpy()]
        contrib = np.zeros(n)
        np.add.at(contrib, dst, b.edge_weight.cpu().numpy() * hh[b.edge_node.cpu().numpy()])
        est += contrib.reshape(copies, 50).sum(0)
    est /= B * copies
    full = np.array([hh[og.indices[og.indptr[v]:og.indptr[v + 1]]].sum() for v in range(50)])
    live = full > 0
    assert np.all(np.abs(est[live] / full[live] - 1) < 0.02), np.abs(est[live] / full[live] - 1).max()


def test_gns_input_node_reduction(P):
    """SPEC.md:287 (Table 3 analog): on a power-law graph (100K nodes, batch
    1000) GNS with cache 1%, fanouts (15, 10) and a cache-only input layer
    needs < 0.5x the input nodes of NS with fanouts (15, 10, 5)."""
    g = P.generate_powerlaw_device(100_000, 250_000, alpha=0.6, offset=10.0, seed=1)
    gns = P.SamplerConfig(strategy="GNS", fanouts=(15, 10), batch_size=1000, cache_frac=0.01, cache_mode="degree",
                          input_layer_cache_only=True)
    ns = P.SamplerConfig(strategy="NS", fanouts=(15, 10, 5), batch_size=1000)
    cache = P.build_cache(g, P.degree_probs(g), 1000, rng_seed=[0, 33, 0])
    rng = np.random.default_rng(0)
    n_g, n_n = [], []
    for t in range(10):
        targets = rng.choice(100_000, 1000, replace=False)
        n_g.append(P.build_minibatch(g, cache, targets, gns, P.BatchRng(0, 0, t)).input_nodes.numel())
        n_n.append(P.build_minibatch(g, None, targets, ns, P.BatchRng(0, 0, t)).input_nodes.numel())
    assert np.mean(n_g) < 0.5 * np.mean(n_n), (np.mean(n_g), np.mean(n_n))


def test_numpy_generator_as_rng(P):
    """A numpy Generator passed as rng (the reference's duck-typed hook,
    sampling.py:93-97) seeds the Philox key: deterministic in its state,
    different for a different state."""
    og = _hub_graph(2000, 5)
    g = P.Graph.from_numpy(og.num_nodes, og.indptr, og.indices)
    cfg = P.SamplerConfig(strategy="NS", fanouts=(5, 3), batch_size=100)

    def draw(seed):
        mb = P.build_minibatch(g, None, np.arange(100), cfg, np.random.default_rng(seed))
        return [{f: getattr(b.to_numpy(), f) for f in FIELDS} for b in mb.blocks]
    a, b, c = draw(5), draw(5), draw(6)
    assert all(np.array_equal(x[f], y[f]) for x, y in zip(a, b) for f in FIELDS)
    assert not all(np.array_equal(x[f], y[f]) for x, y in zip(a, c) for f in ("src_nodes", "edge_src"))


@pytest.mark.parametrize("dtype,C", [(torch.float32, 172), (torch.float64, 47), (torch.float32, 256)])
def test_softmax_xent_bias_fused_equals_separate(P, dtype, C):
    """gns_softmax_xent_bias (one launch: rows, mean loss, output bias
    gradient) == gns_softmax_xent + gns_dense_bwd_bias: dlogits bit for bit,
    the loss and bias gradient to the rounding of their (fixed, different)
    summation orders; repeated launches reuse the ticket counter."""
    from paper_2106_06150_b200 import _lib
    lib = _lib.lib()
    dt = 0 if dtype == torch.float32 else 1
    gen = torch.Generator(device="cuda").manual_seed(C)
    max_rows, pad = 1000, 1024
    labels = torch.randint(0, C, (5000,), device="cuda", dtype=torch.int32, generator=gen)
    targets = torch.randperm(5000, device="cuda", generator=gen)[:max_rows].sort().values.int()
    ws = _lib.workspace(lib.gns_softmax_xent_bias_workspace_size(max_rows, pad, C), "cuda", zero=True)
    ws2 = _lib.workspace(8 * 4096, "cuda")
    wsd = _lib.workspace(lib.gns_dense_bwd_workspace_size(pad, C), "cuda")
    for n in (1000, 777, 1):
        logits = torch.randn((pad, C), dtype=dtype, device="cuda", generator=gen) * 3
        n_dev = torch.tensor([n], dtype=torch.int32, device="cuda")
        g1 = torch.full((pad, C), 7.0, dtype=dtype, device="cuda")
        g2 = torch.full((pad, C), 7.0, dtype=dtype, device="cuda")
        l1 = torch.zeros(1, dtype=torch.float64, device="cuda")
        l2 = torch.zeros(1, dtype=torch.float64, device="cuda")
        b1 = torch.zeros(C, dtype=dtype, device="cuda")
        b2 = torch.zeros(C, dtype=dtype, device="cuda")
        _lib.call("gns_softmax_xent", dt, logits.data_ptr(), C, n_dev.data_ptr(), max_rows, pad, C,
                  labels.data_ptr(), targets.data_ptr(), g1.data_ptr(), l1.data_ptr(), ws2.data_ptr(), ws2.numel(),
                  _lib.stream_ptr())
        _lib.call("gns_dense_bwd_bias", dt, g1.data_ptr(), None, C, None, pad, C, None, b1.data_ptr(),
                  wsd.data_ptr(), wsd.numel(), _lib.stream_ptr())
        for _ in range(2):
            _lib.call("gns_softmax_xent_bias", dt, logits.data_ptr(), C, n_dev.data_ptr(), max_rows, pad, C,
                      labels.data_ptr(), targets.data_ptr(), g2.data_ptr(), l2.data_ptr(), b2.data_ptr(),
                      ws.data_ptr(), ws.numel(), _lib.stream_ptr())
            assert torch.equal(g1, g2)
            assert abs(float(l1) - float(l2)) <= 1e-13 * abs(float(l1))
            ref = g1[:n].double().sum(0)
            eps = 1e-6 if dtype == torch.float32 else 1e-13
            tol = eps * g1[:n].double().abs().sum(0) + eps
            assert torch.all((b2.double() - ref).abs() <= tol)
            assert torch.all((b1.double() - ref).abs() <= tol)
        # the loss is the reference's mean cross-entropy (model.py:189-200)
        lp = torch.log_softmax(logits[:n].double(), 1)
        want = -lp[torch.arange(n), labels[targets[:n].long()].long()].mean()
        assert abs(float(l2) - float(want)) <= (1e-5 if dtype == torch.float32 else 1e-12) * max(1.0, abs(float(want)))


def test_full_batch_forward_rows_of_any_degree(P):
    """evaluate()'s full-neighbourhood forward (model.py:168-186) is built
    from the CSR directly, so rows with more neighbours than the sampler's
    fanout limit (128) work: float64 logits equal (A h)/max(deg, 1) layer by
    layer (scipy order) on a graph with a 2000-neighbour hub."""
    import scipy.sparse as sp
    rng = np.random.default_rng(5)
    n = 3000
    e = np.concatenate([np.stack([np.zeros(2000, dtype=np.int64), rng.choice(np.arange(1, n), 2000, replace=False)], 1),
                        rng.integers(0, n, size=(6000, 2))])
    og = O.build_csr(e, n)
    assert np.diff(og.indptr).max() > 128
    feats = rng.normal(size=(n, 8)).astype(np.float32)
    labels = rng.integers(0, 4, n).astype(np.int32)
    g = P.Graph.from_numpy(n, og.indptr, og.indices, features=feats, labels=labels)
    params = P.init_params((8, 16, 4), seed=0, dtype=torch.float64)
    from paper_2106_06150_b200.train import full_batch_forward
    logits = full_batch_forward(g, params).cpu().numpy()
    w, b = params.model.export()
    h = feats.astype(np.float64)
    norm = np.maximum(np.diff(og.indptr), 1).astype(np.float64)
    adj = sp.csr_matrix((np.ones(og.num_edges), og.indices, og.indptr), shape=(n, n))
    for li in range(2):
        agg = (adj @ h) / norm[:, None]
        z = np.concatenate([h, agg], 1) @ w[li] + b[li]
        h = np.maximum(z, 0) if li == 0 else z
    np.testing.assert_allclose(logits, h, rtol=1e-10, atol=1e-10)


def _fp32_row_mean(indptr, indices, x):
    """float32 (sum over a row's sources in ascending order) / max(deg, 1):
    the kernels' FMA sequence with weight 1 (fma(1, x, acc) = x + acc, one
    float32 rounding per add, as numpy's float32 add)."""
    n = len(indptr) - 1
    deg = np.diff(indptr)
    row = np.repeat(np.arange(n), deg)
    srt = indices[np.lexsort((indices, row))]
    acc = np.zeros((n, x.shape[1]), np.float32)
    for t in range(int(deg.max(initial=0))):
        rows = np.nonzero(deg > t)[0]
        acc[rows] = acc[rows] + x[srt[indptr[rows] + t]]
    return acc / np.maximum(deg, 1).astype(np.float32)[:, None]


@pytest.mark.parametrize("dim", [8, 64, 128, 256, 768])
def test_spmm_fwd_full_block_long_rows_float32(P, dim):
    """float32 aggregation over the whole-graph block (evaluate()'s
    full-neighbourhood forward, model.py:168-186) with rows of 32, 33, 129
    and 2000 edges: every fp32 path (plain, relu input, relu' bits, fused
    gather) walks rows longer than a 32-edge window in ascending source order
    and is bit-identical to the sequential float32 sum."""
    from paper_2106_06150_b200 import _lib
    from paper_2106_06150_b200.train import full_block
    rng = np.random.default_rng(dim)
    n = 3000
    parts = [rng.integers(0, n, size=(6000, 2))]
    for hub, d in ((0, 2000), (1, 129), (2, 33), (3, 32)):
        nb = rng.choice(np.arange(4, n), d, replace=False)
        parts.append(np.stack([np.full(d, hub), nb], 1))
    og = O.build_csr(np.concatenate(parts), n)
    deg = np.diff(og.indptr)
    assert deg[0] >= 2000 and deg[1] >= 129
    g = P.Graph.from_numpy(n, og.indptr, og.indices)
    blk = full_block(g)
    feats = rng.normal(size=(n, dim)).astype(np.float32)
    h = torch.as_tensor(feats, device="cuda")
    for relu in (0, 1):
        x = np.maximum(feats, 0) if relu else feats
        want = np.concatenate([x, _fp32_row_mean(og.indptr, og.indices, x)], 1)
        out = torch.full((n + 3, 2 * dim), 7.0, device="cuda")
        _lib.call("gns_spmm_fwd", 0, h.data_ptr(), dim, dim, relu, blk._c, n, n, out.data_ptr(), 2 * dim,
                  _lib.stream_ptr())
        assert np.array_equal(out[:n].cpu().numpy(), want), relu
        if relu:
            lib = _lib.lib()
            bits = torch.zeros(lib.gns_relu_bits_size(n, dim) // 4, dtype=torch.int32, device="cuda")
            o2 = torch.full((n, 2 * dim), 7.0, device="cuda")
            _lib.call("gns_spmm_fwd_bits", h.data_ptr(), dim, dim, blk._c, n, n, o2.data_ptr(), 2 * dim,
                      bits.data_ptr(), _lib.stream_ptr())
            assert torch.equal(o2, out[:n])
        else:
            o3 = torch.full((n, 2 * dim), 9.0, device="cuda")
            ids = torch.arange(n, dtype=torch.int32, device="cuda")
            _lib.call("gns_spmm_fwd_gather", h.data_ptr(), dim, dim, blk._c, ids.data_ptr(), n, n, 0, 0,
                      o3.data_ptr(), 2 * dim, _lib.stream_ptr())
            assert torch.equal(o3, out[:n])


def test_generate_powerlaw_is_the_reference_graph(P):
    """P.generate_powerlaw (graph.py:172-205: host draws, device CSR) builds
    the reference's preferential-attachment graph: equal to the golden CSRs
    and to the oracle restatement; node data equal the device attribute
    generator's host restatement."""
    from oracle import gen
    with np.load(os.path.join(os.path.dirname(__file__), "golden", "golden_powerlaw.npz")) as z:
        gold = {k: z[k] for k in z.files}
    for tag in ("a", "b"):
        n, m, seed = (int(x) for x in gold[f"{tag}_args"])
        g = P.generate_powerlaw(n, m, seed, feature_dim=6, num_classes=3, train_frac=0.3)
        assert np.array_equal(g.indptr.cpu().numpy(), gold[f"{tag}_indptr"])
        assert np.array_equal(g.indices.cpu().numpy(), gold[f"{tag}_indices"])
        labels, tr, va, te = gen.node_attrs(n, 3, 0.3, seed)
        assert np.array_equal(g.labels.cpu().numpy(), labels)
        assert np.array_equal(g.train_mask.cpu().numpy(), tr)
        f = gen.features(n, 6, 3, labels, 3.0, seed)
        assert np.array_equal(g.features.cpu().numpy().view(np.uint32), f.view(np.uint32))
    with pytest.raises(ValueError):
        P.generate_powerlaw(5, 5, 0)


def test_spmm_bwd_long_transposed_rows(P):
    """Transposed rows of any length (hub sources: the neighbour of thousands
    of dst rows).  Rows of 65..256 entries are sorted by a warp in shared
    memory, longer ones by a CTA (in shared memory up to 8192, in place in
    global memory beyond); rows of more than 16 are summed by 32-entry
    segments spread over all warps.  float64 stays bit-exact with scipy's
    order (model.py:223-225); every float32 path (z mask, relu' bits, every
    lane-staged variant) gives the same dz bit for bit, within float32
    rounding of float64, and repeated launches over one transpose (the
    segments' generation counter) never reuse another launch's partials."""
    import types
    from paper_2106_06150_b200 import _lib
    from paper_2106_06150_b200.train import full_block
    rng = np.random.default_rng(3)
    n = 12000
    parts = [rng.integers(8, n, size=(20000, 2))]
    for hub, d in ((0, n - 1), (1, 3000), (2, 200), (3, 65), (4, 64), (5, 33), (6, 17), (7, 16)):
        nb = np.arange(1, n) if hub == 0 else rng.choice(np.arange(8, n), d, replace=False)
        parts.append(np.stack([np.full(len(nb), hub), nb], 1))
    og = O.build_csr(np.concatenate(parts), n)
    g = P.Graph.from_numpy(n, og.indptr, og.indices)
    blk = full_block(g)
    tlen = np.bincount(og.indices, minlength=n)
    assert tlen.max() > 8192 and np.any((tlen > 256) & (tlen <= 8192)) and np.any((tlen > 64) & (tlen <= 256))
    ref = types.SimpleNamespace(src_nodes=np.arange(n), dst_nodes=np.arange(n), edge_src=og.indices,
                                edge_dst=np.repeat(np.arange(n), np.diff(og.indptr)),
                                edge_weight=np.ones(og.num_edges), dst_degree=np.diff(og.indptr))
    E = og.num_edges
    lib = _lib.lib()
    for dim in (64, 256):
        ws = _lib.workspace(lib.gns_spmm_bwd_workspace_size(n, E, dim), "cuda")
        dcats = [np.random.default_rng(40 + k + dim).normal(size=(n, 2 * dim)) for k in range(2)]
        expect = OM.spmm_mean_bwd(ref, dcats[0], dim)
        dt = torch.as_tensor(dcats[0], device="cuda")
        dh = torch.empty((n, dim), dtype=torch.float64, device="cuda")
        _lib.call("gns_spmm_bwd", 1, dt.data_ptr(), 2 * dim, dim, blk._c, n, n, E, 0, None, None, dh.data_ptr(),
                  dim, ws.data_ptr(), ws.numel(), _lib.stream_ptr())
        assert np.array_equal(dh.cpu().numpy(), expect), dim
        # float32: z-mask path vs the relu'-bits paths
        z = torch.randn((n, dim), device="cuda", generator=torch.Generator(device="cuda").manual_seed(dim))
        bits = torch.zeros(lib.gns_relu_bits_size(n, dim) // 4, dtype=torch.int32, device="cuda")
        cat = torch.empty((n, 2 * dim), device="cuda")
        _lib.call("gns_spmm_fwd_bits", z.data_ptr(), dim, dim, blk._c, n, n, cat.data_ptr(), 2 * dim,
                  bits.data_ptr(), _lib.stream_ptr())
        d32 = [torch.as_tensor(d.astype(np.float32), device="cuda") for d in dcats]
        base = torch.empty((n, dim), device="cuda")
        db0 = torch.empty(dim, device="cuda")
        _lib.call("gns_spmm_bwd", 0, d32[0].data_ptr(), 2 * dim, dim, blk._c, n, n, E, 0, z.data_ptr(),
                  db0.data_ptr(), base.data_ptr(), dim, ws.data_ptr(), ws.numel(), _lib.stream_ptr())
        dz64 = expect * (z.double().cpu().numpy() > 0)
        np.testing.assert_allclose(base.double().cpu().numpy(), dz64, rtol=1e-3, atol=2e-3)
        out = torch.empty((n, dim), device="cuda")
        db = torch.empty(dim, device="cuda")
        try:
            for knob in range(6):
                _lib.call("gns_tune", b"spmm_bwd", knob)
                for k in (1, 0):   # another launch's dcat first, then the checked one
                    out.fill_(float("nan"))
                    _lib.call("gns_spmm_bwd_transposed_bits", d32[k].data_ptr(), 2 * dim, dim, blk._c, n, n, E, 0,
                              bits.data_ptr(), db.data_ptr(), out.data_ptr(), dim, ws.data_ptr(), ws.numel(),
                              _lib.stream_ptr())
                assert torch.equal(out, base), (dim, knob)
                np.testing.assert_allclose(db.cpu().numpy(), db0.cpu().numpy(), rtol=1e-4, atol=1e-2)
        finally:
            _lib.call("gns_tune", b"spmm_bwd", 4)


def test_engine_on_reference_powerlaw_graph(P):
    """The engine on the reference's own preferential-attachment graph
    (graph.py:172-205; hub sources give transposed rows of hundreds of
    entries, so the backward's segmented float32 path runs inside the
    captured steps, across graph replays): per-step losses within 1e-3 of the
    float64 façade on the same Philox batches, as at the bench dims."""
    from paper_2106_06150_b200.engine import GraphedTrainer
    g = P.generate_powerlaw(20000, 10, 0, feature_dim=64, num_classes=16, train_frac=0.5)
    cfg = P.SamplerConfig(strategy="GNS", fanouts=(15, 10, 5), batch_size=1000, cache_frac=0.01,
                          cache_mode="degree", seed=0)
    dims = (64, 256, 256, 16)
    tc = P.TrainConfig(lr=0.003, hidden_dim=256)
    params = P.init_params(dims, seed=0)
    state = P.AdamState.zeros_like(params)
    ref, tmax = [], 0
    for it in P.SamplerPool(g, cfg).iter_epoch(0):
        mb = it.minibatch
        tmax = max(tmax, int(torch.bincount(mb.blocks[1].edge_src.long()).max()))
        loss, grad = P.loss_and_grad(P.forward(mb, g, params), g.labels[mb.targets.long()])
        P.adam_step(params, P.backward(mb, g, params, grad), state, tc)
        ref.append(loss)
    assert tmax > 16   # long transposed rows in a backward block
    tr = GraphedTrainer(g, cfg, dims, tc, seed=0, tf32=False)
    got = []
    tr.run_epoch(0, on_step=lambda e, i, k: got.append(tr.loss_value()))
    assert len(got) == len(ref) >= 10
    np.testing.assert_allclose(got, ref, rtol=1e-3)
