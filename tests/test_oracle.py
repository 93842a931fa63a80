"""CPU tests: the oracle against known answers, golden fixtures and (when the
reference is mounted) the reference itself."""

import os
import re

import numpy as np
import pytest

from oracle import detmath, philox
from oracle import gns as O
from oracle import model as OM

from conftest import ROOT


# ---- Philox / Feistel ----------------------------------------------------------

@pytest.mark.parametrize("ctr,key,expect", [
    ((0, 0, 0, 0), (0, 0), (0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8)),
    ((0xffffffff,) * 4, (0xffffffff,) * 2, (0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd)),
    ((0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344), (0xa4093822, 0x299f31d0),
     (0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1)),
])
def test_philox_kat(ctr, key, expect):
    """Random123 kat_vectors for philox4x32-10."""
    assert tuple(int(x) for x in philox.philox4x32_10(*ctr, *key)) == expect


def test_uniform_is_key53_scaled():
    k = philox.key53(1, 2, 3, philox.stream_word(32, 1, 0), 4, np.arange(100))
    u = philox.uniform(1, 2, 3, philox.stream_word(32, 1, 0), 4, np.arange(100))
    assert np.all(k < 2 ** 53)
    assert np.array_equal(u, k.astype(np.float64) / 2.0 ** 53)
    assert np.all((u >= 0) & (u < 1))


@pytest.mark.parametrize("n", [1, 2, 3, 5, 17, 1000, 4097])
def test_feistel_is_bijection(n):
    p = philox.feistel_permute(np.arange(n), n, 7, 3)
    assert sorted(p.tolist()) == list(range(n))


# ---- deterministic transcendental functions -------------------------------------

def _ulps(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return np.max(np.abs(a - b) / np.spacing(np.maximum(np.abs(a), np.abs(b))))


def test_detmath_close_to_libm():
    rng = np.random.default_rng(1)
    x = np.concatenate([rng.random(50000), 10 ** -rng.uniform(0, 16, 50000), [1.0, 2 ** -53]])
    x = x[x > 0]
    assert _ulps(detmath.det_log(x), np.log(x)) <= 4
    x1 = -np.concatenate([rng.random(50000), 10 ** -rng.uniform(0, 16, 50000), [0.999999999999999, .5]])
    assert _ulps(detmath.det_log1p(x1), np.log1p(x1)) <= 4
    y = -np.concatenate([rng.random(50000) * 50, 10 ** -rng.uniform(0, 16, 50000), [0.5, 40, 45]])
    assert _ulps(detmath.det_expm1(y), np.expm1(y)) <= 4


def test_cuda_constants_match_oracle():
    """The .cuh coefficient tables are the oracle's correctly rounded values."""
    src = open(os.path.join(ROOT, "paper_2106_06150_b200", "csrc", "gns_common.cuh")).read()

    def table(name):
        body = re.search(name + r"\[\d+\] = \{(.*?)\};", src, re.S).group(1)
        return [float.fromhex(t.strip()) for t in body.split(",") if t.strip()]

    assert table("kAtanhC") == detmath.ATANH_C
    assert table("kExpC") == detmath.EXP_C
    for name, val in [("GNS_LN2_HI", detmath.LN2_HI), ("GNS_LN2_LO", detmath.LN2_LO),
                      ("GNS_INV_LN2", detmath.INV_LN2), ("GNS_SQRT_HALF", detmath.SQRT_HALF),
                      ("GNS_ONE_MINUS_1EM15", detmath.ONE_MINUS_1EM15)]:
        m = re.search(r"#define " + name + r" (\S+)", src)
        assert float.fromhex(m.group(1)) == val, name


# ---- KATs (SPEC.md examples) -----------------------------------------------------

def test_spec_kats(golden):
    kat = golden["kat"]
    assert abs(detmath.inclusion_prob(0.01, 100) - 0.63397) < 1e-5
    assert _ulps(detmath.inclusion_prob(0.01, 100), kat["inclusion_0p01_100"]) <= 4
    star = O.build_csr([(0, 1), (0, 2), (0, 3)], 4)
    assert np.array_equal(O.degree_probs(star), kat["star_probs"])
    g = O.build_csr([(0, 1)], 2)
    assert g.indptr.tolist() == [0, 1, 2] and g.indices.tolist() == [1, 0]
    p = kat["incl_p"]
    for cs in (1, 100, 111000):
        assert _ulps(detmath.inclusion_prob(p, cs), kat[f"incl_ref_{cs}"]) <= 4


def test_sample_cache_edge_cases():
    w = np.array([0.0, 0.5, 0.25, 0.25])
    assert O.sample_cache(w, 0).tolist() == []
    assert O.sample_cache(w, 3).tolist() == [1, 2, 3]
    assert O.sample_cache(w, 10).tolist() == [1, 2, 3]
    assert len(O.sample_cache(w, 2, seed=5, epoch=1)) == 2


# ---- oracle vs golden reference outputs -----------------------------------------

def _graph_from(gold):
    return O.OGraph(num_nodes=len(gold["indptr"]) - 1, indptr=gold["indptr"], indices=gold["indices"])


def _cache_from(g, gold, ids):
    mask = np.zeros(g.num_nodes, dtype=bool)
    mask[ids] = True
    return O.OCache(ids=ids, mask=mask, inclusion=gold["cache_inclusion_det"],
                    cached_indptr=gold["cached_indptr"], cached_indices=gold["cached_indices"])


CASES = {"gns": dict(strategy="GNS", fanouts=(15, 10, 5), input_layer_cache_only=True, seed=0),
         "gnsfill": dict(strategy="GNS", fanouts=(6, 4), input_layer_cache_only=False, seed=3),
         "ns": dict(strategy="NS", fanouts=(15, 10, 5), input_layer_cache_only=True, seed=0)}


class _Cfg:
    def __init__(self, **kw):
        self.__dict__.update(kw)


def test_oracle_matches_golden_sampler(golden):
    gold = golden["sampler"]
    g = _graph_from(gold)
    ids = gold["philox_cache_ids"]
    assert np.array_equal(O.sample_cache(O.degree_probs(g), 40, seed=0, epoch=0), ids)
    oc = O.build_cache(g, O.degree_probs(g), 40, ids=ids)
    assert np.array_equal(oc.cached_indptr, gold["cached_indptr"])
    assert np.array_equal(oc.cached_indices, gold["cached_indices"])
    assert _ulps(oc.inclusion, gold["cache_inclusion_ref"]) <= 4
    assert np.array_equal(oc.inclusion, gold["cache_inclusion_det"])
    ci, cx = O.cached_csr_by_filter(g, oc.mask)
    assert np.array_equal(ci, oc.cached_indptr) and np.array_equal(cx, oc.cached_indices)
    cache = _cache_from(g, gold, ids)
    for name, kw in CASES.items():
        cfg = _Cfg(**kw)
        for epoch, index in ((0, 0), (2, 5)):
            mb = O.build_minibatch(g, cache if cfg.strategy == "GNS" else None, gold[f"{name}_targets"], cfg,
                                   O.PhiloxKeys(cfg.seed, epoch, index))
            pre = f"{name}_e{epoch}_i{index}"
            assert len(mb.blocks) == int(gold[f"{pre}_nblocks"])
            for i, b in enumerate(mb.blocks):
                for f in ("dst_nodes", "src_nodes", "edge_src", "edge_dst", "edge_weight", "edge_cached",
                          "dst_degree"):
                    assert np.array_equal(getattr(b, f), gold[f"{pre}_b{i}_{f}"]), (pre, i, f)
            O.validate_minibatch(g, mb)


def test_oracle_model_matches_golden(golden):
    gold = golden["model"]
    g = O.OGraph(num_nodes=len(gold["indptr"]) - 1, indptr=gold["indptr"], indices=gold["indices"],
                 features=gold["features"], labels=gold["labels"], train_mask=gold["train_mask"])
    w = O.degree_probs(g)
    oc = O.build_cache(g, w, 40, ids=gold["cache_ids"])
    cfg = _Cfg(strategy="GNS", fanouts=(5, 3), input_layer_cache_only=True, seed=0)
    params = OM.init_params((16, 32, 4), seed=0)
    st = OM.OAdam.zeros_like(params)
    batches = O.epoch_targets(g, 50, 0, 0)
    losses = []
    for index, targets in enumerate(batches[:6]):
        mb = O.build_minibatch(g, oc, targets, cfg, O.PhiloxKeys(0, 0, index))
        losses.append(OM.train_step(mb, g.features, g.labels, params, st))
    np.testing.assert_allclose(losses, gold["losses"], rtol=1e-12)


# ---- oracle vs the live reference (build container only) -------------------------

def test_oracle_numpy_stream_equals_reference(gb):
    """With the reference's own PCG64 streams the restatement is bit-exact."""
    g = gb.generate_powerlaw(3000, 4, 0)
    cfg = gb.SamplerConfig(strategy="GNS", fanouts=(15, 10, 5), batch_size=100, cache_frac=0.05,
                           cache_mode="degree", seed=0)
    probs = gb.degree_probs(g)
    cs = O.cache_size_for(g, 0.05)
    rc = gb.build_cache(g, probs, cs, epoch=0, rng_seed=[0, 33, 0])
    oc = O.build_cache(g, O.degree_probs(g), cs, numpy_seed=[0, 33, 0])
    assert np.array_equal(oc.ids, rc.nodes.ids)
    assert np.array_equal(oc.cached_indptr, rc.cached_indptr)
    assert np.array_equal(oc.cached_indices, rc.cached_indices)
    oc_ref = O.OCache(ids=rc.nodes.ids, mask=rc.nodes.mask, inclusion=rc.inclusion,
                      cached_indptr=rc.cached_indptr, cached_indices=rc.cached_indices)
    batches = gb.pool.epoch_targets(g, cfg, 0)
    ob = O.epoch_targets(g, 100, 0, 0, numpy_mode=True)
    assert all(np.array_equal(a, b) for a, b in zip(batches, ob))
    for idx in range(2):
        mr = gb.build_minibatch(g, rc, batches[idx], cfg, np.random.default_rng([0, 32, 0, idx]))
        mo = O.build_minibatch(g, oc_ref, batches[idx], cfg, O.NumpyStream(np.random.default_rng([0, 32, 0, idx])))
        for ba, bb in zip(mr.blocks, mo.blocks):
            for f in ("dst_nodes", "src_nodes", "edge_src", "edge_dst", "edge_weight", "edge_cached", "dst_degree"):
                assert np.array_equal(getattr(ba, f), getattr(bb, f)), f


def test_oracle_model_equals_reference(gb):
    g = gb.generate_sbm(300, 3, 0.05, 0.01, seed=2, feature_dim=8)
    cfg = gb.SamplerConfig(strategy="NS", fanouts=(4, 3), batch_size=40, seed=0)
    mb = gb.build_minibatch(g, None, np.arange(0, 300, 7), cfg, np.random.default_rng(0))
    p_ref = gb.init_params((8, 16, 3), seed=0)
    p_or = OM.init_params((8, 16, 3), seed=0)
    lr, _ = OM.forward_pass(mb, g.features, p_or)
    assert np.array_equal(lr, gb.forward(mb, g.features, p_ref))
    loss, grad = OM.loss_and_grad(lr, g.labels[mb.targets])
    loss_r, grad_r = gb.loss_and_grad(lr, g.labels[mb.targets])
    assert loss == loss_r and np.array_equal(grad, grad_r)
    dw, db = OM.backward(mb, g.features, p_or, grad)
    gr = gb.backward(mb, g.features, p_ref, grad)
    for a, b in zip(dw + db, gr.weights + gr.biases):
        assert np.array_equal(a, b)


def test_oracle_random_walk_probs_equals_reference(gb):
    g = gb.generate_powerlaw(2000, 3, 1)
    rng = np.random.default_rng(0)
    mask = rng.random(2000) < 0.1
    g = g.replace(train_mask=mask)
    ts = gb.graph.train_set(g)
    for L, fan in ((1, (3,)), (3, (15, 10, 5))):
        ref = gb.random_walk_probs(g, ts, fan, L).weights
        ours_np = O.random_walk_probs(g, ts.ids, fan, L, device_order=False)
        assert np.array_equal(ref, ours_np)                     # same iterate + same sum
        ours = O.random_walk_probs(g, ts.ids, fan, L)           # build's fixed-order sum
        assert _ulps(ours, ref) <= 4
        assert abs(ours.sum() - 1.0) < 1e-12
    # SPEC.md:144-146 examples: path 0-1-2, train={0}, fanout 1, L=1 -> [2/3, 1/3, 0]
    path = O.build_csr([(0, 1), (1, 2)], 3)
    np.testing.assert_allclose(O.random_walk_probs(path, [0], (1,), 1), [2 / 3, 1 / 3, 0.0], rtol=1e-15)


def test_oracle_isolated_fraction_equals_reference(gb):
    g = gb.generate_powerlaw(500, 3, 2)
    cfg = gb.SamplerConfig(strategy="NS", fanouts=(2, 1), batch_size=50, seed=0)
    mb = gb.build_minibatch(g, None, np.arange(0, 500, 5), cfg, np.random.default_rng(1))
    assert O.isolated_fraction(mb) == gb.isolated_fraction(mb)


def test_oracle_gns_exact_equals_reference(gb):
    """sampling.py:269-296 table + gns-exact weights (sampling.py:238-250)."""
    g = gb.generate_powerlaw(800, 3, 4)
    probs = gb.degree_probs(g)
    w = O.degree_probs(g)
    for k, co in ((5, True), (6, False)):
        ref_t = gb.estimate_edge_inclusion(g, probs, 40, k, co, resamples=8, seed=3)
        ours_t = O.estimate_edge_inclusion(g, w, 40, k, co, resamples=8, numpy_seed=3)
        assert np.array_equal(ref_t, ours_t)
    cfg = gb.SamplerConfig(strategy="GNS", fanouts=(6, 5), batch_size=50, cache_frac=0.05, cache_mode="degree",
                           weight_policy="gns-exact", seed=0)
    # a large cache so every realised cached neighbour has q > 0 (the
    # reference raises InvariantError otherwise, sampling.py:248-249)
    tables = {(6, False): gb.estimate_edge_inclusion(g, probs, 400, 6, False, resamples=64, seed=3),
              (5, True): gb.estimate_edge_inclusion(g, probs, 400, 5, True, resamples=64, seed=3)}
    rc = gb.build_cache(g, probs, 400, epoch=0, rng_seed=[0, 33, 0])
    oc = O.OCache(ids=rc.nodes.ids, mask=rc.nodes.mask, inclusion=rc.inclusion, cached_indptr=rc.cached_indptr,
                  cached_indices=rc.cached_indices)
    targets = np.arange(0, 800, 16)
    mr = gb.build_minibatch(g, rc, targets, cfg, np.random.default_rng(5), exact_tables=tables)
    mo = O.build_minibatch(g, oc, targets, cfg, O.NumpyStream(np.random.default_rng(5)), exact_tables=tables)
    for ba, bb in zip(mr.blocks, mo.blocks):
        for f in ("src_nodes", "edge_src", "edge_dst", "edge_weight", "edge_cached"):
            assert np.array_equal(getattr(ba, f), getattr(bb, f)), f


# ---- host restatement of the synthetic-graph generator (oracle/gen.cc) -------------

@pytest.mark.parametrize("n,m,alpha,offset,seed", [(5000, 20000, 0.6, 10.0, 7), (300000, 400000, 0.6, 300.0, 0),
                                                    (1000, 8000, 0.3, 2.0, 5)])
def test_host_generator_pairs_and_csr(n, m, alpha, offset, seed):
    """oracle/gen.cc pair draw == its numpy restatement (Philox + the
    deterministic pow + Feistel), and its CSR pipeline == the restatement of
    the reference's build_csr (graph.py:142-169) on those pairs."""
    from oracle import gen
    u, v = gen.gen_pairs(n, alpha, offset, seed, 0, m)
    un, vn = gen.gen_pairs_np(n, alpha, offset, seed, 0, m)
    assert np.array_equal(u, un) and np.array_equal(v, vn)
    ip, ix = gen.powerlaw_csr(n, m, alpha, offset, seed, threads=3)
    og = O.build_csr(np.stack([u, v], 1), n)
    assert np.array_equal(ip, og.indptr) and np.array_equal(ix, og.indices)
    ip2, ix2 = gen.build_csr_pairs(n, u, v, threads=2)
    assert np.array_equal(ip2, og.indptr) and np.array_equal(ix2, og.indices)


def test_host_generator_attributes():
    from oracle import gen
    n = 20000
    lab, tr, va, te = gen.node_attrs(n, 13, 0.1, 3)
    ref = gen.node_attrs_np(n, 13, 0.1, 3)
    for a, b in zip((lab, tr, va, te), ref):
        assert np.array_equal(a, b)
    assert lab.min() >= 0 and lab.max() < 13 and not (tr & va).any() and (tr | va | te).all()
    assert abs(tr.mean() - 0.1) < 0.01
    f = gen.features(n, 30, 13, lab, 3.0, 3, threads=4)
    fn = gen.features_np(n, 30, 13, lab, 3.0, 3)
    assert np.array_equal(f.view(np.uint32), fn.view(np.uint32))
    assert f.shape == (n, 32) and not f[:, 30:].any()
    # class-mean + noise: per-class means separate, noise sd ~ 3
    assert 2.5 < f[:, :30].std() < 3.6


def test_detmath_exp_pow_close_to_libm():
    y = np.random.default_rng(0).uniform(-40, 40, 20000)
    np.testing.assert_allclose(detmath.det_exp(y), np.exp(y), rtol=4e-16 * 8)
    a = np.random.default_rng(1).uniform(1.0, 2000.0, 20000)
    np.testing.assert_allclose(detmath.det_pow(a, 2.5), np.power(a, 2.5), rtol=1e-14)


def test_host_cached_csr_equals_build_cache():
    """cache.py:185-197 by filtering (oracle/gen.cc og_cached_csr) equals
    build_cache's gather_rows + lexsort construction."""
    from oracle import gen
    g = gen.powerlaw_graph(20000, 100000, 0.6, 10.0, 3)
    w = O.degree_probs(g)
    c = O.build_cache(g, w, 300, numpy_seed=[0, 33, 0])
    ip, ix = gen.cached_csr(g.indptr, g.indices, c.mask, threads=3)
    assert np.array_equal(ip, c.cached_indptr) and np.array_equal(ix, c.cached_indices)



def _powerlaw_golden():
    with np.load(os.path.join(ROOT, "tests", "golden", "golden_powerlaw.npz")) as z:
        return {k: z[k] for k in z.files}


def test_powerlaw_attach_matches_reference_golden():
    """oracle.gns.generate_powerlaw (graph.py:172-205 restated, batched
    draws) reproduces the reference's graphs: two small CSRs exactly and the
    BASELINE config-1 graph generate_powerlaw(100000, 10, 0) by digest."""
    import hashlib
    gold = _powerlaw_golden()
    for tag in ("a", "b"):
        n, m, seed = (int(x) for x in gold[f"{tag}_args"])
        g = O.generate_powerlaw(n, m, seed)
        assert np.array_equal(g.indptr, gold[f"{tag}_indptr"])
        assert np.array_equal(g.indices, gold[f"{tag}_indices"])
    n, m, seed = (int(x) for x in gold["cfg1_args"])
    g = O.generate_powerlaw(n, m, seed)
    assert len(g.indices) == int(gold["cfg1_num_edges"]) == 1_999_800
    assert hashlib.sha256(np.ascontiguousarray(g.indptr, np.int64)).hexdigest() == str(gold["cfg1_indptr_sha256"])
    assert hashlib.sha256(np.ascontiguousarray(g.indices, np.int64)).hexdigest() == str(gold["cfg1_indices_sha256"])
    with pytest.raises(ValueError):
        O.generate_powerlaw(3, 3, 0)
    with pytest.raises(ValueError):
        O.generate_powerlaw(10, 0, 0)


def test_powerlaw_attach_equals_live_reference(gb):
    for n, m, seed in ((60, 2, 3), (1500, 4, 9)):
        r = gb.generate_powerlaw(n, m, seed)
        o = O.generate_powerlaw(n, m, seed)
        assert np.array_equal(o.indptr, r.indptr) and np.array_equal(o.indices, r.indices)
