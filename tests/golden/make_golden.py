"""Generate golden fixtures by running the REFERENCE (gnsbench) in this container.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py [powerlaw]

The reference is Python and cannot travel to the GPU box, so its outputs on
small inputs are committed here (``golden_*.npz``).  Each fixture records the
inputs (graph CSR, cache ids, targets, Philox key) and the reference's outputs
when fed the build's Philox keys through its duck-typed ``rng.random(n)``
(``sampling.py:166,214,233``) via ``oracle.gns.ReplayRng``.  GPU tests compare
the B200 kernels against these arrays bit for bit.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

import gnsbench as gb  # noqa: E402

from oracle import gns as O  # noqa: E402


def _with_det_inclusion(gb, cache, w):
    from oracle import detmath
    incl = detmath.inclusion_prob(w, len(cache.nodes))
    if len(cache.nodes) >= int((w > 0).sum()):
        incl = np.where(w > 0, 1.0, incl)
    return gb.CacheState(nodes=cache.nodes, inclusion=np.asarray(incl, dtype=np.float64),
                         cached_indptr=cache.cached_indptr, cached_indices=cache.cached_indices,
                         epoch=cache.epoch, source_probs=cache.source_probs)


def _block_arrays(prefix, mb, out):
    for i, b in enumerate(mb.blocks):
        for f in ("dst_nodes", "src_nodes", "edge_src", "edge_dst", "edge_weight", "edge_cached",
                  "dst_degree"):
            out[f"{prefix}_b{i}_{f}"] = np.asarray(getattr(b, f))


def make_sampler_golden():
    out = {}
    g = gb.generate_powerlaw(2000, 4, 0)
    out["indptr"], out["indices"] = g.indptr, g.indices
    probs = gb.degree_probs(g)
    out["probs"] = probs.weights
    cs = 40
    # reference cache draw under its own numpy stream (statistical reference)
    ref_cache = gb.build_cache(g, probs, cs, epoch=0, rng_seed=[0, 33, 0])
    out["ref_cache_ids_numpy"] = ref_cache.nodes.ids
    # the build's Philox cache draw, injected into the reference (cache replay)
    w = O.degree_probs(g)
    ids = O.sample_cache(w, cs, seed=0, epoch=0)
    out["philox_cache_ids"] = ids
    orig = gb.cache.sample_cache
    gb.cache.sample_cache = lambda probs_, size_, seed_: gb.NodeSet.from_ids(ids, g.num_nodes)
    try:
        cache = gb.build_cache(g, probs, cs, epoch=0, rng_seed=[0, 33, 0])
    finally:
        gb.cache.sample_cache = orig
    out["cache_inclusion_ref"] = cache.inclusion
    # "bit-exact given the same inclusion vector": the reference samples with the
    # build's Eq. 9 values (libm vs the deterministic series differ by <= 4 ulp)
    cache = _with_det_inclusion(gb, cache, w)
    out["cache_inclusion_det"] = cache.inclusion
    out["cached_indptr"] = cache.cached_indptr
    out["cached_indices"] = cache.cached_indices
    oc = O.OCache(ids=cache.nodes.ids, mask=cache.nodes.mask, inclusion=cache.inclusion,
                  cached_indptr=cache.cached_indptr, cached_indices=cache.cached_indices)
    cases = [("gns", gb.SamplerConfig(strategy="GNS", fanouts=(15, 10, 5), batch_size=64,
                                      cache_mode="degree", seed=0)),
             ("gnsfill", gb.SamplerConfig(strategy="GNS", fanouts=(6, 4), batch_size=64,
                                          cache_mode="degree", input_layer_cache_only=False, seed=3)),
             ("ns", gb.SamplerConfig(strategy="NS", fanouts=(15, 10, 5), batch_size=64, seed=0))]
    rs = np.random.default_rng(7)
    for name, cfg in cases:
        targets = rs.choice(g.num_nodes, size=64, replace=False)
        out[f"{name}_targets"] = targets
        for epoch, index in ((0, 0), (2, 5)):
            rec = []
            O.build_minibatch(g, oc if cfg.strategy == "GNS" else None, targets, cfg,
                              O.PhiloxKeys(cfg.seed, epoch, index, record=rec))
            mb = gb.build_minibatch(g, cache if cfg.strategy == "GNS" else None, targets, cfg,
                                    O.ReplayRng(rec))
            _block_arrays(f"{name}_e{epoch}_i{index}", mb, out)
            out[f"{name}_e{epoch}_i{index}_nblocks"] = np.array(len(mb.blocks))
    # random-walk cache distribution (cache.py:61-84) with a 10% train set
    wmask = np.random.default_rng(11).random(g.num_nodes) < 0.1
    out["walk_train_ids"] = np.flatnonzero(wmask)
    ts = gb.NodeSet.from_mask(wmask)
    out["walk_probs_L3"] = gb.random_walk_probs(g, ts, (15, 10, 5), 3).weights
    out["walk_probs_L1"] = gb.random_walk_probs(g, ts, (4,), 1).weights
    np.savez_compressed(os.path.join(HERE, "golden_sampler.npz"), **out)


def make_kat_golden():
    out = {
        "inclusion_0p01_100": np.array(gb.inclusion_prob(0.01, 100)),
        "gns_weight_0p01_100_10_4": np.array(gb.gns_weight_paper(0.01, 100, 10, 4)),
        "gns_weight_pc_half": np.array(1.0 / (0.5 * 5 / 5)),
        "star_probs": gb.degree_probs(gb.build_csr([(0, 1), (0, 2), (0, 3)], 4)).weights,
    }
    p = np.concatenate([10.0 ** -np.linspace(0, 12, 200), [0.0, 1.0, 0.5]])
    out["incl_p"] = p
    for cs in (1, 100, 111000):
        out[f"incl_ref_{cs}"] = gb.inclusion_prob(p, cs)
    np.savez_compressed(os.path.join(HERE, "golden_kat.npz"), **out)


def make_model_golden():
    """Reference fp64 trainer (model.py:279-285 loop body) for 6 steps on an SBM
    graph with replayed Philox keys and a Philox cache."""
    out = {}
    g = gb.generate_sbm(400, 4, 0.05, 0.005, seed=1, feature_dim=16)
    out["indptr"], out["indices"] = g.indptr, g.indices
    out["features"], out["labels"] = g.features, g.labels
    out["train_mask"] = g.train_mask
    cfg = gb.SamplerConfig(strategy="GNS", fanouts=(5, 3), batch_size=50, cache_frac=0.1,
                           cache_mode="degree", seed=0)
    w = O.degree_probs(g)
    cs = int(round(cfg.cache_frac * g.num_nodes))
    ids = O.sample_cache(w, cs, seed=0, epoch=0)
    probs = gb.degree_probs(g)
    orig = gb.cache.sample_cache
    gb.cache.sample_cache = lambda probs_, size_, seed_: gb.NodeSet.from_ids(ids, g.num_nodes)
    try:
        cache = gb.build_cache(g, probs, cs, epoch=0, rng_seed=[0, 33, 0])
    finally:
        gb.cache.sample_cache = orig
    cache = _with_det_inclusion(gb, cache, w)
    oc = O.OCache(ids=cache.nodes.ids, mask=cache.nodes.mask, inclusion=cache.inclusion,
                  cached_indptr=cache.cached_indptr, cached_indices=cache.cached_indices)
    dims = (16, 32, 4)
    params = gb.init_params(dims, seed=0)
    state = gb.AdamState.zeros_like(params)
    tc = gb.TrainConfig(lr=0.003)
    batches = O.epoch_targets(g, cfg.batch_size, cfg.seed, 0)
    losses = []
    for index, targets in enumerate(batches[:6]):
        rec = []
        O.build_minibatch(g, oc, targets, cfg, O.PhiloxKeys(cfg.seed, 0, index, record=rec))
        mb = gb.build_minibatch(g, cache, targets, cfg, O.ReplayRng(rec))
        logits = gb.forward(mb, g.features, params)
        loss, grad = gb.loss_and_grad(logits, g.labels[mb.targets])
        grads = gb.backward(mb, g.features, params, grad)
        gb.adam_step(params, grads, state, tc)
        losses.append(loss)
    out["losses"] = np.array(losses)
    for i, (wt, b) in enumerate(zip(params.weights, params.biases)):
        out[f"final_w{i}"], out[f"final_b{i}"] = wt, b
    out["cache_ids"] = ids
    np.savez_compressed(os.path.join(HERE, "golden_model.npz"), **out)


def _philox_cache(g, probs, w, cs, epoch):
    """The build's Philox cache of ``epoch`` (key [0, 33, epoch]) injected into
    the reference's build_cache (cache replay), deterministic inclusion."""
    ids = O.sample_cache(w, cs, seed=0, epoch=epoch)
    orig = gb.cache.sample_cache
    gb.cache.sample_cache = lambda probs_, size_, seed_: gb.NodeSet.from_ids(ids, g.num_nodes)
    try:
        cache = gb.build_cache(g, probs, cs, epoch=epoch, rng_seed=[0, 33, epoch])
    finally:
        gb.cache.sample_cache = orig
    cache = _with_det_inclusion(gb, cache, w)
    oc = O.OCache(ids=cache.nodes.ids, mask=cache.nodes.mask, inclusion=cache.inclusion,
                  cached_indptr=cache.cached_indptr, cached_indices=cache.cached_indices)
    return cache, oc


def make_train_golden():
    """SPEC.md:371-373,519 convergence task: SBM(2000, 4 blocks, 0.02, 0.002),
    16-d features, GNS cache 10% P=1, fanouts (15,10,5), batch 100, hidden 64,
    10 epochs (model.py:257-307).  (a) the reference's fp64 trainer on the
    build's Philox keys (cache, epoch permutation and per-batch keys replayed):
    every step's loss, per-epoch mean loss and micro-F1; (b) the reference
    free-running on its own PCG64 streams (gnsbench.train), GNS and NS: final
    F1 (the SPEC's 2-point tolerance is against these)."""
    out = {}
    g = gb.generate_sbm(2000, 4, 0.02, 0.002, seed=0, feature_dim=16)
    for f in ("indptr", "indices", "features", "labels", "train_mask", "val_mask", "test_mask"):
        out[f] = np.asarray(getattr(g, f))
    cfg = gb.SamplerConfig(strategy="GNS", fanouts=(15, 10, 5), batch_size=100, cache_frac=0.1,
                           cache_period=1, cache_mode="degree", seed=0)
    tc = gb.TrainConfig(epochs=10, seed=0, hidden_dim=64, lr=0.003)
    dims = (16, 64, 64, 4)
    params = gb.init_params(dims, seed=0)
    state = gb.AdamState.zeros_like(params)
    probs = gb.degree_probs(g)
    w = O.degree_probs(g)
    cs = int(round(cfg.cache_frac * g.num_nodes))
    losses, epoch_loss, f1s = [], [], []
    for epoch in range(tc.epochs):
        cache, oc = _philox_cache(g, probs, w, cs, epoch)
        el = []
        for index, targets in enumerate(O.epoch_targets(g, cfg.batch_size, cfg.seed, epoch)):
            rec = []
            O.build_minibatch(g, oc, targets, cfg, O.PhiloxKeys(cfg.seed, epoch, index, record=rec))
            mb = gb.build_minibatch(g, cache, targets, cfg, O.ReplayRng(rec))
            logits = gb.forward(mb, g.features, params)
            loss, grad = gb.loss_and_grad(logits, g.labels[mb.targets])
            grads = gb.backward(mb, g.features, params, grad)
            gb.adam_step(params, grads, state, tc)
            el.append(loss)
        losses += el
        epoch_loss.append(np.mean(el))
        f = gb.model.evaluate(g, params)
        f1s.append([f["train"], f["val"], f["test"]])
    out["losses"] = np.array(losses)
    out["epoch_loss"] = np.array(epoch_loss)
    out["f1"] = np.array(f1s)
    for strat, kw in (("gns", dict(cache_frac=0.1, cache_period=1, cache_mode="degree")), ("ns", {})):
        c2 = gb.SamplerConfig(strategy=strat.upper(), fanouts=(15, 10, 5), batch_size=100, seed=0, **kw)
        rep = gb.train(g, c2, tc)
        out[f"free_{strat}_test_f1"] = np.array(rep.final_test_f1)
        out[f"free_{strat}_epoch_loss"] = np.array([r.loss for r in rep.rows])
    np.savez_compressed(os.path.join(HERE, "golden_train.npz"), **out)


def make_stat_golden():
    """The reference's own cache draw (cache.py:87-103, numpy exponential race
    with seeds [1, 33, e]) repeated R times on a small power-law graph: per-node
    inclusion counts for the two-sample |C| > 1 test of the device draw."""
    g = gb.generate_powerlaw(60, 2, 3)
    probs = gb.degree_probs(g)
    R, cs = 20000, 8
    counts = np.zeros(g.num_nodes, dtype=np.int64)
    for e in range(R):
        counts[gb.sample_cache(probs, cs, [1, 33, e]).ids] += 1
    np.savez_compressed(os.path.join(HERE, "golden_stat.npz"), indptr=g.indptr, indices=g.indices,
                        cache_size=np.array(cs), draws=np.array(R), ref_counts=counts)


def make_format_golden():
    """A GNSG v1 file written by the reference's save_binary (graph.py:283-299)."""
    g = gb.generate_sbm(60, 3, 0.3, 0.05, seed=0, feature_dim=5)
    gb.save_binary(g, os.path.join(HERE, "golden_sbm60.gnsg"))


def make_powerlaw_golden():
    """The reference's preferential-attachment generator (graph.py:172-205):
    two small CSRs, and SHA-256 digests of the BASELINE config-1 graph
    generate_powerlaw(100000, 10, 0) (int64 indptr, int64 indices)."""
    import hashlib
    out = {}
    for tag, (n, m, seed) in {"a": (500, 3, 2), "b": (3000, 10, 0)}.items():
        g = gb.generate_powerlaw(n, m, seed)
        out[f"{tag}_args"] = np.array([n, m, seed])
        out[f"{tag}_indptr"] = g.indptr
        out[f"{tag}_indices"] = g.indices.astype(np.int32)
    g = gb.generate_powerlaw(100000, 10, 0)
    out["cfg1_args"] = np.array([100000, 10, 0])
    out["cfg1_num_edges"] = np.array(len(g.indices))
    out["cfg1_indptr_sha256"] = np.array(hashlib.sha256(np.ascontiguousarray(g.indptr, np.int64)).hexdigest())
    out["cfg1_indices_sha256"] = np.array(hashlib.sha256(np.ascontiguousarray(g.indices, np.int64)).hexdigest())
    np.savez_compressed(os.path.join(HERE, "golden_powerlaw.npz"), **out)


if __name__ == "__main__":
    if sys.argv[1:] == ["powerlaw"]:
        make_powerlaw_golden()
        sys.exit(0)
    make_powerlaw_golden()
    make_format_golden()
    make_kat_golden()
    make_sampler_golden()
    make_model_golden()
    make_train_golden()
    make_stat_golden()
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))
