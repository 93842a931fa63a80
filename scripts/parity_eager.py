"""Eager P.build_minibatch vs the oracle on a bench workload's graph and the
engine's epoch-0 cache, for a few batches, per gns_tune setting; prints the
first mismatching layer/field.

    python scripts/parity_eager.py --config cfg1 "" "warp_sort=0"
"""

from __future__ import annotations

import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("settings", nargs="*", default=[""])
    ap.add_argument("--config", default="cfg1")
    ap.add_argument("--batches", type=int, default=4)
    args = ap.parse_args()
    import bench
    import paper_2106_06150_b200 as P
    from oracle import gns as O
    from paper_2106_06150_b200 import _lib
    from paper_2106_06150_b200.engine import GraphedTrainer

    c = bench.CONFIGS[args.config]
    g, _ = bench.make_graph(P, c)
    cfg = P.SamplerConfig(strategy="GNS", fanouts=bench.FANOUTS, batch_size=bench.BATCH, cache_frac=c["cache"],
                          cache_mode="degree", input_layer_cache_only=True, seed=0)
    dims = (c["dim"], c["hidden"], c["hidden"], c["classes"])
    te = GraphedTrainer(g, cfg, dims, P.TrainConfig(), seed=0, host_targets=True)
    te._begin(0)
    cache = te.cache
    og, oc = bench.host_graph(g), bench.host_cache(cache, g.num_nodes)
    ids = g.train_ids().cpu().numpy().astype(np.int64)
    perm = np.random.default_rng(1).permutation(ids)
    for st in args.settings:
        knobs = dict(kv.split("=") for kv in st.split(",") if kv)
        for k, v in knobs.items():
            _lib.call("gns_tune", k.encode(), int(v))
        bad = 0
        for b in range(args.batches):
            t = perm[b * 1000:(b + 1) * 1000]
            mb = P.build_minibatch(g, cache, t, cfg, P.BatchRng(0, 0, b))
            ref = O.build_minibatch(og, oc, t, cfg, O.PhiloxKeys(0, 0, b))
            for li, (bb, r) in enumerate(zip(mb.blocks, ref.blocks)):
                h = bb.to_numpy()
                for f in bench.BLOCK_FIELDS:
                    x, y = np.asarray(getattr(h, f)), np.asarray(getattr(r, f))
                    if x.shape != y.shape or not np.array_equal(x, y):
                        bad += 1
                        i = (np.flatnonzero(x[:min(len(x), len(y))] != y[:min(len(x), len(y))])[:3]
                             if x.ndim == 1 else None)
                        print(f"  [{st}] batch {b} layer {li} field {f}: {x.shape} vs {y.shape}, first diffs at {i}",
                              flush=True)
        print(f"[{st}] {args.batches} batches, {bad} mismatching fields", flush=True)


if __name__ == "__main__":
    main()
