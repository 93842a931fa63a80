"""Engine parity of the end-to-end path (GraphedTrainer(host_targets=True)
.run_host) on a bench workload: after runs of K steps, the last S trained
batches in the sampler slots vs the oracle (same cache, targets, Philox key).

    python scripts/parity_e2e.py --config cfg1 --runs 4,20,200
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
    ap.add_argument("--config", default="cfg1")
    ap.add_argument("--runs", default="4,20,200")
    ap.add_argument("--env", default="")
    args = ap.parse_args()
    import bench
    import paper_2106_06150_b200 as P
    from oracle import gns as O
    from paper_2106_06150_b200.engine import GraphedTrainer

    c = bench.CONFIGS[args.config]
    g, _ = bench.make_graph(P, c)
    cfg = P.SamplerConfig(strategy="GNS", fanouts=bench.FANOUTS, batch_size=bench.BATCH, cache_frac=c["cache"],
                          cache_mode="degree", input_layer_cache_only=True, seed=0)
    dims = (c["dim"], c["hidden"], c["hidden"], c["classes"])
    te = GraphedTrainer(g, cfg, dims, P.TrainConfig(lr=0.003, hidden_dim=c["hidden"]), seed=0, host_targets=True)
    te._begin(0)
    og, oc = bench.host_graph(g), bench.host_cache(te.cache, g.num_nodes)
    ids = g.train_ids().cpu().numpy().astype(np.int64)
    perm = np.random.default_rng(1).permutation(ids)
    nbh = len(perm) // 1000
    for K in [int(x) for x in args.runs.split(",")]:
        batches = [perm[(j % nbh) * 1000:(j % nbh + 1) * 1000] for j in range(K)]
        te.run_host(batches, epoch=0)
        torch.cuda.synchronize()
        for k in range(K - te.S, K):
            blocks = bench.slot_blocks(te, te.slot_of(k))
            ref = O.build_minibatch(og, oc, batches[k], cfg, O.PhiloxKeys(0, 0, k))
            bad = []
            for li, (b, r) in enumerate(zip(blocks, ref.blocks)):
                for f in bench.BLOCK_FIELDS:
                    x, y = b[f], np.asarray(getattr(r, f))
                    if x.shape != y.shape or not np.array_equal(x, y):
                        bad.append((li, f, x.shape, y.shape))
            print(f"run of {K}: position {k} slot {te.slot_of(k)}: {'OK' if not bad else bad[:6]}", flush=True)


if __name__ == "__main__":
    main()
