"""Per-layer block sizes (dst, src, edges, cached) of the bench workload vs the
static capacities the engine allocates.

    python scripts/block_sizes.py [--config papers100m] [--steps 20]
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
    ap.add_argument("--config", default="papers100m")
    ap.add_argument("--steps", type=int, default=20)
    args = ap.parse_args()
    import bench
    import paper_2106_06150_b200 as P
    from paper_2106_06150_b200 import _lib
    from paper_2106_06150_b200.engine import GraphedTrainer

    c = bench.CONFIGS[args.config]
    g, _ = bench.make_graph(P, c)
    cfg = P.SamplerConfig(strategy="GNS", fanouts=bench.FANOUTS, batch_size=bench.BATCH, cache_frac=c["cache"],
                          cache_mode="degree", seed=0)
    dims = (c["dim"], c["hidden"], c["hidden"], c["classes"])
    tr = GraphedTrainer(g, cfg, dims, P.TrainConfig(), seed=0)
    rec = []

    def on_step(e, i, k):
        rec.append(tr.slots[k % 2].counts.cpu().numpy().copy())
    tr.run(args.steps, on_step=on_step)
    a = np.stack(rec).astype(np.float64)  # steps x L x CNT_N
    L = a.shape[1]
    print(f"{args.config}: sampler layers (output layer first)")
    for l in range(L):
        lb = tr.slots[0].layers[l]
        d, e, cc, s = (a[:, l, _lib.CNT_DST], a[:, l, _lib.CNT_EDGES], a[:, l, _lib.CNT_CACHED],
                       a[:, l, _lib.CNT_SRC])
        print(f" layer {l}: dst {d.mean():9.0f} (cap {lb.max_dst:8d})  src {s.mean():9.0f} (cap {lb.max_src:8d})  "
              f"edges {e.mean():9.0f} (cap {lb.max_edges:8d})  cached-edges {cc.mean():9.0f}  "
              f"max dst/src/edges {d.max():.0f}/{s.max():.0f}/{e.max():.0f}")
        th, wa, hu = a[:, l, 7], a[:, l, 6], a[:, l, _lib.CNT_HUBS]
        print(f"          (row, phase) items: thread tier {th.mean():9.0f}  warp tier {wa.mean():8.0f}  "
              f"hub tier {hu.mean():6.0f}")


if __name__ == "__main__":
    main()
