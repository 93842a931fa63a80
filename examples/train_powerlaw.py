"""Drop-in usage on one B200: a synthetic power-law graph, the reference's
training loop through the module API, then the CUDA-graph engine on the
same graph.

    python examples/train_powerlaw.py [--nodes 200000] [--epochs 3]

1. ``P.train(...)`` — the reference's ``train()`` (model.py:257-307):
   SamplerPool batches, GraphSAGE steps, per-epoch loss / micro-F1.
2. ``GraphedTrainer`` — the throughput path: one CUDA graph per two steps,
   the next batches sampled on a side branch while the current ones train.
"""

from __future__ import annotations

import argparse
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2106_06150_b200 as P  # noqa: E402
from paper_2106_06150_b200.engine import GraphedTrainer  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nodes", type=int, default=200_000)
    ap.add_argument("--epochs", type=int, default=3)
    args = ap.parse_args()
    g = P.generate_powerlaw_device(args.nodes, 8 * args.nodes, alpha=0.6, offset=10.0, seed=0, feature_dim=64,
                                   num_classes=8, train_frac=0.3)
    print(f"graph: {g.num_nodes} nodes, {g.num_edges} directed edges, {g.feature_dim}-d features")
    cfg = P.SamplerConfig(strategy="GNS", fanouts=(15, 10, 5), batch_size=1000, cache_frac=0.01,
                          cache_mode="degree", input_layer_cache_only=True, seed=0)
    tc = P.TrainConfig(epochs=args.epochs, hidden_dim=128, lr=0.003, seed=0)

    # 1. the reference's loop through the drop-in module API (float32 here;
    #    dtype=torch.float64 is the reference's precision)
    t0 = time.perf_counter()
    rep = P.train(g, cfg, tc, dtype=torch.float32)
    for r in rep.rows:
        print(f"epoch {r.epoch}: loss {r.loss:.4f}  train F1 {r.train_f1:.3f}  test F1 {r.test_f1:.3f}  "
              f"mean input nodes {r.mean_input_nodes:.0f}")
    print(f"module API: {time.perf_counter() - t0:.1f} s")

    # 2. the engine: CUDA-graph steps, sampling overlapped with training
    dims = (g.feature_dim, 128, 128, 8)
    tr = GraphedTrainer(g, cfg, dims, tc, seed=0)
    nb = len(tr.batches(0))
    pos = tr.run(nb)                     # one epoch (warm-up, captures)
    tr.prepare(nb)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    losses = []
    e0.record(tr.main)
    tr.run(nb, epoch=pos[0], first=pos[1], on_step=lambda e, i, k: None)
    e1.record(tr.main)
    e1.synchronize()
    ms = e0.elapsed_time(e1)
    losses.append(tr.loss_value())
    print(f"engine: {nb} steps in {ms:.1f} ms = {nb / ms * 1e3:.0f} mini-batches/s, last loss {losses[-1]:.4f}")


if __name__ == "__main__":
    main()
