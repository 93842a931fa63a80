"""Sampler work per layer on the bench workload: rows, positions whose
Philox keys are generated (per phase, per tier), edges emitted — the ALU
work the selection tiers do.

    python scripts/sampler_work.py [--config papers100m] [--batches 4]
"""

from __future__ import annotations

import argparse
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="papers100m")
    ap.add_argument("--batches", type=int, default=4)
    args = ap.parse_args()
    import bench
    import paper_2106_06150_b200 as P
    from paper_2106_06150_b200 import _lib
    from paper_2106_06150_b200.engine import GraphedTrainer

    c = bench.CONFIGS[args.config]
    g, _ = bench.make_graph(P, c)
    cfg = P.SamplerConfig(strategy="GNS", fanouts=bench.FANOUTS, batch_size=bench.BATCH, cache_frac=c["cache"],
                          cache_mode="degree", input_layer_cache_only=True, seed=0)
    dims = (c["dim"], c["hidden"], c["hidden"], c["classes"])
    tr = GraphedTrainer(g, cfg, dims, P.TrainConfig(), seed=0)
    tr.run(4)
    torch.cuda.synchronize()
    cache = tr.cache
    L = tr.L
    for sl in tr.slots[:args.batches]:
        print("--- batch")
        for i, lb in enumerate(sl.layers):
            cnt = lb.counts.tolist()
            nd = cnt[_lib.CNT_DST]
            seeds = sl.seeds0[:nd] if i == 0 else sl.layers[i - 1].src_nodes[:nd]
            s = seeds.long()
            deg = (g.indptr[s + 1] - g.indptr[s])
            nc = (cache.cached_indptr[s + 1] - cache.cached_indptr[s])
            k = lb.k
            m = torch.minimum(nc, torch.full_like(nc, k))
            fill = torch.zeros_like(nc) if lb.cache_only else torch.minimum(k - m, deg - nc)
            cpos = torch.where(m > 0, nc, torch.zeros_like(nc))       # cached phase scans nc
            fpos = torch.where(fill > 0, deg, torch.zeros_like(deg))  # fill phase scans the full row
            def tiers(ln, take):
                act = ln > 0
                stream = act & (take <= 8) & (ln <= 32)
                hub = act & ~stream & (ln > 2048)
                warp = act & ~stream & ~hub
                return {t: (int(msk.sum()), int(ln[msk].sum())) for t, msk in
                        (("stream", stream), ("warp", warp), ("hub", hub))}
            tc, tf = tiers(cpos, m), tiers(fpos, fill)
            print(f"layer {lb.layer}: dst {nd}, edges {cnt[_lib.CNT_EDGES]}, src {cnt[_lib.CNT_SRC]}; "
                  f"keys: cached phase {int(cpos.sum())} {tc}, fill phase {int(fpos.sum())} {tf}; "
                  f"rows taking all cached {int(((m == nc) & (nc > 0)).sum())}, rows with fill {int((fill > 0).sum())}")


if __name__ == "__main__":
    main()
