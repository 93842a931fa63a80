"""Standalone gns_gather_rows on the bench workload's real input-node sets vs
uniformly random sorted id sets of the same size (same feature table), L2
flushed with a 1 GB write between launches.

    python scripts/gather_data_probe.py [--config papers100m]
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
    tr.run(6)
    torch.cuda.synchronize()
    L, D, tab = tr.L, dims[0], g.features
    real = []
    for sl in tr.slots:
        b0 = sl.layers[L - 1]
        n = int(b0.counts[_lib.CNT_SRC])
        if n:
            real.append(b0.src_nodes[:n].clone())
    n = real[0].numel()
    rnd = [torch.sort(torch.randperm(g.num_nodes, device="cuda")[:n].to(torch.int32)).values for _ in range(2)]
    cached = tr.cache.nodes.ids
    print(f"table {tuple(tab.shape)} stride {tab.stride()} ptr%4096={tab.data_ptr() % 4096}; n={n}; "
          f"cached share of input nodes: "
          f"{float(torch.isin(real[0], cached).float().mean()):.3f}")
    ids = real[0].long().cpu().numpy()
    gaps = np.diff(ids)
    print(f"input ids: median gap {np.median(gaps):.0f}, mean gap {gaps.mean():.0f}, "
          f"share of gaps < 8 rows: {(gaps < 8).mean():.3f}")
    out = torch.empty((n + 8, D), device="cuda")
    flush = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
    for name, sets in (("real", real), ("uniform", rnd), ("real", real)):
        ts = []
        for it in range(22):
            ids = sets[it % len(sets)]
            m = ids.numel()
            flush.fill_(it & 255)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            _lib.call("gns_gather_rows", tab.data_ptr(), tab.stride(0), 0, ids.data_ptr(), None, m, D,
                      out.data_ptr(), out.stride(0), 0, _lib.stream_ptr())
            e1.record()
            e1.synchronize()
            if it >= 2:
                ts.append(e0.elapsed_time(e1))
        gb = m * (2 * 4 * D + 4) / 1e9
        print(f"{name:8s} {np.mean(ts) * 1e3:7.1f} us  {gb / (np.mean(ts) / 1e3):7.1f} GB/s")


if __name__ == "__main__":
    main()
