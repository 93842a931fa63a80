"""A/B of the input-layer SpMM variants (gns_tune("spmm_narrow", v)) on the
bench workload's sampled blocks: fused gather (gns_spmm_fwd_gather), L2
flushed (256 MB write) between launches, CUDA events.

    python scripts/spmm_probe.py [--config papers100m] [--reps 20]
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
    ap.add_argument("--reps", type=int, default=20)
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
    L = tr.L
    slots = [sl for sl in tr.slots if int(sl.layers[L - 1].counts[_lib.CNT_DST]) > 0]
    tab = g.features
    D = dims[0]
    cat = torch.empty((tr.npad[0], 2 * D), device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ref = None
    for v in (0, 1):   # 0: generic, 1: register-staged narrow
        _lib.call("gns_tune", b"spmm_narrow", v)
        ts = []
        for it in range(args.reps + 2):
            sl = slots[it % len(slots)]
            flush.fill_(it & 255)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            _lib.call("gns_spmm_fwd_gather", tab.data_ptr(), tab.stride(0), D, sl.layers[L - 1].cblock,
                      sl.layers[L - 2].src_nodes.data_ptr(), tr.cap_dst[0], tr.npad[0], 0, 5, cat.data_ptr(),
                      cat.stride(0), _lib.stream_ptr())
            e1.record()
            e1.synchronize()
            if it >= 2:
                ts.append(e0.elapsed_time(e1))
            if it == len(slots) - 1 + 2 * 0 and it % len(slots) == 0:
                pass
        # equality on slot 0
        sl = slots[0]
        _lib.call("gns_spmm_fwd_gather", tab.data_ptr(), tab.stride(0), D, sl.layers[L - 1].cblock,
                  sl.layers[L - 2].src_nodes.data_ptr(), tr.cap_dst[0], tr.npad[0], 0, 5, cat.data_ptr(),
                  cat.stride(0), _lib.stream_ptr())
        out = cat.clone()
        same = True if ref is None else bool(torch.equal(out, ref))
        ref = out if ref is None else ref
        cnt = sl.layers[L - 1].counts.tolist()
        print(f"narrow={v}: {np.mean(ts) * 1e3:7.1f} us (min {np.min(ts) * 1e3:6.1f})  identical={same}  "
              f"dst={cnt[_lib.CNT_DST]} edges={cnt[_lib.CNT_EDGES]}")
    _lib.call("gns_tune", b"spmm_narrow", 1)


if __name__ == "__main__":
    main()
