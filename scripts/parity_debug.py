"""Engine-slot parity of the bench workload under gns_tune settings: runs the
timed loop (warmup + steps) and compares the last trained batches with the
oracle, bit for bit, per block field.

    python scripts/parity_debug.py --config cfg1 "" "warp_sort=0"
"""

from __future__ import annotations

import argparse
import gc
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
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    args = ap.parse_args()
    import bench
    import paper_2106_06150_b200 as P
    from oracle import gns as O
    from paper_2106_06150_b200 import _lib
    from paper_2106_06150_b200.engine import GraphedTrainer

    c = bench.CONFIGS[args.config]
    g, _ = bench.make_graph(P, c)
    og, oc, _ = bench.host_reference_inputs(c)
    cfg = P.SamplerConfig(strategy="GNS", fanouts=bench.FANOUTS, batch_size=bench.BATCH, cache_frac=c["cache"],
                          cache_mode="degree", input_layer_cache_only=True, seed=0)
    dims = (c["dim"], c["hidden"], c["hidden"], c["classes"])
    from paper_2106_06150_b200.pool import num_batches
    print("batches per epoch", num_batches(g, cfg), "train ids", int(g.train_ids().numel()), flush=True)
    for st in args.settings:
        knobs = dict(kv.split("=") for kv in st.split(",") if kv)
        for k, v in knobs.items():
            _lib.call("gns_tune", k.encode(), int(v))
        tr = GraphedTrainer(g, cfg, dims, P.TrainConfig(lr=0.003, hidden_dim=c["hidden"]), seed=0)
        pos = tr.run(args.warmup)
        tr.prepare(args.steps)
        trained = []
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(tr.main)
        tr.run(args.steps, epoch=pos[0], first=pos[1], on_step=lambda e, i, k: trained.append((e, i, k)))
        e1.record(tr.main)
        e1.synchronize()
        tr.check_errors()
        kept = [(e, i, None, bench.slot_blocks(tr, tr.slot_of(k))) for e, i, k in trained[-tr.S:] if i is not None]
        print(f"[{st}] step {e0.elapsed_time(e1) / args.steps * 1e3:.1f} us; last trained {trained[-tr.S:]}; "
              f"cache epoch {tr.cache.epoch}", flush=True)
        for epoch, index, _, blocks in kept:
            targets = O.epoch_targets(og, cfg.batch_size, cfg.seed, epoch)[index]
            occ = oc if epoch == 0 else None
            if occ is None:
                print("  (epoch > 0: oracle cache not rebuilt here)")
                continue
            ref = O.build_minibatch(og, occ, targets, cfg, O.PhiloxKeys(cfg.seed, epoch, index))
            for li, (b, r) in enumerate(zip(blocks, ref.blocks)):
                bad = [f for f in bench.BLOCK_FIELDS
                       if not (len(b[f]) == len(np.asarray(getattr(r, f))) and np.array_equal(b[f], np.asarray(getattr(r, f))))]
                print(f"  epoch {epoch} index {index} layer {li}: edges {len(b['edge_src'])} vs {len(r.edge_src)}; "
                      f"mismatched fields {bad}", flush=True)
        del tr
        gc.collect()
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
