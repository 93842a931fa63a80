"""A/B of sampler knobs (gns_tune) on the bench workload: for each setting a
fresh GraphedTrainer (knobs are read at capture), the device-timed step over
--steps steps and the sampler chain alone (bench.sampler_throughput).

    python scripts/sampler_ab.py "count_items=4" "count_items=1" "count_items=1,stream_minb=3"
"""

from __future__ import annotations

import argparse
import gc
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("settings", nargs="+")
    ap.add_argument("--config", default="papers100m")
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--repeat", type=int, default=2)
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
    res = {}
    for rep in range(args.repeat):
        for st in args.settings:
            knobs = dict(kv.split("=") for kv in st.split(",") if kv)
            for k, v in knobs.items():
                _lib.call("gns_tune", k.encode(), int(v))
            tr = GraphedTrainer(g, cfg, dims, P.TrainConfig(lr=0.003, hidden_dim=c["hidden"]), seed=0)
            pos = tr.run(10)
            tr.prepare(args.steps)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(tr.main)
            tr.run(args.steps, epoch=pos[0], first=pos[1])
            e1.record(tr.main)
            e1.synchronize()
            step = e0.elapsed_time(e1) / args.steps * 1e3
            smp = bench.sampler_throughput(P, tr, g, cfg)
            res.setdefault(st, []).append((step, smp["ms_per_batch"] * 1e3))
            print(f"{st:40s} step {step:6.1f} us  sampler alone {smp['ms_per_batch'] * 1e3:6.1f} us/batch", flush=True)
            del tr
            gc.collect()
            torch.cuda.empty_cache()
    print("--- mean over repeats")
    for st, v in res.items():
        print(f"{st:40s} step {sum(x for x, _ in v) / len(v):6.1f} us  sampler {sum(y for _, y in v) / len(v):6.1f} us")


if __name__ == "__main__":
    main()
