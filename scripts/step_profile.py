"""Per-kernel device time per training step of the bench's timed loop
(GraphedTrainer.run on the bench workload, CUPTI via torch.profiler), next
to the loop's CUDA-event time per step.  Kernel times of the two branches
overlap, so their sum exceeds the step.

    python scripts/step_profile.py [--config papers100m] [--steps 40]
"""

from __future__ import annotations

import argparse
import collections
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="papers100m")
    ap.add_argument("--steps", type=int, default=40)
    args = ap.parse_args()
    import bench
    import paper_2106_06150_b200 as P
    from paper_2106_06150_b200.engine import GraphedTrainer
    from torch.profiler import ProfilerActivity, profile

    c = bench.CONFIGS[args.config]
    g, _ = bench.make_graph(P, c)
    cfg = P.SamplerConfig(strategy="GNS", fanouts=bench.FANOUTS, batch_size=bench.BATCH, cache_frac=c["cache"],
                          cache_mode="degree", input_layer_cache_only=True, seed=0)
    dims = (c["dim"], c["hidden"], c["hidden"], c["classes"])
    tr = GraphedTrainer(g, cfg, dims, P.TrainConfig(lr=0.003, hidden_dim=c["hidden"]), seed=0)
    pos = tr.run(10)
    tr.prepare(args.steps)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(tr.main)
    pos = tr.run(args.steps, epoch=pos[0], first=pos[1])
    e1.record(tr.main)
    e1.synchronize()
    print(f"step (CUDA events, no profiler): {e0.elapsed_time(e1) / args.steps * 1e3:.1f} us")
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        tr.run(args.steps, epoch=pos[0], first=pos[1])
        torch.cuda.synchronize()
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    t0, t1 = None, None
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            k = e.name.split("(")[0].replace("void ", "")[:72]
            tot[k] += e.device_time / args.steps
            cnt[k] += 1
    print(f"per-kernel device time per step (sum {sum(tot.values()):.1f} us over both branches)")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"  {v:7.1f} us  x{cnt[k] / args.steps:4.1f}  {k}")


if __name__ == "__main__":
    main()
