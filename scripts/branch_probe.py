"""Time the two branches of the captured step separately and together.

    python scripts/branch_probe.py [--config papers100m] [--steps 100]

Captures three graph variants on the same engine state: sample-only,
train-only (gather + layers + backward) and the production step (both,
overlapped), and reports the per-replay device time of each.
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
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--trace", default=None,
                    help="CUPTI per-kernel durations of one variant (sample_only, train_only, production)")
    args = ap.parse_args()
    import bench
    import paper_2106_06150_b200 as P
    from paper_2106_06150_b200.engine import GraphedTrainer

    c = bench.CONFIGS[args.config]
    g, _ = bench.make_graph(P, c)
    cfg = P.SamplerConfig(strategy="GNS", fanouts=bench.FANOUTS, batch_size=bench.BATCH, cache_frac=c["cache"],
                          cache_mode="degree", input_layer_cache_only=True, seed=0)   # bench.py's sampler
    dims = (c["dim"], c["hidden"], c["hidden"], c["classes"])
    tr = GraphedTrainer(g, cfg, dims, P.TrainConfig(), seed=0)
    tr.run(5)
    torch.cuda.synchronize()

    def capture(fn):
        gph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gph, stream=tr.main):
            fn()
        return gph

    tr._set_step(tr.S, 0, 7)
    variants = {
        "sample_only": capture(lambda: tr._sample_body(tr.S)).replay,
        "train_only": capture(lambda: tr._train_body(0, with_adam=False)).replay,
        "gather_only": capture(lambda: tr._gather(0)).replay,
        "production": lambda: tr._replay(0),
    }
    try:
        print("kernel-node |priority| histogram:", tr.kernel_priorities(0))
    except RuntimeError as e:
        print("kernel-node priorities unavailable:", e)
    def production_empty():
        tr._replay(0)

    variants["production, sampling an empty batch"] = production_empty
    if args.trace:
        import collections
        from torch.profiler import ProfilerActivity, profile
        replay = variants[args.trace]
        for _ in range(3):
            replay()
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            with torch.cuda.stream(tr.main):
                for _ in range(10):
                    replay()
            torch.cuda.synchronize()
        tot = collections.defaultdict(float)
        cnt = collections.Counter()
        for e in prof.events():
            if e.device_type == torch.autograd.DeviceType.CUDA:
                k = e.name.split("(")[0].replace("void ", "")[:70]
                tot[k] += e.device_time / 10
                cnt[k] += 1
        print(f"--- {args.trace}: per-kernel device time per replay (sum {sum(tot.values()):.1f} us)")
        for k, v in sorted(tot.items(), key=lambda x: -x[1]):
            print(f"  {v:7.1f} us  x{cnt[k] / 10:4.1f}  {k}")
        return
    for name, replay in variants.items():
        if name.startswith("production, sampling an empty"):
            torch.cuda.synchronize()
            tr._set_step(tr.S, 0, None)
        for _ in range(3):
            replay()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(tr.main)
        with torch.cuda.stream(tr.main):
            for _ in range(args.steps):
                replay()
        e.record(tr.main)
        e.synchronize()
        label = f"production ({tr.S} steps per replay, priority={tr.prio_mode})" if name == "production" else name
        print(f"{label:26s} {s.elapsed_time(e) / args.steps * 1e3:8.1f} us/replay")


if __name__ == "__main__":
    main()
