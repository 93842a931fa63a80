"""Spatial partitioning experiment: the step's sampling branch on a green
context of X SMs (its own graph on a green-context stream) concurrent with
the training graph on the primary context, vs the single-graph step.

    python scripts/partition_probe.py [--config papers100m] [--steps 100]
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
    args = ap.parse_args()
    import bench
    import paper_2106_06150_b200 as P
    from paper_2106_06150_b200.engine import GraphedTrainer
    from torch.cuda.green_contexts import GreenContext

    c = bench.CONFIGS[args.config]
    g, _ = bench.make_graph(P, c)
    cfg = P.SamplerConfig(strategy="GNS", fanouts=bench.FANOUTS, batch_size=bench.BATCH, cache_frac=c["cache"],
                          cache_mode="degree", seed=0)
    dims = (c["dim"], c["hidden"], c["hidden"], c["classes"])
    tr = GraphedTrainer(g, cfg, dims, P.TrainConfig(), seed=0)
    tr.run(5)
    torch.cuda.synchronize()
    tr._set_step(1, 0, 7)

    def timed(fn, stream):
        with torch.cuda.stream(stream):    # CUDAGraph.replay launches on the current stream
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(stream)
            for _ in range(args.steps):
                fn()
            e.record(stream)
            e.synchronize()
        return s.elapsed_time(e) / args.steps * 1e3

    main_s = tr.main
    tg = torch.cuda.CUDAGraph()
    with torch.cuda.graph(tg, stream=main_s):
        tr._train_body(0, with_adam=False)
    print(f"train only: {timed(tg.replay, main_s):.1f} us", flush=True)
    print(f"single-graph step: {timed(lambda: tr._replay(0), main_s):.1f} us", flush=True)
    keep = []
    for X in (16, 24, 32, 48, 64):
        gc = GreenContext.create(X, 0)
        keep.append(gc)
        ss = gc.Stream()
        tr.taux[1] = ss          # transposes inline on the sampling stream
        sg = torch.cuda.CUDAGraph()
        with torch.cuda.stream(ss):
            with torch.cuda.graph(sg, stream=ss):
                tr._sample_body(1)
        t_s = timed(sg.replay, ss)

        def both():
            ev = torch.cuda.Event()
            ev.record(main_s)
            ss.wait_event(ev)
            with torch.cuda.stream(ss):
                sg.replay()
            with torch.cuda.stream(main_s):
                tg.replay()
            ev2 = torch.cuda.Event()
            ev2.record(ss)
            main_s.wait_event(ev2)
        with torch.cuda.stream(main_s):
            t_b = timed(both, main_s)
        print(f"sampler on {X:3d} SMs: alone {t_s:7.1f} us, with training concurrently {t_b:7.1f} us", flush=True)


if __name__ == "__main__":
    main()
