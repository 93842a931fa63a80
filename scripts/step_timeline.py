"""Warm-cache per-call timeline of one engine step, run eagerly on one stream
(no branch overlap): a CUDA event is recorded before and after every libgns
entry point; the time between calls is torch work (cuBLAS GEMMs, copies).

    python scripts/step_timeline.py [--config papers100m] [--reps 10]

Prints the mean duration of every segment of the sampling body (next batch)
and of the training body (current batch), in launch order.
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
    ap.add_argument("--reps", type=int, default=10)
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
    tr = GraphedTrainer(g, cfg, dims, P.TrainConfig(), seed=0, steps_per_graph=1)
    tr.run(4)
    torch.cuda.synchronize()

    orig = _lib.call
    marks = []

    def rec(label):
        e = torch.cuda.Event(enable_timing=True)
        e.record(torch.cuda.current_stream())
        marks.append((label, e))

    def call(name, *a):
        rec("torch/copy")
        orig(name, *a)
        rec(name)

    totals = {"sample": collections.defaultdict(float), "train": collections.defaultdict(float)}
    order = {"sample": [], "train": []}
    _lib.call = call
    try:
        for it in range(args.reps + 1):
            for phase, fn in (("sample", lambda: tr._sample_body(1)),
                              ("train", lambda: tr._train_body(1, with_adam=True))):
                if phase == "sample":
                    tr._set_step(1, 0, 100 + it)
                marks.clear()
                with torch.cuda.stream(tr.main):
                    rec("start")
                    fn()
                    rec("end")
                torch.cuda.synchronize()
                seen = collections.Counter()
                for (l0, e0), (l1, e1) in zip(marks, marks[1:]):
                    dt = e0.elapsed_time(e1) * 1e3
                    if l1 == "torch/copy" and dt < 1.0:
                        continue
                    seen[l1] += 1
                    key = f"{l1}#{seen[l1]}"
                    if it > 0:
                        totals[phase][key] += dt / args.reps
                    if it == 1:
                        order[phase].append(key)
    finally:
        _lib.call = orig
    for phase in ("sample", "train"):
        tot = sum(totals[phase].values())
        print(f"--- {phase}: {tot:.1f} us (eager, one stream, warm)")
        for k in order[phase]:
            print(f"  {totals[phase][k]:8.1f} us  {k}")


if __name__ == "__main__":
    main()
