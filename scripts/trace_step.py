"""In-graph kernel timeline of the production step (CUPTI via torch.profiler):
per-kernel durations as replayed inside the CUDA graph, which branch
(stream) they ran on, and how much of each branch overlapped the other.

    python scripts/trace_step.py [--config papers100m] [--replays 5]
"""
from __future__ import annotations

import argparse
import collections
import json
import os
import sys
import tempfile

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="papers100m")
    ap.add_argument("--replays", type=int, default=5)
    ap.add_argument("--dump", action="store_true")
    ap.add_argument("--sampler-only", action="store_true")
    args = ap.parse_args()
    import bench
    import paper_2106_06150_b200 as P
    from paper_2106_06150_b200.engine import GraphedTrainer

    c = bench.CONFIGS[args.config]
    g, _ = bench.make_graph(P, c)
    cfg = P.SamplerConfig(strategy="GNS", fanouts=bench.FANOUTS, batch_size=bench.BATCH, cache_frac=c["cache"],
                          cache_mode="degree", seed=0)
    dims = (c["dim"], c["hidden"], c["hidden"], c["classes"])
    tr = GraphedTrainer(g, cfg, dims, P.TrainConfig(), seed=0)
    pos = tr.run(6)
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        if args.sampler_only:
            # the sampling body alone, eagerly (per-kernel device durations
            # without the training branch's contention)
            with torch.cuda.stream(tr.main):
                for i in range(args.replays):
                    tr._set_step(1, pos[0], 10 + i)
                    tr._sample_body(1)
        else:
            tr.run(args.replays, epoch=pos[0], first=pos[1])
        torch.cuda.synchronize()
    path = os.path.join(tempfile.mkdtemp(), "trace.json")
    prof.export_chrome_trace(path)
    allev = [e for e in json.load(open(path))["traceEvents"] if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")
             and "dur" in e]
    allev.sort(key=lambda e: e["ts"])
    ev = [e for e in allev if e.get("cat") == "kernel"]
    if "--dump" in sys.argv:
        # the GPU activity around the 4th epoch_targets (a replay start)
        starts = [i for i, e in enumerate(allev) if "epoch_targets" in e["name"]]
        i0 = starts[min(3, len(starts) - 1)]
        base = allev[i0]["ts"]
        for e in allev[max(0, i0 - 12):i0 + 14]:
            print(f"  {e['ts'] - base:9.1f} +{e['dur']:7.1f}  s{e['args'].get('stream')}  {e['cat'][:10]:10s} "
                  f"{e['name'].split('(')[0][:60]}")
    # split into replays by gaps > 20 us between kernel end and next start on any stream
    t0, t1 = ev[0]["ts"], max(e["ts"] + e["dur"] for e in ev)
    span = (t1 - t0) / args.replays
    print(f"{len(ev)} kernels, {span:.1f} us per step (wall span / replays)")
    streams = collections.Counter(e["args"].get("stream") for e in ev)
    main_stream = max(streams, key=lambda s: sum(e["dur"] for e in ev if e["args"].get("stream") == s))
    by = collections.defaultdict(lambda: [0.0, 0])
    for e in ev:
        name = e["name"].split("(")[0].replace("void ", "")[:60]
        st = "main" if e["args"].get("stream") == main_stream else "side"
        by[(st, name)][0] += e["dur"] / args.replays
        by[(st, name)][1] += 1 / args.replays
    for st in ("main", "side"):
        tot = sum(v[0] for (s, _), v in by.items() if s == st)
        print(f"--- {st} branch: sum of kernel time {tot:.1f} us per step")
        for (s, name), (d, n) in sorted(by.items(), key=lambda x: -x[1][0]):
            if s == st and d > 2:
                print(f"  {d:7.1f} us  x{n:4.1f}  {name}")
    # busy time of each class and their overlap (union of intervals)
    def union(iv):
        iv = sorted(iv)
        tot, cs, ce = 0.0, None, None
        for a, b in iv:
            if cs is None or a > ce:
                if cs is not None:
                    tot += ce - cs
                cs, ce = a, b
            else:
                ce = max(ce, b)
        return tot + ((ce - cs) if cs is not None else 0.0)
    # one replay's timeline (the 4th), with idle gaps > 1 us
    idle_at = []
    cover = sorted((e["ts"], e["ts"] + e["dur"], e) for e in ev)
    cur_end = cover[0][1]
    for a, b, e in cover[1:]:
        if a > cur_end + 1.0:
            idle_at.append((cur_end, a - cur_end, e["name"].split("(")[0][:50]))
        cur_end = max(cur_end, b)
    gaps = collections.Counter()
    for _, d, nm in idle_at:
        gaps[nm] += d / args.replays
    print("idle gaps (> 1 us) per step, by the kernel that ends the gap:")
    for nm, d in gaps.most_common(15):
        print(f"  {d:6.1f} us before {nm}")
    # per replay (split at the first sampler kernel of each replay): when the
    # training kernels and the sampling kernels end, relative to replay start
    samp = ("sample_", "layer_count", "enumerate_", "relabel", "batch_targets", "batch_slice", "tsort", "tscan",
            "tscatter", "tcount", "unique_small")
    starts = [i for i, e in enumerate(ev) if "batch_targets" in e["name"] or "batch_slice" in e["name"]]
    rows = []
    for a, b in zip(starts, starts[1:] + [len(ev)]):
        seg = ev[a:b]
        t0_ = min(e["ts"] for e in seg)
        tr_end = max((e["ts"] + e["dur"] for e in seg if not any(k in e["name"] for k in samp)), default=t0_)
        sa_end = max((e["ts"] + e["dur"] for e in seg if any(k in e["name"] for k in samp)), default=t0_)
        rows.append((tr_end - t0_, sa_end - t0_))
    if rows:
        print("per replay (us from its first kernel): train ends / sampler ends: " +
              ", ".join(f"{x:.0f}/{y:.0f}" for x, y in rows))
    mi = [(e["ts"], e["ts"] + e["dur"]) for e in ev if e["args"].get("stream") == main_stream]
    si = [(e["ts"], e["ts"] + e["dur"]) for e in ev if e["args"].get("stream") != main_stream]
    um, us_, ua = union(mi), union(si), union(mi + si)
    print(f"busy per step: main {um / args.replays:.1f} us, side {us_ / args.replays:.1f} us, "
          f"either {ua / args.replays:.1f} us, both {(um + us_ - ua) / args.replays:.1f} us, "
          f"idle {(t1 - t0 - ua) / args.replays:.1f} us")


if __name__ == "__main__":
    main()
