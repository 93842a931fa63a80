"""A/B of the transposed-SpMM variants (gns_tune("spmm_bwd", v)) on the bench
workload: for each variant a fresh GraphedTrainer (the knob is read at
capture), the device-timed step over --steps steps, the layer-1 transposed
SpMM timed by CUDA events inside the step graph, and the same kernel
standalone on a sampled slot with L2 flushed (256 MB write) between launches;
dz compared bit for bit with variant 0 (the per-row kernel).

    python scripts/bwd_probe.py [--config papers100m] [--variants 0,1,2,3,4,5]
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
    ap.add_argument("--variants", default="0,1,2,3,4,5")
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--ncu", action="store_true",
                    help="only the standalone launches, inside cudaProfilerStart/Stop (ncu --profile-from-start off)")
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
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ref = None
    for v in [int(x) for x in args.variants.split(",")]:
        _lib.call("gns_tune", b"spmm_bwd", v)
        tr = GraphedTrainer(g, cfg, dims, P.TrainConfig(lr=0.003, hidden_dim=c["hidden"]), seed=0)
        pos = tr.run(10)
        if args.ncu:
            torch.cuda.synchronize()
            L = tr.L
            si = next(i for i, sl in enumerate(tr.slots) if int(sl.layers[L - 2].counts[_lib.CNT_SRC]) > 0)
            blk, ws = tr.slots[si].layers[L - 2], tr.tws[si][1]
            torch.cuda.profiler.start()
            for _ in range(2):
                _lib.call("gns_spmm_bwd_transposed_bits", tr.dcat[1].data_ptr(), tr.dcat[1].stride(0), dims[1],
                          blk.cblock, tr.cap_dst[1], tr.cap_src[1], tr.cap_edges[1], 0, tr.relu_bits[1].data_ptr(),
                          None, tr.dz[0].data_ptr(), tr.dz[0].stride(0), ws.data_ptr(), ws.numel(),
                          _lib.stream_ptr())
            torch.cuda.synchronize()
            torch.cuda.profiler.stop()
            del tr
            continue
        tr.prepare(args.steps)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(tr.main)
        pos = tr.run(args.steps, epoch=pos[0], first=pos[1])
        e1.record(tr.main)
        e1.synchronize()
        step_ms = e0.elapsed_time(e1) / args.steps
        tr.capture_profiled()
        ing = []
        tr.run(20 * tr.S, epoch=pos[0], first=pos[1],
               on_step=lambda e, i, k: ing.append(tr.bwd1_ms()) if k % tr.S == 0 else None)
        torch.cuda.synchronize()
        # standalone on a filled slot's layer-1 block (its transpose is in tws[slot][1])
        L = tr.L
        si = next(i for i, sl in enumerate(tr.slots) if int(sl.layers[L - 2].counts[_lib.CNT_SRC]) > 0)
        sl = tr.slots[si]
        blk = sl.layers[L - 2]
        ws = tr.tws[si][1]
        dcat = tr.dcat[1]
        gen = torch.Generator(device="cuda").manual_seed(5)
        dcat.copy_(torch.randn(dcat.shape, device="cuda", generator=gen))
        out = torch.empty_like(tr.dz[0])
        db = torch.empty(dims[1], device="cuda")
        ts = []
        for it in range(args.reps + 2):
            flush.fill_(it & 255)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            _lib.call("gns_spmm_bwd_transposed_bits", dcat.data_ptr(), dcat.stride(0), dims[1], blk.cblock,
                      tr.cap_dst[1], tr.cap_src[1], tr.cap_edges[1], 0, tr.relu_bits[1].data_ptr(), db.data_ptr(),
                      out.data_ptr(), out.stride(0), ws.data_ptr(), ws.numel(), _lib.stream_ptr())
            b.record()
            b.synchronize()
            if it >= 2:
                ts.append(a.elapsed_time(b))
        n = int(blk.counts[_lib.CNT_SRC])
        ne = int(blk.counts[_lib.CNT_EDGES])
        deg = torch.bincount(blk.edge_src[:ne].long(), minlength=n)
        hist = {f">={t}": int((deg >= t).sum()) for t in (2, 4, 16, 64, 256)}
        print(f"  transposed rows: max edges {int(deg.max())}, rows with {hist}, edges in rows >=16: "
              f"{int(deg[deg >= 16].sum())}, rows with 0 edges {int((deg == 0).sum())}", flush=True)
        o = out[:n].clone()
        same = True if ref is None else bool(torch.equal(o, ref))
        if ref is None:
            ref = o
        cnt = blk.counts.tolist()
        byts = 4 * 2 * dims[1] * cnt[_lib.CNT_DST] + 4 * dims[1] * cnt[_lib.CNT_SRC] + 12 * cnt[_lib.CNT_EDGES]
        print(f"spmm_bwd={v}: step {step_ms:.4f} ms  in-graph {np.mean(ing) * 1e3:6.1f} us  "
              f"standalone {np.mean(ts) * 1e3:6.1f} us (min {np.min(ts) * 1e3:5.1f}, "
              f"{byts / np.mean(ts) / 1e6:6.0f} GB/s)  identical={same}  src={cnt[_lib.CNT_SRC]} "
              f"dst={cnt[_lib.CNT_DST]} edges={cnt[_lib.CNT_EDGES]}", flush=True)
        del tr
        import gc
        gc.collect()
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
