"""GNS mini-batch training throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config papers100m]
                    [--impl ours|reference] [--no-cpu-baseline]

One step = sample one mini-batch (3-layer GNS, fanouts 15,10,5, batch 1000,
input layer cache-only) + gather its input features + one GraphSAGE training
step (forward, loss, backward, Adam), on a synthetic power-law graph of the
named shape generated on the device.  N>1: one process per GPU (torchrun),
rank r takes batches r, r+W, ... (pool.py:80 striding), NCCL gradient
all-reduce; time = max over ranks.  Prints ONE JSON line on rank 0.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GNS mini-batches/sec (sample+gather+train) at 1/2/4/8 B200; gather HBM GB/s"
UNIT = "mini-batches/s"

CONFIGS = {
    # name: nodes, undirected pairs drawn, feature dim, classes, train fraction, hidden, cache frac, alpha, offset
    "cfg1": dict(label="synthetic power-law 100K nodes / 2M directed edges, 64-d (BASELINE configs[0])",
                 nodes=100_000, pairs=1_000_000, dim=64, classes=16, train=0.5, hidden=64, cache=0.01,
                 alpha=0.6, offset=10.0, cpu_batches=12),
    "products": dict(label="ogbn-products-shaped synthetic: 2.4M nodes, ~124M directed edges, 100-d",
                     nodes=2_400_000, pairs=62_000_000, dim=100, classes=47, train=0.10, hidden=256,
                     cache=0.01, alpha=0.6, offset=30.0, cpu_batches=6),
    "papers100m": dict(label="ogbn-papers100M-shaped synthetic: 111M nodes, ~3.2B directed edges, 128-d",
                       nodes=111_000_000, pairs=1_615_000_000, dim=128, classes=172, train=0.01,
                       hidden=256, cache=0.01, alpha=0.6, offset=300.0, cpu_batches=4),
    "oag": dict(label="OAG-paper-shaped synthetic: 15M nodes, ~220M directed edges, 768-d",
                nodes=15_000_000, pairs=110_000_000, dim=768, classes=146, train=0.43, hidden=256,
                cache=0.01, alpha=0.6, offset=100.0, cpu_batches=4),
}
FANOUTS = (15, 10, 5)
BATCH = 1000


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self.proc = None

    def start(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.samples.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(2)
        except Exception:
            self.proc.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def make_graph(P, c, seed=0):
    t0 = time.perf_counter()
    g = P.generate_powerlaw_device(c["nodes"], c["pairs"], alpha=c["alpha"], offset=c["offset"], seed=seed,
                                   feature_dim=c["dim"], num_classes=c["classes"], train_frac=c["train"])
    torch.cuda.synchronize()
    return g, time.perf_counter() - t0


def batch_stream(pool, start_epoch=0):
    epoch = start_epoch
    while True:
        n = 0
        for item in pool.iter_epoch(epoch):
            n += 1
            yield item
        if n == 0:
            raise RuntimeError("empty epoch")
        epoch += 1


def host_graph(g):
    """Reference-layout numpy copy of the device graph (CPU baseline input)."""
    from oracle import gns as O
    h = g.to_host()
    return O.OGraph(num_nodes=h.num_nodes, indptr=h.indptr, indices=h.indices, features=h.features,
                    labels=h.labels, train_mask=h.train_mask)


def host_cache(cache, n):
    from oracle import gns as O
    ids = cache.nodes.ids.cpu().numpy().astype(np.int64)
    mask = np.zeros(n, dtype=bool)
    mask[ids] = True
    return O.OCache(ids=ids, mask=mask, inclusion=cache.inclusion.cpu().numpy(),
                    cached_indptr=cache.cached_indptr.cpu().numpy(),
                    cached_indices=cache.cached_indices.cpu().numpy())


def cpu_reference_run(P, g, c, cfg, cache, n_batches, warmup=1, host=None):
    """The reference's CPU algorithm (oracle port: pool.py fork workers + the
    float64 trainer loop body) on this host's cores."""
    from oracle import cpu_pipeline, gns as O
    og, oc = host if host is not None else host_inputs(g, cache)
    batches = O.epoch_targets(og, cfg.batch_size, cfg.seed, 0, numpy_mode=True)
    batches = batches[:n_batches + warmup]
    dims = (c["dim"], c["hidden"], c["hidden"], c["classes"])
    r = cpu_pipeline.run(og, oc, cfg, dims, batches, epoch=0, warmup=warmup)
    r["cores"] = r["workers"] + 1
    return r


def host_inputs(g, cache):
    return host_graph(g), (host_cache(cache, g.num_nodes) if cache is not None else None)


def full_size_parity(P, g, cfg, cache, og, oc, n_batches=1):
    """One mini-batch of the bench workload sampled on the device (libgns)
    and by the oracle restatement of the reference (Philox keys): every block
    field must be bit-identical."""
    from oracle import gns as O
    fields = ("dst_nodes", "src_nodes", "edge_src", "edge_dst", "edge_weight", "edge_cached", "dst_degree")
    train = np.flatnonzero(og.train_mask)
    ok = True
    for b in range(n_batches):
        targets = np.random.default_rng(1000 + b).choice(train, cfg.batch_size, replace=False)
        mb = P.build_minibatch(g, cache, targets, cfg, P.BatchRng(cfg.seed, 0, b))
        ref = O.build_minibatch(og, oc, targets, cfg, O.PhiloxKeys(cfg.seed, 0, b))
        for bg, br in zip(mb.blocks, ref.blocks):
            h = bg.to_numpy()
            ok &= all(np.array_equal(getattr(h, f), np.asarray(getattr(br, f))) for f in fields)
    return {"batches": n_batches, "bit_exact": bool(ok), "fields": list(fields),
            "vs": "oracle restatement of sampling.py:189-336 with the same Philox keys, full-size graph"}


def gather_microbench(tr, D, reps=24):
    """features[input_nodes] (model.py:146) through gns_gather_rows on the
    input nodes of the batches currently held in the engine's sampler slots;
    a 256 MB copy between launches flushes L2.  Returns [(bytes, ms)]."""
    from paper_2106_06150_b200 import _lib
    L = len(FANOUTS)
    # the engine's last replay may still be sampling into a slot on its side
    # stream: settle every stream before reading the slots' device counts
    torch.cuda.synchronize()
    sets = []
    for sl in tr.slots:
        b0 = sl.layers[L - 1]
        n = int(b0.counts[_lib.CNT_SRC])
        if n:
            sets.append((b0.src_nodes, b0.counts[_lib.CNT_SRC:_lib.CNT_SRC + 1], n))
    tab = tr.g.features
    out = torch.empty((max(n for _, _, n in sets), D), dtype=torch.float32, device=tab.device)
    # L2 flush: copy 256 MB of random bytes (a constant memset can be
    # absorbed without displacing L2 lines; a real read+write stream cannot)
    flush = torch.randint(0, 256, (256 << 20,), dtype=torch.uint8, device=tab.device)
    scratch = torch.empty_like(flush)
    s = torch.cuda.current_stream()
    res = []
    for it in range(reps + 2):
        ids, n_dev, n = sets[it % len(sets)]
        scratch.copy_(flush)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        _lib.call("gns_gather_rows", tab.data_ptr(), tab.stride(0), 0, ids.data_ptr(), n_dev.data_ptr(), out.shape[0],
                  D, out.data_ptr(), out.stride(0), 0, _lib.stream_ptr(s))
        e1.record(s)
        e1.synchronize()
        if it >= 2:
            res.append((n * (2 * 4 * D + 4), e0.elapsed_time(e1)))
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default=os.environ.get("GNS_BENCH_CONFIG", "papers100m"), choices=list(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--workers", type=int, default=2, help="sampling slots in flight (SamplerPool num_workers)")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    c = CONFIGS[args.config]

    if args.impl == "reference" and rank != 0:
        return
    import paper_2106_06150_b200 as P
    from paper_2106_06150_b200 import _lib

    from paper_2106_06150_b200 import dist as gdist
    torch.cuda.set_device(local)
    force_dist = os.environ.get("GNS_FORCE_DIST", "0") == "1"   # captured NCCL path at N=1 (testing)
    if (world > 1 or force_dist) and args.impl == "ours":
        gdist.init_from_env("nccl")
    distributed = dist.is_initialized()
    g, gen_s = make_graph(P, c, seed=0)
    cfg = P.SamplerConfig(strategy="GNS", fanouts=FANOUTS, batch_size=BATCH, cache_frac=c["cache"],
                          cache_mode="degree", input_layer_cache_only=True, seed=0)
    dims = (c["dim"], c["hidden"], c["hidden"], c["classes"])
    config = {"workload": c["label"], "config": args.config, "nodes": g.num_nodes, "edges": g.num_edges,
              "feature_dim": c["dim"], "fanouts": list(FANOUTS), "global_batch": BATCH * world,
              "cache_frac": c["cache"], "cache_mode": "degree", "hidden": c["hidden"],
              "classes": c["classes"], "parallelism": f"dp{world}",
              "l2": "inputs larger than L2 (feature table + CSR >> 126 MB); no flush",
              "graph_gen_s": round(gen_s, 2)}

    if args.impl == "reference":
        pool = P.SamplerPool(g, cfg)
        pool._refresh_cache(0)
        n = max(1, min(args.steps, c["cpu_batches"] * 2))
        r = cpu_reference_run(P, g, c, cfg, pool.cache, n, warmup=min(args.warmup, 1))
        cpu = {"value": r["value"], "unit": UNIT, "cores": r["cores"], "kind": "port",
               "sample": f"{r['steps']} mini-batches of the same workload (epoch 0), oracle port of pool.py "
                         f"fork workers ({r['workers']}) + float64 trainer loop body; "
                         f"sample {r['sample_ms']:.0f} ms/batch/worker, train {r['train_ms']:.0f} ms/batch"}
        line = {"impl": "reference", "metric": METRIC, "value": r["value"], "unit": UNIT, "n_gpus": world,
                "steps": r["steps"], "warmup": 1, "ms_per_step": 1e3 / r["value"], "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": config,
                "cpu_baseline": cpu,
                "e2e": {"value": r["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    tc = P.TrainConfig(lr=0.003, hidden_dim=c["hidden"])

    from paper_2106_06150_b200.engine import GraphedTrainer
    allreduce = gdist.make_allreduce(force=force_dist) if distributed else None
    tr = GraphedTrainer(g, cfg, dims, tc, rank=rank, world_size=world, allreduce=allreduce, seed=0)
    pos = tr.run(args.warmup, epoch=0, first=0)
    tr.prepare(args.steps)
    torch.cuda.synchronize()
    if distributed:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    l0 = _lib.launch_counter[0]
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record(tr.main)
    pos = tr.run(args.steps, epoch=pos[0], first=pos[1])
    t_end.record(tr.main)
    t_end.synchronize()
    clk = clocks.stop()
    launches = _lib.launch_counter[0] - l0
    # graph replays launch the captured kernels: count them per step
    per_step = tr.kernels_per_step()
    launches_total = int(round(launches + per_step * args.steps))
    ms = gdist.max_over_ranks(t_start.elapsed_time(t_end), device="cuda")
    value = args.steps * world / (ms / 1e3)
    tr.check_errors()

    # per-kernel rooflines: the step graph re-captured with timing events
    # around the input-layer kernels of the first step of each replay
    # (gns_gather_rows + gns_spmm_fwd, or the fused gns_spmm_fwd_gather)
    peak, peak_kind = load_peaks()
    tr.capture_profiled()
    nprof = min(30, args.steps) * tr.S
    gather_ms, spmm_ms, spmm_bytes, n_in = [], [], [], []
    D = c["dim"]

    def on_step(e, i, k):
        if k % tr.S:          # the events time the first step of each replay
            return
        if not tr.fused_gather:
            gather_ms.append(tr.gather_ms())
        spmm_ms.append(tr.spmm0_ms())
        cnt = tr.slots[tr.slot_of(k)].counts[len(FANOUTS) - 1].tolist()
        n_in.append(cnt[_lib.CNT_SRC])
        nd, ne = cnt[_lib.CNT_DST], cnt[_lib.CNT_EDGES]
        # input-layer SpMM, algorithmic bytes: every
        # distinct input row read once (n_src; a batch's repeated rows are L2
        # hits, ncu DRAM traffic ~ this) + the cat rows written, incl. the zero
        # padding the GEMM reads (up to the size-switched row count) +
        # per-edge index/weight (4 + 8 B) + row scan (+ dst id, fused gather)
        C = tr.switch_chunk
        rows_w = min(tr.npad[0], -(-nd // C) * C) if tr.use_switch else tr.npad[0]
        spmm_bytes.append(cnt[_lib.CNT_SRC] * 4 * D + rows_w * 2 * 4 * D + 12 * ne
                          + (12 if tr.fused_gather else 8) * nd)
    pos = tr.run(nprof, epoch=pos[0], first=pos[1], on_step=on_step)
    n_in = np.array(n_in, dtype=np.float64)
    gbytes = n_in * (2 * 4 * D + 4)     # rows read + rows written + int32 ids
    if not tr.fused_gather:
        g_ms = np.array(gather_ms)
        g_how = f"CUDA events around the gather inside the captured step graph, {len(g_ms)} replays"
    else:
        g_ms, g_how = gather_microbench(tr, D), ("gns_gather_rows (reference-API gather) on the input nodes of the "
                                                 "engine's sampled batches, CUDA events, L2 flushed between launches")
        gbytes = np.array([gather_bytes for gather_bytes, _ in g_ms])
        g_ms = np.array([t for _, t in g_ms])
    gather_gbs = float(gbytes.sum() / (g_ms.sum() / 1e3) / 1e9)
    spmm_gbs = float(np.sum(spmm_bytes) / (np.sum(spmm_ms) / 1e3) / 1e9)
    gather_k = {"kernel": "gns_gather_rows (gather_f32x4_kernel)", "bound": "hbm", "achieved": round(gather_gbs, 1),
                "peak": peak, "peak_kind": peak_kind, "unit": "GB/s", "frac": round(gather_gbs / peak, 4),
                "traffic": None, "algorithmic_bytes_per_launch": float(gbytes.mean()),
                "avg_launch_ms": float(g_ms.mean()), "measured": g_how}
    spmm_name = "gns_spmm_fwd_gather (input layer, fused feature gather)" if tr.fused_gather else \
        "gns_spmm_fwd (input layer)"
    spmm_k = {"kernel": spmm_name, "bound": "hbm", "achieved": round(spmm_gbs, 1), "peak": peak,
              "peak_kind": peak_kind, "unit": "GB/s", "frac": round(spmm_gbs / peak, 4), "traffic": None,
              "algorithmic_bytes_per_launch": float(np.mean(spmm_bytes)), "avg_launch_ms": float(np.mean(spmm_ms)),
              "share_of_step": float(np.mean(spmm_ms) / (ms / args.steps)),
              "measured": f"CUDA events around the kernel inside the captured step graph, {len(spmm_ms)} replays"}
    if not tr.fused_gather:
        gather_k["share_of_step"] = float(g_ms.mean() / (ms / args.steps))
    # the dominant HBM kernel of the step: the fused gather+aggregate when the
    # gather is fused, else the gather (as in round 1)
    roofline = spmm_k if tr.fused_gather else gather_k
    kernels = {"gns_gather_rows": gather_k, "gns_spmm_fwd (input layer)": spmm_k}
    prof_path = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(prof_path):
        try:
            tj = json.load(open(prof_path)).get(args.config, {})
            for kk, name in ((gather_k, "gather_f32x4_kernel"), (spmm_k, "spmm_fwd_gather" if tr.fused_gather
                                                                     else "spmm_fwd_kernel")):
                if tj.get(name):
                    kk["traffic"] = tj[name]
        except Exception:
            pass
    pool = tr

    # end-to-end through the public API with host buffers: targets from pinned
    # host memory every step (read by a copy kernel in the graph), every
    # step's loss back in pinned host memory and read by the host; the timed
    # run_host call includes its eager prologue (sampling the first batch)
    e2e = None
    k2 = args.e2e_steps if args.e2e_steps is not None else max(5, args.steps)
    if k2 > 0:
        ids_host = g.train_ids().cpu().numpy().astype(np.int64)
        perm = np.random.default_rng(1).permutation(ids_host)
        nb = len(perm) // BATCH
        te = GraphedTrainer(g, cfg, dims, tc, rank=rank, world_size=world, allreduce=allreduce, seed=0,
                            host_targets=True)
        # warm-up: captures both graph parities and brings the clocks back up
        # after the host-only parity check (a cold start skews a short run)
        nw = 4 * te.S * max(1, 48 // (4 * te.S))
        k2 = -(-k2 // te.S) * te.S   # whole replays in the timed region
        # rank r's host batches: r, r+W, ... of the permutation (pool.py:80)
        batches = [perm[((j * world + rank) % nb) * BATCH:((j * world + rank) % nb + 1) * BATCH]
                   for j in range(k2 + nw)]
        te.cache = tr.cache
        te.run_host(batches[:nw], epoch=0)
        torch.cuda.synchronize()
        if distributed:
            dist.barrier()
        w0 = time.perf_counter()
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        s0.record(te.main)
        te.run_host(batches[nw:], epoch=0)
        s1.record(te.main)
        s1.synchronize()
        wall = gdist.max_over_ranks(time.perf_counter() - w0, device="cuda")
        e2e = {"value": k2 * world / wall, "unit": UNIT, "h2d_bytes_per_step": BATCH * 4 + 4 + 32,
               "d2h_bytes_per_step": 8, "steps": k2,
               "path": "GraphedTrainer(host_targets=True).run_host: pinned host targets read by a copy kernel in "
                       "the step graph, every step's loss written to pinned host memory by the graph and read "
                       "by the host one replay late; wall clock, max over ranks",
               "device_ms_per_step": s0.elapsed_time(s1) / k2}
        del te

    cpu = None
    parity = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        host = host_inputs(g, pool.cache)
        parity = full_size_parity(P, g, cfg, pool.cache, *host)
        r = cpu_reference_run(P, g, c, cfg, pool.cache, c["cpu_batches"], host=host)
        cpu = {"value": r["value"], "unit": UNIT, "cores": r["cores"], "kind": "port",
               "sample": f"{r['steps']} mini-batches of this workload (epoch 0, after 1 warm-up), oracle port "
                         f"of pool.py fork workers ({r['workers']}) + float64 trainer loop body; sample "
                         f"{r['sample_ms']:.0f} ms/batch/worker, train {r['train_ms']:.0f} ms/batch"}

    if rank == 0:
        line = {"metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 4), "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic", "config": config,
                "roofline": roofline, "kernels": kernels, "cpu_baseline": cpu, "parity": parity, "e2e": e2e,
                "gpu_launches": launches_total,
                "gpu_launches_per_step": launches_total / args.steps, "clocks": clk,
                "per_step": {"input_nodes": float(n_in.mean()), "gather_ms": float(g_ms.mean()),
                             "fused_gather": tr.fused_gather,
                             "graph_replays": -(-args.steps // tr.S), "steps_per_graph": tr.S,
                             "step_priority": tr.prio_mode}}
        print(json.dumps(line), flush=True)
    if distributed:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
