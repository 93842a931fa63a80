"""GNS mini-batch training throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config papers100m]
                    [--impl ours|reference] [--precision tf32|fp32]
                    [--no-cpu-baseline] [--no-extras]

One step = sample one mini-batch (3-layer GNS, fanouts 15,10,5, batch 1000,
input layer cache-only) + gather its input features + one GraphSAGE training
step (forward, loss, backward, Adam), on a synthetic power-law graph of the
named shape (device generator; oracle/gen.cc rebuilds the same graph bit for
bit on the host for the CPU arm).  N>1: one process per GPU (torchrun; spawned
by this script when WORLD_SIZE is unset), rank r takes batches r, r+W, ...
(pool.py:80 striding, padded to equal step counts), NCCL gradient all-reduce
captured in the step graph; time = max over ranks.  Prints ONE JSON line on
rank 0.

``--impl reference`` is the CPU arm: the reference's algorithm (oracle port
of pool.py fork workers + the float64 trainer loop body, numpy PCG64 streams)
on this host's cores, on the same graph (built on the host by oracle/gen.cc:
this process never loads libgns.so or touches the GPU).
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GNS mini-batches/sec (sample+gather+train) at 1/2/4/8 B200; gather HBM GB/s"
UNIT = "mini-batches/s"
L2_BYTES = 126 << 20

CONFIGS = {
    # name: nodes, undirected pairs drawn, feature dim, classes, train fraction, hidden, cache frac, alpha, offset
    # cfg1 is the reference's own graph: generate_powerlaw(100000, 10, 0)
    # (graph.py:172-205, preferential attachment, 1,999,800 directed entries)
    "cfg1": dict(label="reference generate_powerlaw(100000, 10, seed 0): 100K nodes / 2M directed edges, 64-d "
                       "(BASELINE configs[0])",
                 nodes=100_000, attach=10, dim=64, classes=16, train=0.5, hidden=64, cache=0.01, cpu_batches=12),
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
BLOCK_FIELDS = ("dst_nodes", "src_nodes", "edge_src", "edge_dst", "edge_weight", "edge_cached", "dst_degree")


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


def workload_config(name, c, nodes, edges, world):
    """The ``config`` object of both arms (identical for the same workload)."""
    ld = (c["dim"] + 3) // 4 * 4
    resident = nodes * ld * 4 + edges * 4 + (nodes + 1) * 8
    l2 = ("inputs larger than L2 (feature table + CSR >> 126 MB); no flush" if resident > 4 * L2_BYTES else
          "inputs fit in L2 (feature table + CSR < 4x 126 MB): L2-resident numbers, no flush")
    return {"workload": c["label"], "config": name, "nodes": int(nodes), "edges": int(edges),
            "feature_dim": c["dim"], "fanouts": list(FANOUTS), "global_batch": BATCH * world,
            "cache_frac": c["cache"], "cache_mode": "degree", "hidden": c["hidden"], "classes": c["classes"],
            "parallelism": f"dp{world}", "l2": l2}


def free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


# ---------------------------------------------------------------------------
# CPU arm (the reference algorithm on the host; no libgns, no GPU)
# ---------------------------------------------------------------------------

class RefConfig:
    """The fields of the reference's SamplerConfig (sampling.py:80-126) the
    oracle sampler reads."""

    def __init__(self, cache_frac, seed=0):
        self.strategy, self.fanouts, self.batch_size = "GNS", FANOUTS, BATCH
        self.cache_frac, self.cache_period, self.cache_mode = cache_frac, 1, "degree"
        self.input_layer_cache_only, self.seed, self.weight_policy = True, seed, "gns-paper"


def host_reference_inputs(c, seed=0, threads=None):
    """The bench graph rebuilt on the host (oracle/gen.cc, bit-identical to
    the device generator) and the epoch-0 cache drawn the reference's way
    (cache.py:87-103: numpy exponential race + argpartition, seed
    [seed, 33, 0]; inclusion Eq. 9 on the cached ids, the only entries the
    sampler reads, sampling.py:253; cached CSR = the full CSR filtered by the
    cache mask, cache.py:185-197)."""
    from oracle import detmath, gen, gns as O
    t0 = time.perf_counter()
    if "attach" in c:
        # the reference's generator restated (oracle.gns, graph.py:172-205) +
        # the device attribute generator's host restatement (oracle/gen.cc)
        top = O.generate_powerlaw(c["nodes"], c["attach"], seed)
        labels, tr, va, te = gen.node_attrs(c["nodes"], c["classes"], c["train"], seed, threads)
        og = O.OGraph(num_nodes=top.num_nodes, indptr=top.indptr, indices=top.indices.astype(np.int32),
                      features=gen.features(c["nodes"], c["dim"], c["classes"], labels, 3.0, seed, threads),
                      labels=labels, train_mask=tr, val_mask=va, test_mask=te)
    else:
        og = gen.powerlaw_graph(c["nodes"], c["pairs"], c["alpha"], c["offset"], seed, feature_dim=c["dim"],
                                num_classes=c["classes"], train_frac=c["train"], threads=threads)
    t1 = time.perf_counter()
    w = O.degree_probs(og)
    cs = O.cache_size_for(og, c["cache"])
    ids = O.sample_cache(w, cs, numpy_seed=[seed, 33, 0])
    mask = np.zeros(og.num_nodes, dtype=bool)
    mask[ids] = True
    incl = np.zeros(og.num_nodes, dtype=np.float64)
    incl[ids] = detmath.inclusion_prob(w[ids], len(ids))
    c_indptr, c_indices = gen.cached_csr(og.indptr, og.indices, mask, threads=threads)
    oc = O.OCache(ids=ids, mask=mask, inclusion=incl, cached_indptr=c_indptr, cached_indices=c_indices, epoch=0)
    return og, oc, {"graph_s": round(t1 - t0, 1), "cache_s": round(time.perf_counter() - t1, 1)}


def reference_arm(args, name, c, world, rank):
    """``--impl reference``: rank 0 alone, the host's cores, K timed steps
    after W warm-up steps (the same K and W as our arm)."""
    if rank != 0:
        return
    from oracle import cpu_pipeline, gns as O
    og, oc, setup = host_reference_inputs(c)
    cfg = RefConfig(c["cache"])
    batches = O.epoch_targets(og, BATCH, cfg.seed, 0, numpy_mode=True)      # pool.py:60-66
    need = args.steps + args.warmup
    batches = (batches * (-(-need // len(batches))))[:need]
    dims = (c["dim"], c["hidden"], c["hidden"], c["classes"])
    r = cpu_pipeline.run(og, oc, cfg, dims, batches, epoch=0, warmup=args.warmup)
    cores = r["workers"] + 1
    sample = (f"{r['steps']} mini-batches of this workload after {args.warmup} warm-up (epoch 0): oracle port of "
              f"pool.py fork workers ({r['workers']}, numpy PCG64 streams) + the float64 trainer loop body "
              f"(model.py:279-285); sample {r['sample_ms']:.0f} ms/batch/worker, train {r['train_ms']:.0f} "
              f"ms/batch; graph rebuilt on the host by oracle/gen.cc")
    line = {"impl": "reference", "metric": METRIC, "value": r["value"], "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 / r["value"], "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(name, c, og.num_nodes, og.num_edges, world),
            "cpu_baseline": {"value": r["value"], "unit": UNIT, "cores": cores, "kind": "port", "sample": sample},
            "e2e": {"value": r["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "setup": setup, "gpu_launches": 0}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def make_graph(P, c, seed=0):
    import torch
    t0 = time.perf_counter()
    if "attach" in c:
        g = P.generate_powerlaw(c["nodes"], c["attach"], seed, feature_dim=c["dim"], num_classes=c["classes"],
                                train_frac=c["train"])
    else:
        g = P.generate_powerlaw_device(c["nodes"], c["pairs"], alpha=c["alpha"], offset=c["offset"], seed=seed,
                                       feature_dim=c["dim"], num_classes=c["classes"], train_frac=c["train"])
    torch.cuda.synchronize()
    return g, time.perf_counter() - t0


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


def slot_blocks(tr, slot):
    """Host copy of the batch held in an engine sampler slot (the exact
    buffers the captured training step read)."""
    mb = tr.slots[slot].snapshot()
    out = []
    for b in mb.blocks:
        h = b.to_numpy()
        out.append({f: getattr(h, f) for f in BLOCK_FIELDS} | {"self_pos": b.self_pos.long().cpu().numpy()})
    return out


def engine_parity(og, oc, cfg, kept):
    """``kept``: [(epoch, index, targets or None, blocks)] read from the
    engine's slots after the timed runs.  Each must equal the oracle's
    build_minibatch (sampling.py:299-336 restated) on the same Philox key
    (seed, epoch, index) and the same targets (the Feistel epoch slice,
    pool.py:60-66, or the host's target array) — every block field and the
    relabel map self_pos, bit for bit."""
    from oracle import gns as O
    perms = {}
    ok, checked = True, []
    for epoch, index, targets, blocks in kept:
        if targets is None:
            if epoch not in perms:
                perms[epoch] = O.epoch_targets(og, cfg.batch_size, cfg.seed, epoch)
            targets = perms[epoch][index]
        ref = O.build_minibatch(og, oc, targets, cfg, O.PhiloxKeys(cfg.seed, epoch, index))
        same = len(ref.blocks) == len(blocks)
        for b, r in zip(blocks, ref.blocks):
            same &= all(np.array_equal(b[f], np.asarray(getattr(r, f))) for f in BLOCK_FIELDS)
            same &= np.array_equal(b["self_pos"], np.searchsorted(np.asarray(r.src_nodes), np.asarray(r.dst_nodes)))
        ok &= bool(same)
        checked.append({"epoch": epoch, "index": index, "bit_exact": bool(same),
                        "edges": int(sum(len(b["edge_src"]) for b in blocks))})
    return ok, checked


def gather_microbench(tr, D, reps=24):
    """features[input_nodes] (model.py:146) through gns_gather_rows on the
    input nodes of the batches currently held in the engine's sampler slots;
    a 256 MB copy between launches flushes L2.  Returns [(bytes, ms)]."""
    import torch
    from paper_2106_06150_b200 import _lib
    L = len(FANOUTS)
    torch.cuda.synchronize()
    sets = []
    for sl in tr.slots:
        b0 = sl.layers[L - 1]
        n = int(b0.counts[_lib.CNT_SRC])
        if n:
            sets.append((b0.src_nodes, b0.counts[_lib.CNT_SRC:_lib.CNT_SRC + 1], n))
    tab = tr.g.features
    out = torch.empty((max(n for _, _, n in sets), D), dtype=torch.float32, device=tab.device)
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


def kernel_line(name, nbytes, ms, peak, peak_kind, how, step_ms=None):
    gbs = float(np.sum(nbytes) / (np.sum(ms) / 1e3) / 1e9)
    d = {"kernel": name, "bound": "hbm", "achieved": round(gbs, 1), "peak": peak, "peak_kind": peak_kind,
         "unit": "GB/s", "frac": round(gbs / peak, 4), "traffic": None,
         "algorithmic_bytes_per_launch": float(np.mean(nbytes)), "avg_launch_ms": float(np.mean(ms)),
         "measured": how}
    if step_ms:
        d["share_of_step"] = float(np.mean(ms) / step_ms)
    return d


def sampler_throughput(P, tr, g, cfg, n_batches=24):
    """The sampling branch alone (K5 sampler + K6 dedup/relabel, all layers of
    one mini-batch) on one stream, batch after batch: mini-batches/s and
    sampled edges/s (north star), plus the bytes lower bound of SURVEY.md
    §8(d) (seed offsets, the sampled edges' output, relabel reads/writes)."""
    import torch
    from paper_2106_06150_b200 import _lib
    from paper_2106_06150_b200.sampling import MiniBatchSampler
    sl = MiniBatchSampler(g, cfg)
    perm = tr.epoch_perm
    nb = perm.numel() // cfg.batch_size
    # one gns_step_t per batch, on the device before the timed chain starts
    steps = torch.zeros((n_batches + 2, 4), dtype=torch.int64)
    for it in range(n_batches + 2):
        idx = (it * 7) % nb
        steps[it, 0] = (cfg.seed & 0xFFFFFFFF) | ((tr._perm_epoch & 0xFFFFFFFF) << 32)
        steps[it, 1], steps[it, 2], steps[it, 3] = idx, idx * cfg.batch_size, cfg.batch_size
    steps = steps.to(g.device)
    s = torch.cuda.Stream(device=g.device)
    cache = tr.cache
    edges = seeds = srcs = 0
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        for it in range(n_batches + 2):
            if it == 2:
                t0.record(s)
            sl.enqueue_device(None, steps[it], cache, epoch_perm=perm)
        t1.record(s)
    t1.synchronize()
    ms = t0.elapsed_time(t1) / n_batches
    # counts of the last batch (representative; every batch is ~the same size)
    c = sl.counts.cpu().numpy()
    for layer in range(len(cfg.fanouts)):
        edges += int(c[layer][_lib.CNT_EDGES])
        seeds += int(c[layer][_lib.CNT_DST])
        srcs += int(c[layer][_lib.CNT_SRC])
    # lower bound (SURVEY §8(d) K5 + K6): indptr + cached_indptr per seed,
    # per-edge output (src id, row, fp64 weight, flag = 17 B), relabel:
    # 4 (E + seeds) read + 4 src + 4 E written
    nbytes = 16 * seeds + 17 * edges + 4 * (edges + seeds) + 4 * srcs + 4 * edges
    # K6 alone: gns_relabel on each layer of the last batch
    # (mark seeds + sampled ids in the two-level bitmap, enumerate, rank),
    # CUDA events, 20 launches per layer; recomputes the same src_nodes /
    # edge_src.  Algorithmic bytes: the summary bitmap (N/256 B) scanned twice
    # (tile counts, then ranks) with the 16-B bitmap pieces under set summary
    # bits (<= 16 n_src B, twice) + ids read to mark and to rank (2 x 4 (n +
    # E)) + rank words read per id (8 (n + E)) + edge_src / self_pos written
    # (4 (n + E)) + src_nodes and rank words written (12 n_src).  A chain of
    # four dependent launches: latency-bound, the fraction is low by design
    k6 = []
    N = g.num_nodes
    with torch.cuda.stream(s):
        for li, lb in enumerate(sl.layers):
            if li == 0:
                sd, nsd = sl.seeds0, sl.n_seeds0
            else:
                prev = sl.layers[li - 1]
                sd, nsd = prev.src_nodes, prev.counts[_lib.CNT_SRC:_lib.CNT_SRC + 1]
            cl = [int(x) for x in lb.counts.tolist()]
            n_l, e_l, s_l = cl[_lib.CNT_DST], cl[_lib.CNT_EDGES], cl[_lib.CNT_SRC]
            b = 2 * (N // 256 + 16 * s_l) + 8 * (n_l + e_l) + 8 * (n_l + e_l) + 4 * (n_l + e_l) + 12 * s_l
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            for it in range(22):
                if it == 2:
                    a0.record(s)
                _lib.call("gns_relabel", N, sd.data_ptr(), nsd.data_ptr(), lb.max_dst, lb.cblock, lb.max_edges,
                          sl.ws_relabel.data_ptr(), sl.ws_relabel.numel(), _lib.stream_ptr(s))
            a1.record(s)
            a1.synchronize()
            t_ms = a0.elapsed_time(a1) / 20
            gbs = b / (t_ms / 1e3) / 1e9
            k6.append({"layer": lb.layer, "dst": n_l, "edges": e_l, "src": s_l, "us": round(t_ms * 1e3, 1),
                       "algorithmic_bytes": b, "achieved_gbs": round(gbs, 1), "frac": round(gbs / load_peaks()[0], 4)})
    return {"ms_per_batch": round(ms, 4), "mini_batches_per_s": round(1e3 / ms, 1),
            "relabel_k6": k6,
            "sampled_edges_per_batch": edges, "sampled_edges_per_s": round(edges / (ms / 1e3), 1),
            "bytes_lower_bound_per_batch": nbytes, "achieved_gbs_lower_bound": round(nbytes / (ms / 1e3) / 1e9, 1),
            "how": f"one sampler chain (gns_batch_slice_sorted + 3 x gns_sample_layer), {n_batches} batches back to "
                   "back on one stream, CUDA events; the engine runs it concurrently with training on a "
                   "low-priority branch"}


def refresh_timing(P, tr, g, reps=3):
    """Per-epoch cache refresh at full size (K1-K3: exponential-race draw over
    N nodes, Eq. 9 inclusion, cached CSR by filtering all E entries) into a
    spare cache set, CUDA events.  Algorithmic bytes per SURVEY.md §8(d):
    4N (deg) + 8N (keys) + 4E (scan indices) + 8N (cached indptr) + 4 nnz_C."""
    import torch
    from paper_2106_06150_b200 import cache as C
    st = C.empty_like(tr.cache, g)
    probs = tr._probs
    cs = tr._cache_size()
    res = []
    for r in range(reps + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        C.refresh_cache(st, g, probs, cs, 100 + r, [tr.cfg.seed, 33, 100 + r], positions=tr._positions)
        e1.record()
        e1.synchronize()
        if r:
            res.append(e0.elapsed_time(e1))
    n, E = g.num_nodes, g.num_edges
    nnz = int(st.cached_indices.numel())
    nbytes = 4 * n + 8 * n + 4 * E + 8 * n + 4 * nnz
    ms = float(np.mean(res))
    del st
    return {"ms": round(ms, 3), "algorithmic_bytes": nbytes, "gbs": round(nbytes / (ms / 1e3) / 1e9, 1),
            "cache_size": cs, "cached_csr_nnz": nnz,
            "how": "cache.refresh_cache (gns_cache_draw + gns_inclusion + gns_cached_csr_count/fill) into a spare "
                   "set exactly as the engine refreshes (cached-CSR positions only for gns-exact), "
                   "host-synchronised (the engine prefetches it on a low-priority stream during the previous "
                   "epoch instead)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default=os.environ.get("GNS_BENCH_CONFIG", "papers100m"), choices=list(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--precision", default="tf32", choices=["tf32", "fp32"],
                    help="GEMM precision of the headline engine (the sampler, gather, SpMMs, loss and Adam are "
                         "fp32/int either way); fp32 and fp64 lines are added at N=1 unless --no-extras")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the precision / epoch / mixed / sampler extras")
    ap.add_argument("--e2e-steps", type=int, default=None)
    args = ap.parse_args()
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        # one process per GPU: re-launch under torchrun (127.0.0.1 rendezvous)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
        raise SystemExit(subprocess.call(cmd))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    name = args.config
    c = CONFIGS[name]
    if args.impl == "reference":
        reference_arm(args, name, c, world, rank)
        return
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}: refusing to report n_gpus != N")
    ours_arm(args, name, c, world, rank, local)


def ours_arm(args, name, c, world, rank, local):
    import torch
    import torch.distributed as dist

    import paper_2106_06150_b200 as P
    from paper_2106_06150_b200 import _lib
    from paper_2106_06150_b200 import dist as gdist
    from paper_2106_06150_b200.engine import GraphedTrainer

    if torch.cuda.device_count() <= local:
        raise SystemExit(f"rank {rank}: no CUDA device {local}")
    torch.cuda.set_device(local)
    force_dist = os.environ.get("GNS_FORCE_DIST", "0") == "1"   # captured NCCL path at N=1 (testing)
    if world > 1 or force_dist:
        gdist.init_from_env("nccl")
    distributed = dist.is_initialized()
    g, gen_s = make_graph(P, c, seed=0)
    cfg = P.SamplerConfig(strategy="GNS", fanouts=FANOUTS, batch_size=BATCH, cache_frac=c["cache"],
                          cache_mode="degree", input_layer_cache_only=True, seed=0)
    dims = (c["dim"], c["hidden"], c["hidden"], c["classes"])
    config = workload_config(name, c, g.num_nodes, g.num_edges, world)
    tc = P.TrainConfig(lr=0.003, hidden_dim=c["hidden"])
    allreduce = gdist.make_allreduce(force=force_dist) if distributed else None
    solo = rank == 0 and world == 1
    extras = solo and not args.no_extras

    tr = GraphedTrainer(g, cfg, dims, tc, rank=rank, world_size=world, allreduce=allreduce, seed=0,
                        tf32=args.precision == "tf32")
    pos = tr.run(args.warmup, epoch=0, first=0)
    tr.prepare(args.steps)
    torch.cuda.synchronize()
    if distributed:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    l0 = _lib.launch_counter[0]
    trained = []
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record(tr.main)
    pos = tr.run(args.steps, epoch=pos[0], first=pos[1], on_step=lambda e, i, k: trained.append((e, i, k)))
    t_end.record(tr.main)
    t_end.synchronize()
    clk = clocks.stop()
    launches = _lib.launch_counter[0] - l0
    per_step = tr.kernels_per_step()     # graph replays launch the captured kernels
    launches_total = int(round(launches + per_step * args.steps))
    ms = gdist.max_over_ranks(t_start.elapsed_time(t_end), device="cuda")
    value = args.steps * world / (ms / 1e3)
    step_ms = ms / args.steps
    tr.check_errors()
    # the last replay's training slots still hold the batches it trained on
    kept = []
    if solo:
        for e, i, k in trained[-tr.S:]:
            if i is not None and e == 0:
                kept.append((e, i, None, slot_blocks(tr, tr.slot_of(k))))

    # ---- per-kernel rooflines: the step graph re-captured with CUDA events
    peak, peak_kind = load_peaks()
    tr.capture_profiled()
    nprof = min(30, args.steps) * tr.S
    spmm_ms, spmm_bytes, n_in, bwd_ms, bwd_bytes = [], [], [], [], []
    D, H = c["dim"], c["hidden"]

    rep = {}

    def on_step(e, i, k):
        # the events time every step of a replay; their per-replay means
        # (read once, at the replay's first step) pair with each step's bytes
        if k % tr.S == 0:
            rep["spmm"], rep["bwd"] = tr.spmm0_ms(), tr.bwd1_ms()
        spmm_ms.append(rep["spmm"])
        bwd_ms.append(rep["bwd"])
        sl = tr.slots[tr.slot_of(k)]
        cnt = sl.counts[len(FANOUTS) - 1].tolist()
        n_in.append(cnt[_lib.CNT_SRC])
        nd, ne = cnt[_lib.CNT_DST], cnt[_lib.CNT_EDGES]
        # input-layer SpMM, algorithmic bytes: every
        # distinct input row read once (a batch's repeated rows are L2 hits) +
        # the cat rows written incl. the zero padding the size-switched GEMM
        # reads + per-edge index/weight (4 + 8 B) + row scan + dst id
        C = tr.switch_chunk
        rows_w = min(tr.npad[0], -(-nd // C) * C) if tr.use_switch else tr.npad[0]
        spmm_bytes.append(cnt[_lib.CNT_SRC] * 4 * D + rows_w * 2 * 4 * D + 12 * ne + 12 * nd)
        # layer 1's transposed SpMM (K8 bwd): dcat rows (self + neighbour
        # halves) of its dst rows, dz rows written for its src rows, 12 B/edge
        c1 = sl.counts[len(FANOUTS) - 2].tolist()
        bwd_bytes.append(4 * 2 * H * c1[_lib.CNT_DST] + 4 * H * c1[_lib.CNT_SRC] + 12 * c1[_lib.CNT_EDGES])
    pos = tr.run(nprof, epoch=pos[0], first=pos[1], on_step=on_step)
    n_in = np.array(n_in, dtype=np.float64)
    g_res = gather_microbench(tr, D)
    spmm_k = kernel_line("gns_spmm_fwd_gather (input layer: feature gather fused with the mean aggregation)",
                         spmm_bytes, spmm_ms, peak, peak_kind,
                         f"CUDA events around the kernel inside the captured step graph, every step of "
                         f"{len(spmm_ms) // tr.S} replays",
                         step_ms)
    bwd_k = kernel_line("gns_spmm_bwd_transposed_bits (model layer 1 backward, hidden 256)", bwd_bytes, bwd_ms,
                        peak, peak_kind, f"CUDA events inside the captured step graph, every step of {len(bwd_ms) // tr.S} replays",
                        step_ms)
    gather_k = kernel_line("gns_gather_rows (reference-API gather features[input_nodes], gather_f32x4_kernel)",
                           [b for b, _ in g_res], [t for _, t in g_res], peak, peak_kind,
                           "standalone on the input nodes of the engine's sampled batches, CUDA events, L2 flushed "
                           "(256 MB copy) between launches")
    kernels = {"spmm_fwd_gather": spmm_k, "spmm_bwd_transposed": bwd_k, "gather_rows": gather_k}
    prof_path = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(prof_path):
        try:
            tj = json.load(open(prof_path)).get(name, {})
            for kk, key in ((gather_k, "gather_f32x4_kernel"), (spmm_k, "spmm_fwd_gather"),
                            (bwd_k, "spmm_bwd_transposed")):
                if tj.get(key):
                    kk["traffic"] = tj[key]
        except Exception:
            pass
    roofline = spmm_k

    extra = {}
    if extras:
        extra["sampler"] = sampler_throughput(P, tr, g, cfg)
        extra["cache_refresh"] = refresh_timing(P, tr, g)
        # a window of whole epochs including their boundaries: the epoch
        # permutation (gns_epoch_targets) and the cache refresh of every
        # epoch (pool.py:133-135; prefetched into the idle set during the
        # previous epoch) are inside the timed region
        tr._free_execs()          # the profiled graphs carry events
        tr._prof_events = None
        # two untimed epochs capture the step graphs of both cache sets (the
        # double buffer alternates sets at every refresh)
        e0 = pos[0] + 1
        nsteps = 2 * len(tr.batches(e0))
        tr.run(nsteps, epoch=e0, first=0)
        e0 += 2
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(tr.main)
        tr.run(nsteps, epoch=e0, first=0)
        a1.record(tr.main)
        a1.synchronize()
        wall = time.perf_counter() - w0
        extra["epochs"] = {"epochs": [e0, e0 + 1], "steps": nsteps, "wall_s": round(wall, 4),
                           "mini_batches_per_s": round(nsteps / wall, 1),
                           "device_ms_per_step": round(a0.elapsed_time(a1) / nsteps, 4),
                           "refreshes": [x for x in tr.refresh_log if x[0] >= e0],
                           "how": "GraphedTrainer.run over two whole epochs from the first batch: every step, the "
                                  "epoch permutations and both epoch-start cache refreshes inside the window "
                                  "(host wall clock, incl. graph re-captures when a refreshed cached CSR outgrew "
                                  "its buffer)"}
    S, prio = tr.S, tr.prio_mode
    del tr
    torch.cuda.empty_cache()

    # ---- end to end through the public API with host buffers: targets from
    # pinned host memory every step (read by a copy kernel in the graph), every
    # step's loss back in pinned host memory and read by the host
    e2e = None
    k2 = args.e2e_steps if args.e2e_steps is not None else max(5, args.steps)
    ids_host = g.train_ids().cpu().numpy().astype(np.int64)
    perm = np.random.default_rng(1).permutation(ids_host)
    nbh = len(perm) // BATCH

    def run_e2e(te, k2, tag):
        nw = 4 * te.S * max(1, 48 // (4 * te.S))
        k2 = -(-k2 // te.S) * te.S   # whole replays in the timed region
        # rank r's host batches: r, r+W, ... of the permutation (pool.py:80)
        S = te.S
        batches = [perm[((j * world + rank) % nbh) * BATCH:((j * world + rank) % nbh + 1) * BATCH]
                   for j in range(k2 + nw + S)]
        # one continuous loop over host batches split at the timed window: each
        # call samples the next call's first S batches ahead (lookahead), so
        # the window holds exactly k2 target reads from pinned memory and k2
        # loss reads, as a steady-state training loop does
        te.run_host(batches[:nw], epoch=0, lookahead=batches[nw:nw + S])
        torch.cuda.synchronize()
        if distributed:
            dist.barrier()
        w0 = time.perf_counter()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(te.main)
        te.run_host(batches[nw:nw + k2], epoch=0, base=nw, lookahead=batches[nw + k2:nw + k2 + S])
        s1.record(te.main)
        s1.synchronize()
        wall = gdist.max_over_ranks(time.perf_counter() - w0, device="cuda")
        got = []
        if solo:   # the last replay's slots: its batches k2-S .. k2-1 (Philox batch = nw + position)
            for k in range(k2 - S, k2):
                got.append((0, nw + k, batches[nw + k], slot_blocks(te, te.slot_of(k))))
        return {"value": k2 * world / wall, "unit": UNIT, "h2d_bytes_per_step": BATCH * 4 + 4 + 32,
                "d2h_bytes_per_step": 8, "steps": k2, "device_ms_per_step": s0.elapsed_time(s1) / k2,
                "path": f"GraphedTrainer(host_targets=True{tag}).run_host: pinned host targets read by a copy kernel "
                        "in the step graph, every step's loss written to pinned host memory by the graph and read "
                        "by the host one replay late; wall clock, max over ranks"}, got

    cache0 = None
    if k2 > 0:
        te = GraphedTrainer(g, cfg, dims, tc, rank=rank, world_size=world, allreduce=allreduce, seed=0,
                            host_targets=True, tf32=args.precision == "tf32")
        te._begin(0)
        cache0 = te.cache
        e2e, got = run_e2e(te, k2, "")
        kept += got
        del te
    torch.cuda.empty_cache()

    precisions = None
    if extras and k2 > 0:
        precisions = {args.precision: {"value": round(value, 3), "ms_per_step": round(step_ms, 4),
                                       "e2e": round(e2e["value"], 3)}}
        other = "fp32" if args.precision == "tf32" else "tf32"
        t2 = GraphedTrainer(g, cfg, dims, tc, seed=0, host_targets=True, tf32=other == "tf32")
        t2.cache = cache0
        e2b, _ = run_e2e(t2, k2, f", tf32={other == 'tf32'}")
        precisions[other] = {"e2e": round(e2b["value"], 3), "device_ms_per_step": round(e2b["device_ms_per_step"], 4),
                             "how": "same engine, GEMMs " + ("TF32 tensor cores" if other == "tf32" else
                                                            "full fp32 (no TF32)")}
        del t2
        torch.cuda.empty_cache()
        precisions["fp64"] = fp64_e2e(P, g, cfg, dims, tc, cache0, perm, min(k2, 40))

    mixed = None
    if extras and os.environ.get("GNS_BENCH_MIXED", "1") == "1":
        mixed = mixed_placement(P, g, cfg, dims, tc, cache0, min(args.steps, 200), args.warmup)

    cpu = None
    parity = None
    if solo and not args.no_cpu_baseline:
        og, oc = host_graph(g), host_cache(cache0, g.num_nodes)
        ok, checked = engine_parity(og, oc, cfg, kept)
        parity = {"batches": len(checked), "bit_exact": bool(ok), "fields": list(BLOCK_FIELDS) + ["self_pos"],
                  "checked": checked,
                  "vs": "the engine's sampler-slot buffers of the last trained batches (device-timed run: Feistel "
                        "epoch slices; end-to-end run: host target arrays) vs the oracle restatement of "
                        "sampling.py:299-336 on the same (seed, epoch, batch) Philox keys, full-size graph"}
        from oracle import cpu_pipeline, gns as O
        batches = O.epoch_targets(og, BATCH, 0, 0, numpy_mode=True)[:c["cpu_batches"] + 1]
        r = cpu_pipeline.run(og, oc, cfg, dims, batches, epoch=0, warmup=1)
        cpu = {"value": r["value"], "unit": UNIT, "cores": r["workers"] + 1, "kind": "port",
               "sample": f"{r['steps']} mini-batches of this workload (epoch 0, after 1 warm-up), oracle port "
                         f"of pool.py fork workers ({r['workers']}) + float64 trainer loop body; sample "
                         f"{r['sample_ms']:.0f} ms/batch/worker, train {r['train_ms']:.0f} ms/batch"}

    if rank == 0:
        dtype = {"tf32": "tf32", "fp32": "f32"}[args.precision]
        line = {"metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": round(step_ms, 4), "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": dtype,
                "precision_detail": "sampler ids int32, weights/inclusion f64 (bit-exact to the reference); gather, "
                                    "SpMMs, loss, Adam f32; linear-layer GEMMs " +
                                    ("TF32 tensor cores (fp32 accumulate)" if args.precision == "tf32" else "fp32"),
                "data": "synthetic", "config": config, "roofline": roofline, "kernels": kernels,
                "cpu_baseline": cpu, "parity": parity, "e2e": e2e, "precisions": precisions,
                "mixed_placement": mixed, "gpu_launches": launches_total,
                "gpu_launches_per_step": launches_total / args.steps, "clocks": clk,
                "setup": {"graph_gen_s": round(gen_s, 2)},
                "per_step": {"input_nodes": float(n_in.mean()), "fused_gather": True,
                             "graph_replays": -(-args.steps // S), "steps_per_graph": S,
                             "step_priority": prio}} | extra
        print(json.dumps(line), flush=True)
    if distributed:
        dist.barrier()
        dist.destroy_process_group()


def fp64_e2e(P, g, cfg, dims, tc, cache, perm, steps):
    """The reference-parity precision end to end through the reference-API
    façade: build_minibatch(host targets) + GraphSAGE(float64).train_step
    (fp64 gather, the bit-exact fp64 SpMM, fp64 GEMMs, fp64 loss and Adam) +
    the loss read back, per step (model.py:279-285 loop body)."""
    import torch
    model = P.GraphSAGE(dims, dtype=torch.float64, seed=0)
    nb = len(perm) // BATCH
    batches = [perm[(j % nb) * BATCH:(j % nb + 1) * BATCH] for j in range(steps + 3)]
    for j in range(3):
        float(model.train_step(P.build_minibatch(g, cache, batches[j], cfg, P.BatchRng(0, 0, j)), g, tc))
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    for j in range(3, steps + 3):
        mb = P.build_minibatch(g, cache, batches[j], cfg, P.BatchRng(0, 0, j))
        float(model.train_step(mb, g, tc))
    wall = time.perf_counter() - w0
    return {"e2e": round(steps / wall, 3), "steps": steps, "dtype": "f64",
            "how": "eager reference-API path: P.build_minibatch(g, cache, host targets, cfg, BatchRng) + "
                   "GraphSAGE(dtype=float64).train_step + float(loss) per step (fp64 GEMMs, bit-exact fp64 SpMM); "
                   "wall clock — the like-for-like precision of the float64 reference"}


def mixed_placement(P, g, cfg, dims, tc, cache, steps, warmup):
    """North-star subsystem 1 / paper §3.1: the feature table in pinned host
    memory; the cached rows refreshed into an HBM table (gns_cache_refresh_rows
    over the host link) and read from HBM, uncached input rows read over the
    host link by the mixed gather (gns_gather_rows_mixed)."""
    import torch
    from paper_2106_06150_b200 import _lib
    from paper_2106_06150_b200.engine import GraphedTrainer
    t0 = time.perf_counter()
    hf = torch.empty(tuple(g.features.shape), dtype=torch.float32, pin_memory=True)
    hf.copy_(g.features)
    pin_s = time.perf_counter() - t0
    tm = GraphedTrainer(g, cfg, dims, tc, seed=0, feature_placement="mixed", host_features=hf)
    # feature refresh over the host link, timed alone
    tm.cache = cache
    torch.cuda.synchronize()
    r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    r0.record()
    tm._fill_table(tm.cur, torch.cuda.current_stream())
    r1.record()
    r1.synchronize()
    refresh_ms = r0.elapsed_time(r1)
    ld = g.features.shape[1]
    refresh_bytes = cache.nodes.ids.numel() * ld * 4
    pos = tm.run(warmup, epoch=0)
    tm.prepare(steps)
    torch.cuda.synchronize()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record(tm.main)
    host_rows = []
    tm.run(steps, epoch=pos[0], first=pos[1])
    s1.record(tm.main)
    s1.synchronize()
    ms = s0.elapsed_time(s1) / steps
    # input rows read over the host link per step (the uncached ones), from the
    # slots of the last replay
    for sl in tm._group(0) + tm._group(1):
        mb = tm.slots[sl].snapshot()
        ids = mb.input_nodes
        if ids.numel():
            host_rows.append(int((~cache.nodes.contains(ids)).sum()))
    rows = float(np.mean(host_rows)) if host_rows else 0.0
    del tm, hf
    torch.cuda.empty_cache()
    return {"mini_batches_per_s": round(1e3 / ms, 1), "ms_per_step": round(ms, 4), "steps": steps,
            "host_rows_per_step": rows, "host_link_gbs": round(rows * ld * 4 / (ms / 1e3) / 1e9, 2),
            "feature_refresh": {"ms": round(refresh_ms, 3), "bytes": refresh_bytes,
                                "gbs": round(refresh_bytes / (refresh_ms / 1e3) / 1e9, 2)},
            "pin_s": round(pin_s, 1),
            "how": "GraphedTrainer(feature_placement='mixed'): 57 GB feature table in pinned host memory; cached "
                   "rows in an HBM table refreshed from host at each cache refresh; uncached input rows read over "
                   "the host link by the gather inside the step graph; device-timed"}


if __name__ == "__main__":
    main()
