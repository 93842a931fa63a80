import os, sys, torch, numpy as np
sys.path.insert(0, os.getcwd())
import bench
import paper_2106_06150_b200 as P
from paper_2106_06150_b200 import _lib
from oracle import gns as O
c = bench.CONFIGS["cfg1"]
g, _ = bench.make_graph(P, c)
ip = g.indptr.cpu().numpy(); ix = g.indices.cpu().numpy()
rows_sorted = all(np.all(np.diff(ix[ip[v]:ip[v+1]]) > 0) for v in range(0, g.num_nodes, 97))
print("N", g.num_nodes, "E", len(ix), "sampled rows strictly sorted:", rows_sorted, flush=True)
try:
    P.validate_graph(g); print("validate_graph ok", flush=True)
except Exception as e:
    print("validate_graph FAILED", e, flush=True)
og = O.OGraph(num_nodes=g.num_nodes, indptr=ip, indices=ix)
cfg = P.SamplerConfig(strategy="GNS", fanouts=bench.FANOUTS, batch_size=bench.BATCH, cache_frac=c["cache"], cache_mode="degree", seed=0)
cs = O.cache_size_for(og, cfg.cache_frac)
cache = P.build_cache(g, P.degree_probs(g), cs, rng_seed=[0, 33, 0])
oc = O.build_cache(og, O.degree_probs(og), cs, seed=0, epoch=0)
print("cache ids equal", np.array_equal(cache.nodes.ids.cpu().numpy(), oc.ids), flush=True)
for bi in range(4):
    targets = np.random.default_rng(bi).choice(g.num_nodes, 1000, replace=False)
    mb = P.build_minibatch(g, cache, targets, cfg, P.BatchRng(0, 0, bi))
    ref = O.build_minibatch(og, oc, targets, cfg, O.PhiloxKeys(0, 0, bi))
    for li, (bg, br) in enumerate(zip(mb.blocks, ref.blocks)):
        h = bg.to_numpy()
        diffs = [f for f in ("dst_nodes","src_nodes","edge_src","edge_dst","edge_weight","edge_cached","dst_degree") if getattr(h, f).shape != np.asarray(getattr(br, f)).shape or not np.array_equal(getattr(h, f), getattr(br, f))]
        print("batch", bi, "block", li, "diffs", diffs, "src", len(h.src_nodes), len(br.src_nodes), "edges", len(h.edge_src), len(br.edge_src), flush=True)
