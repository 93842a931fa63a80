"""Where the device generator and oracle/gen.cc differ (debug helper)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2106_06150_b200 as P
from oracle import gen
n, m, alpha, offset, seed = 20000, 150000, 0.6, 50.0, 3
g = P.generate_powerlaw_device(n, m, alpha=alpha, offset=offset, seed=seed, feature_dim=30, num_classes=7, train_frac=0.2)
og = gen.powerlaw_graph(n, m, alpha, offset, seed, feature_dim=30, num_classes=7, train_frac=0.2)
ip = g.indptr.cpu().numpy()
print("indptr eq", np.array_equal(ip, og.indptr), "nnz", ip[-1], og.indptr[-1])
d = np.flatnonzero(np.diff(ip) != np.diff(og.indptr))
print("rows differing", d.size, d[:10])
print("labels eq", np.array_equal(g.labels.cpu().numpy(), og.labels))
print("train eq", np.array_equal(g.train_mask.cpu().numpy(), og.train_mask))
f = g.features.cpu().numpy()
print("feat shape", f.shape, og.features.shape, "eq", np.array_equal(f.view(np.uint32), og.features[:, :30].view(np.uint32)))
