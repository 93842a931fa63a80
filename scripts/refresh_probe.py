"""Per-kernel times of one full-size cache refresh (papers100M shape):
run under ncu for the launch list, or alone for the CUDA-event total.

    python scripts/refresh_probe.py [reps]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2106_06150_b200 as P
from paper_2106_06150_b200 import cache as C

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
g = P.generate_powerlaw_device(111_000_000, 1_615_000_000, alpha=0.6, offset=300.0, seed=0, feature_dim=0,
                               num_classes=172, train_frac=0.01)
probs = P.degree_probs(g)
cs = 1_110_000
st = C.build_cache(g, probs, cs, epoch=0, rng_seed=[0, 33, 0], positions=False)
torch.cuda.synchronize()
for r in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    C.refresh_cache(st, g, probs, cs, 1 + r, [0, 33, 1 + r], positions=False)
    e1.record()
    e1.synchronize()
    print(f"refresh {r}: {e0.elapsed_time(e1):.2f} ms, nnz_C {st.cached_indices.numel()}")
