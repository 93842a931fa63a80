"""One eager sampler chain of the bench workload (gns_batch_slice_sorted +
3 x gns_sample_layer + the block transposes) inside cudaProfilerStart/Stop,
for `ncu --profile-from-start off`.

    ncu --set full --clock-control none --profile-from-start off -o rep \
        python scripts/sampler_ncu.py [--config papers100m]
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
    args = ap.parse_args()
    import bench
    import paper_2106_06150_b200 as P
    from paper_2106_06150_b200.engine import GraphedTrainer

    c = bench.CONFIGS[args.config]
    g, _ = bench.make_graph(P, c)
    cfg = P.SamplerConfig(strategy="GNS", fanouts=bench.FANOUTS, batch_size=bench.BATCH, cache_frac=c["cache"],
                          cache_mode="degree", input_layer_cache_only=True, seed=0)
    dims = (c["dim"], c["hidden"], c["hidden"], c["classes"])
    tr = GraphedTrainer(g, cfg, dims, P.TrainConfig(), seed=0)
    tr.run(4)
    torch.cuda.synchronize()
    sl = tr._group(0)[0]
    tr._set_step(sl, 0, 9)
    torch.cuda.profiler.start()
    with torch.cuda.stream(tr.main):
        tr._sample_body(sl)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()


if __name__ == "__main__":
    main()
