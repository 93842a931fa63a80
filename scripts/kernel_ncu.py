"""The training branch's HBM kernels of the bench workload launched eagerly
with exactly the arguments the captured step graph gives them (size-switched
zero fill included), inside cudaProfilerStart/Stop — ncu cannot replay kernel
nodes of graphs that hold conditional (SWITCH) nodes, so this is how the
timed configuration gets its `ncu --set full` capture:

    ncu --set full --clock-control none --profile-from-start off -o rep \
        python scripts/kernel_ncu.py [--config papers100m]

Prints the algorithmic bytes of each launch (bench.py's formulas) so the
ncu DRAM bytes can be set against them.
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
    from paper_2106_06150_b200 import _lib
    from paper_2106_06150_b200.engine import GraphedTrainer

    c = bench.CONFIGS[args.config]
    g, _ = bench.make_graph(P, c)
    cfg = P.SamplerConfig(strategy="GNS", fanouts=bench.FANOUTS, batch_size=bench.BATCH, cache_frac=c["cache"],
                          cache_mode="degree", input_layer_cache_only=True, seed=0)
    dims = (c["dim"], c["hidden"], c["hidden"], c["classes"])
    tr = GraphedTrainer(g, cfg, dims, P.TrainConfig(lr=0.003, hidden_dim=c["hidden"]), seed=0)
    tr.run(12)
    torch.cuda.synchronize()
    L = tr.L
    si = next(i for i, sl in enumerate(tr.slots) if int(sl.layers[L - 1].counts[_lib.CNT_DST]) > 0)
    sl = tr.slots[si]
    b0, b1 = sl.layers[L - 1], sl.layers[L - 2]
    D, H = dims[0], dims[1]
    tab = g.features
    s = _lib.stream_ptr()
    c0, c1 = b0.counts.tolist(), b1.counts.tolist()
    nd, ne = c0[_lib.CNT_DST], c0[_lib.CNT_EDGES]
    C = tr.switch_chunk
    rows_w = min(tr.npad[0], -(-nd // C) * C) if tr.use_switch else tr.npad[0]
    print(f"spmm_fwd_gather algorithmic bytes {c0[_lib.CNT_SRC] * 4 * D + rows_w * 2 * 4 * D + 12 * ne + 12 * nd}")
    print(f"spmm_bwd_transposed algorithmic bytes "
          f"{4 * 2 * H * c1[_lib.CNT_DST] + 4 * H * c1[_lib.CNT_SRC] + 12 * c1[_lib.CNT_EDGES]}")
    print(f"gather_rows algorithmic bytes {c0[_lib.CNT_SRC] * (2 * 4 * D + 4)}")
    out = torch.empty((tr.cap_src[0], D), device="cuda")
    torch.cuda.profiler.start()
    # input layer: fused gather + aggregation into cat0 (engine._train_rest, li = 0)
    _lib.call("gns_spmm_fwd_gather", tab.data_ptr(), tab.stride(0), D, b0.cblock, b1.src_nodes.data_ptr(),
              tr.cap_dst[0], tr.npad[0], C if tr.use_switch else 0, b0.k, tr.cat[0].data_ptr(),
              tr.cat[0].stride(0), s)
    # hidden layer 1 forward (relu on load + relu' bits)
    _lib.call("gns_spmm_fwd_bits", tr.z[0].data_ptr(), tr.z[0].stride(0), H, b1.cblock, tr.cap_dst[1], tr.npad[1],
              tr.cat[1].data_ptr(), tr.cat[1].stride(0), tr.relu_bits[1].data_ptr(), s)
    # layer 1 backward: transposed SpMM + relu' + bias gradient partials
    ws = tr.tws[si][1]
    _lib.call("gns_spmm_bwd_transposed_bits", tr.dcat[1].data_ptr(), tr.dcat[1].stride(0), H, b1.cblock,
              tr.cap_dst[1], tr.cap_src[1], tr.cap_edges[1], 0, tr.relu_bits[1].data_ptr(),
              tr.model.gbiases[0].data_ptr(), tr.dz[0].data_ptr(), tr.dz[0].stride(0), ws.data_ptr(), ws.numel(), s)
    # the reference-API gather features[input_nodes]
    _lib.call("gns_gather_rows", tab.data_ptr(), tab.stride(0), 0, b0.src_nodes.data_ptr(),
              b0.counts[_lib.CNT_SRC:_lib.CNT_SRC + 1].data_ptr(), out.shape[0], D, out.data_ptr(), out.stride(0), 0,
              s)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()


if __name__ == "__main__":
    main()
