#!/bin/bash
# A/B two builds of libgns.so on one box (run under gpurun from the repo root):
#   bash scripts/ab_lib.sh ab/libgns_head.so [bench args...]
# alternates the given build (A) and the in-tree build (B), 3 runs each.
A=$1; shift
mkdir -p gpurun_out/ab
for i in 1 2 3; do
  GNS_LIB=$PWD/$A timeout 600 python bench.py --no-extras "$@" > gpurun_out/ab/A_$i.log 2>&1
  timeout 600 python bench.py --no-extras "$@" > gpurun_out/ab/B_$i.log 2>&1
done
python - <<'PY'
import json, glob
for tag in "AB":
    for f in sorted(glob.glob(f"gpurun_out/ab/{tag}_*.log")):
        d = json.loads(open(f).read().strip().splitlines()[-1])
        k = d.get("kernels", {})
        print(tag, f[-5:], round(d["value"], 1), round(d["ms_per_step"], 4), "e2e", round(d["e2e"]["value"], 1),
              "bwd", round(1e3 * k.get("spmm_bwd_transposed", {}).get("avg_launch_ms", 0), 1),
              "gather", round(1e3 * k.get("spmm_fwd_gather", {}).get("avg_launch_ms", 0), 1))
PY
