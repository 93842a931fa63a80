"""Turn a round_profile.sh output directory into the committed evidence under
profiles/: bench JSON lines, the launch-list summary, ncu metric tables and
traffic.json (DRAM bytes per launch for the roofline kernels).

    python scripts/summarize_profiles.py gpurun_out/r1d r1
"""

from __future__ import annotations

import collections
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")

METRICS = [
    ("gpu__time_duration.sum", "us", 1e-3),
    ("dram__bytes_read.sum", "DRAM read MB", 1e-6),
    ("dram__bytes_write.sum", "DRAM write MB", 1e-6),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "% dram peak", 1),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "% warps active", 1),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "long-sb stall/issue", 1),
    ("launch__registers_per_thread", "regs", 1),
    ("launch__grid_size", "grid", 1),
]


def last_json(path):
    try:
        lines = [ln for ln in open(path).read().splitlines() if ln.startswith("{")]
        return json.loads(lines[-1]) if lines else None
    except OSError:
        return None


def ncu_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return []
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(h, r))
        d["_units"] = dict(zip(h, units))
        res.append(d)
    return res


def num(d, key):
    v = d.get(key, "")
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return None
    u = d["_units"].get(key, "")
    scale = {"nsecond": 1.0, "ns": 1.0, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6, "byte": 1.0,
             "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1.0)
    return x * scale


def launch_table(path, steps=5):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[hi + 1:]:
        v = float(r[vi].replace(",", ""))
        v = v / 1e3 if r[ui] in ("nsecond", "ns") else v * 1e3 if r[ui] in ("msecond", "ms") else v
        name = r[ki].split("(")[0].replace("void ", "").strip()[:58]
        tot[name] += v
        cnt[name] += 1
    T = sum(tot.values())
    lines = [f"| kernel | share | µs / step | µs / launch | launches / step |", "|---|---:|---:|---:|---:|"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1])[:24]:
        lines.append(f"| `{k}` | {v / T * 100:.1f}% | {v / steps:.1f} | {v / cnt[k]:.1f} | {cnt[k] / steps:.1f} |")
    return T / steps, "\n".join(lines)


def main():
    src, tag = sys.argv[1], sys.argv[2]
    os.makedirs(os.path.join(PROF, "bench"), exist_ok=True)
    rnd = tag[1:].split("_")[0].rstrip("abcdefghijklmnopqrstuvwxyz") if tag.startswith("r") else "?"
    md = [f"# Profiles — round {rnd} (`{tag}`, {os.path.basename(src)})", ""]
    md.append("Produced by `scripts/round_profile.sh` on one B200 (gpurun) and summarised by "
              "`scripts/summarize_profiles.py`.  ncu numbers are serialised, cold-cache replays: "
              "compare shares, not absolutes, with the in-graph CUDA-event timings of bench.py.")
    md.append("")
    md.append("## Bench lines (`profiles/bench/`)")
    md.append("")
    md.append("| config | mini-batches/s | ms/step | e2e mb/s | dominant kernel frac | gather frac | parity | "
              "CPU port mb/s (cores) |")
    md.append("|---|---:|---:|---:|---:|---:|---|---:|")
    for cfg in ("papers100m", "products", "oag", "cfg1"):
        d = last_json(os.path.join(src, f"bench_{cfg}.log"))
        if not d:
            continue
        with open(os.path.join(PROF, "bench", f"{tag}_{cfg}.json"), "w") as f:
            f.write(json.dumps(d) + "\n")
        cpu = d.get("cpu_baseline") or {}
        md.append(f"| {cfg} | {d['value']:.1f} | {d['ms_per_step']:.3f} | {d['e2e']['value']:.1f} | "
                  f"{d['roofline']['frac']:.3f} | {d['kernels']['gather_rows']['frac']:.3f} | "
                  f"{(d.get('parity') or {}).get('bit_exact')} | {cpu.get('value', float('nan')):.3f} "
                  f"({cpu.get('cores')}) |")
    ref = last_json(os.path.join(src, "bench_papers100m_reference.log"))
    if ref:
        with open(os.path.join(PROF, "bench", f"{tag}_papers100m_reference_arm.json"), "w") as f:
            f.write(json.dumps(ref) + "\n")
        md.append("")
        md.append(f"Reference arm (`bench.py --impl reference`, papers100M-shaped): {ref['value']:.3f} mb/s on "
                  f"{ref['cpu_baseline']['cores']} host cores ({ref['cpu_baseline']['kind']}).")
    lp = os.path.join(src, "launches_papers100m.csv")
    if os.path.exists(lp):
        shutil.copy(lp, os.path.join(PROF, f"{tag}_launches_papers100m.csv"))
        per_step, table = launch_table(lp)
        md += ["", "## Launch list, papers100M-shaped (`ncu --metrics gpu__time_duration.sum`, 5 steps, "
               "size-switched GEMMs off: ncu cannot replay graphs with conditional nodes)", "",
               f"Serialised cold sum {per_step:.0f} µs per step (the graph overlaps the sampling branch with "
               "training).", "", table]
    traffic = {}
    for rep, title, keep in (("ncu_full_kernels.ncu-rep", "training-branch HBM kernels in the timed configuration "
                              "(`scripts/kernel_ncu.py`: eager launches with the step graph's arguments)", None),
                             ("ncu_full_sampler.ncu-rep", "sampling-branch kernels, one chain "
                              "(`scripts/sampler_ncu.py`; selection tiers and enumeration kept)",
                              "sample_warp|sample_stream|enumerate_apply"),
                             ("ncu_full_step.ncu-rep", "training-branch SpMM kernels", None),
                             ("ncu_full_gather.ncu-rep", "reference-API gather", None)):
        path = os.path.join(src, rep)
        if not os.path.exists(path):
            continue
        dst = os.path.join(PROF, f"{tag}_{rep}")
        if keep:   # commit the main kernels only (the full report stays in gpurun_out/)
            subprocess.run(["ncu", "-i", path, "-k", f"regex:{keep}", "--export", dst, "-f"], capture_output=True)
        else:
            shutil.copy(path, dst)
        rows = ncu_rows(path)
        if keep:
            import re
            rows = [d for d in rows if re.search(keep, d.get("Kernel Name", ""))]
        md += ["", f"## `ncu --set full`: {title} (`profiles/{tag}_{rep}`)", "",
               "| kernel | grid | " + " | ".join(u for _, u, _ in METRICS[:-1]) + " |",
               "|---|---:|" + "---:|" * (len(METRICS) - 1)]
        for d in rows:
            name = d.get("Kernel Name", "?").split("(")[0].replace("void ", "")[:50]
            vals = []
            for key, unit, sc in METRICS[:-1]:
                x = num(d, key)
                vals.append("—" if x is None else f"{x * sc:.1f}")
            md.append(f"| `{name}` | {d.get('launch__grid_size', '')} | " + " | ".join(vals) + " |")
            rd, wr = num(d, "dram__bytes_read.sum"), num(d, "dram__bytes_write.sum")
            if rd is not None and wr is not None:
                kn = d.get("Kernel Name", "")
                if "spmm_fwd_chunk_kernel<0, 1" in kn or "spmm_fwd_chunk_kernel<false, true" in kn:
                    traffic.setdefault("spmm_fwd_gather", int(rd + wr))
                if "spmm_bwd_rows_kernel" in kn:
                    traffic.setdefault("spmm_bwd_transposed", int(rd + wr))
                if "gather_f32x4" in d.get("Kernel Name", ""):
                    traffic.setdefault("gather_f32x4_kernel", int(rd + wr))
    if traffic:
        with open(os.path.join(PROF, "traffic.json"), "w") as f:
            json.dump({"_note": f"dram__bytes_read.sum + dram__bytes_write.sum per launch, first launch of each "
                                f"kernel in profiles/{tag}_ncu_full_kernels.ncu-rep (papers100M-shaped bench, "
                                f"the timed configuration's arguments)",
                       "papers100m": traffic}, f, indent=1)
            f.write("\n")
    with open(os.path.join(PROF, "README.md"), "w") as f:
        f.write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
