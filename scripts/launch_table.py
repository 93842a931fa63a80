"""Summarise an ncu --csv launch list (gpu__time_duration.sum): per-kernel
totals/averages and one step's launch sequence.

    python scripts/launch_table.py gpurun_out/launches.csv [steps] [--seq N]
"""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ki, vi, ui, gi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit"), h.index("Grid Size")
    out = []
    for r in rows[hi + 1:]:
        v = float(r[vi].replace(",", ""))
        v = v / 1000 if r[ui] == "nsecond" else v * 1000 if r[ui] == "msecond" else v
        out.append((r[ki], r[gi], v))
    return out


def main():
    data = load(sys.argv[1])
    steps = int(sys.argv[2]) if len(sys.argv) > 2 and not sys.argv[2].startswith("-") else 5
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for k, _, v in data:
        name = k.split("(")[0].replace("void ", "")[:60]
        tot[name] += v
        cnt[name] += 1
    T = sum(tot.values())
    print(f"{len(data)} launches, {T / steps:.1f} us per step (serialised, cold), {steps} steps")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{v / T * 100:5.1f}%  {v / steps:7.1f} us/step  {v / cnt[k]:7.1f} us x{cnt[k] / steps:4.1f}/step  {k}")
    if "--seq" in sys.argv:
        n = int(sys.argv[sys.argv.index("--seq") + 1])
        for k, g, v in data[:n]:
            print(f"{v:8.1f} {g:>14s} {k.split('(')[0][:70]}")


if __name__ == "__main__":
    main()
