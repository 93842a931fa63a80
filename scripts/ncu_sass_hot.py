"""Top SASS lines of an ncu report by warp-stall samples, per kernel
instance (the report's source page lists one block per profiled launch):

    python scripts/ncu_sass_hot.py rep.ncu-rep [N] [name-substring] [instance]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
name = sys.argv[3] if len(sys.argv) > 3 else ""
inst = int(sys.argv[4]) if len(sys.argv) > 4 else -1
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
blocks, cur = [], None
for r in csv.reader(io.StringIO(out)):
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}
        blocks.append(cur)
    elif cur is not None:
        cur["rows"].append(r)
sel = [b for b in blocks if name in b["name"]]
if not sel:
    sys.exit(f"no kernel matching {name!r}: {[b['name'][:60] for b in blocks]}")
b = sel[inst]
hdr = b["rows"][0]
ix = {h: i for i, h in enumerate(hdr)}
S, I = ix["Warp Stall Sampling (All Samples)"], ix["Instructions Executed"]
data = [r for r in b["rows"][1:] if len(r) == len(hdr)]
tot_s = sum(int(r[S] or 0) for r in data)
tot_i = sum(int(r[I] or 0) for r in data)
print(f"{b['name'][:100]} (instance {inst} of {len(sel)})\n samples {tot_s}, warp instructions {tot_i}")
data.sort(key=lambda r: -int(r[S] or 0))
for r in data[:n]:
    print(f"{r[0][-5:]} {r[1][:64]:64s} stall {r[S]:>6s} inst {r[I]:>8s}")

if "--ranges" in sys.argv or True:
    # instructions and stall samples by address range (0x200 bytes = 32 SASS lines)
    agg = {}
    for r in data:
        a = int(r[0], 16) >> 9
        x = agg.setdefault(a, [0, 0, r[1][:40]])
        x[0] += int(r[I] or 0)
        x[1] += int(r[S] or 0)
    print("--- by 0x200-byte range: instructions, stall samples, first SASS line")
    for a in sorted(agg):
        if agg[a][0] > tot_i * 0.01 or agg[a][1] > tot_s * 0.01:
            print(f"{(a << 9) & 0xfffff:05x} inst {agg[a][0]:>9d} ({agg[a][0] / tot_i:5.1%})  stall {agg[a][1]:>5d} "
                  f"({agg[a][1] / max(tot_s, 1):5.1%})  {agg[a][2]}")
