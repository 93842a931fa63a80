"""SASS lines of one kernel in an ncu report executed at least N times
(instruction count, stall samples), offsets relative to the kernel start:

    python scripts/ncu_hot_lines.py rep.ncu-rep name-substring [min_count] [instance]
"""
import csv
import io
import subprocess
import sys

rep, name = sys.argv[1], sys.argv[2]
mn = int(sys.argv[3]) if len(sys.argv) > 3 else 0
inst = int(sys.argv[4]) if len(sys.argv) > 4 else 0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
blocks, cur = [], None
for r in csv.reader(io.StringIO(out)):
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}
        blocks.append(cur)
    elif cur is not None:
        cur["rows"].append(r)
b = [x for x in blocks if name in x["name"]][inst]
hdr = b["rows"][0]
ix = {h: i for i, h in enumerate(hdr)}
I, S = ix["Instructions Executed"], ix["Warp Stall Sampling (All Samples)"]
rows = [r for r in b["rows"][1:] if len(r) == len(hdr)]
base = int(rows[0][0], 16)
tot = sum(int(r[I] or 0) for r in rows)
print(b["name"][:100], "total instructions", tot)
for r in rows:
    n = int(r[I] or 0)
    if n >= mn and n > 0:
        print(f"{int(r[0], 16) - base:05x} {n:9d} {r[S]:>5s}  {r[1][:72]}")
