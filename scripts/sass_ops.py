"""Executed warp instructions of an ncu SASS page grouped by opcode (python scripts/sass_ops.py rep [n])."""
import collections
import csv
import io
import subprocess
import sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
agg, tot = collections.Counter(), 0
for r in rows[2:]:
    if len(r) != len(hdr):
        continue
    t = r[ix["Source"]].strip().split()
    if t and t[0].startswith("@"):
        t = t[1:]
    n = int(r[ix["Instructions Executed"]])
    agg[t[0] if t else "?"] += n
    tot += n
print(f"total {tot:.4e}")
for o, n in agg.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 40):
    print(f"{o:24s} {100 * n / tot:6.2f}%")
