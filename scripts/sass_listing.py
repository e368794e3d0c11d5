"""Annotated SASS listing of k_simulate<16, true> for a source-line range: executed count per
instruction from an ncu report, source line from nvdisasm -g of the same libsamu.so.
  python scripts/sass_listing.py report.ncu-rep libsamu.so first_line last_line [min_count]"""
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

rep, so, a, b = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
mn = float(sys.argv[5]) if len(sys.argv) > 5 else 0
fn = sys.argv[6] if len(sys.argv) > 6 else "_Z10k_simulateILi16ELb1ELi1EEv9SimLaunch"
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=tmp, capture_output=True)
cub = [f for f in os.listdir(tmp) if f.startswith("k_simulate") and f.endswith(".cubin")][0]
sass = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cub)], capture_output=True, text=True).stdout
line_of, cur, inside = {}, None, False
for ln in sass.splitlines():
    if ln.startswith(".text."):
        inside = ln.startswith(f".text.{fn}:")
        continue
    if not inside:
        continue
    m = re.search(r'//## File "(.*)", line (\d+)', ln)
    if m:
        cur = int(m.group(2)) if os.path.basename(m.group(1)) == "k_simulate.cu" else -int(m.group(2))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
    if m:
        line_of[int(m.group(1), 16)] = cur
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows[2:] if len(r) == len(hdr)]
base = int(data[0][ix["Address"]], 16)
mx = max(int(r[ix["Instructions Executed"]]) for r in data)
last_in = False
for r in data:
    off = int(r[ix["Address"]], 16) - base
    l = line_of.get(off)
    n = int(r[ix["Instructions Executed"]])
    inr = l is not None and a <= abs(l) <= b if l and l > 0 else last_in
    if l is not None and l > 0:
        last_in = a <= l <= b
    if inr and n >= mn * mx:
        print(f"{off:06x} {l if l else '':>6} {n:>12d}  {r[ix['Source']].strip()}")
