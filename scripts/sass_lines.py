"""Aggregate an ncu SASS source page (instructions executed, stall samples) by CUDA source line.

  python scripts/sass_lines.py report.ncu-rep libsamu.so [top]

The SASS addresses of the ncu page are mapped to k_simulate<true>'s line table from
`nvdisasm -g` of the same libsamu.so (build with -lineinfo), so the per-line split needs no
source import.  Prints the top lines by executed warp instructions and a per-range summary.
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

rep, so = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
fn = sys.argv[4] if len(sys.argv) > 4 else "_Z10k_simulateILi16ELb1ELi1EEv9SimLaunch"

tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=tmp, capture_output=True)
cub = [f for f in os.listdir(tmp) if f.startswith("k_simulate") and f.endswith(".cubin")][0]
sass = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cub)], capture_output=True, text=True).stdout
line_of = {}
cur_line, inside = None, False
for ln in sass.splitlines():
    if ln.startswith(".text."):
        inside = ln.startswith(f".text.{fn}:")
        continue
    if not inside:
        continue
    m = re.search(r'//## File "(.*)", line (\d+)', ln)
    if m:
        f = os.path.basename(m.group(1))
        cur_line = int(m.group(2)) if f == "k_simulate.cu" else (f, int(m.group(2)))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
    if m:
        line_of[int(m.group(1), 16)] = cur_line

raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[1]
ia, ie, iss = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
data = [r for r in rows[2:] if len(r) == len(hdr)]
base = int(data[0][ia], 16)
inst, samp, hdr_i = collections.Counter(), collections.Counter(), collections.Counter()
tot_i = tot_s = 0
for r in data:
    off = int(r[ia], 16) - base
    line = line_of.get(off, -1)
    if isinstance(line, tuple):
        hdr_i[line[0]] += int(r[ie])
    i, s = int(r[ie]), int(r[iss])
    inst[line] += i
    samp[line] += s
    tot_i += i
    tot_s += s
# SAMU_SRC: the k_simulate.cu the .so was built from (default: the working tree's)
src = open(os.environ.get("SAMU_SRC") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "..",
                                                      "paper_2503_16893_b200", "csrc", "k_simulate.cu")).read().splitlines()
print(f"total warp instructions {tot_i:.4e}, stall samples {tot_s}")
for line, i in inst.most_common(top):
    if isinstance(line, tuple):
        txt, line = f"[{line[0]}:{line[1]}]", 0
    else:
        txt = src[line - 1].strip()[:90] if 0 < line <= len(src) else "?"
    print(f"{line:5d} {100 * i / tot_i:6.2f}% inst {100 * samp[line] / max(tot_s, 1):6.2f}% samp  {txt}")
print("header intrinsics:", {k: f"{100 * v / tot_i:.2f}%" for k, v in hdr_i.most_common()})
if len(sys.argv) > 5:
    ranges = [tuple(map(int, x.split("-"))) for x in sys.argv[5].split(",")]
    for a, b in ranges:
        i = sum(v for k, v in inst.items() if isinstance(k, int) and a <= k <= b)
        s = sum(v for k, v in samp.items() if isinstance(k, int) and a <= k <= b)
        print(f"lines {a}-{b}: {100 * i / tot_i:6.2f}% inst {100 * s / max(tot_s, 1):6.2f}% samp")
