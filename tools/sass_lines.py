"""Attribute ncu per-instruction counts/stalls to source lines (no GPU needed).

usage: python tools/sass_lines.py <report.ncu-rep> <kernel-substring> [lib.so] [top]
Maps each SASS offset of the profiled kernel to the file:line nvdisasm -g reports
for the same cubin (built with -lineinfo), then sums instructions and stall
samples per line.
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

rep, kname = sys.argv[1], sys.argv[2]
lib = sys.argv[3] if len(sys.argv) > 3 else os.path.join(os.path.dirname(__file__), "..", "paper_2510_14982_b200",
                                                         "libapo_b200.so")
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
cubin = [os.path.join(tmp, f) for f in os.listdir(tmp) if f.endswith(".cubin")][0]
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
# find the function section
line_of = {}
cur_fn = None
cur_line = None
for ln in dis.splitlines():
    m = re.match(r"\s*\.text\.(\S+):", ln)
    if m:
        cur_fn = m.group(1)
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur_line = f"{os.path.basename(m.group(1))}:{m.group(2)}"
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s", ln)
    if m and cur_fn and kname in cur_fn:
        line_of[int(m.group(1), 16)] = cur_line
sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                      text=True).stdout
rows = list(csv.reader(io.StringIO(sass)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows[2:] if len(r) >= len(hdr)]
base = int(data[0][ix["Address"]], 16)
inst = collections.Counter()
stall = collections.Counter()
T = S = 0.0
for r in data:
    off = int(r[ix["Address"]], 16) - base
    key = line_of.get(off, "?")
    n = float(r[ix["Instructions Executed"]] or 0)
    s = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    inst[key] += n
    stall[key] += s
    T += n
    S += s
print(f"mapped {len(line_of)} offsets; total inst {T:.4g}, stall samples {S:.4g}")
keys = sorted(set(inst) | set(stall), key=lambda k: -(stall[k] / max(S, 1) + inst[k] / max(T, 1)))
for k in keys[:top]:
    print(f"  {k:28s} inst {100 * inst[k] / T:5.1f}%  stall {100 * stall[k] / S:5.1f}%")
