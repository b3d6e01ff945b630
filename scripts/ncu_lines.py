"""Aggregate ncu stall samples per CUDA source line (needs -lineinfo builds).

  python scripts/ncu_lines.py <report.ncu-rep> <object.o> <kernel-substring> <source.cu> [top]
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

rep, obj, kern, src = sys.argv[1:5]
top = int(sys.argv[5]) if len(sys.argv) > 5 else 30
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, check=True, capture_output=True)
cubin = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
dis = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cubin)], capture_output=True, text=True).stdout
lines, inside, cur = {}, False, None
for l in dis.splitlines():
    if l.startswith(".text."):
        inside = kern in l
        continue
    if not inside:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (os.path.basename(m.group(1)), int(m.group(2)))
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
    if m and cur:
        lines[int(m.group(1), 16)] = cur
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, data = rows[1], rows[2:]
ia, isamp, iex = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
base = int(data[0][ia], 16)
tot = sum(float(r[isamp] or 0) for r in data)
agg, ex = collections.Counter(), collections.Counter()
for r in data:
    ln = lines.get(int(r[ia], 16) - base)
    agg[ln] += float(r[isamp] or 0)
    ex[ln] += int(r[iex] or 0)
text = {os.path.basename(src): open(src).read().split("\n")}
for ln, s in sorted(agg.items(), key=lambda x: -x[1])[:top]:
    code = text.get(ln[0], [""] * (ln[1] + 1))[ln[1] - 1].strip()[:80] if ln else ""
    print(f"{100 * s / tot:5.1f}% {ex[ln]:>12} {ln}: {code}")
