#!/usr/bin/env python3
"""Stall samples and instruction counts of one ncu capture per CUDA source
line: aligns ncu's SASS source page (instruction order) with `nvdisasm -g`
of the same kernel in the built library (line-info comments), then sums per
source line.

    python scripts/ncu_lines.py <rep.ncu-rep> <lib.so> <kernel-mangled-substring> [top]
"""
import collections
import csv
import glob
import io
import os
import re
import subprocess
import sys
import tempfile

rep, lib, kname = sys.argv[1:4]
lib = os.path.abspath(lib)
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     check=True, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h, data = rows[1], rows[2:]
ix = {k: i for i, k in enumerate(h)}


def num(r, k):
    try:
        return float(r[ix[k]].replace(",", ""))
    except (KeyError, ValueError, IndexError):
        return 0.0


stall_cols = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", lib], cwd=tmp, capture_output=True)
dis = None
for cub in glob.glob(os.path.join(tmp, "*.cubin")):
    out = subprocess.run(["nvdisasm", "-g", "-c", "-fun", kname, cub], capture_output=True, text=True)
    if out.returncode == 0 and out.stdout.strip():
        # -fun takes a function index or name; fall back to the full listing
        dis = out.stdout
        break
if dis is None:
    for cub in glob.glob(os.path.join(tmp, "*.cubin")):
        out = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
        if kname in out:
            dis = out
            break
# the kernel's section: from its .text label to the next section banner
start = dis.find(".text." + kname) if (".text." + kname) in dis else dis.find(kname)
sec = dis[start:]
end = sec.find("//---------------------", 10)
sec = sec[:end] if end > 0 else sec
lines_of = []
cur = None
for ln in sec.splitlines():
    m = re.search(r'//## File "(.*?)", line (\d+)', ln)
    if m:
        cur = (os.path.basename(m.group(1)), int(m.group(2)))
        continue
    if re.match(r"\s*/\*[0-9a-f]{4,}\*/", ln):
        lines_of.append(cur)
n = min(len(lines_of), len(data))
agg = collections.defaultdict(lambda: [0.0, 0.0, collections.Counter()])
for i in range(n):
    r = data[i]
    a = agg[lines_of[i]]
    a[0] += num(r, "Warp Stall Sampling (All Samples)")
    a[1] += num(r, "Instructions Executed")
    for k in stall_cols:
        a[2][k] += num(r, k)
tot_s = sum(v[0] for v in agg.values()) or 1
tot_i = sum(v[1] for v in agg.values()) or 1
srcs = {}
for m in re.finditer(r'//## File "(.*?)"', sec):
    b = os.path.basename(m.group(1))
    if b not in srcs:
        try:
            srcs[b] = dict(enumerate(open(m.group(1)).read().splitlines(), 1))
        except Exception:
            srcs[b] = {}
print(f"aligned {n} of {len(data)} ncu SASS rows with {len(lines_of)} nvdisasm instructions\n")
print("| line | samples % | instr % | top stalls | source |")
print("|---|---|---|---|---|")
for key, (s, ins, c) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    st = ", ".join(f"{k[6:]} {100 * v / max(s, 1):.0f}%" for k, v in c.most_common(2))
    f, line = key if key else ("?", 0)
    text = srcs.get(f, {}).get(line, "").strip().replace("|", "\\|")[:70]
    print(f"| {f}:{line} | {100 * s / tot_s:.1f} | {100 * ins / tot_i:.1f} | {st} | `{text}` |")
