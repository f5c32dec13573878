#!/usr/bin/env python3
"""Instruction-level hot spots of one `ncu --set full --import-source on`
capture: warp-instruction counts grouped by how often an instruction runs
(which tells the loop level it belongs to), stall reasons, and the top SASS
lines by stall samples.

    python scripts/ncu_hotspots.py gpurun_out/prof_c3.ncu-rep > profiles/r01_c3_hotspots.md
"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     check=True, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
kernel = rows[0][1] if rows and len(rows[0]) > 1 else "?"
h, data = rows[1], rows[2:]
ix = {k: i for i, k in enumerate(h)}
S, I = "Warp Stall Sampling (All Samples)", "Instructions Executed"


def f(r, k):
    try:
        return float(r[ix[k]].replace(",", ""))
    except (KeyError, ValueError, IndexError):
        return 0.0


tot_s = sum(f(r, S) for r in data) or 1.0
tot_i = sum(f(r, I) for r in data)
print(f"# ncu source hot spots: `{kernel}`\n")
print(f"{tot_i / 1e6:.1f} M warp-instructions, {int(tot_s)} stall samples.\n")
print("## Stall reasons (share of samples)\n\n| reason | % |\n|---|---|")
stalls = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
agg = {k: sum(f(r, k) for r in data) for k in stalls}
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:10]:
    print(f"| {k} | {v / tot_s * 100:.1f} |")
# group instructions by execution count (same count = same loop level)
print("\n## Execution-count classes\n\n| executions per instruction | static instrs | warp-instr (M) | % instr | % samples |")
print("|---|---|---|---|---|")
cls = collections.defaultdict(lambda: [0, 0.0, 0.0])
for r in data:
    n = f(r, I)
    if n <= 0:
        continue
    key = int(round(n, -int(max(0, len(str(int(n))) - 2))))  # 2 significant digits
    cls[key][0] += 1
    cls[key][1] += n
    cls[key][2] += f(r, S)
for key, (cnt, n, smp) in sorted(cls.items(), key=lambda x: -x[1][1])[:12]:
    print(f"| ~{key:,} | {cnt} | {n / 1e6:.1f} | {n / tot_i * 100:.1f} | {smp / tot_s * 100:.1f} |")
print("\n## Top 25 SASS lines by stall samples\n\n| address | SASS | samples | executions | top stall |\n|---|---|---|---|---|")
for r in sorted(data, key=lambda r: -f(r, S))[:25]:
    st = max(stalls, key=lambda k: f(r, k)) if stalls else ""
    src = r[ix["Source"]].strip().replace("|", "\\|")[:60]
    print(f"| {r[ix['Address']][-5:]} | `{src}` | {int(f(r, S))} | {int(f(r, I))} | {st} |")
