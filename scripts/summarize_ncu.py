#!/usr/bin/env python3
"""Summarise ncu captures from gpurun_out/ into profiles/ (tracked).

    python scripts/summarize_ncu.py r01 c2:prof_c2 c5:prof_c5 c4:prof_c4

For each config: the `--set full` report gpurun_out/<rep>.ncu-rep and the
launch list gpurun_out/launches_<cfg>.csv.  Writes
profiles/<round>_ncu_summary.md, copies the launch lists to
profiles/<round>_launches_<cfg>.csv and updates profiles/traffic.json
(dram read+write bytes per launch of the dominant kernel, keyed
"<cfg>:<kernel name as reported by hpar_last_kernel>").
"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

RAW = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
       "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
       "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
       "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_sector_hit_rate.pct"]
KERNEL_NAMES = {"rowwise": "rowwise_tma_dsmem", "flat_tma": "flat_tma", "hist": "hist256_lanepriv_tma",
                "segmented": "segmented_csr", "teams": "teams_threads", "stencil5": "stencil5_tma", "generic": "generic"}


def unit_scale(unit: str) -> float:
    return {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-9, "us": 1e-6,
            "ms": 1e-3, "s": 1.0}.get(unit, 1.0)


def raw_metrics(rep: str) -> tuple[str, dict]:
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    name = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
    out = {}
    for k in RAW:
        if k in hdr:
            i = hdr.index(k)
            v = vals[i].replace(",", "")
            try:
                out[k] = (float(v) * unit_scale(units[i]), units[i])
            except ValueError:
                out[k] = (v, units[i])
    return name, out


def main():
    rnd = sys.argv[1]
    os.makedirs(PROF, exist_ok=True)
    tpath = os.path.join(PROF, "traffic.json")
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    lines = [f"# ncu summary, {rnd}", "",
             "Captured with `ncu --set full --clock-control none --import-source on` under gpurun on one B200",
             "(scripts/profile_all.sh), after the same command exited 0 without ncu.  Times are from a",
             "serialised, profiled replay: compare shares, not absolutes.  Bytes are per launch.", ""]
    # sections of configs not re-captured this time are kept from the existing file
    sections = {}
    spath = os.path.join(PROF, f"{rnd}_ncu_summary.md")
    if os.path.exists(spath):
        cur = None
        for ln in open(spath).read().split("\n"):
            if ln.startswith("## "):
                cur = ln[3:].split(":")[0]
                sections[cur] = []
            if cur is not None:
                sections[cur].append(ln)
    for spec in sys.argv[2:]:
        cfg, rep = spec.split(":")
        body = []
        sections[cfg] = body
        path = os.path.join(OUT, rep + ".ncu-rep")
        if not os.path.exists(path):
            continue
        name, m = raw_metrics(path)
        short = next((v for k, v in KERNEL_NAMES.items() if k in name), name)
        rd = m.get("dram__bytes_read.sum", (0,))[0]
        wr = m.get("dram__bytes_write.sum", (0,))[0]
        dur = m.get("gpu__time_duration.sum", (0,))[0]
        traffic[f"{cfg}:{short}"] = int(rd + wr)
        body.append(f"## {cfg}: `{name[:110]}`")
        body.append("")
        body.append("| metric | value |")
        body.append("|---|---|")
        for k, (v, u) in m.items():
            if isinstance(v, float):
                if u.endswith("byte"):
                    v = f"{v:,.0f} B"
                elif u in ("ns", "us", "ms", "s"):
                    v = f"{v * 1e6:,.2f} us"
                else:
                    v = f"{v:,.2f} {u}"
            body.append(f"| {k} | {v} |")
        if dur:
            body.append(f"| DRAM read+write / duration | {(rd + wr) / dur / 1e9:,.0f} GB/s |")
        body.append("")
        lc = os.path.join(OUT, f"launches_{cfg}.csv")
        if os.path.exists(lc):
            shutil.copy(lc, os.path.join(PROF, f"{rnd}_launches_{cfg}.csv"))
    for cfg in sorted(sections):
        body = sections[cfg]
        while body and body[-1] == "":
            body.pop()
        lines += body + [""]
    open(spath, "w").write("\n".join(lines) + "\n")
    json.dump(traffic, open(tpath, "w"), indent=1, sort_keys=True)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
