#!/usr/bin/env python
"""Summarise ncu captures into profiles/ (run here, on the CPU box).

    python scripts/ncu_summary.py TAG KEY gpurun_out/prof_X.ncu-rep [launches.csv]

Writes profiles/TAG_ncu_summary.md (per-kernel duration, DRAM bytes,
DRAM % of peak, occupancy, top stall reasons) and records the dominant
streaming kernel's DRAM read+write bytes per launch under KEY (e.g.
"dsymv_32768") in profiles/traffic.json, which bench.py reports as
roofline.traffic.
"""

from __future__ import annotations

import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [dict(zip(hdr, r)) for r in rows[2:]], dict(zip(hdr, units))


def num(v):
    try:
        return float(str(v).replace(",", ""))
    except ValueError:
        return float("nan")


def main():
    tag, key, rep = sys.argv[1], sys.argv[2], sys.argv[3]
    launches = sys.argv[4] if len(sys.argv) > 4 else None
    rows, units = raw_rows(rep)
    lines = [f"# ncu summary `{tag}` ({os.path.basename(rep)})", "",
             "Captured with `ncu --set full --clock-control none --import-source on` under gpurun "
             "(cold caches, one kernel at a time: compare shares, not absolute step times).", "",
             "| kernel | time (us) | DRAM read (MB) | DRAM write (MB) | DRAM % peak | occupancy % | regs | top stalls (per issue) |",
             "|---|---|---|---|---|---|---|---|"]
    main_bytes, main_name = None, None
    for d in rows:
        name = d["Kernel Name"]
        t = num(d.get("gpu__time_duration.sum")) * {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3,
                                                     "ms": 1e3}.get(units.get("gpu__time_duration.sum"), 1.0)
        rd = num(d.get("dram__bytes_read.sum"))
        wr = num(d.get("dram__bytes_write.sum"))
        scale_r = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(units.get("dram__bytes_read.sum"), 1.0)
        scale_w = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(units.get("dram__bytes_write.sum"), 1.0)
        stalls = []
        for k, v in d.items():
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                x = num(v)
                if x == x and x > 0.3:
                    stalls.append((x, k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
        stalls.sort(reverse=True)
        lines.append(f"| `{name[:70]}` | {t:.1f} | {rd * scale_r:.1f} | {wr * scale_w:.2f} | "
                     f"{num(d.get('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed')):.1f} | "
                     f"{num(d.get('sm__warps_active.avg.pct_of_peak_sustained_active')):.1f} | "
                     f"{d.get('launch__registers_per_thread', '')} | "
                     + ", ".join(f"{n} {x:.1f}" for x, n in stalls[:4]) + " |")
        # the streaming kernel's bytes per call: the first streaming row,
        # plus every later row of the same kernel (the tail grid of a split
        # SYMV call; capture exactly one call's grids, e.g. -k regex:symv_kernel -c 2)
        if "epilogue" not in name and "scal" not in name:
            if main_bytes is None:
                main_name, main_bytes = name, 0
            if name == main_name:
                main_bytes += int((rd * scale_r + wr * scale_w) * 1e6)
    if launches:
        agg = defaultdict(list)
        rws = list(csv.reader(open(launches)))
        i = [k for k, r in enumerate(rws) if r and r[0] == "ID"][0]
        h = rws[i]
        idx = {k: j for j, k in enumerate(h)}
        for r in rws[i + 1:]:
            if len(r) < len(h) or r[idx["Metric Name"]] != "gpu__time_duration.sum":
                continue
            agg[r[idx["Kernel Name"]].split("(")[0]].append(num(r[idx["Metric Value"]]))
        tot = sum(sum(v) for k, v in agg.items() if "kb::" in k or "kernel" in k)
        lines += ["", f"Launch list (`{os.path.basename(launches)}`, `--metrics gpu__time_duration.sum`): "
                  "share of the library's kernel time", "", "| kernel | launches | mean (us) | share |", "|---|---|---|---|"]
        for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
            if "kb::" not in k:
                continue
            lines.append(f"| `{k}` | {len(v)} | {sum(v) / len(v) / 1e3:.1f} | {sum(v) / tot:.3f} |")
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", f"{tag}_ncu_summary.md"), "w") as fh:
        fh.write("\n".join(lines) + "\n")
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    traffic = json.load(open(tp)) if os.path.exists(tp) else {}
    if main_bytes:
        traffic[key] = main_bytes
        json.dump(traffic, open(tp, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
