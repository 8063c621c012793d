"""Turn ncu outputs from gpurun_out/ into the committed summaries in profiles/.

    python profiles/summarize.py <tag> <launches.csv> <full.ncu-rep>

Writes profiles/<tag>_launches.csv (kernel, grid, block, duration per launch,
our kernels and torch setup kernels alike) and profiles/<tag>_ncu.md (per
kernel: duration, DRAM bytes, achieved DRAM throughput, occupancy, issue
activity, top stall reasons) from one `ncu --set full` capture.
"""
from __future__ import annotations

import csv
import io
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__grid_size", "grid"),
    ("sm__warps_active.avg.per_cycle_active", "warps active/SM"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("lts__t_bytes.sum", "L2 bytes"),
]
STALLS = ["long_scoreboard", "wait", "short_scoreboard", "not_selected", "math_pipe_throttle",
          "branch_resolving", "lg_throttle", "mio_throttle", "dispatch_stall", "no_instruction"]


def launches(src: str, dst: str) -> None:
    rows = []
    with open(src) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(io.StringIO("".join(lines))):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"]
        short = name.split("(")[0].replace("void ", "").split("::")[-1][:60]
        rows.append([r["ID"], short, r["Grid Size"], r["Block Size"], r["Metric Value"]])
    with open(dst, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["launch", "kernel", "grid", "block", "duration_ns"])
        w.writerows(rows)


def full(rep: str, dst: str, tag: str) -> None:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    lines = [f"# ncu --set full summary ({tag})", "",
             "Captured with `ncu --set full --clock-control none --import-source on` on one B200 "
             "(gpurun), BERT-Large compression-stage steps (`bench.py --steps 3 --warmup 3`).", ""]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")
        lines.append(f"## {name}")
        lines.append("")
        lines.append("| metric | value |")
        lines.append("|---|---|")
        for m, label in METRICS:
            if m in hdr:
                lines.append(f"| {label} (`{m}`) | {r[hdr.index(m)]} {units[hdr.index(m)]} |")
        st = []
        for s in STALLS:
            k = f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"
            if k in hdr:
                try:
                    st.append((float(r[hdr.index(k)]), s))
                except ValueError:
                    pass
        st.sort(reverse=True)
        lines.append(f"| top stalls (warps per issue) | " +
                     ", ".join(f"{s} {v:.2f}" for v, s in st[:4]) + " |")
        lines.append("")
    with open(dst, "w") as f:
        f.write("\n".join(lines))
    traffic = {}
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "").split("::")[-1]
        base = name.split("<")[0]
        rd = float(r[hdr.index("dram__bytes_read.sum")])
        wr = float(r[hdr.index("dram__bytes_write.sum")])
        scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
        u_r = scale[units[hdr.index("dram__bytes_read.sum")]]
        u_w = scale[units[hdr.index("dram__bytes_write.sum")]]
        traffic[base] = {"kernel": name, "dram_bytes": rd * u_r + wr * u_w}
    with open(os.path.join(HERE, f"{tag}_traffic.json"), "w") as f:
        json.dump(traffic, f, indent=1)


if __name__ == "__main__":
    tag, lcsv, rep = sys.argv[1:4]
    launches(lcsv, os.path.join(HERE, f"{tag}_launches.csv"))
    full(rep, os.path.join(HERE, f"{tag}_ncu.md"), tag)
    print("wrote", tag)
