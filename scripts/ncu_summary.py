"""Summarise ncu artefacts into profiles/ (run here, on the CPU box).

    python scripts/ncu_summary.py report.ncu-rep out.md        # --set full capture
    python scripts/ncu_summary.py launches.csv out.md           # gpu__time_duration launch list
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_active.avg", "sm__cycles_active.max", "sm__cycles_active.min",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "launch__grid_size", "launch__block_size",
]


def rep_summary(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    lines = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        lines.append(f"### {d.get('Kernel Name', '?')[:120]}\n")
        for k in KEYS:
            if k in d:
                lines.append(f"- `{k}` = {d[k]} {u.get(k, '')}")
        stalls = []
        for k, v in d.items():
            if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("_per_issue_active.ratio"):
                try:
                    if float(v) > 0.1:
                        stalls.append((float(v), k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")))
                except ValueError:
                    pass
        if stalls:
            lines.append("- stalls (warps per issue): " + ", ".join(f"{n} {v:.2f}" for v, n in sorted(stalls, reverse=True)))
        rd = float(d.get("dram__bytes_read.sum", "0") or 0)
        wr = float(d.get("dram__bytes_write.sum", "0") or 0)
        lines.append(f"- DRAM traffic per launch = {rd + wr:.1f} {u.get('dram__bytes_read.sum', '')}\n")
    return "\n".join(lines)


def launches_summary(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = defaultdict(list)
    for r in rows[hdr + 1:]:
        if len(r) > vi:
            agg[r[ki][:70]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    lines = ["| kernel | launches | mean us | share |", "|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"| `{k}` | {len(v)} | {sum(v) / len(v) / 1e3:.1f} | {100 * sum(v) / tot:.1f}% |")
    return "\n".join(lines)


if __name__ == "__main__":
    src, dst = sys.argv[1], sys.argv[2]
    body = rep_summary(src) if src.endswith(".ncu-rep") else launches_summary(src)
    with open(dst, "w") as fh:
        fh.write(f"# ncu summary of `{src.split('/')[-1]}`\n\n{body}\n")
    print(dst)
