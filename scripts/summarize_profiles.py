"""Summarise an ncu launch list (CSV) and an ncu --set full report into markdown.

    python scripts/summarize_profiles.py LAUNCHES.csv REPORT.ncu-rep OUT.md [title]
"""

import csv
import subprocess
import sys
from collections import defaultdict

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe active %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("launch__registers_per_thread", "registers"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "active lanes / instr"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall short_scoreboard"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall long_scoreboard"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall wait"),
    ("smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio", "stall math_pipe_throttle"),
]


def launches(path):
    rows = list(csv.reader(open(path)))
    h = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr = rows[h]
    ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
    t, n = defaultdict(float), defaultdict(int)
    for r in rows[h + 1:]:
        try:
            v = float(r[iv].replace(",", ""))
        except (ValueError, IndexError):
            continue
        k = r[ik].split("(")[0].replace("void ", "")
        t[k] += v
        n[k] += 1
    return t, n


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")}
        for m, name in METRICS:
            if m in hdr:
                u = units[hdr.index(m)]
                d[name] = r[hdr.index(m)] + (f" {u}" if u else "")
        res.append(d)
    return res


def main():
    lpath, rpath, opath = sys.argv[1:4]
    title = sys.argv[4] if len(sys.argv) > 4 else "profile"
    lines = [f"# {title}", ""]
    if lpath != "-":
        t, n = launches(lpath)
        tot = sum(t.values())
        lines += ["## Launch list (ncu gpu__time_duration.sum, cold-cache, serialised: compare shares)", "",
                  "| kernel | launches | total us | share |", "|---|---|---|---|"]
        for k in sorted(t, key=lambda k: -t[k]):
            lines.append(f"| {k} | {n[k]} | {t[k] / 1e3:.1f} | {100 * t[k] / tot:.1f}% |")
        lines.append("")
    if rpath != "-":
        lines += ["## ncu --set full (selected metrics)", ""]
        for d in full(rpath):
            lines.append(f"### {d['kernel']}")
            for _, name in METRICS:
                if name in d:
                    lines.append(f"- {name}: {d[name]}")
            lines.append("")
    open(opath, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
