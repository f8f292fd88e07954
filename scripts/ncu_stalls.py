"""Summarise an ncu report: per kernel, duration, key metrics, top stall reasons,
opcode mix and stall reasons by opcode (SASS source page).

    python scripts/ncu_stalls.py REPORT.ncu-rep [kernel-regex]
"""
import csv
import io
import re
import subprocess
import sys
from collections import Counter, defaultdict


def ncu(*args):
    return subprocess.run(["ncu", "-i", *args], capture_output=True, text=True, cwd="/tmp").stdout


def main():
    import os
    rep = os.path.abspath(sys.argv[1])
    kre = sys.argv[2] if len(sys.argv) > 2 else "."
    raw = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    h, u = raw[0], raw[1]
    names = []
    for row in raw[2:]:
        name = row[h.index("Kernel Name")]
        if not re.search(kre, name) or name in names:
            continue
        names.append(name)
        g = lambda m: row[h.index(m)] if m in h else "NA"
        print(f"## {name[:90]}")
        for m in ("gpu__time_duration.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
                  "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
                  "launch__registers_per_thread", "smsp__thread_inst_executed_per_inst_executed.ratio",
                  "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "dram__bytes_read.sum", "dram__bytes_write.sum"):
            print(f"  {m}: {g(m)} {u[h.index(m)] if m in h else ''}")
        st = [x for x in h if x.startswith("smsp__average_warps_issue_stalled_") and x.endswith("_per_issue_active.ratio")]
        vals = sorted(((float(row[h.index(x)] or 0), x) for x in st), reverse=True)[:8]
        print("  stalls/issue: " + ", ".join(f"{x.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')} {v:.2f}" for v, x in vals))
        src = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source", "sass",
                                               "--kernel-name", "regex:" + re.escape(name.split("(")[0].split("<")[0].split()[-1])))))
        if len(src) < 3:
            continue
        sh = src[1]
        ix = {k: j for j, k in enumerate(sh)}
        opc, samp = Counter(), Counter()
        by = defaultdict(Counter)
        keys = [k for k in sh if k.startswith("stall_") and "Not Issued" not in k]
        for r in src[2:]:
            if len(r) < len(sh):
                continue
            toks = r[ix["Source"]].strip().split()
            if not toks:
                continue
            op = (toks[1] if toks[0].startswith("@") else toks[0]).split(".")[0]
            try:
                opc[op] += int(r[ix["Instructions Executed"]] or 0)
                for k in keys:
                    by[k][op] += int(r[ix[k]] or 0)
            except ValueError:  # repeated header of the next kernel section
                continue
        tot = sum(opc.values())
        print("  opcode mix: " + ", ".join(f"{o} {v / tot:.3f}" for o, v in opc.most_common(10)))
        for k in sorted(keys, key=lambda k: -sum(by[k].values()))[:5]:
            print(f"  {k} by opcode: " + ", ".join(f"{o} {v}" for o, v in by[k].most_common(5)))


if __name__ == "__main__":
    main()
