"""Summarise ncu reports / launch lists into profiles/ (run here, no GPU).

    python tools/ncu_summary.py gpurun_out/r01_retain.ncu-rep ...   -> markdown table
    python tools/ncu_summary.py --launches gpurun_out/r01_launches_c3.csv
"""

from __future__ import annotations

import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid size"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "global load sectors"),
    ("l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum", "global store sectors"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
]


def raw(rep: str) -> list[dict]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"Kernel Name": r[h.index("Kernel Name")]}
        for k, _ in KEYS:
            if k in h:
                i = h.index(k)
                d[k] = (r[i], units[i])
        res.append(d)
    return res


def report(reps: list[str]) -> str:
    lines = []
    for rep in reps:
        for d in raw(rep):
            lines.append(f"### `{d['Kernel Name'][:90]}`  ({rep.split('/')[-1]})\n")
            lines.append("| metric | value |\n|---|---|")
            for k, label in KEYS:
                if k in d:
                    v, u = d[k]
                    lines.append(f"| {label} (`{k}`) | {v} {u} |")
            lines.append("")
    return "\n".join(lines)


def launches(path: str) -> str:
    rows = list(csv.reader([l for l in open(path) if not l.startswith("==")]))
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    tot, cnt = defaultdict(float), defaultdict(int)
    for r in rows[1:]:
        name = r[ki].split("(")[0]
        tot[name] += float(r[vi].replace(",", ""))
        cnt[name] += 1
    T = sum(tot.values())
    out = ["| kernel | launches | total ms | mean ms | share |", "|---|---|---|---|---|"]
    for k in sorted(tot, key=lambda k: -tot[k]):
        out.append(f"| `{k}` | {cnt[k]} | {tot[k] / 1e6:.3f} | {tot[k] / cnt[k] / 1e6:.3f} | {tot[k] / T:.3f} |")
    return "\n".join(out)


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        print(launches(sys.argv[2]))
    else:
        print(report(sys.argv[1:]))
