#!/usr/bin/env python
"""Summarise ncu reports / launch lists into markdown for profiles/ (offline, no GPU).

  ncu_summary.py full <report.ncu-rep>       key counters of every profiled launch
  ncu_summary.py launches <launches.csv>     per-kernel totals of a gpu__time_duration launch list
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = [("gpu__time_duration.sum", "duration"), ("launch__grid_size", "grid"), ("launch__block_size", "block"),
        ("launch__registers_per_thread", "regs"), ("launch__shared_mem_per_block_dynamic", "dyn smem"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
        ("sm__inst_executed.avg.per_cycle_active", "IPC"),
        ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM thru %"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM thru %"),
        ("dram__bytes_read.sum", "DRAM read"), ("dram__bytes_write.sum", "DRAM write"),
        ("smsp__inst_executed.sum", "warp inst")]


def full(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    idx = {n: i for i, n in enumerate(h)}
    print("| kernel | " + " | ".join(k[1] for k in KEYS) + " |")
    print("|---" * (len(KEYS) + 1) + "|")
    for r in rows[2:]:
        name = r[idx["Kernel Name"]].split("(")[0]
        cells = []
        for k, _ in KEYS:
            i = idx.get(k)
            cells.append("%s %s" % (r[i], units[i]) if i is not None else "-")
        print("| %s | %s |" % (name, " | ".join(cells)))


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows[hi + 1:]:
        v = float(r[vi].replace(",", ""))
        unit = r[ui]
        ms = v / 1e6 if unit == "ns" else (v / 1e3 if unit in ("us", "usecond") else v)
        name = r[ki].split("(")[0]
        tot[name] += ms
        cnt[name] += 1
    allms = sum(tot.values())
    print("| kernel | launches | total ms | share |")
    print("|---|---|---|---|")
    for name, ms in sorted(tot.items(), key=lambda kv: -kv[1]):
        print("| %s | %d | %.3f | %.1f%% |" % (name, cnt[name], ms, 100 * ms / allms))
    print("| **all** | %d | %.3f | 100%% |" % (sum(cnt.values()), allms))


if __name__ == "__main__":
    {"full": full, "launches": launches}[sys.argv[1]](sys.argv[2])
