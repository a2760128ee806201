#!/usr/bin/env python
"""Per CUDA source line stall samples of one kernel in an ncu report (offline): the report's own
source correlation (ncu --import-source on, -lineinfo).  usage: ncu_lines.py <report> [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur, hdr, agg = None, None, {}
for r in csv.reader(io.StringIO(out)):
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 5 or not r[0].isdigit():
        continue
    try:
        st = int(r[4] or 0)
    except ValueError:
        continue
    key = (cur, int(r[0]))
    a = agg.setdefault(key, [0, r[1][:120]])
    a[0] += st
tot = sum(v[0] for v in agg.values()) or 1
for (f, ln), (st, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print("%5.1f%%  %s:%d  %s" % (100.0 * st / tot, f, ln, src.strip()))
