#!/usr/bin/env python
"""Attribute ncu SASS-level stall samples to CUDA source lines (offline, no GPU).

usage: sass_lines.py <ncu report> <kernel regex> <libdh2.so> [launch index]
SRC_DIR overrides the source directory used to print the lines (the sources the .so was
built from).  Extracts the cubin from the .so, disassembles the kernel with line info (nvdisasm -g) and
joins it with the per-instruction samples of `ncu -i --page source --print-source sass`.
"""
import collections
import csv
import glob
import io
import os
import re
import subprocess
import sys
import tempfile

rep, kre, so = sys.argv[1], sys.argv[2], sys.argv[3]
launch = int(sys.argv[4]) if len(sys.argv) > 4 else 0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--kernel-name",
                      "regex:" + kre, "--launch-skip", str(launch), "--launch-count", "1"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
kname = rows[0][1]
h = rows[1]
ai, si, ns, ie = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
data = []
for r in rows[2:]:
    try:
        data.append((int(r[ai], 16), int(r[ns] or 0), int(r[ie] or 0), r[si]))
    except Exception:
        pass
base = data[0][0]
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=tmp, capture_output=True)
mangled = None
lines = {}
for cub in glob.glob(os.path.join(tmp, "*.cubin")):
    syms = subprocess.run(["cuobjdump", "-symbols", cub], capture_output=True, text=True).stdout
    for s in re.findall(r"STT_FUNC\s+\S+\s+\S+\s+(\S+)", syms):
        dem = subprocess.run(["cu++filt", s], capture_output=True, text=True).stdout.strip()
        if dem.replace(" ", "") == kname.replace(" ", ""):
            mangled = s
            dis = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
            cur = None
            inside = False
            for ln in dis.splitlines():
                if ".section" in ln and ".text." in ln:
                    inside = ln.strip().endswith(".text." + s) or (".text." + s + ",") in ln
                    continue
                if not inside:
                    continue
                m = re.search(r'line (\d+)', ln)
                if "//##" in ln and m:
                    f = re.search(r'File "([^"]+)"', ln)
                    cur = (os.path.basename(f.group(1)) if f else "?", int(m.group(1)))
                m2 = re.search(r"/\*([0-9a-f]{4,})\*/", ln)
                if m2 and cur:
                    lines[int(m2.group(1), 16)] = cur
            break
    if mangled:
        break
print("kernel:", kname, "->", mangled, file=sys.stderr)
agg = collections.Counter()
aggi = collections.Counter()
tot = sum(d[1] for d in data) or 1
for addr, samp, inst, _ in data:
    key = lines.get(addr - base, ("?", 0))
    agg[key] += samp
    aggi[key] += inst
srcs = {}
for key, v in agg.most_common(30):
    f, l = key
    txt = ""
    srcdir = os.environ.get("SRC_DIR") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_1809_04384_b200", "csrc")
    for cand in glob.glob(os.path.join(srcdir, f)):
        srcs.setdefault(cand, open(cand).read().splitlines())
        if 0 < l <= len(srcs[cand]):
            txt = srcs[cand][l - 1].strip()
    print("%5.1f%%  inst %12d  %s:%d  %s" % (100.0 * v / tot, aggi[key], f, l, txt[:100]))
