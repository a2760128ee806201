"""Markdown table of a round's bench lines (offline).  usage: round_summary.py TAG [DIR]
reads DIR/TAG_bench_{c4,c5,c3,c2}.json (DIR defaults to profiles/)."""
import json
import os
import sys

tag = sys.argv[1]
d = sys.argv[2] if len(sys.argv) > 2 else "profiles"
print("| config | n | device step | Mdof/s | e2e Mdof/s | dominant class: TF/s (of measured DMMA peak) | HBM passes (of measured) | nearfield matvec |")
print("|---|---|---|---|---|---|---|---|")
for c in ("c4", "c5", "c3", "c2"):
    p = os.path.join(d, "%s_bench_%s.json" % (tag, c))
    if not os.path.exists(p):
        continue
    j = json.loads(open(p).read().strip().splitlines()[-1])
    r = j["roofline"]
    hb = ", ".join("%s %.2f" % (k.replace("setup_", ""), v["frac_of_hbm"]) for k, v in r["hbm_passes"]["passes"].items())
    nf = j.get("nearfield", {})
    print("| %s | %d | %.1f ms | %.4f | %.4f | %s %.1f (%.3f) | %s | %.2f of HBM (%.3f ms) |" % (
        c.upper(), j["config"]["n"], j["ms_per_step"], j["value"], j["e2e"]["value"], r["kernel"], r["achieved"], r["frac"],
        hb, nf.get("matvec_near_frac_of_hbm", 0.0), nf.get("matvec_near_ms", 0.0)))
