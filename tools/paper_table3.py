"""The paper's own parameter setting (m = 4, leaf 32, eta1 = 10, eta2 = 1, eps = 1e-4;
PAPER.md §5) on the sphere sizes of Table 3, storage in KB/DoF against
the table's columns (hardware-independent).  ORIG storage needs no GPU (structure-only context);
the recompressed columns run the CUDA path (sizes that fit one GPU: n = 8192, 32768).

  python tools/paper_table3.py [--gpu]      (prints one JSON line per size)"""
import json, os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_1809_04384_b200 import DH2
from synth import mesh_for

# Table 3: orig basis, orig matrix, recomp rank, recomp basis, recomp matrix
TABLE3 = {8192: (16.0, 4.9, 205.5, 12, 0.2, 120.6), 32768: (32.0, 45.7, 1450.8, 15, 1.7, 312.3),
          131072: (64.0, 98.4, 5114.2, 21, 3.9, 586.7)}
gpu = "--gpu" in sys.argv
for n, (kappa, ob, om, rk, rb, rm) in TABLE3.items():
    q = int(round((n / 8) ** 0.5))
    xyz, tri = mesh_for(dict(mesh="sphere", q=q))
    line = {"n": n, "kappa": kappa, "paper": {"orig_basis": ob, "orig_matrix": om, "rank": rk, "recomp_basis": rb,
                                              "recomp_matrix": rm}}
    h = DH2(xyz, tri, kappa, 4, 32, 10.0, 1.0, device=-1)
    r = h.storage(0)
    s = h.stats()
    line["structure"] = {"blocks": s["blocks"], "near": s["near"], "row_pairs": s["row_pairs"], "device_bytes": s["device_bytes"]}
    line["ours_orig"] = {"basis": r["kb_per_dof_basis"], "matrix": r["kb_per_dof_matrix"]}
    h.close()
    if gpu and s["device_bytes"] < 150e9:
        g = DH2(xyz, tri, kappa, 4, 32, 10.0, 1.0)
        for mode in ("SPEC_BLOCKREL", "FROB_BLOCKREL"):
            t0 = time.perf_counter()
            g.recompress(1e-4, mode)
            dt = time.perf_counter() - t0
            rr = g.storage(1)
            line["ours_recomp_" + mode] = {"basis": rr["kb_per_dof_basis"], "matrix": rr["kb_per_dof_matrix"],
                                           "max_rank": rr["max_rank"], "mean_rank": rr["mean_rank"], "seconds": dt}
        g.close()
    print(json.dumps(line), flush=True)
