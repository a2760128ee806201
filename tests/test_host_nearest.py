"""The tiled search of nearest() (dh2_host.cpp) returns exactly the direction of the exhaustive
search (P:396-403 with the tie rule R4) — C++ check built with g++ against the library's host
source, on the C2 sphere at kappa 16 and 43 (every level with <= 12000 directions)."""
import os
import subprocess

import numpy as np

from synth import get_config, mesh_for

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_nearest_tiles_equal_exhaustive(tmp_path):
    cfg = get_config("C2")
    xyz, tri = mesh_for(cfg)
    np.ascontiguousarray(xyz, dtype=np.float64).tofile(tmp_path / "xyz.bin")
    np.ascontiguousarray(tri, dtype=np.int64).tofile(tmp_path / "tri.bin")
    exe = tmp_path / "nearest_check"
    src = os.path.join(ROOT, "paper_1809_04384_b200", "csrc")
    subprocess.run(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-fopenmp", "-I", src,
                    os.path.join(ROOT, "tests", "host", "nearest_check.cpp"), os.path.join(src, "dh2_host.cpp"),
                    "-o", str(exe)], check=True)
    r = subprocess.run([str(exe), str(tmp_path / "xyz.bin"), str(tmp_path / "tri.bin"), str(xyz.shape[0]),
                        str(tri.shape[0])], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "mismatches 0" in r.stdout
