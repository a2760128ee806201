"""The subtree partition on one GPU: a context in the virtual mode runs all P
shards phase by phase with the same shard code and exchange items as the NCCL mode (only the
transport differs).  Per-pair kernels see identical inputs, so the recompressed matrix must be
BITWISE identical to the single-shard run: matvec outputs, ranks; certified sums up to the
summation order; and the single-shard run is itself parity-checked against the oracle
(tests/test_gpu_parity.py)."""
import numpy as np
import pytest

from synth import get_config, mesh_for, seeded_vector

pytestmark = pytest.mark.gpu

_RUNS = {}


def run(name, world):
    from paper_1809_04384_b200 import DH2
    key = (name, world)
    if key not in _RUNS:
        cfg = get_config(name)
        xyz, tri = mesh_for(cfg)
        h = DH2(xyz, tri, cfg["kappa"], cfg["m"], cfg["leaf"], cfg["eta1"], cfg["eta2"], world=world)
        h.recompress(cfg["eps"])
        _RUNS[key] = h
    return _RUNS[key]


CASES = [(n, w) for n in ["P1", "P2", "P3", "P4", "C1"] for w in (2, 4)] + [("C2", 2), ("C2", 4), ("C2", 8)]


@pytest.mark.parametrize("name,world", CASES)
def test_sharded_equals_single(name, world):
    h1, hp = run(name, 1), run(name, world)
    s1, sp = h1.stats(), hp.stats()
    assert sp["transport"] == "virtual" and sp["shards_here"] == world and sp["world"] == world
    assert sp["exchange_bytes"] > 0
    for side in ("row", "col"):
        assert np.array_equal(h1.export("rank_" + side, np.int32), hp.export("rank_" + side, np.int32)), side
    for key in ("E_row", "E_col", "far2"):
        assert abs(sp[key] - s1[key]) <= 1e-13 * max(abs(s1[key]), 1e-300), key
    for seed in (1, 2):
        x = seeded_vector(h1.n, seed)
        assert np.array_equal(h1.matvec(x, 1), hp.matvec(x, 1)), "RECOMP matvec differs"
        assert np.array_equal(h1.matvec(x, 0), hp.matvec(x, 0)), "ORIG matvec differs"
    r1, rp = h1.storage(1), hp.storage(1)
    for f in ("row_basis_bytes", "col_basis_bytes", "coupling_bytes", "nearfield_bytes", "max_rank"):
        assert r1[f] == rp[f], f
    assert abs(r1["mean_rank"] - rp["mean_rank"]) <= 1e-12 * r1["mean_rank"]


def test_sharded_device_pointers():
    """matvec with device pointers (bench path) on the virtual partition."""
    import torch
    h1, hp = run("P2", 1), run("P2", 4)
    x = torch.from_numpy(seeded_vector(h1.n, 3)).to("cuda")
    y1, yp = torch.empty_like(x), torch.empty_like(x)
    h1.matvec_device(x.data_ptr(), y1.data_ptr(), 1)
    hp.matvec_device(x.data_ptr(), yp.data_ptr(), 1)
    torch.cuda.synchronize()
    assert torch.equal(y1, yp)
