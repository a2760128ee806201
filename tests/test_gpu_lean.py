"""The memory-lean chunked plan (SURVEY §7.4 rules 2-7) against the full plan.

Every per-pair computation of the lean plan is the full plan's, with the same kernels and the same
inputs (leaf V and S_b regenerated bitwise, weights of the direct pairs kept, the rest chunk-local),
so ranks, singular values, certified sums, the recompressed matrix and its matvec must be BITWISE
equal for any number of chunks; the full plan itself is checked against the oracle
(tests/test_gpu_parity.py).  A direct oracle check of the lean plan is added on top."""
import numpy as np
import pytest

from synth import get_config, mesh_for, seeded_vector
from oracle import ops

from conftest import oracle_run

pytestmark = pytest.mark.gpu

_RUNS = {}


def _run(name, chunks, fuse=0):
    from paper_1809_04384_b200 import DH2
    key = (name, chunks, fuse)
    if key not in _RUNS:
        cfg = get_config(name)
        xyz, tri = mesh_for(cfg)
        h = DH2(xyz, tri, cfg["kappa"], cfg["m"], cfg["leaf"], cfg["eta1"], cfg["eta2"])
        h.set_option("fuse_leaf_weights", fuse)
        if chunks:
            h.set_option("lean_chunks", chunks)
        h.recompress(cfg["eps"])
        s = h.stats()
        assert s["lean"]["on"] == bool(chunks)
        _RUNS[key] = (h, s)
    return _RUNS[key]


def _factors(h, side="row"):
    """(rank, sigma per pair, Q/F per pair, S~ per block) read through the exported offsets/lds."""
    rank = h.export("rank_" + side, np.int32)
    nsig = h.export("nsig_" + side, np.int32)
    sig = h.export("sigma_" + side, np.float64)
    sig_off = h.export("sig_off_" + side, np.int64)
    Q = h.export("Q_" + side, np.complex128)
    Q_off = h.export("Q_off_" + side, np.int64)
    rowsb = h.export("rowsb_" + side, np.int32)
    child0 = h.export("child0_" + side, np.int32)
    child1 = h.export("child1_" + side, np.int32)
    pairs = h.export(side + "_pairs", np.int64).reshape(-1, 3)
    c_begin, c_end = h.export("c_begin", np.int64), h.export("c_end", np.int64)
    sigmas, qs = [], []
    for p in range(len(rank)):
        sigmas.append(sig[sig_off[p]:sig_off[p] + nsig[p]])
        t = int(pairs[p, 1])
        rows = int(c_end[t] - c_begin[t]) if child0[p] < 0 else int(rank[child0[p]] + rank[child1[p]])
        ld = int(rowsb[p])
        kk = int(rank[p])
        qs.append(Q[Q_off[p]:Q_off[p] + ld * kk].reshape(kk, ld).T[:rows] if kk else np.zeros((rows, 0)))
    return rank, sigmas, qs


def _st_blocks(h):
    St = h.export("St", np.complex128)
    off = h.export("blk_St_off", np.int64)
    prow, pcol = h.export("blk_prow", np.int32), h.export("blk_pcol", np.int32)
    kr, kc = h.export("rank_row", np.int32), h.export("rank_col", np.int32)
    kb = h.export("kb_row", np.int32)
    blocks = h.export("blocks", np.int64).reshape(-1, 3)
    out = {}
    for b in range(len(blocks)):
        a, c, ld = int(kr[prow[b]]), int(kc[pcol[b]]), int(kb[prow[b]])
        out[tuple(int(v) for v in blocks[b])] = St[off[b]:off[b] + ld * c].reshape(c, ld).T[:a] if a and c else np.zeros((a, c))
    return out


@pytest.mark.parametrize("name,chunks,fuse", [("P1", 1, 0), ("P1", 3, 0), ("P2", 4, 0), ("P4", 2, 0), ("P6", 1, 0),
                                              ("P7", 5, 0), ("P8", 3, 0), ("C1", 8, 0), ("C2", 1, 0), ("C2", 16, 0),
                                              ("C4s", 7, 0), ("C4s", 3, 2), ("P7", 2, 2), ("P2", 3, 1)])
def test_lean_bitwise_equal_to_full(name, chunks, fuse):
    """(fuse: dh2_set_option fuse_leaf_weights on both plans: the leaf total weights folded into the
    truncation, leaf Zhat never formed)"""
    hf, sf = _run(name, 0, fuse)
    hl, sl = _run(name, chunks, fuse)
    if fuse:
        assert sl["fused_leaf_levels_row"] and sl["fused_leaf_levels_row"] == sf["fused_leaf_levels_row"]
    assert sl["lean"]["chunks"] >= 1
    for key in ("E_row", "E_col", "far2"):
        assert sl[key] == sf[key], key
    rf, sgf, qf = _factors(hf)
    rl, sgl, ql = _factors(hl)
    assert np.array_equal(rf, rl)
    for a, b in zip(sgf, sgl):
        assert np.array_equal(a, b)
    for a, b in zip(qf, ql):
        assert np.array_equal(a, b)
    assert np.array_equal(hf.export("rank_col", np.int32), hl.export("rank_col", np.int32))
    stf, stl = _st_blocks(hf), _st_blocks(hl)
    assert stf.keys() == stl.keys()
    for key in stf:
        assert np.array_equal(stf[key], stl[key]), key
    for seed in (1, 2):
        x = seeded_vector(hf.n, seed)
        assert np.array_equal(hf.matvec(x, 1), hl.matvec(x, 1))
    assert hf.storage(1) == hl.storage(1)


@pytest.mark.parametrize("name,chunks", [("P2", 3), ("P4", 2)])
def test_lean_against_oracle(name, chunks):
    """G3/G4 of tests/test_gpu_parity.py directly on the lean plan."""
    h, s = _run(name, chunks)
    rc = oracle_run(name)
    st = rc.st
    pairs = h.export("row_pairs", np.int64).reshape(-1, 3)
    rank = h.export("rank_row", np.int32)
    for p, (_, t, c) in enumerate(pairs):
        assert rank[p] == rc.row.rank[(int(t), int(c))]
    for seed in (1, 2, 3):
        x = seeded_vector(st.n, seed)
        yo = ops.matvec(rc, x, "orig")
        yr = ops.matvec(rc, x, "recomp")
        assert np.linalg.norm(h.matvec(x, 1) - yr) <= 1e-10 * np.linalg.norm(yo)
    assert abs(s["far2"] - rc.far_norm2()) <= 1e-12 * rc.far_norm2()


def test_lean_state_errors():
    from paper_1809_04384_b200 import DH2Error
    h, _ = _run("P1", 3)
    x = seeded_vector(h.n, 1)
    with pytest.raises(DH2Error):
        h.matvec(x, 0)  # ORIG needs V and S resident
    with pytest.raises(DH2Error):
        h.set_option("adjoint_symmetry", 0)


@pytest.mark.parametrize("name,world,chunks", [("P2", 2, 3), ("P4", 2, 2), ("C1", 4, 2), ("C2", 4, 3), ("C4s", 2, 5)])
def test_lean_sharded_bitwise_equal_to_full(name, world, chunks):
    """The lean plan on every shard of the subtree partition (virtual mode: the shards run on this GPU
    with device-to-device exchanges of R (s,-c), ranks and compact C'): the same matrix, bitwise."""
    from paper_1809_04384_b200 import DH2
    hf, sf = _run(name, 0)
    cfg = get_config(name)
    xyz, tri = mesh_for(cfg)
    h = DH2(xyz, tri, cfg["kappa"], cfg["m"], cfg["leaf"], cfg["eta1"], cfg["eta2"], world=world)
    h.set_option("lean_chunks", chunks)
    h.recompress(cfg["eps"])
    s = h.stats()
    assert s["lean"]["on"] and s["shards_here"] == world and s["exchange_bytes"] > 0
    for key in ("E_row", "E_col", "far2"):
        assert s[key] == pytest.approx(sf[key], rel=1e-14), key
    assert np.array_equal(h.export("rank_row", np.int32), hf.export("rank_row", np.int32))
    for seed in (1, 2):
        x = seeded_vector(hf.n, seed)
        assert np.array_equal(h.matvec(x, 1), hf.matvec(x, 1))
    assert h.storage(1) == hf.storage(1)
    h.close()
