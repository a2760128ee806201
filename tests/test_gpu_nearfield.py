"""Parity of the nearfield (NEXT-4) through the C ABI with oracle/nearfield.py:
the assembled inadmissible leaves entrywise (Sauter-Schwab n_q = 5 for touching pairs, Duffy-Gauss
n_q = 3 otherwise, the same rules on both sides: only the summation order differs), the nearfield
matvec and the full product G x = G_far x + N x, the shard partition, and the error paths.

Tolerance: each block to 1e-12 of its largest entry.  An entry is a sum of at most 6 x 625 terms of
one sign pattern per region; rounding of that sum is ~1e-15 relative to the sum of magnitudes,
and within a near block the entries vary by less than 1e3, so 1e-12 leaves a margin of 10.
"""
import numpy as np
import pytest

from synth import get_config, mesh_for, seeded_vector
from oracle import nearfield as nf
from oracle import ops
from oracle.structure import DH2Structure

from conftest import oracle_run, release_gpu_contexts

pytestmark = pytest.mark.gpu

_RUNS = {}


def near_run(name, world=1):
    from paper_1809_04384_b200 import DH2
    key = (name, world)
    if key not in _RUNS:
        cfg = get_config(name)
        xyz, tri = mesh_for(cfg)
        h = DH2(xyz, tri, cfg["kappa"], cfg["m"], cfg["leaf"], cfg["eta1"], cfg["eta2"], world=world)
        h.nearfield_assemble()
        _RUNS[key] = (h, cfg, xyz, tri)
    return _RUNS[key]


def _blocks_gpu(h):
    near = h.export("near", np.int64).reshape(-1, 2)
    off = h.export("near_off", np.int64)
    val = h.export("near_values", np.complex128)
    return near, off, val


def _check_block(cfg, xyz, tri, st, t, s, got):
    ct = st.ct
    rows = np.asarray(ct.perm[ct.begin[t]: ct.begin[t] + ct.size(t)])
    cols = np.asarray(ct.perm[ct.begin[s]: ct.begin[s] + ct.size(s)])
    ref = nf.near_block(xyz, tri, rows, cols, cfg["kappa"])
    G = got.reshape(len(cols), len(rows)).T
    err = np.abs(G - ref).max() / np.abs(ref).max()
    assert err <= 1e-12, (t, s, err)


@pytest.mark.parametrize("name", ["P1", "P3", "C1", "P8"])
def test_nearfield_blocks_all(name):
    h, cfg, xyz, tri = near_run(name)
    st = DH2Structure(xyz, tri, cfg["kappa"], cfg["m"], cfg["leaf"], cfg["eta1"], cfg["eta2"])
    near, off, val = _blocks_gpu(h)
    assert np.array_equal(near, np.asarray(st.near).reshape(-1, 2))
    ct = st.ct
    sizes = [ct.size(int(t)) * ct.size(int(s)) for t, s in near]
    assert np.array_equal(off, np.concatenate([[0], np.cumsum(sizes)[:-1]]))
    assert len(val) == sum(sizes)
    assert h.storage(0)["nearfield_bytes"] == 16.0 * len(val)
    for b, (t, s) in enumerate(near):
        _check_block(cfg, xyz, tri, st, int(t), int(s), val[off[b]: off[b] + sizes[b]])


def test_nearfield_blocks_sampled_c2():
    h, cfg, xyz, tri = near_run("C2")
    st = oracle_run("C2").st
    near, off, val = _blocks_gpu(h)
    rng = np.random.default_rng(7)
    ct = st.ct
    for b in rng.choice(len(near), 150, replace=False):
        t, s = (int(v) for v in near[b])
        _check_block(cfg, xyz, tri, st, t, s, val[off[b]: off[b] + ct.size(t) * ct.size(s)])


@pytest.mark.parametrize("name", ["P2", "C1"])
def test_full_matvec(name):
    """G x = G_far x + N x for the interpolation (ORIG) and the recompressed (RECOMP) matrix."""
    h, cfg, xyz, tri = near_run(name)
    rc = oracle_run(name)
    h.recompress(cfg["eps"])
    blocks = nf.nearfield_blocks(rc.st, xyz, tri, cfg["kappa"])
    for seed in (1, 2):
        x = seeded_vector(h.n, seed)
        yn = nf.near_matvec(rc.st, blocks, x)
        for which, tag in ((0, "orig"), (1, "recomp")):
            yf = ops.matvec(rc, x, tag)
            y = h.matvec(x, which, add_near=True)
            tol = 1e-12 if which == 0 else 1e-10  # north_star's far-field tolerance for RECOMP
            assert np.linalg.norm(y - (yf + yn)) <= tol * np.linalg.norm(yf + yn)
            d = y - h.matvec(x, which)  # the nearfield part alone
            assert np.linalg.norm(d - yn) <= 1e-12 * np.linalg.norm(yn)


def test_shards_bitwise():
    h1, cfg, xyz, tri = near_run("C1")
    h2, _, _, _ = near_run("C1", world=2)
    h1.recompress(cfg["eps"])
    h2.recompress(cfg["eps"])
    x = seeded_vector(h1.n, 3)
    assert np.array_equal(h1.matvec(x, 1, add_near=True), h2.matvec(x, 1, add_near=True))
    a = np.concatenate([h2.export("near_values", np.complex128, shard=p) for p in (0, 1)])
    assert np.array_equal(a, h1.export("near_values", np.complex128))


def test_errors():
    from paper_1809_04384_b200 import DH2
    from paper_1809_04384_b200.dh2 import DH2Error
    cfg = get_config("P1")
    xyz, tri = mesh_for(cfg)
    h = DH2(xyz, tri, cfg["kappa"], cfg["m"], cfg["leaf"], cfg["eta1"], cfg["eta2"])
    x = seeded_vector(h.n, 1)
    with pytest.raises(DH2Error, match="DH2_ESTATE"):
        h.matvec(x, 0, add_near=True)
    with pytest.raises(DH2Error, match="DH2_EINVAL"):
        h.nearfield_assemble(0, 3)
    with pytest.raises(DH2Error, match="DH2_EINVAL"):
        h.nearfield_assemble(5, 9)
    h.nearfield_assemble(5, 3)
    h.nearfield_assemble(5, 3)  # re-assembly
    h.matvec(x, 0, add_near=True)
    h.close()


@pytest.mark.parametrize("name", ["C4", "C5"])
def test_full_size_sampled(name):
    """BASELINE's full-size meshes (after the recompression, memory-lean plan): sampled blocks."""
    release_gpu_contexts()
    from paper_1809_04384_b200 import DH2
    cfg = get_config(name)
    xyz, tri = mesh_for(cfg)
    h = DH2(xyz, tri, cfg["kappa"], cfg["m"], cfg["leaf"], cfg["eta1"], cfg["eta2"])
    h.recompress(cfg["eps"])
    h.nearfield_assemble()
    near = h.export("near", np.int64).reshape(-1, 2)
    off = h.export("near_off", np.int64)
    perm = h.export("perm", np.int64)
    begin = h.export("c_begin", np.int64)
    end = h.export("c_end", np.int64)
    rng = np.random.default_rng(11)
    for b in rng.choice(len(near), 12, replace=False):
        t, s = (int(v) for v in near[b])
        nt, ns = end[t] - begin[t], end[s] - begin[s]
        got = h.export("near_values@%d:%d" % (off[b], nt * ns), np.complex128)
        ref = nf.near_block(xyz, tri, perm[begin[t]:end[t]], perm[begin[s]:end[s]], cfg["kappa"])
        G = got.reshape(ns, nt).T
        assert np.abs(G - ref).max() <= 1e-12 * np.abs(ref).max()
    x = seeded_vector(h.n, 1)
    y = h.matvec(x, 1, add_near=True)
    assert np.all(np.isfinite(y))
    st = h.stats()
    assert st["kernels"]["nearfield"]["launches"] >= 3 and st["nearfield"]["assembled"]
    assert st["nearfield"]["touching_entries"] > h.n
    h.close()


@pytest.mark.parametrize("name", ["P1", "P8", "C1", "P6", "P7"])
def test_near_matvec_tma_and_direct(name):
    """Both forms of the nearfield matvec (option near_tma: 1 = blocks streamed through shared memory
    by cp.async.bulk stages, 0 = direct global loads) against the oracle's N x; leaves of 8, 15 (ragged,
    cut mesh), 16 and 64 triangles, i.e. both row widths of the kernel and chunks that end inside a
    stage.  The two forms sum each row in a different order: equal to rounding, not bitwise."""
    h, cfg, xyz, tri = near_run(name)
    st = DH2Structure(xyz, tri, cfg["kappa"], cfg["m"], cfg["leaf"], cfg["eta1"], cfg["eta2"])
    blocks = nf.nearfield_blocks(st, xyz, tri, cfg["kappa"])
    for seed in (1, 2):
        x = seeded_vector(h.n, seed)
        yn = nf.near_matvec(st, blocks, x)
        far = h.matvec(x, 0)
        got = {}
        for tma in (1, 0):
            h.set_option("near_tma", tma)
            got[tma] = h.matvec(x, 0, add_near=True) - far
            assert np.linalg.norm(got[tma] - yn) <= 1e-12 * np.linalg.norm(yn)
        assert np.linalg.norm(got[1] - got[0]) <= 1e-13 * np.linalg.norm(yn)
    h.set_option("near_tma", 1)
    from paper_1809_04384_b200.dh2 import DH2Error
    with pytest.raises(DH2Error, match="DH2_EINVAL"):
        h.set_option("near_tma", 2)
