"""C-ABI checks that need no GPU: libdh2.so loads and exports every symbol include/dh2.h
declares, errors are reported through return codes, and the host structures built by the
C++ library (structure-only context, device = DH2_DEVICE_NONE) are bit-identical to the
oracle's independent construction (parity gate G0: exact)."""
import ctypes
import os
import re

import numpy as np
import pytest

from synth import get_config, mesh_for
from oracle.structure import DH2Structure
from oracle.recompress import Recompression
from oracle import ops

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_1809_04384_b200 import build
    build.build()
    from paper_1809_04384_b200 import dh2
    return dh2.load_library()


def test_header_symbols_exported(lib):
    hdr = open(os.path.join(ROOT, "include", "dh2.h")).read()
    declared = set(re.findall(r"\b(dh2_[a-z_]+)\s*\(", hdr))
    from paper_1809_04384_b200.dh2 import EXPORTED
    assert declared == set(EXPORTED)
    for name in declared:
        assert hasattr(lib, name), name


def _structure_ctx(cfg):
    from paper_1809_04384_b200.dh2 import DH2
    xyz, tri = mesh_for(cfg)
    return DH2(xyz, tri, cfg["kappa"], cfg["m"], cfg["leaf"], cfg["eta1"], cfg["eta2"], device=-1), xyz, tri


def test_invalid_arguments(lib):
    from paper_1809_04384_b200.dh2 import DH2, DH2Error, DH2_EINVAL, DH2_ENOTIMPL, DH2_ESTATE
    xyz = np.array([[0.0, 0, 0], [1, 0, 0], [0, 1, 0]])
    with pytest.raises(DH2Error) as e:
        DH2(xyz, np.array([[0, 1, 3]]), 1.0, 3, 8, device=-1)  # index out of range
    assert e.value.code == DH2_EINVAL
    with pytest.raises(DH2Error) as e:
        DH2(xyz, np.array([[0, 1, 1]]), 1.0, 3, 8, device=-1)  # zero area
    assert e.value.code == DH2_EINVAL
    with pytest.raises(DH2Error) as e:
        DH2(xyz, np.array([[0, 1, 2]]), 1.0, 6, 8, device=-1)  # m = 6 (k = 216) beyond the grid tables
    assert e.value.code == DH2_ENOTIMPL
    h = DH2(xyz, np.array([[0, 1, 2]]), 1.0, 3, 8, device=-1)
    with pytest.raises(DH2Error) as e:
        h.recompress(1e-4)
    assert e.value.code == DH2_ESTATE
    with pytest.raises(DH2Error) as e:
        h.matvec(np.zeros(1, dtype=complex))
    assert e.value.code == DH2_ESTATE


def test_no_gpu_fails_loudly(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_1809_04384_b200.dh2 import DH2, DH2Error, DH2_ECUDA
    xyz, tri = mesh_for(get_config("C1"))
    with pytest.raises(DH2Error) as e:
        DH2(xyz, tri, 4.0, 3, 16, device=0)
    assert e.value.code == DH2_ECUDA


def _pairs(P):
    return np.array([(l, t, c) for l, lv in enumerate(P) for (t, c) in lv], dtype=np.int64).reshape(-1, 3)


@pytest.mark.parametrize("name", ["P0", "P1", "P2", "P3", "P8", "C1", "C2"])
def test_structure_bit_identical_to_oracle(lib, name):
    cfg = get_config(name)
    h, xyz, tri = _structure_ctx(cfg)
    st = DH2Structure(xyz, tri, cfg["kappa"], cfg["m"], cfg["leaf"], cfg["eta1"], cfg["eta2"])
    ct = st.ct
    assert np.array_equal(h.export("perm", np.int64), ct.perm)
    assert np.array_equal(h.export("c_begin", np.int64), ct.begin)
    assert np.array_equal(h.export("c_end", np.int64), ct.end)
    assert np.array_equal(h.export("c_level", np.int64), ct.level)
    assert np.array_equal(h.export("c_lo", np.float64).reshape(-1, 3), ct.lo)
    assert np.array_equal(h.export("c_hi", np.float64).reshape(-1, 3), ct.hi)
    assert np.array_equal(h.export("mdir", np.int32), np.array(st.mdir, dtype=np.int32))
    blocks = h.export("blocks", np.int64).reshape(-1, 3)
    assert np.array_equal(blocks, st.blocks)
    assert np.array_equal(h.export("near", np.int64).reshape(-1, 2), st.near)
    assert np.array_equal(h.export("row_pairs", np.int64).reshape(-1, 3), _pairs(st.row_pairs))
    assert np.array_equal(h.export("col_pairs", np.int64).reshape(-1, 3), _pairs(st.col_pairs))
    assert np.array_equal(h.export("basis_pairs", np.int64).reshape(-1, 3), _pairs(st.basis_pairs))
    dir_off = h.export("dir_off", np.int64)
    dirs = h.export("dirs", np.float64).reshape(-1, 3)
    for l in st.active_levels:
        D = dirs[dir_off[l]:dir_off[l] + st.dirs[l].shape[0]]
        assert np.array_equal(D, st.dirs[l])


def test_storage_orig_matches_oracle(lib):
    cfg = get_config("P1")
    h, xyz, tri = _structure_ctx(cfg)
    st = DH2Structure(xyz, tri, cfg["kappa"], cfg["m"], cfg["leaf"], cfg["eta1"], cfg["eta2"])
    rc = Recompression(st, cfg["eps"])
    ref = ops.storage(rc, "orig")
    got = h.storage(0)
    for key in ("row_basis_bytes", "col_basis_bytes", "coupling_bytes", "nearfield_bytes", "kb_per_dof_matrix"):
        assert got[key] == ref[key], key


@pytest.mark.parametrize("name", ["P0", "P1", "P2", "P3", "P8", "C1", "C2"])
def test_adjoint_symmetry_structure(name):
    """SURVEY NEXT-1 precondition, checked by the library on the host structure: every block
    has its antipodal mirror (s,t,-c) and every column pair (s,c) corresponds to the row pair
    (s,-c) with the same blocks (mirrored), parents, children and bounds."""
    h, _, _ = _structure_ctx(get_config(name))
    s = h.stats()
    assert s["mirror_missing"] == 0
    assert s["adjoint_symmetry"]["available"], s["adjoint_symmetry"]
    assert s["row_pairs"] == s["col_pairs"]
    with pytest.raises(Exception):
        h.set_option("adjoint_symmetry", 2)
    with pytest.raises(Exception):
        h.set_option("no_such_option", 1)
    h.close()
