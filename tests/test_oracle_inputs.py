"""Pins of the synthetic workload meshes (SPEC geometry examples)."""
import numpy as np
import pytest

from synth import sphere_mesh, cube_mesh, seeded_vector


def _edges(tri):
    e = {}
    for a, b, c in tri:
        for u, v in ((a, b), (b, c), (c, a)):
            e.setdefault((min(u, v), max(u, v)), []).append((u, v))
    return e


def _area(xyz, tri):
    v = xyz[tri]
    cr = np.cross(v[:, 1] - v[:, 0], v[:, 2] - v[:, 0])
    return 0.5 * np.linalg.norm(cr, axis=1), cr


@pytest.mark.parametrize("q", [1, 2, 4, 8])
def test_sphere_closed_oriented(q):
    xyz, tri = sphere_mesh(q)
    assert tri.shape == (8 * q * q, 3)
    assert np.max(np.abs(np.linalg.norm(xyz, axis=1) - 1.0)) <= 1e-12
    edges = _edges(tri)
    assert all(len(v) == 2 for v in edges.values())
    # consistent orientation: shared edges traversed in opposite directions
    assert all(v[0] == (v[1][1], v[1][0]) for v in edges.values())
    assert xyz.shape[0] - len(edges) + tri.shape[0] == 2  # Euler characteristic
    area, cr = _area(xyz, tri)
    assert area.min() > 0
    cen = xyz[tri].mean(axis=1)
    assert np.all(np.einsum("ij,ij->i", cr, cen) > 0)  # outward


def test_sphere_area_increases_to_4pi():
    a = [(_area(*sphere_mesh(q))[0]).sum() for q in (4, 8, 16)]
    assert a[0] < a[1] < a[2] < 4 * np.pi


@pytest.mark.parametrize("q", [1, 3, 8])
def test_cube_closed_area6(q):
    xyz, tri = cube_mesh(q)
    assert tri.shape == (12 * q * q, 3)
    edges = _edges(tri)
    assert all(len(v) == 2 for v in edges.values())
    assert all(v[0] == (v[1][1], v[1][0]) for v in edges.values())
    assert xyz.shape[0] - len(edges) + tri.shape[0] == 2
    area, cr = _area(xyz, tri)
    assert abs(area.sum() - 6.0) <= 1e-12
    cen = xyz[tri].mean(axis=1) - 0.5
    assert np.all(np.einsum("ij,ij->i", cr, cen) > 0)


def test_paper_mesh_sizes():
    # PAPER Table 3 first row n = 2048 (sphere q = 16); Table 1 first row n = 2352 (cube q = 14)
    assert sphere_mesh(16)[1].shape[0] == 2048
    assert cube_mesh(14)[1].shape[0] == 2352


def test_seeded_vector_reproducible():
    x = seeded_vector(100, 1)
    assert np.array_equal(x, seeded_vector(100, 1))
    assert np.all(np.abs(x.real) <= 1) and np.all(np.abs(x.imag) <= 1)
    assert not np.array_equal(x, seeded_vector(100, 2))
