"""Invariants of the seeded synthetic meshes (inputs/meshes.py)."""
import numpy as np
import pytest

from inputs import meshes


def _check_closed(m, chi):
    t = m.tris
    e = np.sort(np.concatenate([t[:, [0, 1]], t[:, [1, 2]], t[:, [2, 0]]]), axis=1)
    _, cnt = np.unique(e, axis=0, return_counts=True)
    assert np.all(cnt == 2), "every edge shared by exactly two triangles"
    de = np.concatenate([t[:, [0, 1]], t[:, [1, 2]], t[:, [2, 0]]])
    _, dc = np.unique(de, axis=0, return_counts=True)
    assert np.all(dc == 1), "consistent winding"
    nv = len(np.unique(t))
    assert nv - cnt.size + m.n == chi
    v = m.verts
    a = np.linalg.norm(np.cross(v[t[:, 1]] - v[t[:, 0]], v[t[:, 2]] - v[t[:, 0]]), axis=1)
    assert a.min() > 0
    # outward orientation: divergence theorem volume > 0
    vol = np.einsum("ij,ij->i", v[t[:, 0]], np.cross(v[t[:, 1]], v[t[:, 2]])).sum() / 6
    assert vol > 0
    return cnt.size


def test_bar():
    m = meshes.bar()
    assert m.n == 2100
    ne = _check_closed(m, 2)
    assert ne == 3150
    assert len(m.ports[0][1]) == 50 and len(m.ports[0][2]) == 50


def test_coils():
    m = meshes.coils()
    _check_closed(m, 4)  # two spheres
    assert 120_000 < m.n < 140_000
    for _, p, q in m.ports:
        assert len(p) == 8 and len(q) == 8


def test_bga_small():
    m = meshes.bga(nb=3)
    # 9 balls (chi 2 each) + two plates of genus 9 (chi -16 each)
    _check_closed(m, 9 * 2 - 2 * 16)
    assert m.n == 9 * 1280 + 2 * (9 * (2 * 160 + 32)) + 2 * 4 * 3 * 4 * 2


def test_pop_small_and_determinism():
    m1 = meshes.pop(n_traces=40, n_vias=20, domain=2e-3)
    m2 = meshes.pop(n_traces=40, n_vias=20, domain=2e-3)
    assert np.array_equal(m1.tris, m2.tris) and np.array_equal(m1.verts, m2.verts)
    c = m1.verts[m1.tris].mean(axis=1)
    assert np.unique(np.round(c / 1e-12), axis=0).shape[0] == m1.n, "no coincident centroids"


def test_make_x():
    x = meshes.make_x(2, 1000)
    assert x.dtype == np.complex64 and x.shape == (3, 1000)
    assert np.abs(x.real).max() <= 1 and np.abs(x.imag).max() <= 1
    assert np.array_equal(x, meshes.make_x(2, 1000))
