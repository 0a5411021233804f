"""Pins of the oracle's tangent mode (caller-given `dirs` per triangle; PREDICATES §7 and §12,
`P:183` "tangent ... of the surface", `P:549` anisotropic brushed metal; DESIGN D8).

In tangent mode a triangle's contribution to voxel v is M_v = A_v d^ d^T with
d^ = dirs[t] / |dirs[t]| (the caller's direction normalised, not the face normal). The pins
below fix that against closed forms computed here in fp64 from small integer directions:

* every voxel of a triangle carries M/mass = d^ d^T of *its own* triangle's dirs row (three
  disjoint, non-axis-aligned triangles with three different, non-unit dirs: an unnormalised,
  ignored or mis-indexed `dirs` fails);
* the total mass is the triangle's area (grid units), the total M is area * d^ d^T;
* zero-norm or non-finite dirs rows are rejected;
* the same for the sampling front end (§12 `sample_triangles`).
"""
import numpy as np
import pytest

import oracle

N = 64
BBOX = np.array([0, 0, 0, 1, 1, 1], np.float32)

# non-unit integer directions with integer norms: |d| = 5, 6, 7
DIRS = np.array([[3.0, 0.0, 4.0], [2.0, 4.0, 4.0], [-2.0, 3.0, 6.0]], np.float32)


def _tris():
    """Three tilted triangles in disjoint corners of the unit box (world units)."""
    base = np.array([[0.05, 0.06, 0.07], [0.21, 0.09, 0.12], [0.08, 0.23, 0.19]], np.float64)
    offs = [np.array([0.0, 0.0, 0.0]), np.array([0.55, 0.1, 0.3]), np.array([0.2, 0.6, 0.55])]
    return np.stack([base + o for o in offs]).astype(np.float32)


def _area_grid(t):
    g = t.astype(np.float64) * N
    return 0.5 * np.linalg.norm(np.cross(g[1] - g[0], g[2] - g[0]))


def _dd(d):
    u = d.astype(np.float64) / np.linalg.norm(d.astype(np.float64))
    return np.array([u[0] * u[0], u[1] * u[1], u[2] * u[2], u[0] * u[1], u[0] * u[2], u[1] * u[2]])


def _owner(tris):
    """Voxel key -> index of the triangle whose candidate box holds it (boxes are disjoint)."""
    own = {}
    for t, tri in enumerate(tris):
        g = tri.astype(np.float64) * N
        lo = np.floor(g.min(0)).astype(int) - 1
        hi = np.floor(g.max(0)).astype(int) + 1
        for i in range(lo[0], hi[0] + 1):
            for j in range(lo[1], hi[1] + 1):
                for k in range(lo[2], hi[2] + 1):
                    key = oracle.morton(i, j, k)
                    assert key not in own
                    own[key] = t
    return own


def _check_level0(L0, tris, dirs, own):
    ok = L0["mass"] > 1e-4
    assert ok.sum() > 20
    for key, mass, m6 in zip(L0["key"][ok], L0["mass"][ok], L0["m6"][ok]):
        t = own[int(key)]
        np.testing.assert_allclose(m6 / mass, _dd(dirs[t]), rtol=2e-5, atol=2e-6)
    # per triangle: total mass = area, total M = area * d^d^T (exact integer sums of §8)
    for t, tri in enumerate(tris):
        sel = np.array([own[int(k)] == t for k in L0["key"]])
        acc = L0["acc"][sel].astype(np.float64).sum(0) / 2 ** 32
        area = _area_grid(tri)
        assert acc[0] == pytest.approx(area, rel=1e-5)
        np.testing.assert_allclose(acc[1:], area * _dd(dirs[t]), rtol=1e-4, atol=1e-5 * area)


def test_tangent_mode_exact_overlap():
    tris = _tris()
    own = _owner(tris)
    o = oracle.Oracle(N, BBOX)
    o.add_triangles(tris, DIRS)
    o.build(0)
    _check_level0(o.level(0), tris, DIRS, own)
    # the dirs are not the face normals: normal mode gives a different M on every triangle
    n = oracle.Oracle(N, BBOX)
    n.add_triangles(tris)
    n.build(0)
    assert not np.array_equal(n.level(0)["acc"][:, 1:], o.level(0)["acc"][:, 1:])


def test_tangent_mode_scale_invariant_and_per_row():
    """dirs scaled per row by positive powers of two give bit-identical accumulators
    (normalisation), and permuting triangles together with their dirs rows changes nothing."""
    tris = _tris()
    a = oracle.Oracle(N, BBOX)
    a.add_triangles(tris, DIRS)
    a.build(2)
    b = oracle.Oracle(N, BBOX)
    perm = [2, 0, 1]
    b.add_triangles(tris[perm], (DIRS * np.array([[0.25], [8.0], [2.0]], np.float32))[perm])
    b.build(2)
    for l in range(3):
        assert np.array_equal(a.level(l)["key"], b.level(l)["key"])
        assert np.array_equal(a.level(l)["acc"], b.level(l)["acc"])


@pytest.mark.parametrize("bad", [[0.0, 0.0, 0.0], [np.nan, 1.0, 0.0], [np.inf, 0.0, 1.0]])
def test_tangent_mode_rejects_bad_dirs(bad):
    tris = _tris()
    d = DIRS.copy()
    d[1] = bad
    with pytest.raises(oracle.OracleError):
        oracle.Oracle(N, BBOX).add_triangles(tris, d)
    with pytest.raises(oracle.OracleError):
        oracle.Oracle(N, BBOX).sample_triangles(tris, d, 16)


def test_tangent_mode_sampling_front_end():
    tris = _tris()
    own = _owner(tris)
    o = oracle.Oracle(N, BBOX)
    o.sample_triangles(tris, DIRS, 256)
    o.build(0)
    L0 = o.level(0)
    ok = L0["mass"] > 0
    assert ok.sum() > 10
    for key, mass, m6 in zip(L0["key"][ok], L0["mass"][ok], L0["m6"][ok]):
        np.testing.assert_allclose(m6 / mass, _dd(DIRS[own[int(key)]]), rtol=2e-5, atol=2e-6)
    # each triangle's samples carry its whole area (f = A / n_t per sample)
    for t, tri in enumerate(tris):
        sel = np.array([own[int(k)] == t for k in L0["key"]])
        assert L0["acc"][sel, 0].astype(np.float64).sum() / 2 ** 32 == pytest.approx(_area_grid(tri), rel=1e-5)
