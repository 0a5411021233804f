"""Pins of the oracle's sampling front end (docs/PREDICATES.md §12; the
paper's own voxelization): Catmull-Rom end-point and midpoint properties (SPEC
subdivide_spline examples), the SPEC sample-count examples, Heitz's map keeping samples
inside the triangle and spreading them uniformly (area fractions), closed-form per-voxel
masses of a straight piece, exact mass totals, and convergence of the sampled voxel masses
to the exact-overlap path of §4-§7 as the sample count grows."""
import numpy as np
import pytest

import gen
import oracle


def test_spline_endpoints_and_midpoint():
    rng = np.random.default_rng(0)
    for _ in range(20):
        G = rng.uniform(0, 8, (4, 3)).astype(np.float32)
        p0, _ = oracle.spline_eval(G, 0.0)
        p1, _ = oracle.spline_eval(G, 1.0)
        assert np.array_equal(p0, G[1])                           # t = 0 -> P1 (exactly)
        assert np.abs(p1 - G[2]).max() <= 1e-5 * (1 + np.abs(G).max())   # t = 1 -> P2
        # tangent at t = 0 is parallel to (P2 - P0) (Catmull-Rom derivative 0.5 (P2 - P0))
        _, t0 = oracle.spline_eval(G, 0.0)
        d = (G[2] - G[0]).astype(np.float64)
        assert np.abs(t0 - d / np.linalg.norm(d)).max() < 1e-6
    # collinear, equally spaced controls: t = 0.5 is the midpoint, the tangent the direction
    a, b = np.array([1.0, 2.0, 3.0]), np.array([0.5, -0.25, 1.0])
    G = np.stack([a + b * k for k in range(4)]).astype(np.float32)
    p, t = oracle.spline_eval(G, 0.5)
    assert np.abs(p - (a + 1.5 * b)).max() < 1e-6
    assert np.abs(t - b / np.linalg.norm(b)).max() < 1e-6


def test_triangle_sample_counts_spec():
    assert oracle.tri_samples(2.0, 2.0, 64) == 64          # area = max -> the whole budget
    assert oracle.tri_samples(1.0, 2.0, 100) == 50         # half the area -> half the samples
    assert oracle.tri_samples(1e-6, 2.0, 100) == 1         # at least one for a positive area
    assert oracle.tri_samples(0.0, 2.0, 100) == 0          # zero-area triangles emit nothing


def test_heitz_map_inside_and_uniform():
    rng = np.random.default_rng(1)
    g = rng.uniform(0, 10, 9).astype(np.float32)
    n = 20000
    P = oracle.tri_sample_points(g, n).astype(np.float64)
    V = g.reshape(3, 3).astype(np.float64)
    # barycentric coordinates by an independent solve
    Mt = np.stack([V[0] - V[2], V[1] - V[2]], 1)
    lam, *_ = np.linalg.lstsq(Mt, (P - V[2]).T, rcond=None)
    b = np.vstack([lam, 1 - lam.sum(0)])
    assert b.min() >= -1e-5 and np.abs(b.sum(0) - 1).max() < 1e-6
    assert np.abs(Mt @ lam + V[2][:, None] - P.T).max() < 1e-4   # points lie in the plane
    # uniform in area: the corner sub-triangle {b_m > 1/2} holds a quarter of the area
    for m in range(3):
        assert abs((b[m] > 0.5).mean() - 0.25) < 0.01


def test_straight_piece_masses_closed_form():
    # a straight, evenly parameterised piece along x from 0.25 to 3.75 (grid units) in a
    # 8^3 grid: the voxel x = i receives the samples with x_s in [i, i+1)
    N = 8
    bbox = np.array([0, 0, 0, N, N, N], np.float32)      # world = grid units
    a, b = np.array([0.25, 4.5, 4.5]), np.array([3.75, 4.5, 4.5])
    d = (b - a) / 1.0
    ctrl = np.stack([a - d, a, b, b + d])[None].astype(np.float32)
    r = np.array([0.5], np.float32)
    n = 1000
    o = oracle.Oracle(N, bbox)
    o.sample_splines(ctrl, r, n)
    o.build(0)
    L = o.level(0)
    x = a[0] + (b[0] - a[0]) * (np.arange(n) + 0.5) / n
    cnt = np.bincount(np.floor(x).astype(int), minlength=N)
    mp = np.float32(np.float32(np.float32(np.pi) * r[0]) * r[0]) * np.float32(3.5)
    f = np.float32(mp / np.float32(n))
    keys = [oracle.morton(i, 4, 4) for i in range(4)]
    assert L["key"].tolist() == keys
    for i in range(4):
        assert L["acc"][i, 0] == cnt[i] * int(np.rint(np.float64(f) * 2 ** 32))
        # M_xx = mass (tangent = x), other moments 0
        assert L["acc"][i, 1] == L["acc"][i, 0] and np.all(L["acc"][i, 2:] == 0)
    # voxel masses are length fractions of pi r^2 |d| within one sample
    assert np.abs(L["mass"] - mp * np.array([0.75, 1.0, 1.0, 0.75]) / 3.5).max() <= f * 1.01


def test_triangle_sampled_mass_total_and_convergence():
    c = gen.config(1)
    res = {}
    exact = oracle.Oracle(c["grid_res"], c["bbox"])
    exact.add_triangles(c["tris"])
    exact.build(0)
    E = exact.level(0)
    for budget in (16, 256, 4096):
        o = oracle.Oracle(c["grid_res"], c["bbox"])
        o.sample_triangles(c["tris"], None, budget)
        o.build(0)
        res[budget] = o.level(0)
    # total mass = total area (sum of n_t * fl(A/n_t) per triangle, so equal up to rounding)
    tot_exact = E["acc"][:, 0].sum() / 2 ** 32
    for budget, L in res.items():
        assert abs(L["acc"][:, 0].sum() / 2 ** 32 - tot_exact) < 1e-4 * tot_exact
    # per-voxel masses converge to the exact clipped areas (L1 error shrinks with the budget)
    def l1(L):
        m = dict(zip(E["key"].tolist(), E["mass"].astype(np.float64)))
        s = dict(zip(L["key"].tolist(), L["mass"].astype(np.float64)))
        ks = set(m) | set(s)
        return sum(abs(m.get(k, 0.0) - s.get(k, 0.0)) for k in ks) / tot_exact
    errs = [l1(res[b]) for b in (16, 256, 4096)]
    assert errs[0] > errs[1] > errs[2] and errs[2] < 0.1
    # every sampled voxel is also an exact-overlap key (samples lie on the triangles)
    assert set(res[4096]["key"].tolist()) <= set(E["key"].tolist())


def test_spline_sampled_masses_converge_to_exact_centerline():
    # thin straight fibers (r = 0.001 voxel) cut into equal collinear pieces, where the
    # Catmull-Rom curve is the polyline itself: the exact capsule path's ball-touch lengths
    # approach the centerline length per voxel, the quantity the samples estimate
    N = 64
    rng = np.random.default_rng(3)
    segs = []
    for _ in range(24):
        a = rng.uniform(0.1, 0.9, 3)
        b = np.clip(a + rng.normal(0, 0.25, 3), 0.05, 0.95)
        nodes = a + (b - a) * np.linspace(0, 1, 11)[:, None]
        segs.append(np.stack([nodes[:-1], nodes[1:]], 1))
    s = np.concatenate(segs).astype(np.float32)
    r = np.full(len(s), 0.001 / N, np.float32)
    bbox = np.array([0, 0, 0, 1, 1, 1], np.float32)
    ctrl = gen.splines_from_segments(s)
    ex = oracle.Oracle(N, bbox)
    ex.add_fibers(s, r)
    ex.build(0)
    E = ex.level(0)
    tot = E["mass"].astype(np.float64).sum()

    def l1(n):
        o = oracle.Oracle(N, bbox)
        o.sample_splines(ctrl, r, n)
        o.build(0)
        L = o.level(0)
        m = dict(zip(E["key"].tolist(), E["mass"].astype(np.float64)))
        q = dict(zip(L["key"].tolist(), L["mass"].astype(np.float64)))
        return sum(abs(m.get(k, 0.0) - q.get(k, 0.0)) for k in set(m) | set(q)) / tot
    e = [l1(n) for n in (2, 16, 256)]
    assert e[0] > e[1] > e[2] and e[2] < 0.02, e
