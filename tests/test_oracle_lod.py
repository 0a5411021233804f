"""Pins of the oracle's LoD pyramid and SGGX-H (docs/PREDICATES.md §8-§9; P:364,
P:371-389) against the mathematics of SGGX and the SPEC's worked examples."""
import json
import math
import os

import numpy as np
import pytest

import gen
import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
Q = 2.0 ** 32


def acc(w, S6):
    """(w, M = w S) as int64 accumulators (§8 quantisation of fp32 values)."""
    m = np.float32(w) * np.asarray(S6, np.float32)
    return oracle.acc_from_float(np.float32(w), m)


DIR = {"x": [1, 0, 0, 0, 0, 0], "y": [0, 1, 0, 0, 0, 0], "z": [0, 0, 1, 0, 0, 0]}


def fib_theta64():
    """Independent fp64 spherical-Fibonacci slice table (PREDICATES §9 definition)."""
    k = np.arange(32)
    z = 1 - (k + 0.5) / 32
    phi = k * math.pi * (3 - math.sqrt(5))
    rho = np.sqrt(1 - z * z)
    return np.stack([rho * np.cos(phi), rho * np.sin(phi), z], 1)


def test_theta_table_is_unit_hemisphere():
    th, coef = oracle.theta()
    th64 = fib_theta64()
    assert np.allclose(th, th64, atol=1e-7)
    assert np.all(th[:, 2] > 0) and np.allclose(np.linalg.norm(th.astype(np.float64), axis=1), 1, atol=1e-6)
    # coefficients are the quadratic form of theta: q_k(S) = theta^T S theta
    S = np.array([[0.3, 0.1, -0.2], [0.1, 0.5, 0.05], [-0.2, 0.05, 0.2]])
    s6 = np.array([S[0, 0], S[1, 1], S[2, 2], S[0, 1], S[0, 2], S[1, 2]])
    assert np.allclose(coef.astype(np.float64) @ s6, np.einsum("ki,ij,kj->k", th64, S, th64), atol=1e-6)


@pytest.mark.parametrize("case", GOLD["projected_area"]["cases"])
def test_sigma_is_projected_area(case):
    """sigma(w) = sqrt(w^T S w); checked on the slice directions."""
    S6 = np.asarray(case["S"], np.float64)
    S = np.array([[S6[0], S6[3], S6[4]], [S6[3], S6[1], S6[5]], [S6[4], S6[5], S6[2]]])
    w = np.asarray(case["w"], np.float64)
    assert math.sqrt(w @ S @ w) == pytest.approx(case["sigma"])   # the SPEC's value
    sig = oracle.sigma(acc(1.0, S6))
    th = fib_theta64()
    assert np.allclose(sig, np.sqrt(np.maximum(np.einsum("ki,ij,kj->k", th, S, th), 0)), atol=2e-6)


def test_sigma_random_psd_fp64_shadow():
    rng = np.random.default_rng(2)
    th = fib_theta64()
    for _ in range(200):
        A = rng.normal(size=(3, 3)); S = A @ A.T; S /= np.trace(S)
        w = rng.uniform(0.1, 10)
        a = acc(w, [S[0, 0], S[1, 1], S[2, 2], S[0, 1], S[0, 2], S[1, 2]])
        sig = oracle.sigma(a)
        want = np.sqrt(np.maximum(np.einsum("ki,ij,kj->k", th, S, th), 0))
        assert np.allclose(sig, want, atol=1e-5)


def test_distance_worked_value_and_metric():
    g = GOLD["sigma_distance_dx_dy"]
    th = fib_theta64()
    closed = float(np.abs(np.abs(th[:, 0]) - np.abs(th[:, 1])).sum())   # sigma(delta_x) = |theta_x|
    assert closed == pytest.approx(g["value"], abs=g["tol"])
    assert oracle.distance(acc(1, DIR["x"]), acc(1, DIR["y"])) == pytest.approx(closed, abs=1e-5)
    rng = np.random.default_rng(4)
    def rnd():
        A = rng.normal(size=(3, 3)); S = A @ A.T; S /= np.trace(S)
        return acc(rng.uniform(0.5, 3), [S[0, 0], S[1, 1], S[2, 2], S[0, 1], S[0, 2], S[1, 2]])
    for _ in range(300):
        a, b, c = rnd(), rnd(), rnd()
        dab, dba = oracle.distance(a, b), oracle.distance(b, a)
        assert dab == dba and oracle.distance(a, a) == 0.0
        assert oracle.distance(a, c) <= dab + oracle.distance(b, c) + 1e-5


def _dir_of(cl):
    S = cl[1:4] / cl[0]
    return "xyz"[int(np.argmax(S))]


@pytest.mark.parametrize("name", ["two_x_y_z_k3", "perpendicular_k3", "checkerboard_k3"])
def test_spec_merge_examples(name):
    ex = GOLD["merge_examples"][name]
    cl = np.stack([acc(w, DIR[d]) for d, w in zip(ex["inputs"], ex["weights"])])
    out = oracle.sggxh(cl, 3)
    got = [[_dir_of(c), round(c[0] / Q)] for c in out]
    assert got == ex["expected"]


def test_identical_pair_merges_first_and_refit_is_exact():
    """S1 = S2 != S3 -> merges (1,2); the merged S equals S1."""
    S1 = [0.2, 0.3, 0.5, 0.1, 0.0, -0.05]
    S3 = [0.9, 0.05, 0.05, 0.0, 0.0, 0.0]
    cl = np.stack([acc(1.0, S1), acc(1.0, S1), acc(1.0, S3)])
    out = oracle.sggxh(cl, 2)
    assert len(out) == 2
    assert np.array_equal(out[0], cl[0] + cl[1]) and np.array_equal(out[1], cl[2])
    assert np.allclose(out[0][1:] / out[0][0], cl[0][1:] / cl[0][0], rtol=1e-6)


def test_k1_is_naive_root_and_weights_conserved():
    rng = np.random.default_rng(8)
    for n in range(2, 25):
        cl = np.stack([acc(rng.uniform(0.1, 2), np.r_[rng.dirichlet([1, 1, 1]), 0, 0, 0]) for _ in range(n)])
        root = oracle.sggxh(cl, 1)
        assert len(root) == 1 and np.array_equal(root[0], cl.sum(0))
        for K in (2, 3, 5):
            out = oracle.sggxh(cl, K)
            assert len(out) == min(n, K)                                   # merge count = n - K
            assert np.array_equal(out.sum(0), cl.sum(0))                   # exact conservation


def test_dominance_multimodal():
    """SPEC dominance restated with the sigma distance: on multi-modal voxels the
    K=3 SGGX-H lobes, each summarising only its members, stay closer to every leaf lobe than the
    single naive SGGX does."""
    rng = np.random.default_rng(12)
    th = fib_theta64()
    def sig6(S6):
        M = np.array([[S6[0], S6[3], S6[4]], [S6[3], S6[1], S6[5]], [S6[4], S6[5], S6[2]]])
        return np.sqrt(np.maximum(np.einsum("ki,ij,kj->k", th, M, th), 0))
    wins = 0
    for trial in range(25):
        modes = rng.normal(size=(rng.integers(2, 4), 3))
        leaves = []
        for _ in range(8):
            t = modes[rng.integers(len(modes))] + 0.05 * rng.normal(size=3)
            t /= np.linalg.norm(t)
            T = np.outer(t, t)
            leaves.append(acc(rng.uniform(0.5, 1.5), [T[0, 0], T[1, 1], T[2, 2], T[0, 1], T[0, 2], T[1, 2]]))
        leaves = np.stack(leaves)
        out = oracle.sggxh(leaves, 3)
        naive = leaves.sum(0)
        # assign each leaf to its nearest output lobe; error = weighted sigma distance to it
        def err(lobes):
            tot = 0.0
            for c in leaves:
                s = sig6(c[1:] / c[0])
                tot += c[0] / Q * min(np.abs(s - sig6(l[1:] / l[0])).sum() for l in lobes)
            return tot
        e3, e1 = err(out), err([naive])
        assert e3 <= e1 + 1e-6
        wins += e3 < e1 - 1e-6
    assert wins >= 0.9 * 25


def _build(segs=None, radii=None, tris=None, N=32, levels=5, k=3):
    o = oracle.Oracle(N, np.array([0, 0, 0, 1, 1, 1], np.float32), k)
    if segs is not None:
        o.add_fibers(segs, radii)
    if tris is not None:
        o.add_triangles(tris)
    o.build(levels)
    return o


def test_pyramid_conservation_and_parents():
    import gen
    o = _build(tris=gen.icosphere(1), N=64, levels=6)
    total = None
    prev = None
    for l in range(7):
        L = o.level(l)
        s = L["acc"].sum(0)
        if total is None:
            total = s
        assert np.array_equal(s, total)                          # exact mass/M conservation
        if prev is not None:
            assert np.array_equal(L["key"], np.unique(prev["key"] >> np.uint64(3)))
            assert len(L["key"]) <= len(prev["key"])
        # clusters sum to the naive aggregate exactly
        assert np.array_equal(L["cl_acc"].sum(1), L["acc"])
        assert np.all(L["ncl"] <= 3)
        prev = L
    assert len(o.level(6)["key"]) == 1


def test_naive_aggregate_delta_x_delta_y():
    """a delta-x child and a delta-y child with equal weights -> naive S = diag(1/2,1/2,0)."""
    N = 64
    s = np.array([[[10.2, 20.5, 20.5], [10.8, 20.5, 20.5]],          # along x in voxel (10,20,20)
                  [[11.5, 20.2, 20.5], [11.5, 20.8, 20.5]]], np.float32) / N   # along y in (11,20,20)
    o = _build(s, np.full(2, 0.01 / N, np.float32), N=N, levels=1)
    L1 = o.level(1)
    a = L1["acc"][L1["key"] == (oracle.morton(10, 20, 20) >> 3)][0]
    # both fibers have equal length and radius -> equal mass (S_p normalisation, §5)
    S = a[1:] / a[0]
    assert np.allclose(S, GOLD["interpolate_delta_xy"]["S_expected"], atol=1e-6)
    # SGGX-H with K=3 keeps both lobes (n = 2 <= K), strictly less isotropic than the naive S
    assert L1["ncl"][L1["key"] == (oracle.morton(10, 20, 20) >> 3)][0] == 2


def test_build_from_equals_build():
    """orc_build_from (chained parity at full size) starts from given level records and must
    reproduce build() exactly: config 1 and a small weave, from every start level, both
    distance modes."""
    c = gen.config(1)
    for distance in ("sigma", "hist"):
        o = oracle.Oracle(c["grid_res"], c["bbox"], distance=distance, hist_samples=200)
        o.add_triangles(c["tris"])
        o.build(6)
        for l0 in range(0, 6):
            L = o.level(l0)
            o2 = oracle.Oracle(c["grid_res"], c["bbox"], distance=distance, hist_samples=200)
            o2.build_from(l0, L["key"], L["acc"], L["ncl"], L["cl_acc"], 6)
            for l in range(l0, 7):
                a, b = o.level(l), o2.level(l)
                for f in ("key", "acc", "ncl", "cl_acc", "cl"):
                    assert np.array_equal(a[f], b[f]), (distance, l0, l, f)
    s, r = gen.plain_weave(n_warp=8, n_weft=8, n_seg=16, pitch=1 / 8)
    o = oracle.Oracle(64, np.array([0, 0, 0, 1, 1, 1], np.float32))
    o.add_fibers(s, r)
    o.build(6)
    L = o.level(2)
    o2 = oracle.Oracle(64, np.array([0, 0, 0, 1, 1, 1], np.float32))
    o2.build_from(2, L["key"], L["acc"], L["ncl"], L["cl_acc"], 6)
    for l in range(2, 7):
        assert np.array_equal(o.level(l)["cl_acc"], o2.level(l)["cl_acc"]), l
    # unsorted keys are rejected
    with pytest.raises(oracle.OracleError):
        o2.build_from(2, L["key"][::-1].copy(), L["acc"][::-1].copy(), L["ncl"], L["cl_acc"], 6)
