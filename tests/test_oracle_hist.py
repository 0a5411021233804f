"""Pins of the oracle's histogram distance (docs/PREDICATES.md §10):
the paper's own SGGX similarity -- N whole-sphere samples per SGGX, a
5x5x5 histogram, a Wasserstein distance between histograms (sliced
over 32 directions). Each test pins the oracle to something other than
itself: closed forms (Archimedes' hat-box theorem, rank-1 SGGX, one-bin shifts), an
independent sampler (eigen square root + Gaussian directions, numpy), an independent 1-D
optimal-transport routine (scipy.stats.wasserstein_distance), and the SPEC examples."""
import numpy as np
import pytest
from scipy.spatial.transform import Rotation
from scipy.stats import wasserstein_distance

import oracle

N = oracle.HIST_N_DEFAULT
SCALE = 32 * 5 * 65536          # d_hist = SCALE * N * (mean sliced W1), up to fixed-point rounding


def _acc(S):
    S = np.asarray(S, np.float64)
    return oracle.acc_from_float(1.0, [S[0, 0], S[1, 1], S[2, 2], S[0, 1], S[0, 2], S[1, 2]])


def _bins(d):
    b = np.clip(np.floor((d + 1.0) * 2.5).astype(int), 0, 4)
    return b[:, 0] + 5 * b[:, 1] + 25 * b[:, 2]


def _centres():
    b = np.arange(125)
    return np.stack([(2 * (b % 5) - 4) / 5, (2 * ((b // 5) % 5) - 4) / 5, (2 * (b // 25) - 4) / 5], 1)


def test_sample_table_uniform_on_sphere():
    u = oracle.sample_table(N).astype(np.float64)
    assert u.shape == (N, 3)
    assert np.abs(np.linalg.norm(u, axis=1) - 1).max() < 1e-6
    # Archimedes: the area fraction of the cap z > t is (1 - t) / 2
    for t in (-0.8, -0.3, 0.0, 0.45, 0.9):
        assert abs((u[:, 2] > t).mean() - (1 - t) / 2) < 2.0 / N
    # z levels symmetric, azimuths balanced
    assert np.abs(u[:, 2] + u[::-1, 2]).max() < 1e-7
    assert np.abs(u.mean(0)).max() < 1e-3


@pytest.mark.parametrize("axis", [0, 1, 2])
def test_hist_rank1_sggx_is_two_antipodal_cells(axis):
    # S = e e^T: every sample normalize(L u) is +-e (SPEC antipodal example, cells (2,2,4), (2,2,0) for z)
    S = np.zeros((3, 3))
    S[axis, axis] = 1.0
    h = oracle.hist(_acc(S), N)
    u = oracle.sample_table(N)
    hi = [2, 2, 2]
    hi[axis] = 4
    lo = [2, 2, 2]
    lo[axis] = 0
    cell = lambda c: c[0] + 5 * c[1] + 25 * c[2]
    assert int(h.sum()) == N
    assert h[cell(hi)] == int((u[:, axis] > 0).sum())
    assert h[cell(lo)] == int((u[:, axis] < 0).sum())
    # u_axis == 0 exactly (s = 0 has phi = 0, so u_y = 0) gives v = 0: the centre cell by definition
    assert h[62] == int((u[:, axis] == 0).sum())
    assert h[cell(hi)] + h[cell(lo)] + h[62] == N


def test_hist_isotropic_is_binned_sample_table():
    # S = I/3: L = I/sqrt(3), samples are the table points themselves
    h = oracle.hist(_acc(np.eye(3) / 3), N).astype(np.int64)
    u = oracle.sample_table(N).astype(np.float64)
    ref = np.bincount(_bins(u / np.linalg.norm(u, axis=1, keepdims=True)), minlength=125)
    assert int(h.sum()) == N
    assert np.abs(h - ref).sum() <= 6          # a few points may sit on a bin face (fp32 vs fp64)
    assert h.max() <= 0.10 * N                  # SPEC: no single cell holds > 10% for S = identity
    # cells that do not meet the unit sphere stay empty (98 cells do)
    assert int((h > 0).sum()) <= 98 and h[62] == 0


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_hist_matches_independent_sggx_sampler(seed):
    # generic anisotropic S; the reference distribution of normalize(S^1/2 g), g Gaussian, uses the
    # eigen square root (not Cholesky) -- same law, independent construction
    rng = np.random.default_rng(seed)
    Q = Rotation.from_euler("xyz", rng.uniform(-np.pi, np.pi, 3)).as_matrix()
    S = Q @ np.diag([1.0, 10 ** rng.uniform(-2, -0.5), 10 ** rng.uniform(-3.5, -2)]) @ Q.T
    S /= np.trace(S)
    h = oracle.hist(_acc(S), N).astype(np.float64) / N
    w, V = np.linalg.eigh(S)
    Sh = V @ np.diag(np.sqrt(np.maximum(w, 0))) @ V.T
    g = rng.standard_normal((1_000_000, 3))

    def law(M):
        v = g @ M.T
        return np.bincount(_bins(v / np.linalg.norm(v, axis=1, keepdims=True)), minlength=125) / len(v)

    p = law(Sh)
    assert 0.5 * np.abs(h - p).sum() < 0.03
    # the test is sensitive to a transposed factor (a plausible mistake): L^T u has another law
    L = np.linalg.cholesky(S + 1e-12 * np.eye(3))
    assert 0.5 * np.abs(law(L.T) - p).sum() > 0.1


def test_sw_tables_are_sorted_projections():
    perm, gap = oracle.sw_tables()
    theta, _ = oracle.theta()
    c = _centres() * 5
    for k in range(32):
        assert sorted(perm[k].tolist()) == list(range(125))
        proj = c @ theta[k].astype(np.float64) * 65536
        sp = proj[perm[k]]
        assert np.all(np.diff(sp) >= -1.0)                     # ascending up to the rounding to integers
        assert np.all(gap[k] >= 0)
        assert abs(gap[k].sum() - (proj.max() - proj.min())) <= 1.0


def _scipy_sw(h1, h2):
    theta, _ = oracle.theta()
    c = _centres()
    return np.mean([wasserstein_distance(c @ theta[k].astype(np.float64), c @ theta[k].astype(np.float64),
                                         h1.astype(np.float64), h2.astype(np.float64)) for k in range(32)])


@pytest.mark.parametrize("seed", range(4))
def test_hist_distance_is_sliced_w1(seed):
    rng = np.random.default_rng(seed)
    h1 = rng.multinomial(N, rng.dirichlet(np.ones(125) * 0.3)).astype(np.uint16)
    h2 = rng.multinomial(N, rng.dirichlet(np.ones(125) * 0.3)).astype(np.uint16)
    d = oracle.hist_distance(h1, h2)
    assert d == oracle.hist_distance(h2, h1)
    assert oracle.hist_distance(h1, h1) == 0
    sw = _scipy_sw(h1, h2)              # on the normalized histograms (weights are normalized by scipy)
    assert abs(d / (SCALE * N) - sw) < 2e-6


def test_hist_distance_one_bin_shift():
    # SPEC: two delta histograms one bin apart along x -> one bin width (2/5) x mean |theta_x|
    theta, _ = oracle.theta()
    for a, b in (((3, 2, 4), (4, 2, 4)), ((0, 1, 1), (1, 1, 1))):
        h1 = np.zeros(125, np.uint16)
        h2 = np.zeros(125, np.uint16)
        h1[a[0] + 5 * a[1] + 25 * a[2]] = N
        h2[b[0] + 5 * b[1] + 25 * b[2]] = N
        want = 0.4 * np.abs(theta[:, 0].astype(np.float64)).mean()
        assert abs(oracle.hist_distance(h1, h2) / (SCALE * N) - want) < 2e-6


def test_sggxh_hist_merges_identical_pair_first():
    x = np.diag([1.0, 0, 0]); y = np.diag([0, 1.0, 0]); z = np.diag([0, 0, 1.0])
    # S1 = S2 != S3 -> (1, 2) merged (SPEC merge_closest example)
    out = oracle.sggxh_hist(np.stack([_acc(x), _acc(x), _acc(z)]), k=2)
    assert np.array_equal(out, np.stack([_acc(x) * 2, _acc(z)]))
    # two identical pairs, k = 2: (0,2) then (1,2) of the shifted list
    out = oracle.sggxh_hist(np.stack([_acc(x), _acc(y), _acc(x), _acc(y)]), k=2)
    assert np.array_equal(out, np.stack([_acc(x) * 2, _acc(y) * 2]))
    # three perpendicular deltas, k = 3: nothing merged
    out = oracle.sggxh_hist(np.stack([_acc(x), _acc(y), _acc(z)]), k=3)
    assert np.array_equal(out, np.stack([_acc(x), _acc(y), _acc(z)]))


def test_sggxh_hist_first_merge_is_brute_force_argmin():
    rng = np.random.default_rng(5)
    accs = []
    for _ in range(6):
        d = rng.standard_normal((4, 3))
        d /= np.linalg.norm(d, axis=1, keepdims=True)
        accs.append(_acc(d.T @ d / 4))
    accs = np.stack(accs)
    hs = [oracle.hist(a) for a in accs]
    D = {(i, j): oracle.hist_distance(hs[i], hs[j]) for i in range(6) for j in range(i + 1, 6)}
    i, j = min(D, key=lambda ij: (D[ij], ij))
    out = oracle.sggxh_hist(accs, k=5)
    want = [accs[c] for c in range(6) if c != j]
    want[i] = accs[i] + accs[j]
    assert np.array_equal(out, np.stack(want))


def test_hist_mode_level_build_invariants():
    import gen
    c = gen.config(1)
    res = {}
    for mode in ("sigma", "hist"):
        o = oracle.Oracle(c["grid_res"], c["bbox"], k=3, distance=mode)
        o.add_triangles(c["tris"], c["dirs"])
        o.build(3)
        res[mode] = [o.level(l) for l in range(4)]
        o.close()
    for l in range(1, 4):
        a, b = res["sigma"][l], res["hist"][l]
        assert np.array_equal(a["key"], b["key"]) and np.array_equal(a["acc"], b["acc"])
        # lobes conserve the voxel's moments exactly in both modes
        assert np.array_equal(b["cl_acc"].sum(1), b["acc"])
        # parents with n <= K are untouched by the distance: identical lobes in both modes
        assert np.all(b["ncl"] <= 3)
    # some parents differ between the two distances (they are different measures)
    assert any(not np.array_equal(res["sigma"][l]["cl_acc"], res["hist"][l]["cl_acc"]) for l in range(1, 4))
