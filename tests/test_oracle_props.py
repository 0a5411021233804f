"""Order/split invariance and moment properties of the oracle (PREDICATES §8; D19, D20)."""
import numpy as np
import pytest

import gen
import oracle


def _leaf(segs, radii, N=128, parts=1, levels=3):
    o = oracle.Oracle(N, np.array([0, 0, 0, 1, 1, 1], np.float32))
    for p in np.array_split(np.arange(len(segs)), parts):
        o.add_fibers(segs[p], radii[p])
    o.build(levels)
    return [o.level(l) for l in range(levels + 1)]


@pytest.fixture(scope="module")
def weave_small():
    s, r = gen.plain_weave(n_warp=16, n_weft=16, n_seg=32, pitch=1 / 16)
    return s, r


def test_permutation_and_split_invariance(weave_small):
    s, r = weave_small
    base = _leaf(s, r)
    perm = np.random.default_rng(0).permutation(len(s))
    for got in (_leaf(s[perm], r[perm]), _leaf(s, r, parts=5)):
        for a, b in zip(base, got):
            for k in a:
                assert np.array_equal(a[k], b[k]), k


def test_trace_psd(weave_small):
    s, r = weave_small
    L0 = _leaf(s, r, levels=0)[0]
    m6 = L0["m6"].astype(np.float64)
    tr = m6[:, :3].sum(1)
    ok = L0["mass"] > 0
    assert np.allclose(tr[ok], L0["mass"][ok], rtol=1e-6, atol=1e-30)
    for mass, v in zip(L0["mass"], m6):
        M = np.array([[v[0], v[3], v[4]], [v[3], v[1], v[5]], [v[4], v[5], v[2]]])
        assert np.linalg.eigvalsh(M)[0] >= -1e-6 * max(mass, 1e-30)


def test_empty_and_degenerate_inputs():
    o = oracle.Oracle(16, np.array([0, 0, 0, 1, 1, 1], np.float32))
    o.add_fibers(np.zeros((0, 6), np.float32), np.zeros(0, np.float32))
    o.build(4)
    for l in range(5):
        assert len(o.level(l)["key"]) == 0
    # zero-length segment = sphere: keys with zero mass (D25)
    o = oracle.Oracle(16, np.array([0, 0, 0, 16, 16, 16], np.float32))
    o.add_fibers(np.array([[8.5, 8.5, 8.5, 8.5, 8.5, 8.5]], np.float32), np.array([0.7], np.float32))
    o.build(1)
    L0 = o.level(0)
    assert len(L0["key"]) == 7 and not L0["acc"].any()        # centre + 6 face neighbours
    assert o.level(1)["ncl"].sum() == 0
    # geometry outside the grid is culled
    o = oracle.Oracle(16, np.array([0, 0, 0, 1, 1, 1], np.float32))
    o.add_fibers(np.array([[3, 3, 3, 4, 4, 4]], np.float32), np.array([0.01], np.float32))
    o.build(0)
    assert len(o.level(0)["key"]) == 0
    with pytest.raises(oracle.OracleError):
        o.add_fibers(np.array([[0.1, 0.1, 0.1, 0.2, np.nan, 0.2]], np.float32), np.array([0.01], np.float32))
    with pytest.raises(oracle.OracleError):
        o.add_fibers(np.array([[0.1, 0.1, 0.1, 0.2, 0.2, 0.2]], np.float32), np.array([-0.01], np.float32))


def test_window_matches_full_run(weave_small):
    """Windowed oracle (used for full-size parity): cell c at level L equals the full run
    restricted to that cell, at every level <= L."""
    s, r = weave_small
    N = 128
    full = oracle.Oracle(N, np.array([0, 0, 0, 1, 1, 1], np.float32))
    full.add_fibers(s, r)
    full.build(4)
    for cell in (0, 77, 300):
        w = oracle.Oracle(N, np.array([0, 0, 0, 1, 1, 1], np.float32))
        w.set_window(4, cell)
        w.add_fibers(s, r)
        w.build(4)
        for l in range(5):
            F, Wl = full.level(l), w.level(l)
            sel = (F["key"] >> np.uint64(3 * (4 - l))) == cell
            for k in F:
                assert np.array_equal(F[k][sel], Wl[k]), (cell, l, k)
