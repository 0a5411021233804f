"""GPU parity of SGGX-H with the paper's histogram distance (distance_mode = hist,
docs/PREDICATES.md §10): the CUDA path through the C ABI against the
oracle, every level bit-exact (keys, accumulators, lobe counts, lobes). The histograms and
distances are integers, so agreement is exact by construction once the pinned fp32 sampling
agrees; these tests check that it does, over leaf and non-leaf levels, K = 1..8, N = 32..8160."""
import numpy as np
import pytest
import torch

import gen
import oracle
from windowing import chain_levels

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    from paper_2604_13191_b200 import build
    build.build()
    import paper_2604_13191_b200 as P
    return P


def _cmp(v, o, levels, tag):
    for l in range(levels + 1):
        g, r = v.level(l), o.level(l)
        assert np.array_equal(g["key"].cpu().numpy().astype(np.uint64), r["key"]), (tag, l, "keys")
        assert np.array_equal(g["acc"].cpu().numpy(), r["acc"]), (tag, l, "acc")
        if l > 0:
            assert np.array_equal(g["ncl"].cpu().numpy(), r["ncl"]), (tag, l, "ncl")
            assert np.array_equal(g["cl"].cpu().numpy(), r["cl"]), (tag, l, "lobes")


def _run(P, N, bbox, levels, segs=None, radii=None, tris=None, dirs=None, k=3, n=5000):
    v = P.Vox(N, bbox, k=k, distance="hist", hist_samples=n)
    o = oracle.Oracle(N, np.asarray(bbox, np.float32), k, distance="hist", hist_samples=n)
    if segs is not None:
        v.voxelize_fibers(torch.from_numpy(segs).cuda(), torch.from_numpy(radii).cuda())
        o.add_fibers(segs, radii)
    if tris is not None:
        v.voxelize_triangles(torch.from_numpy(tris).cuda(), None if dirs is None else torch.from_numpy(dirs).cuda())
        o.add_triangles(tris, dirs)
    v.build_lod(levels)
    o.build(levels)
    return v, o


def test_hist_config1_all_levels(P):
    c = gen.config(1)
    v, o = _run(P, c["grid_res"], c["bbox"], c["levels"], tris=c["tris"])
    _cmp(v, o, c["levels"], "icosphere")
    # the two distances do differ somewhere (the mode is really switched)
    s = P.Vox(c["grid_res"], c["bbox"])
    s.voxelize_triangles(torch.from_numpy(c["tris"]).cuda())
    s.build_lod(c["levels"])
    assert any(not torch.equal(s.level(l)["cl"], v.level(l)["cl"]) for l in range(1, c["levels"] + 1))


@pytest.mark.parametrize("k,n", [(1, 5000), (2, 32), (3, 8160), (5, 1000), (8, 5000)])
def test_hist_weave_k_and_n(P, k, n):
    s, r = gen.plain_weave(n_warp=8, n_weft=8, n_seg=16, pitch=1 / 8)
    v, o = _run(P, 64, np.array([0, 0, -0.1, 1, 1, 0.1], np.float32), 5, segs=s, radii=r, k=k, n=n)
    _cmp(v, o, 5, f"weave k={k} n={n}")


def test_hist_triangles_tangent_dirs(P):
    t, d = gen.ridge_mesh(24, 24, seed=3)
    bbox = np.concatenate([t.reshape(-1, 3).min(0), t.reshape(-1, 3).max(0)]).astype(np.float32)
    v, o = _run(P, 64, bbox, 6, tris=t, dirs=d)
    _cmp(v, o, 6, "ridge")


def test_hist_config4_windowed(P):
    # bench workload, full size; oracle recomputes one level-4 Morton cell (16^3 leaves)
    c = gen.config(4)
    v = P.Vox(c["grid_res"], c["bbox"], distance="hist")
    v.voxelize_fibers(torch.from_numpy(c["segments"]).cuda(), torch.from_numpy(c["radii"]).cuda())
    v.build_lod(c["levels"])
    k0 = v.level(0)["key"].cpu().numpy().astype(np.uint64)
    cells, cnt = np.unique(k0 >> np.uint64(12), return_counts=True)
    cell = int(cells[np.argsort(-cnt)[len(cnt) // 3]])
    N, bbox = c["grid_res"], c["bbox"]
    E = float(np.max(bbox[3:] - bbox[:3]))
    i, j, kk = oracle.unmorton(cell)
    lo_box = np.array([i, j, kk], np.float64) * 16 * E / N + bbox[:3] - 2 * E / N
    hi_box = lo_box + 20 * E / N
    s, r = c["segments"], c["radii"]
    sel = np.all((np.maximum(s[:, 0], s[:, 1]) + r[:, None] >= lo_box) &
                 (np.minimum(s[:, 0], s[:, 1]) - r[:, None] <= hi_box), axis=1)
    o = oracle.Oracle(N, bbox, 3, distance="hist")
    o.set_window(4, cell)
    o.add_fibers(np.ascontiguousarray(s[sel]), np.ascontiguousarray(r[sel]))
    o.build(4)
    for l in range(5):
        g, rr = v.level(l), o.level(l)
        m = (g["key"] >> (3 * (4 - l))) == cell
        assert np.array_equal(g["key"][m].cpu().numpy().astype(np.uint64), rr["key"]), l
        assert np.array_equal(g["acc"][m].cpu().numpy(), rr["acc"]), l
        if l > 0:
            assert np.array_equal(g["ncl"][m].cpu().numpy(), rr["ncl"]), l
            assert np.array_equal(g["cl"][m].cpu().numpy(), rr["cl"]), l
    assert int((o.level(1)["ncl"] == 3).sum()) > 50      # the window holds real SGGX-H work
    chain_levels(v, c, 5)   # levels 6..12 over the whole grid, the oracle from the GPU's level 5
