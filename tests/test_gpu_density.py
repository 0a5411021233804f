"""GPU parity of the sub-voxel occupancy and axis-projected densities (vox_density_*,
docs/PREDICATES.md §13) against the oracle: the 512-bit masks,
occupancy and axis densities bit-exact at every level, for fibers, triangles (normal and
tangent mode), and at config 4's full size inside oracle windows."""
import numpy as np
import pytest
import torch

import gen
import oracle
from windowing import window_oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    from paper_2604_13191_b200 import build
    build.build()
    import paper_2604_13191_b200 as P
    return P


def _cmp(v, o, l, sel=None, tag=""):
    g = v.density_level(l, masks=True)
    r = o.density_level(l)
    s = (lambda t: t) if sel is None else (lambda t: t[sel])
    assert np.array_equal(s(g["mask"]).cpu().numpy().view(np.uint64), r["mask"]), (tag, l, "masks")
    assert np.array_equal(s(g["occ"]).cpu().numpy(), r["occ"]), (tag, l, "occupancy")
    assert np.array_equal(s(g["axis"]).cpu().numpy(), r["axis"]), (tag, l, "axis densities")


def test_density_fibers_all_levels(P):
    s, r = gen.plain_weave(n_warp=8, n_weft=8, n_seg=32, pitch=1 / 8)
    s = (s + np.float32(0.0071)).astype(np.float32)
    bbox = np.array([0, 0, 0, 1, 1, 1], np.float32)
    v = P.Vox(32, bbox)
    S, R = torch.from_numpy(s).cuda(), torch.from_numpy(r).cuda()
    v.voxelize_fibers(S, R)
    v.build_lod(5)
    v.density_fibers(S, R)
    o = oracle.Oracle(32, bbox)
    o.add_fibers(s, r)
    o.build(5)
    o.density_fibers(s, r)
    for l in range(6):
        _cmp(v, o, l, tag="weave")
    assert float(v.density_level(0)["occ"].max()) > 0.1


@pytest.mark.parametrize("tangent", [False, True])
def test_density_triangles_all_levels(P, tangent):
    t = gen.icosphere(2, 0.4)
    d = None
    if tangent:
        t, d = gen.ridge_mesh(12, 6, height=0.05, seed=2)
    bbox = np.concatenate([t.reshape(-1, 3).min(0) - 0.01, t.reshape(-1, 3).max(0) + 0.01]).astype(np.float32)
    v = P.Vox(16, bbox)
    T = torch.from_numpy(t).cuda()
    v.voxelize_triangles(T, None if d is None else torch.from_numpy(d).cuda())
    v.build_lod(4)
    v.density_triangles(T)
    o = oracle.Oracle(16, bbox)
    o.add_triangles(t, d)
    o.build(4)
    o.density_triangles(t)
    for l in range(5):
        _cmp(v, o, l, tag=f"tris tangent={tangent}")


def test_density_config4_windowed(P):
    c = gen.config(4)
    v = P.Vox(c["grid_res"], c["bbox"], profile=True)
    S, R = torch.from_numpy(c["segments"]).cuda(), torch.from_numpy(c["radii"]).cuda()
    v.voxelize_fibers(S, R)
    v.build_lod(3)
    v.density_fibers(S, R)
    k0 = v.level(0)["key"]
    cells, cnt = torch.unique(k0 >> 9, return_counts=True)
    for cell in (int(cells[torch.argmax(cnt)]), int(cells[len(cells) // 2])):
        o = window_oracle(c, 3, cell)
        s, r = c["segments"], c["radii"]
        o.density_fibers(s[_touching(c, 3, cell)], r[_touching(c, 3, cell)])
        for l in range(4):
            sel = (v.level(l)["key"] >> (3 * (3 - l))) == cell
            _cmp(v, o, l, sel=sel, tag="config4")
    assert v.stats()["ms_density"] > 0


def _touching(c, level, cell):
    N, bbox = c["grid_res"], c["bbox"]
    E = float(np.max(bbox[3:] - bbox[:3]))
    i, j, k = oracle.unmorton(cell)
    lo_box = np.array([i, j, k], np.float64) * (1 << level) * E / N + bbox[:3] - 2 * E / N
    hi_box = lo_box + ((1 << level) + 4) * E / N
    s, r = c["segments"], c["radii"]
    lo = np.minimum(s[:, 0], s[:, 1]) - r[:, None]
    hi = np.maximum(s[:, 0], s[:, 1]) + r[:, None]
    return np.all((hi >= lo_box) & (lo <= hi_box), axis=1)


def test_density_states(P):
    v = P.Vox(16, [0, 0, 0, 1, 1, 1])
    with pytest.raises(P.VoxError):
        v.density_level(0)
    S = torch.tensor([[[0.2, 0.2, 0.2], [0.8, 0.7, 0.6]]], device="cuda")
    R = torch.tensor([0.05], device="cuda")
    with pytest.raises(P.VoxError):
        v.density_fibers(S, R)            # before any voxelize call
    v.voxelize_fibers(S, R)
    v.density_fibers(S, R)
    v.build_lod(2)
    assert v.density_level(2)["occ"].numel() == v.size(2)


@pytest.mark.parametrize("seed", [0, 1])
def test_density_fibers_at_max_coordinates(P, seed):
    """Random fibers in the far corner of an 8192^3 grid (fine-grid coordinates near 8N =
    65536, where fp32 spacing is coarsest), axis-parallel and oblique, radii 0 to 2 voxels:
    the conservative sure-hit / sure-miss shortcuts of the density kernel never contradict
    the pinned predicate (bit-exact masks against the oracle)."""
    rng = np.random.default_rng(100 + seed)
    n = 300
    a = rng.uniform(0.996, 0.9995, (n, 3))
    d = rng.normal(0, 1, (n, 3))
    d[: n // 4, 1:] = 0.0                      # along x
    d[n // 4: n // 3, :2] *= 1e-4               # nearly along z
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    b = a + d * rng.uniform(0.0, 6.0, (n, 1)) / 8192
    s = np.stack([a, b], 1).astype(np.float32)
    r = (rng.uniform(0.0, 2.0, n) / 8192).astype(np.float32)
    bbox = np.array([0, 0, 0, 1, 1, 1], np.float32)
    v = P.Vox(8192, bbox)
    S, R = torch.from_numpy(s).cuda(), torch.from_numpy(r).cuda()
    v.voxelize_fibers(S, R)
    v.build_lod(1)
    v.density_fibers(S, R)
    o = oracle.Oracle(8192, bbox)
    o.add_fibers(s, r)
    o.build(1)
    o.density_fibers(s, r)
    _cmp(v, o, 0, tag=f"corner{seed}")
    _cmp(v, o, 1, tag=f"corner{seed}")
    assert float(v.density_level(0)["occ"].max()) > 0.1
