"""GPU parity of the paper's sampling front end (vox_sample_splines / vox_sample_triangles,
docs/PREDICATES.md §12) against the oracle: every level bit-exact (keys,
accumulators, lobes), alone, mixed with the exact path, sharded, and at the edges (one sample,
budget 1, pieces leaving the grid)."""
import numpy as np
import pytest
import torch

import gen
import oracle

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
        assert np.array_equal(g["mass"].cpu().numpy(), r["mass"]), (tag, l, "mass")
        if l > 0:
            assert np.array_equal(g["ncl"].cpu().numpy(), r["ncl"]), (tag, l, "ncl")
            assert np.array_equal(g["cl"].cpu().numpy(), r["cl"]), (tag, l, "lobes")


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("n", [1, 8, 33])
def test_splines_weave_all_levels(P, n):
    c = gen.config(2)
    ctrl = gen.splines_from_segments(c["segments"])
    v = P.Vox(c["grid_res"], c["bbox"])
    v.sample_splines(_cuda(ctrl), _cuda(c["radii"]), n)
    v.build_lod(c["levels"])
    o = oracle.Oracle(c["grid_res"], c["bbox"])
    o.sample_splines(ctrl, c["radii"], n)
    o.build(c["levels"])
    _cmp(v, o, c["levels"], f"weave splines n={n}")


@pytest.mark.parametrize("cfg,budget", [(1, 1), (1, 64), (3, 16)])
def test_triangles_all_levels(P, cfg, budget):
    c = gen.config(cfg)
    v = P.Vox(c["grid_res"], c["bbox"])
    v.sample_triangles(_cuda(c["tris"]), None if c["dirs"] is None else _cuda(c["dirs"]), budget)
    v.build_lod(c["levels"])
    o = oracle.Oracle(c["grid_res"], c["bbox"])
    o.sample_triangles(c["tris"], c["dirs"], budget)
    o.build(c["levels"])
    _cmp(v, o, c["levels"], f"tris cfg={cfg} budget={budget}")


def test_mixed_exact_and_sampled_and_out_of_grid(P):
    s, r = gen.plain_weave(n_warp=16, n_weft=16, n_seg=32, pitch=1 / 16)
    rng = np.random.default_rng(4)
    ctrl = gen.splines_from_segments(s)
    ctrl[::7] += rng.normal(0, 0.3, ctrl[::7].shape).astype(np.float32)   # some pieces leave the grid
    bbox = np.array([0, 0, -0.1, 1, 1, 0.1], np.float32)
    t, d = gen.ridge_mesh(8, 8, seed=1)
    t = (t * 0.5 + 0.25).astype(np.float32)
    v = P.Vox(128, bbox)
    o = oracle.Oracle(128, bbox)
    v.voxelize_fibers(_cuda(s), _cuda(r))
    o.add_fibers(s, r)
    v.sample_splines(_cuda(ctrl), _cuda(r), 5)
    o.sample_splines(ctrl, r, 5)
    v.sample_triangles(_cuda(t), _cuda(d), 7)
    o.sample_triangles(t, d, 7)
    v.build_lod(7)
    o.build(7)
    _cmp(v, o, 7, "mixed")


def test_sampled_fake_world_sharding(P):
    c = gen.config(2)
    ctrl, R = _cuda(gen.splines_from_segments(c["segments"])), _cuda(c["radii"])
    N, L = c["grid_res"], c["levels"]
    full = P.Vox(N, c["bbox"])
    full.sample_splines(ctrl, R, 4)
    full.build_lod(L)
    world = 3
    shards = [P.Vox(N, c["bbox"], rank=q, world=world) for q in range(world)]
    for v in shards:
        v.sample_splines(ctrl, R, 4)
        v.build_lod(L)
    lt = shards[0].built_levels()
    for l in range(lt + 1):
        ref = full.level(l)
        for key in ("key", "acc", "ncl", "cl"):
            assert torch.equal(torch.cat([v.level(l)[key] for v in shards]), ref[key]), (l, key)


def test_sampling_errors(P):
    v = P.Vox(64, [0, 0, 0, 1, 1, 1])
    ctrl = torch.zeros((4, 4, 3), device="cuda")
    r = torch.full((4,), 0.01, device="cuda")
    with pytest.raises(P.VoxError):
        v.sample_splines(ctrl, r, 0)
    bad = ctrl.clone()
    bad[1, 2, 0] = float("nan")
    with pytest.raises(P.VoxError):
        v.sample_splines(bad, r, 4)
    with pytest.raises(P.VoxError):
        v.sample_triangles(torch.zeros((2, 3, 3), device="cuda"), None, 0)
