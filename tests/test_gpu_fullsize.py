"""Parity at BASELINE.json's full sizes, in bench.py's launch configuration, on sampled
outputs: the GPU builds the whole config; the oracle recomputes whole Morton cells (every
primitive touching a cell, LoD inside it) and every level <= the cell level is compared
bit-for-bit inside those cells (windowed parity). The levels above the
window are chained: the oracle starts from the GPU's records of a middle level (whose own
values the windows and the exact conservation sums check) and builds every level above it
with its own arithmetic, compared bit-for-bit over the whole level."""
import numpy as np
import pytest
import torch

import gen
import oracle
from windowing import chain_levels, window_oracle

pytestmark = pytest.mark.gpu


def _cells(keys0, level, count, rng):
    cells, cnt = np.unique(keys0 >> np.uint64(3 * level), return_counts=True)
    order = np.argsort(-cnt, kind="stable")
    pick = [cells[order[0]], cells[order[len(order) // 2]]]          # densest and a median cell
    pick += list(rng.choice(cells, size=max(0, count - 2), replace=False))
    return [int(c) for c in pick]


def _check(v, c, level, cells):
    levels = [v.level(l) for l in range(level + 1)]      # device copies; cells selected on the GPU
    for cell in cells:
        o = window_oracle(c, level, cell)
        for l in range(level + 1):
            g = levels[l]
            sel = (g["key"] >> (3 * (level - l))) == cell
            r = o.level(l)
            assert np.array_equal(g["key"][sel].cpu().numpy().astype(np.uint64), r["key"]), (cell, l, "keys")
            assert np.array_equal(g["acc"][sel].cpu().numpy(), r["acc"]), (cell, l, "acc")
            assert np.array_equal(g["mass"][sel].cpu().numpy(), r["mass"]), (cell, l, "mass")
            if l > 0:
                assert np.array_equal(g["ncl"][sel].cpu().numpy(), r["ncl"]), (cell, l, "ncl")
                assert np.array_equal(g["cl"][sel].cpu().numpy(), r["cl"]), (cell, l, "cl")
        o.close()


@pytest.fixture(scope="module")
def P():
    from paper_2604_13191_b200 import build
    build.build()
    import paper_2604_13191_b200 as P
    return P


def test_config4_fullsize_windowed(P):
    c = gen.config(4)                                   # 10.28M segments at 4096^3, bench workload
    v = P.Vox(c["grid_res"], c["bbox"])
    v.voxelize_fibers(torch.from_numpy(c["segments"]).cuda(), torch.from_numpy(c["radii"]).cuda())
    v.build_lod(c["levels"])
    L0 = v.level(0)
    k0 = L0["key"].cpu().numpy().astype(np.uint64)
    assert len(k0) > 10_000_000
    # mass conservation at full size (exact integers), every level
    tot = L0["acc"].sum(0)
    del L0
    for l in range(1, c["levels"] + 1):
        assert torch.equal(v.level(l)["acc"].sum(0), tot)
    _check(v, c, 6, _cells(k0, 6, 4, np.random.default_rng(0)))
    chain_levels(v, c, 3)   # levels 4..12 over the whole grid (332k .. 1 voxels)


def test_config3_fullsize_windowed(P):
    c = gen.config(3)                                   # 100,352 triangles at 2048^3, tangent mode
    v = P.Vox(c["grid_res"], c["bbox"])
    v.voxelize_triangles(torch.from_numpy(c["tris"]).cuda(), torch.from_numpy(c["dirs"]).cuda())
    v.build_lod(c["levels"])
    k0 = v.level(0)["key"].cpu().numpy().astype(np.uint64)
    _check(v, c, 7, _cells(k0, 7, 3, np.random.default_rng(1)))


def test_config5_8192_windowed(P):
    # the largest grid of BASELINE's sweep: 32^3 voxel bins (15 local key bits), 13 levels
    c = gen.config(5, n_segments=4_000_000, grid_res=8192)
    v = P.Vox(c["grid_res"], c["bbox"])
    v.voxelize_fibers(torch.from_numpy(c["segments"]).cuda(), torch.from_numpy(c["radii"]).cuda())
    v.build_lod(c["levels"])
    L0 = v.level(0)
    k0 = L0["key"].cpu().numpy().astype(np.uint64)
    tot = L0["acc"].sum(0)
    del L0
    for l in (1, 5, 9, c["levels"]):
        assert torch.equal(v.level(l)["acc"].sum(0), tot)
    _check(v, c, 5, _cells(k0, 5, 3, np.random.default_rng(2)))
