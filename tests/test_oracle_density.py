"""Pins of the oracle's sub-voxel density (docs/PREDICATES.md §13; the
paper's occupancy O = hits / Res_3^3 and axis-projected densities): SPEC's
closed-form occupancy examples built from exact primitives, identity with an
independent key voxelization of the 8N grid (bit indexing, voxel assignment, scaling), and
the level-l masks against a brute-force coarsening of that fine key set."""
import numpy as np
import pytest

import gen
import oracle


def _one(o, key):
    L = o.level(0)
    idx = int(np.searchsorted(L["key"], np.uint64(key)))
    assert L["key"][idx] == key
    return idx


def test_spec_occupancy_examples():
    N = 8
    bbox = np.array([0, 0, 0, N, N, N], np.float32)     # world = grid units
    v = (2, 2, 2)
    key = oracle.morton(*v)
    cases = []
    # one sub-voxel: a tiny sphere in the interior of sub-voxel (3, 4, 5)
    c = np.array(v) + (np.array([3, 4, 5]) + 0.5) / 8
    cases.append((np.stack([c, c])[None], np.array([0.01]), 1 / 512, (1 / 64, 1 / 64, 1 / 64)))
    # a z-column: a thin fiber through sub-column (3, 4) from inside the bottom to the top layer
    a = np.array([v[0] + 3.5 / 8, v[1] + 4.5 / 8, v[2] + 0.01])
    b = a + [0, 0, 0.98]
    cases.append((np.stack([a, b])[None], np.array([0.01]), 8 / 512, (8 / 64, 8 / 64, 1 / 64)))
    # the whole voxel: a fat fiber through it
    a = np.array(v) + [-1.0, 0.5, 0.5]
    cases.append((np.stack([a, a + [3, 0, 0]])[None], np.array([2.0]), 1.0, (1.0, 1.0, 1.0)))
    for seg, r, occ, axis in cases:
        seg = seg.astype(np.float32); r = r.astype(np.float32)
        o = oracle.Oracle(N, bbox)
        o.add_fibers(seg, r)
        o.build(0)
        o.density_fibers(seg, r)
        d = o.density_level(0)
        i = _one(o, key)
        assert d["occ"][i] == np.float32(occ)
        assert tuple(d["axis"][i].tolist()) == tuple(np.float32(axis).tolist())
    # a triangle pair covering the voxel in the interior of sub-layer z = 4: one full layer
    z = v[2] + 4.5 / 8
    q = np.array([[1.5, 1.5, z], [3.5, 1.5, z], [3.5, 3.5, z], [1.5, 3.5, z]], np.float32)
    tris = np.stack([q[[0, 1, 2]], q[[0, 2, 3]]]).astype(np.float32)
    o = oracle.Oracle(N, bbox)
    o.add_triangles(tris)
    o.build(0)
    o.density_triangles(tris)
    d = o.density_level(0)
    i = _one(o, key)
    assert d["occ"][i] == np.float32(64 / 512)
    assert d["axis"][i].tolist() == [np.float32(8 / 64), np.float32(8 / 64), 1.0]
    assert d["mask"][i].tolist() == [0, 0, 0, 0, 2 ** 64 - 1, 0, 0, 0]


def _fine_keys(kind, prims, N, bbox):
    o8 = oracle.Oracle(8 * N, bbox)
    if kind == "fiber":
        o8.add_fibers(*prims)
    else:
        o8.add_triangles(prims[0])
    o8.build(0)
    k = o8.level(0)["key"]
    ijk = np.array([oracle.unmorton(int(x)) for x in k], np.int64).reshape(-1, 3)
    return ijk


@pytest.mark.parametrize("kind", ["fiber", "tri"])
def test_masks_equal_the_8n_key_voxelization(kind):
    N = 16
    if kind == "fiber":
        s, r = gen.plain_weave(n_warp=4, n_weft=4, n_seg=16, pitch=1 / 4)
        s = (s + np.float32(0.013)).astype(np.float32)
        bbox = np.array([0, 0, 0, 1, 1, 1], np.float32)
        prims = (s, (r * 0.6).astype(np.float32))
    else:
        c = gen.config(1)
        bbox = c["bbox"]
        prims = (c["tris"],)
    o = oracle.Oracle(N, bbox)
    if kind == "fiber":
        o.add_fibers(*prims)
    else:
        o.add_triangles(prims[0])
    o.build(3)
    if kind == "fiber":
        o.density_fibers(*prims)
    else:
        o.density_triangles(prims[0])
    fine = _fine_keys(kind, prims, N, bbox)
    keys0 = set(o.level(0)["key"].tolist())
    fine = fine[[oracle.morton(*(x >> 3)) in keys0 for x in fine]]
    for l in range(4):
        d = o.density_level(l)
        L = o.level(l)
        # brute force: set bit (A,B,C) of the level-l voxel for every fine key x with x >> l
        want = {}
        for x in fine:
            cx = x >> l
            vk = oracle.morton(*(cx >> 3))
            A, B, C = cx & 7
            w = want.setdefault(vk, np.zeros(8, np.uint64))
            w[C] |= np.uint64(1) << np.uint64(A + 8 * B)
        got = {int(k): d["mask"][i] for i, k in enumerate(L["key"])}
        assert set(want) <= set(got)
        for k, m in got.items():
            assert np.array_equal(m, want.get(k, np.zeros(8, np.uint64))), (l, k)
        pop = np.array([sum(bin(int(w)).count("1") for w in m) for m in d["mask"]])
        assert np.array_equal(d["occ"], (pop / 512).astype(np.float32))
        assert np.all(d["axis"] >= d["occ"][:, None])       # a projected cell covers <= 8 hits: h/512 <= p/64
