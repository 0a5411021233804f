"""GPU parity: the CUDA path (through the C ABI) against the oracle, element by element.

Key sets bit-exact; mass/M and every lobe bit-exact by construction (PREDICATES §8), which
implies north_star's 1e-5 relative tolerance (asserted separately on the fp32 outputs)."""
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


def _cmp_level(g, r, l, tag=""):
    gk = g["key"].cpu().numpy().astype(np.uint64)
    assert gk.shape == r["key"].shape, f"{tag} level {l}: {gk.shape} vs {r['key'].shape} voxels"
    assert np.array_equal(gk, r["key"]), f"{tag} level {l} keys"
    assert np.array_equal(g["acc"].cpu().numpy(), r["acc"]), f"{tag} level {l} accumulators"
    gm, rm = g["mass"].cpu().numpy(), r["mass"]
    assert np.allclose(gm, rm, rtol=1e-5, atol=0), f"{tag} level {l} mass (1e-5)"
    assert np.array_equal(gm, rm) and np.array_equal(g["m6"].cpu().numpy(), r["m6"])
    if l > 0:
        assert np.array_equal(g["ncl"].cpu().numpy(), r["ncl"]), f"{tag} level {l} ncl"
        assert np.array_equal(g["cl"].cpu().numpy(), r["cl"]), f"{tag} level {l} lobes"


def _run_both(P, N, bbox, levels, segs=None, radii=None, tris=None, dirs=None, k=3, parts=1):
    v = P.Vox(N, bbox, k=k)
    o = oracle.Oracle(N, np.asarray(bbox, np.float32), k)
    if segs is not None:
        for idx in np.array_split(np.arange(len(segs)), parts):
            v.voxelize_fibers(torch.from_numpy(np.ascontiguousarray(segs[idx])).cuda(),
                              torch.from_numpy(np.ascontiguousarray(radii[idx])).cuda())
        o.add_fibers(segs, radii)
    if tris is not None:
        v.voxelize_triangles(torch.from_numpy(tris).cuda(), None if dirs is None else torch.from_numpy(dirs).cuda())
        o.add_triangles(tris, dirs)
    v.build_lod(levels)
    o.build(levels)
    return v, o


def test_config1_icosphere_all_levels(P):
    c = gen.config(1)
    v, o = _run_both(P, c["grid_res"], c["bbox"], c["levels"], tris=c["tris"])
    for l in range(c["levels"] + 1):
        _cmp_level(v.level(l), o.level(l), l, "icosphere")


def test_config2_plain_weave_all_levels(P):
    c = gen.config(2)
    v, o = _run_both(P, c["grid_res"], c["bbox"], c["levels"], segs=c["segments"], radii=c["radii"])
    for l in range(c["levels"] + 1):
        _cmp_level(v.level(l), o.level(l), l, "weave")
    st = v.stats()
    assert st["pairs"] <= st["candidates"]


@pytest.mark.parametrize("seed,n,N,rscale", [(0, 1, 32, 1.0), (1, 37, 64, 0.3), (2, 1000, 64, 1.0),
                                               (3, 4099, 128, 2.0), (4, 20000, 256, 0.7)])
def test_random_fibers_ragged(P, seed, n, N, rscale):
    """Random segments incl. ones straddling or outside the bbox, zero-length and r = 0."""
    rng = np.random.default_rng(seed)
    a = rng.uniform(-0.1, 1.1, (n, 3))
    b = a + rng.normal(0, 3.0 / N, (n, 3))
    segs = np.stack([a, b], 1).astype(np.float32)
    radii = (rng.uniform(0.0, 1.5, n) * rscale / N).astype(np.float32)
    if n > 10:
        segs[3, 1] = segs[3, 0]        # zero-length (sphere)
        radii[5] = 0.0                 # r = 0 (zero-volume fiber)
    L = int(np.log2(N))
    v, o = _run_both(P, N, [0, 0, 0, 1, 1, 1], L, segs=segs, radii=radii)
    for l in range(L + 1):
        _cmp_level(v.level(l), o.level(l), l, f"fibers{seed}")


def test_fibers_on_grid_planes_and_axes(P):
    """Adversarial fibers for the pinned predicate's branches (PREDICATES §4): axis-aligned
    segments (one or two fixed axes), endpoints exactly on voxel faces / corners (slab
    parameters exactly 0 or 1), lines at exactly r = 1/2 voxel from a row of voxel faces
    (tangent keys), diagonals through corners, spheres on corners; all levels bit-exact."""
    N = 64
    h = 1.0 / N
    segs, radii = [], []
    for ax in range(3):   # along each axis: on a grid line, on a face, inside; r tangent or not
        for off, r in ((0.0, 0.5), (0.5, 0.5), (0.25, 0.5), (0.0, 0.25), (0.5, 1.0), (0.3, 0.0)):
            a = np.array([20.0, 30.0, 40.0]) + off
            b = a.copy()
            b[ax] += 7.0
            segs.append([a * h, b * h])
            radii.append(r * h)
    for d in ((1, 1, 0), (1, 1, 1), (2, 1, 0), (0, 1, 1)):   # through corners, two or one fixed axes
        a = np.array([10.0, 12.0, 14.0])
        b = a + 5.0 * np.array(d, float)
        for r in (0.5, 0.7071067811865476, 0.25):
            segs.append([a * h, b * h])
            radii.append(r * h)
    for c in ((8.0, 8.0, 8.0), (8.5, 8.0, 8.0), (63.0, 63.0, 63.0), (0.0, 0.0, 0.0)):   # spheres
        p = np.array(c) * h
        segs.append([p, p])
        radii.append(0.5 * h)
        segs.append([p, p + np.array([0.0, 0.0, 1.0]) * h])   # unit segment from a corner
        radii.append(0.5 * h)
    segs = np.asarray(segs, np.float32)
    radii = np.asarray(radii, np.float32)
    L = int(np.log2(N))
    v, o = _run_both(P, N, [0, 0, 0, 1, 1, 1], L, segs=segs, radii=radii)
    for l in range(L + 1):
        _cmp_level(v.level(l), o.level(l), l, "grid-planes")


def test_triangles_tangent_mode_and_k(P):
    t, d = gen.ridge_mesh(n_quads=40, ridges=10, height=4 / 256, noise_amp=0.5 / 256)
    for k in (1, 2, 3, 8):
        v, o = _run_both(P, 256, [0, 0, 0, 1, 1, 1], 8, tris=t, dirs=d, k=k)
        for l in range(9):
            _cmp_level(v.level(l), o.level(l), l, f"ridge k={k}")


def test_mixed_and_split_calls(P):
    s, r = gen.plain_weave(n_warp=16, n_weft=16, n_seg=32, pitch=1 / 16)
    tris = gen.icosphere(2, radius=0.3)
    v = P.Vox(128, [0, 0, 0, 1, 1, 1])
    o = oracle.Oracle(128, np.array([0, 0, 0, 1, 1, 1], np.float32))
    perm = np.random.default_rng(1).permutation(len(s))
    for idx in np.array_split(perm, 3):
        v.voxelize_fibers(torch.from_numpy(s[idx]).cuda(), torch.from_numpy(r[idx]).cuda())
    v.voxelize_triangles(torch.from_numpy(tris).cuda())
    o.add_fibers(s, r)
    o.add_triangles(tris)
    v.build_lod(7)
    o.build(7)
    for l in range(8):
        _cmp_level(v.level(l), o.level(l), l, "mixed")


@pytest.mark.parametrize("part", [1, 5000, 60000])
def test_morton_parts_equal_one_pass(P, part):
    """A call cut into Morton parts (part_candidates; the > 2^32-candidate path of config 5 at
    8192^3) gives the oracle's result: fibers, then triangles accumulating into the same leaves,
    with part = 1 forcing one part per non-empty top cell."""
    s, r = gen.plain_weave(n_warp=16, n_weft=16, n_seg=32, pitch=1 / 16)
    tris = gen.icosphere(2, radius=0.3)
    v = P.Vox(128, [0, 0, 0, 1, 1, 1], part_candidates=part)
    o = oracle.Oracle(128, np.array([0, 0, 0, 1, 1, 1], np.float32))
    v.voxelize_fibers(torch.from_numpy(s).cuda(), torch.from_numpy(r).cuda())
    st = v.stats()
    assert st["candidates"] > part
    v.voxelize_triangles(torch.from_numpy(tris).cuda())
    o.add_fibers(s, r)
    o.add_triangles(tris)
    v.build_lod(7)
    o.build(7)
    for l in range(8):
        _cmp_level(v.level(l), o.level(l), l, f"parts{part}")


def test_host_entry_points(P):
    c = gen.config(1)
    v = P.Vox(c["grid_res"], c["bbox"])
    v.voxelize_triangles_host(c["tris"])
    v.build_lod(6)
    o = oracle.Oracle(c["grid_res"], c["bbox"])
    o.add_triangles(c["tris"])
    o.build(6)
    for l in range(7):
        _cmp_level(v.level(l, device="cpu"), o.level(l), l, "host")
    # asynchronous D2H on a side stream, interleaved with the build of further levels
    w = P.Vox(c["grid_res"], c["bbox"])
    w.voxelize_triangles_host(c["tris"])
    side = torch.cuda.Stream()
    outs = {}
    n0 = w.size(0)   # the leaf level: fp32 views formed on the side stream from the accumulators
    outs[0] = {"key": torch.empty(n0, dtype=torch.int64).pin_memory(),
               "mass": torch.empty(n0, dtype=torch.float32).pin_memory(),
               "m6": torch.empty((n0, 6), dtype=torch.float32).pin_memory()}
    w.copy_level_async(0, outs[0], side)
    for l in range(1, 7):
        w.build_lod(l)
        n = w.size(l)
        outs[l] = {"key": torch.empty(n, dtype=torch.int64).pin_memory(),
                   "mass": torch.empty(n, dtype=torch.float32).pin_memory(),
                   "m6": torch.empty((n, 6), dtype=torch.float32).pin_memory(),
                   "ncl": torch.empty(n, dtype=torch.uint8).pin_memory(),
                   "cl": torch.empty((n, 3, 7), dtype=torch.float32).pin_memory()}
        w.copy_level_async(l, outs[l], side)
    side.synchronize()
    r = o.level(0)
    assert np.array_equal(outs[0]["key"].numpy().astype(np.uint64), r["key"])
    assert np.array_equal(outs[0]["mass"].numpy(), r["mass"]) and np.array_equal(outs[0]["m6"].numpy(), r["m6"])
    # borrowed views: the first read forms the level's fp32 arrays on the ctx stream, later
    # copies read those arrays
    for l in (0, 3):
        assert int(w.view(l)["n"]) == w.size(l)
        _cmp_level(w.level(l, device="cpu"), o.level(l), l, "view")
    # an async copy of a level whose views a read formed copies those views, after the read
    n3 = w.size(3)
    again = {"key": torch.empty(n3, dtype=torch.int64).pin_memory(),
             "mass": torch.empty(n3, dtype=torch.float32).pin_memory(),
             "m6": torch.empty((n3, 6), dtype=torch.float32).pin_memory(),
             "ncl": torch.empty(n3, dtype=torch.uint8).pin_memory(),
             "cl": torch.empty((n3, 3, 7), dtype=torch.float32).pin_memory()}
    w.copy_level_async(3, again, side)
    side.synchronize()
    r = o.level(3)
    assert np.array_equal(again["mass"].numpy(), r["mass"]) and np.array_equal(again["m6"].numpy(), r["m6"])
    assert np.array_equal(again["cl"].numpy(), r["cl"])
    for l in range(1, 7):
        r = o.level(l)
        assert np.array_equal(outs[l]["key"].numpy().astype(np.uint64), r["key"])
        assert np.array_equal(outs[l]["mass"].numpy(), r["mass"]) and np.array_equal(outs[l]["m6"].numpy(), r["m6"])
        assert np.array_equal(outs[l]["ncl"].numpy(), r["ncl"]) and np.array_equal(outs[l]["cl"].numpy(), r["cl"])


def test_overlapped_contexts_async_copies(P):
    """The e2e pattern of bench.py: consecutive jobs whose contexts overlap -- job i's level
    copies (vox_copy_level_async on a high-priority side stream, fp32 views formed there) are
    still in flight while job i+1 uploads from host buffers and builds -- each job's host
    results equal the oracle's, bit for bit."""
    c = gen.config(2)
    N, L = c["grid_res"], c["levels"]
    o = oracle.Oracle(N, c["bbox"])
    o.add_fibers(c["segments"], c["radii"])
    o.build(L)
    pa = torch.from_numpy(c["segments"]).pin_memory()
    pb = torch.from_numpy(c["radii"]).pin_memory()
    side = torch.cuda.Stream(priority=-1)
    jobs = []
    for _ in range(3):
        v = P.Vox(N, c["bbox"])
        v.voxelize_fibers_host(pa, pb)
        outs = {}
        for l in range(L + 1):
            if l:
                v.build_lod(l)
            n = v.size(l)
            outs[l] = {"key": torch.empty(n, dtype=torch.int64).pin_memory(),
                       "mass": torch.empty(n, dtype=torch.float32).pin_memory(),
                       "m6": torch.empty((n, 6), dtype=torch.float32).pin_memory()}
            if l:
                outs[l]["ncl"] = torch.empty(n, dtype=torch.uint8).pin_memory()
                outs[l]["cl"] = torch.empty((n, 3, 7), dtype=torch.float32).pin_memory()
            v.copy_level_async(l, outs[l], side)
        ev = torch.cuda.Event()
        ev.record(side)
        jobs.append((v, ev, outs))
        if len(jobs) > 1:   # release the previous job once its copies have landed
            pv, pe, _ = jobs[-2]
            pe.synchronize()
            pv.close()
    jobs[-1][1].synchronize()
    jobs[-1][0].close()
    for _, _, outs in jobs:
        for l in range(L + 1):
            r = o.level(l)
            assert np.array_equal(outs[l]["key"].numpy().astype(np.uint64), r["key"]), l
            assert np.array_equal(outs[l]["mass"].numpy(), r["mass"]), l
            assert np.array_equal(outs[l]["m6"].numpy(), r["m6"]), l
            if l:
                assert np.array_equal(outs[l]["ncl"].numpy(), r["ncl"]), l
                assert np.array_equal(outs[l]["cl"].numpy(), r["cl"]), l


def test_errors_and_states(P):
    v = P.Vox(64, [0, 0, 0, 1, 1, 1])
    bad = torch.tensor([[[0.1, 0.1, 0.1], [0.2, float("nan"), 0.2]]], device="cuda")
    with pytest.raises(P.VoxError) as e:
        v.voxelize_fibers(bad, torch.tensor([0.01], device="cuda"))
    assert e.value.name == "VOX_ERR_INVALID_ARG"
    ok = torch.tensor([[[0.1, 0.1, 0.1], [0.2, 0.2, 0.2]]], device="cuda")
    with pytest.raises(P.VoxError):
        v.voxelize_fibers(ok, torch.tensor([-0.01], device="cuda"))
    with pytest.raises(P.VoxError):
        v.voxelize_triangles(torch.rand(2, 3, 3, device="cuda"), torch.zeros(2, 3, device="cuda"))
    assert v.level(0)["key"].numel() == 0                      # unchanged after errors
    v.voxelize_fibers(torch.zeros(0, 2, 3, device="cuda"), torch.zeros(0, device="cuda"))   # S = 0 no-op
    with pytest.raises(P.VoxError) as e:
        v.level(1)
    assert e.value.name == "VOX_ERR_LEVEL"
    with pytest.raises(P.VoxError) as e:
        v.build_lod(7)
    assert e.value.name == "VOX_ERR_LEVEL"
    v.voxelize_fibers(ok, torch.tensor([0.01], device="cuda"))
    v.build_lod(6)
    with pytest.raises(P.VoxError) as e:
        v.voxelize_fibers(ok, torch.tensor([0.01], device="cuda"))
    assert e.value.name == "VOX_ERR_STATE"
    # capacity cap refuses before allocating
    w = P.Vox(64, [0, 0, 0, 1, 1, 1], max_bytes=1000)
    with pytest.raises(P.VoxError) as e:
        w.voxelize_fibers(ok, torch.tensor([0.05], device="cuda"))
    assert e.value.name == "VOX_ERR_CAPACITY"


def test_fake_world_sharding_equals_unsharded(P):
    """T4 fake world: R Morton shards run one after another on one GPU; the
    union of their local levels and the gathered top levels equal the unsharded result."""
    s, r = gen.plain_weave(n_warp=32, n_weft=32, n_seg=64, pitch=1 / 32)
    S, R = torch.from_numpy(s).cuda(), torch.from_numpy(r).cuda()
    N, L = 256, 8
    full = P.Vox(N, [0, 0, 0, 1, 1, 1])
    full.voxelize_fibers(S, R)
    full.build_lod(L)
    # anchor: the unsharded result is the oracle's, level by level (so every comparison of the
    # shards with `full` below is a comparison with the oracle)
    o = oracle.Oracle(N, np.array([0, 0, 0, 1, 1, 1], np.float32))
    o.add_fibers(s, r)
    o.build(L)
    for l in range(L + 1):
        _cmp_level(full.level(l), o.level(l), l, "unsharded weave")
    for world, part in ((2, 0), (3, 0), (8, 0), (3, 20000)):   # part: Morton parts inside each shard
        shards = [P.Vox(N, [0, 0, 0, 1, 1, 1], rank=q, world=world, part_candidates=part) for q in range(world)]
        for v in shards:
            v.voxelize_fibers(S, R)
            v.build_lod(L)                      # stops at log2(N) - T without the gather
        T = shards[0].stats()["top_depth"]
        lt = L - T
        assert all(v.built_levels() == lt for v in shards)
        for l in range(lt + 1):
            got = [v.level(l) for v in shards]
            ref = full.level(l)
            for key in ("key", "acc", "mass", "m6", "ncl", "cl"):
                assert torch.equal(torch.cat([g[key] for g in got]), ref[key]), (world, l, key)
        recs = torch.cat([v.export_level(lt) for v in shards])   # = the all-gather, in rank order
        for v in shards:
            v.import_level(lt, recs)
            v.build_lod(L)
            for l in range(lt, L + 1):
                g, ref = v.level(l), full.level(l)
                for key in ("key", "acc", "ncl", "cl"):
                    assert torch.equal(g[key], ref[key]), (world, l, key)


def test_fake_world_triangles(P):
    """Sharded triangle voxelization (primitives outside a shard are skipped by its emit):
    the union of the shards' local levels equals the unsharded result."""
    c = gen.config(1)
    T = torch.from_numpy(c["tris"]).cuda()
    full = P.Vox(c["grid_res"], c["bbox"])
    full.voxelize_triangles(T)
    full.build_lod(c["levels"])
    o = oracle.Oracle(c["grid_res"], c["bbox"])
    o.add_triangles(c["tris"])
    o.build(c["levels"])
    for l in range(c["levels"] + 1):
        _cmp_level(full.level(l), o.level(l), l, "unsharded icosphere")
    for world in (2, 5):
        shards = [P.Vox(c["grid_res"], c["bbox"], rank=q, world=world) for q in range(world)]
        for v in shards:
            v.voxelize_triangles(T)
            v.build_lod(c["levels"])
        lt = shards[0].built_levels()
        for l in range(lt + 1):
            for key in ("key", "acc", "ncl", "cl"):
                assert torch.equal(torch.cat([v.level(l)[key] for v in shards]), full.level(l)[key]), (world, l, key)


def test_deterministic_repeat(P):
    c = gen.config(2)
    outs = []
    for _ in range(2):
        v = P.Vox(c["grid_res"], c["bbox"])
        v.voxelize_fibers(torch.from_numpy(c["segments"]).cuda(), torch.from_numpy(c["radii"]).cuda())
        v.build_lod(9)
        outs.append([v.level(l) for l in range(10)])
    for a, b in zip(*outs):
        for k in a:
            assert torch.equal(a[k], b[k])


def test_edge_cases_new_entry_points(P):
    """Empty and degenerate inputs through the NEXT-row entry points: no-ops where nothing is
    hit, exact agreement with the oracle where something is."""
    bbox = np.array([0, 0, 0, 1, 1, 1], np.float32)
    v = P.Vox(16, bbox)
    # nothing inside the grid: every primitive outside the bbox
    far = torch.tensor([[[5.0, 5.0, 5.0], [6.0, 6.0, 6.0]]], device="cuda")
    v.voxelize_fibers(far, torch.tensor([0.1], device="cuda"))
    v.sample_splines(torch.tensor([[[5.0, 5, 5], [6, 6, 6], [7, 7, 7], [8, 8, 8]]], device="cuda"),
                     torch.tensor([0.1], device="cuda"), 4)
    v.build_lod(4)
    assert all(v.size(l) == 0 for l in range(5))
    assert v.encode_level(2)["sggx6"].numel() == 0
    v.density_fibers(far, torch.tensor([0.1], device="cuda"))
    assert v.density_level(3)["occ"].numel() == 0
    # zero-area and zero-length primitives: keys without mass, zero samples
    w = P.Vox(16, bbox)
    o = oracle.Oracle(16, bbox)
    tri = np.array([[[0.3, 0.3, 0.3], [0.3, 0.3, 0.3], [0.3, 0.3, 0.3]],
                    [[0.1, 0.2, 0.5], [0.8, 0.3, 0.5], [0.4, 0.9, 0.5]]], np.float32)
    w.sample_triangles(torch.from_numpy(tri).cuda(), None, 9)
    o.sample_triangles(tri, None, 9)
    seg = np.array([[[0.5, 0.5, 0.5], [0.5, 0.5, 0.5]]], np.float32)
    w.voxelize_fibers(torch.from_numpy(seg).cuda(), torch.tensor([0.03], device="cuda"))
    o.add_fibers(seg, np.array([0.03], np.float32))
    w.build_lod(4)
    o.build(4)
    for l in range(5):
        _cmp_level(w.level(l), o.level(l), l, "edge")
    codes, _ = oracle.encode(o.level(0)["acc"])
    assert np.array_equal(w.encode_level(0)["sggx6"].cpu().numpy(), codes)
