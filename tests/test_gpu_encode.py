"""GPU parity of the SGGX finalisation and 6-byte compact form (vox_encode_level,
docs/PREDICATES.md §11) against the oracle's encoding of its own levels:
bytes and jitter flags bit-exact at every level (leaf aggregates, parent aggregates, lobes)."""
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


def _oracle_codes(r, k, leaf):
    agg, fa = oracle.encode(r["acc"])
    if leaf:
        return agg, None, fa
    cl, fc = oracle.encode(r["cl_acc"].reshape(-1, 7))
    cl = cl.reshape(-1, k, 6)
    fc = fc.reshape(-1, k)
    used = np.arange(k)[None, :] < r["ncl"][:, None]
    flags = fa.astype(np.int64)
    for q in range(k):
        flags |= ((fc[:, q] & used[:, q]).astype(np.int64) << (q + 1))
    return agg, cl, flags.astype(np.uint8)


def _cmp_codes(v, r, l, k, sel=None, tag=""):
    g = v.encode_level(l)
    s = (lambda t: t) if sel is None else (lambda t: t[sel])
    agg, cl, fl = _oracle_codes(r, k, l == 0)
    assert np.array_equal(s(g["sggx6"]).cpu().numpy(), agg), (tag, l, "aggregate bytes")
    if l == 0:
        lead = s(g["cl6"]).cpu().numpy()
        assert np.array_equal(lead[:, 0], agg), (tag, l, "leaf lobe = aggregate")
        assert np.array_equal(s(g["flags"]).cpu().numpy() & 1, fl), (tag, l, "flags")
    else:
        assert np.array_equal(s(g["cl6"]).cpu().numpy(), cl), (tag, l, "lobe bytes")
        assert np.array_equal(s(g["flags"]).cpu().numpy(), fl), (tag, l, "flags")


@pytest.mark.parametrize("k", [1, 3, 8])
def test_encode_weave_all_levels(P, k):
    s, r = gen.plain_weave(n_warp=16, n_weft=16, n_seg=32, pitch=1 / 16)
    bbox = np.array([0, 0, -0.1, 1, 1, 0.1], np.float32)
    v = P.Vox(128, bbox, k=k)
    v.voxelize_fibers(torch.from_numpy(s).cuda(), torch.from_numpy(r).cuda())
    v.build_lod(7)
    o = oracle.Oracle(128, bbox, k)
    o.add_fibers(s, r)
    o.build(7)
    for l in range(8):
        _cmp_codes(v, o.level(l), l, k, tag=f"weave k={k}")


def test_encode_config1_and_degenerate_jitter(P):
    c = gen.config(1)
    v = P.Vox(c["grid_res"], c["bbox"])
    v.voxelize_triangles(torch.from_numpy(c["tris"]).cuda())
    v.build_lod(c["levels"])
    o = oracle.Oracle(c["grid_res"], c["bbox"])
    o.add_triangles(c["tris"])
    o.build(c["levels"])
    for l in range(c["levels"] + 1):
        _cmp_codes(v, o.level(l), l, 3, tag="icosphere")
    # flat faces: a leaf's normal distribution is a delta -> jittered
    assert int((v.encode_level(0)["flags"] & 1).sum()) > 0


def test_encode_config4_windowed(P):
    c = gen.config(4)
    v = P.Vox(c["grid_res"], c["bbox"])
    v.voxelize_fibers(torch.from_numpy(c["segments"]).cuda(), torch.from_numpy(c["radii"]).cuda())
    v.build_lod(c["levels"])
    k0 = v.level(0)["key"]
    cells, cnt = torch.unique(k0 >> 15, return_counts=True)
    cell = int(cells[torch.argmax(cnt)])
    o = window_oracle(c, 5, cell)
    for l in range(6):
        sel = (v.level(l)["key"] >> (3 * (5 - l))) == cell
        _cmp_codes(v, o.level(l), l, 3, sel=sel, tag="config4")
    st = v.stats()
    assert st["launches"] > 0
