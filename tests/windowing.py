"""Windowed oracle runs (test helper): the oracle recomputes one Morton cell of a full-size
workload -- every primitive touching the cell (plus a 2-voxel margin) is voxelized, values are
kept inside the cell only, and the LoD is built inside it."""
import numpy as np

import oracle


def window_oracle(c, level, cell, **okw):
    N, bbox = c["grid_res"], c["bbox"]
    E = float(np.max(bbox[3:] - bbox[:3]))
    i, j, k = oracle.unmorton(cell)
    lo_box = np.array([i, j, k], np.float64) * (1 << level) * E / N + bbox[:3] - 2 * E / N
    hi_box = lo_box + ((1 << level) + 4) * E / N
    o = oracle.Oracle(N, bbox, **okw)
    o.set_window(level, cell)
    if c["kind"] == "fiber":
        s, r = c["segments"], c["radii"]
        lo = np.minimum(s[:, 0], s[:, 1]) - r[:, None]
        hi = np.maximum(s[:, 0], s[:, 1]) + r[:, None]
        sel = np.all((hi >= lo_box) & (lo <= hi_box), axis=1)
        o.add_fibers(np.ascontiguousarray(s[sel]), np.ascontiguousarray(r[sel]))
    else:
        t = c["tris"]
        sel = np.all((t.max(1) >= lo_box) & (t.min(1) <= hi_box), axis=1)
        d = None if c["dirs"] is None else np.ascontiguousarray(c["dirs"][sel])
        o.add_triangles(np.ascontiguousarray(t[sel]), d)
    o.build(level)
    return o


def chain_levels(v, c, l0, k=3, hist_samples=5000):
    """Oracle levels l0+1..top from the GPU's level-l0 records vs the GPU's own levels."""
    rec = v.export_level(l0).cpu().numpy().view(np.int64)
    words = 9 + 7 * k
    rec = rec.reshape(-1, words)
    o = oracle.Oracle(c["grid_res"], c["bbox"], k, distance=v.distance, hist_samples=hist_samples)
    o.build_from(l0, rec[:, 0].view(np.uint64), rec[:, 1:8], rec[:, 8].astype(np.uint8),
                 rec[:, 9:].reshape(-1, k, 7), c["levels"])
    for l in range(l0 + 1, c["levels"] + 1):
        g, r = v.level(l, device="cpu"), o.level(l)
        assert np.array_equal(g["key"].numpy().astype(np.uint64), r["key"]), (l, "keys")
        assert np.array_equal(g["acc"].numpy(), r["acc"]), (l, "acc")
        assert np.array_equal(g["ncl"].numpy(), r["ncl"]), (l, "ncl")
        assert np.array_equal(g["cl"].numpy(), r["cl"]), (l, "lobes")
    o.close()
