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
