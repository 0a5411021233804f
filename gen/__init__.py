"""Seeded synthetic workloads for the five BASELINE.json configs.

This module only builds geometry (numpy, fp64 internally, returned as fp32 world units).
It holds none of the method's arithmetic (no grid transform, overlap test, weight or
clustering), so both the CUDA path and the oracle may consume its outputs.

Every function is deterministic for a given argument set (explicit numpy Generator seeds).
"""
from __future__ import annotations

import math

import numpy as np

__all__ = ["icosphere", "plain_weave", "ridge_mesh", "knit", "config", "CONFIGS"]


# --------------------------------------------------------------------------- config 1

def icosphere(subdiv: int = 1, radius: float = 0.4, center=(0.5, 0.5, 0.5)):
    """Regular icosahedron subdivided `subdiv` times, projected to a sphere.

    subdiv=1 -> 42 vertices, 80 faces (config 1). Returns triangle soup f32 [T,3,3]
    ("points that are not shared between different triangles").
    """
    t = (1.0 + 5.0 ** 0.5) / 2.0
    V = [(-1, t, 0), (1, t, 0), (-1, -t, 0), (1, -t, 0), (0, -1, t), (0, 1, t), (0, -1, -t), (0, 1, -t),
         (t, 0, -1), (t, 0, 1), (-t, 0, -1), (-t, 0, 1)]
    V = [np.array(v, dtype=np.float64) / np.linalg.norm(v) for v in V]
    F = [(0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11), (1, 5, 9), (5, 11, 4), (11, 10, 2),
         (10, 7, 6), (7, 1, 8), (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8), (3, 8, 9), (4, 9, 5), (2, 4, 11),
         (6, 2, 10), (8, 6, 7), (9, 8, 1)]
    for _ in range(subdiv):
        cache = {}

        def mid(a, b):
            key = (min(a, b), max(a, b))
            if key not in cache:
                m = V[a] + V[b]
                V.append(m / np.linalg.norm(m))
                cache[key] = len(V) - 1
            return cache[key]

        nf = []
        for a, b, c in F:
            ab, bc, ca = mid(a, b), mid(b, c), mid(c, a)
            nf += [(a, ab, ca), (b, bc, ab), (c, ca, bc), (ab, bc, ca)]
        F = nf
    P = np.array(V) * radius + np.asarray(center, dtype=np.float64)
    return P[np.array(F)].astype(np.float32)


# --------------------------------------------------------------------------- config 2

def plain_weave(n_warp: int = 128, n_weft: int = 128, n_seg: int = 256, pitch: float = 1.0 / 128,
                amp_frac: float = 0.3, radius_frac: float = 0.28):
    """Plain-weave patch over [0,1]^2 at z = 1/2: warp fibers along x, weft along y.

    Warp j: y = (j+1/2)p, z = 1/2 + A cos(pi (x/p - 1/2) + pi j); weft i: x = (i+1/2)p,
    z = 1/2 - A cos(pi (y/p - 1/2) + pi i); A = amp_frac*p, r = radius_frac*p.
    Each fiber is n_seg equal-parameter segments over [0,1]. Returns (segments f32
    [S,2,3], radii f32 [S]); no RNG.
    """
    A = amp_frac * pitch
    s = np.linspace(0.0, 1.0, n_seg + 1)
    segs = []
    for j in range(n_warp):
        x = s
        y = np.full_like(s, (j + 0.5) * pitch)
        z = 0.5 + A * np.cos(np.pi * (x / pitch - 0.5) + np.pi * j)
        P = np.stack([x, y, z], 1)
        segs.append(np.stack([P[:-1], P[1:]], 1))
    for i in range(n_weft):
        y = s
        x = np.full_like(s, (i + 0.5) * pitch)
        z = 0.5 - A * np.cos(np.pi * (y / pitch - 0.5) + np.pi * i)
        P = np.stack([x, y, z], 1)
        segs.append(np.stack([P[:-1], P[1:]], 1))
    seg = np.concatenate(segs).astype(np.float32)
    rad = np.full(seg.shape[0], radius_frac * pitch, dtype=np.float32)
    return seg, rad


# --------------------------------------------------------------------------- config 3

def _value_noise(x, y, cells: int, rng):
    g = rng.uniform(-1.0, 1.0, size=(cells + 2, cells + 2))
    fx, fy = x * cells, y * cells
    ix, iy = np.floor(fx).astype(int), np.floor(fy).astype(int)
    tx, ty = fx - ix, fy - iy
    sx, sy = tx * tx * (3 - 2 * tx), ty * ty * (3 - 2 * ty)
    a = g[ix, iy] * (1 - sx) + g[ix + 1, iy] * sx
    b = g[ix, iy + 1] * (1 - sx) + g[ix + 1, iy + 1] * sx
    return a * (1 - sy) + b * sy


def ridge_mesh(n_quads: int = 224, ridges: int = 56, height: float = 4.0 / 2048,
               noise_amp: float = 0.5 / 2048, seed: int = 3, noise_cells: int = 32):
    """Brushed-metal ridge heightfield over [0,1]^2 (config 3 stand-in for the steel table,
    P:516-551): z = 1/2 + h*tri(ridges*x) + value-noise, 2 triangles per quad.

    Returns (tris f32 [T,3,3], dirs f32 [T,3]) with dirs = the ridge direction (0,1,0)
    projected onto each facet (tangent mode).
    """
    rng = np.random.default_rng(seed)
    u = np.linspace(0.0, 1.0, n_quads + 1)
    X, Y = np.meshgrid(u, u, indexing="ij")
    ph = ridges * X
    tri = 2.0 * np.abs(ph - np.floor(ph + 0.5))          # triangle wave in [0,1], ridges along y
    Z = 0.5 + height * tri + noise_amp * _value_noise(X, Y, noise_cells, rng)
    P = np.stack([X, Y, Z], -1)
    a, b, c, d = P[:-1, :-1], P[1:, :-1], P[1:, 1:], P[:-1, 1:]
    t1 = np.stack([a, b, c], -2).reshape(-1, 3, 3)
    t2 = np.stack([a, c, d], -2).reshape(-1, 3, 3)
    tris = np.concatenate([t1, t2])
    n = np.cross(tris[:, 1] - tris[:, 0], tris[:, 2] - tris[:, 1])
    n /= np.linalg.norm(n, axis=1, keepdims=True)
    ydir = np.array([0.0, 1.0, 0.0])
    dirs = ydir - (n @ ydir)[:, None] * n
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    return tris.astype(np.float32), dirs.astype(np.float32)


# --------------------------------------------------------------------------- configs 4, 5

def _knit_centerline(course: int, n_wales: int, theta: np.ndarray, W: float, H: float, depth: float):
    """Closed-form weft-knit course: one loop per 2*pi of theta, loops interlock with the
    next course (they rise 1.25 H above their base and fold back in x)."""
    x = W * (theta / (2 * np.pi) + 0.14 * np.sin(2 * theta))
    y = H * (course + 0.5 - 0.75 * np.cos(theta))
    z = depth * np.cos(2 * theta + np.pi * course)
    return np.stack([x, y, z], -1)


def knit(n_segments: int = 10_000_000, seed: int = 4, grid_res: int = 4096, seg_len_vox: float = 3.0,
         radius_vox: float = 0.5, courses: int = 16, wales: int = 16, yarn_radius_frac: float = 0.18,
         fibers_per_yarn: int | None = None, max_fibers_per_yarn: int | None = None):
    """Explicit-fiber knit patch (config 4; config 5 with other sizes).

    16 courses x 16 wales of interlooped yarn loops over roughly [0,1]^2; each course yarn
    holds F fibers at cross-section offsets rho = R_y sqrt(u), phase phi ~ U(0, 2pi), with
    one twist turn per loop; each fiber is resampled at arclength L = seg_len_vox voxels;
    r = r0 U(0.9, 1.1), r0 = radius_vox voxels. F is chosen so the segment count is
    n_segments (+-0.5%) unless given. Returns (segments f32 [S,2,3], radii f32 [S], bbox f32 [6]).
    The bbox is the cubic hull of the patch (fixed world patch for every S and N), so the
    voxel size is E/grid_res.
    """
    rng = np.random.default_rng(seed)
    W = H = 1.0 / max(courses, wales)
    Ry = yarn_radius_frac * W
    depth = 0.35 * W
    # cubic hull of the patch (independent of F and S)
    lo = np.array([-0.2 * W - Ry, -0.3 * H - Ry, -depth - Ry])
    hi = np.array([wales * W + 0.2 * W + Ry, (courses + 1.3) * H + Ry, depth + Ry])
    E = float((hi - lo).max())
    c = 0.5 * (lo + hi)
    bbox = np.concatenate([c - E / 2, c + E / 2]).astype(np.float32)
    vox = E / grid_res
    L = seg_len_vox * vox
    # dense centerline per course, its arclength parameterisation
    nd = 4096 * wales
    th = np.linspace(0.0, 2 * np.pi * wales, nd + 1)
    cl = [_knit_centerline(cc, wales, th, W, H, depth) for cc in range(courses)]
    dl = [np.linalg.norm(np.diff(p, axis=0), axis=1) for p in cl]
    yarn_len = sum(float(d.sum()) for d in dl)
    if fibers_per_yarn is None:
        F = max(1, int(round(n_segments / (yarn_len / L))))
    else:
        F = fibers_per_yarn
    if max_fibers_per_yarn is not None:
        F = min(F, max_fibers_per_yarn)
    segs = []
    radii = []
    for cc in range(courses):
        P = cl[cc]
        s_acc = np.concatenate([[0.0], np.cumsum(dl[cc])])
        T = np.gradient(P, axis=0)
        T /= np.linalg.norm(T, axis=1, keepdims=True)
        Nrm = np.cross(T, np.array([0.0, 0.0, 1.0]))
        Nrm /= np.linalg.norm(Nrm, axis=1, keepdims=True)
        Bn = np.cross(T, Nrm)
        rho = Ry * np.sqrt(rng.uniform(0.0, 1.0, F))
        phi = rng.uniform(0.0, 2 * np.pi, F)
        r = radius_vox * vox * rng.uniform(0.9, 1.1, F)
        for f in range(F):
            ang = phi[f] + th            # one twist turn per loop
            Q = P + rho[f] * (np.cos(ang)[:, None] * Nrm + np.sin(ang)[:, None] * Bn)
            dq = np.linalg.norm(np.diff(Q, axis=0), axis=1)
            qa = np.concatenate([[0.0], np.cumsum(dq)])
            m = max(1, int(qa[-1] / L))
            tq = np.linspace(0.0, qa[-1], m + 1)
            R = np.stack([np.interp(tq, qa, Q[:, a]) for a in range(3)], 1)
            segs.append(np.stack([R[:-1], R[1:]], 1).astype(np.float32))
            radii.append(np.full(m, r[f], dtype=np.float32))
    seg = np.concatenate(segs)
    rad = np.concatenate(radii)
    return seg, rad, bbox


# --------------------------------------------------------------------------- configs

CONFIGS = {
    1: "icosphere mesh, 80 triangles, voxelized at 64^3 with density+SGGX and 6 LoD levels",
    2: "procedural plain-weave fabric patch, 256 fibers x 256 segments at 512^3",
    3: "100k-triangle synthetic brushed-metal ridge mesh at 2048^3 with full LoD pyramid",
    4: "explicit-fiber knit fabric, 10M fiber segments at 4096^3, 1 GPU vs 8 GPU Morton-range shards",
    5: "sparsity/resolution sweep: 1M-50M fiber segments at 1024^3-8192^3 across 1/2/4/8 B200",
}


def config(n: int, **kw) -> dict:
    """Inputs of BASELINE.json config n as a dict:
    {kind: 'tri'|'fiber', grid_res, bbox, levels, tris/dirs or segments/radii}."""
    if n == 1:
        return dict(kind="tri", grid_res=64, levels=6, bbox=np.array([0, 0, 0, 1, 1, 1], np.float32),
                    tris=icosphere(1), dirs=None)
    if n == 2:
        s, r = plain_weave()
        return dict(kind="fiber", grid_res=512, levels=9, bbox=np.array([0, 0, 0, 1, 1, 1], np.float32),
                    segments=s, radii=r)
    if n == 3:
        t, d = ridge_mesh()
        return dict(kind="tri", grid_res=2048, levels=11, bbox=np.array([0, 0, 0, 1, 1, 1], np.float32),
                    tris=t, dirs=d)
    if n == 4:
        S = kw.get("n_segments", 10_000_000)
        s, r, bb = knit(S, seed=4, grid_res=4096, **{k: v for k, v in kw.items() if k != "n_segments"})
        return dict(kind="fiber", grid_res=4096, levels=12, bbox=bb, segments=s, radii=r)
    if n == 5:
        S = kw.get("n_segments", 1_000_000)
        N = kw.get("grid_res", 1024)
        s, r, bb = knit(S, seed=5, grid_res=N, seg_len_vox=3.0 * N / 4096, radius_vox=0.5 * N / 4096)
        return dict(kind="fiber", grid_res=N, levels=int(math.log2(N)), bbox=bb, segments=s, radii=r)
    raise ValueError(n)


def splines_from_segments(seg):
    """Catmull-Rom controls [S,4,3] for consecutive fiber segments [S,2,3] (input preparation
    for the sampling front end, PREDICATES §12): piece i runs seg[i,0] -> seg[i,1]; its outer
    controls are the neighbouring nodes of the same fiber (segments chained end to start), or
    the end node reflected (2 P1 - P2, 2 P2 - P1) at a fiber end."""
    seg = np.asarray(seg, np.float32)
    P1, P2 = seg[:, 0], seg[:, 1]
    prev_ok = np.zeros(len(seg), bool)
    prev_ok[1:] = np.all(seg[:-1, 1] == seg[1:, 0], axis=1)
    next_ok = np.zeros(len(seg), bool)
    next_ok[:-1] = prev_ok[1:]
    P0 = np.where(prev_ok[:, None], np.roll(P1, 1, axis=0), 2 * P1 - P2)
    P3 = np.where(next_ok[:, None], np.roll(P2, -1, axis=0), 2 * P2 - P1)
    return np.ascontiguousarray(np.stack([P0, P1, P2, P3], 1).astype(np.float32))

