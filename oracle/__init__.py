"""CPU oracle of the hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import this package. The product package
``paper_2604_13191_b200`` never imports it, and this package never imports the product.

This module is argument marshalling over ``oracle/oracle.c`` (plain C, pinned fp32 per
``docs/PREDICATES.md``, exact ``__int128`` sums). See the C file's header for what is
computed and how it is pinned.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
K_DEFAULT = 3
HIST_N_DEFAULT = 5000   # P:389 "N=5000 samples for each S"


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so (gcc, -ffp-contract=off, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(
            ["gcc", "-std=c11", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
             "-o", _LIB, _SRC, "-lm"])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB)
        f32p = C.POINTER(C.c_float)
        i64p = C.POINTER(C.c_int64)
        u64p = C.POINTER(C.c_uint64)
        u8p = C.POINTER(C.c_uint8)
        L.orc_create.restype = C.c_void_p
        L.orc_create.argtypes = [C.c_uint32, f32p, C.c_int]
        L.orc_destroy.argtypes = [C.c_void_p]
        L.orc_set_window.argtypes = [C.c_void_p, C.c_int, C.c_uint64]
        L.orc_add_fibers.argtypes = [C.c_void_p, f32p, f32p, C.c_uint64]
        L.orc_add_triangles.argtypes = [C.c_void_p, f32p, f32p, C.c_uint64]
        L.orc_build.argtypes = [C.c_void_p, C.c_int]
        L.orc_build_from.argtypes = [C.c_void_p, C.c_int, C.c_uint64, u64p, i64p, u8p, i64p, C.c_int]
        L.orc_level_size.restype = C.c_uint64
        L.orc_level_size.argtypes = [C.c_void_p, C.c_int]
        L.orc_level_copy.argtypes = [C.c_void_p, C.c_int, u64p, i64p, f32p, f32p, u8p, i64p, f32p]
        L.orc_morton.restype = C.c_uint64
        L.orc_morton.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32]
        L.orc_unmorton.argtypes = [C.c_uint64] + [C.POINTER(C.c_uint32)] * 3
        L.orc_grid.argtypes = [f32p, C.c_uint32, f32p, f32p]
        L.orc_fiber_eval.argtypes = [f32p, f32p, C.c_float, C.c_int64, C.c_int64, C.c_int64, f32p]
        L.orc_tri_sat.argtypes = [f32p, C.c_int64, C.c_int64, C.c_int64]
        L.orc_tri_area.restype = C.c_float
        L.orc_tri_area.argtypes = [f32p, C.c_int64, C.c_int64, C.c_int64]
        L.orc_theta.argtypes = [f32p, f32p]
        L.orc_sggxh.argtypes = [C.c_int, i64p, C.c_int, i64p]
        L.orc_sigma.argtypes = [i64p, f32p]
        L.orc_distance.restype = C.c_float
        L.orc_distance.argtypes = [i64p, i64p]
        u16p = C.POINTER(C.c_uint16)
        L.orc_set_distance.argtypes = [C.c_void_p, C.c_int, C.c_int]
        L.orc_sample_table.argtypes = [C.c_int, f32p]
        L.orc_sw_tables.argtypes = [u8p, i64p]
        L.orc_hist.argtypes = [i64p, C.c_int, u16p]
        L.orc_hist_distance.restype = C.c_int64
        L.orc_hist_distance.argtypes = [u16p, u16p]
        L.orc_sggxh_hist.argtypes = [C.c_int, i64p, C.c_int, C.c_int, i64p]
        L.orc_jacobi.argtypes = [f32p, f32p]
        L.orc_encode.argtypes = [C.c_uint64, i64p, u8p, u8p]
        L.orc_finalize.argtypes = [i64p, f32p]
        L.orc_spline_eval.argtypes = [f32p, C.c_float, f32p, f32p]
        L.orc_density_fibers.argtypes = [C.c_void_p, f32p, f32p, C.c_uint64]
        L.orc_density_triangles.argtypes = [C.c_void_p, f32p, C.c_uint64]
        L.orc_density_level.argtypes = [C.c_void_p, C.c_int, u64p, f32p, f32p]
        L.orc_sample_splines.argtypes = [C.c_void_p, f32p, f32p, C.c_uint64, C.c_int]
        L.orc_sample_triangles.argtypes = [C.c_void_p, f32p, f32p, C.c_uint64, C.c_int]
        L.orc_tri_samples.argtypes = [C.c_float, C.c_float, C.c_int]
        L.orc_tri_sample_points.argtypes = [f32p, C.c_int, f32p]
        _lib = L
    return _lib


def _f32(a):
    a = np.ascontiguousarray(a, dtype=np.float32)
    return a, a.ctypes.data_as(C.POINTER(C.c_float))


def _i64(a):
    a = np.ascontiguousarray(a, dtype=np.int64)
    return a, a.ctypes.data_as(C.POINTER(C.c_int64))


class OracleError(RuntimeError):
    pass


def _check(rc, what):
    if rc != 0:
        raise OracleError(f"{what} failed with oracle status {rc}")


class Oracle:
    """Plain CPU voxelizer + LoD builder (docs/PREDICATES.md §1-§9)."""

    def __init__(self, grid_res: int, bbox, k: int = K_DEFAULT, distance: str = "sigma",
                 hist_samples: int = HIST_N_DEFAULT):
        bb, p = _f32(np.asarray(bbox, dtype=np.float32).reshape(6))
        self._bb = bb
        self.k = int(k)
        self.grid_res = int(grid_res)
        self._h = lib().orc_create(int(grid_res), p, int(k))
        if not self._h:
            raise OracleError("orc_create rejected (grid_res, bbox, k)")
        if distance not in ("sigma", "hist"):
            raise OracleError(f"unknown distance {distance!r}")
        _check(lib().orc_set_distance(self._h, 1 if distance == "hist" else 0, int(hist_samples)), "set_distance")

    def close(self):
        if self._h:
            lib().orc_destroy(self._h)
            self._h = None

    __del__ = close

    def set_window(self, level: int, cell: int):
        _check(lib().orc_set_window(self._h, int(level), int(cell)), "set_window")

    def add_fibers(self, segments, radii):
        s, sp = _f32(np.asarray(segments).reshape(-1, 6))
        r, rp = _f32(np.asarray(radii).reshape(-1))
        assert s.shape[0] == r.shape[0]
        _check(lib().orc_add_fibers(self._h, sp, rp, s.shape[0]), "add_fibers")

    def add_triangles(self, tris, dirs=None):
        t, tp = _f32(np.asarray(tris).reshape(-1, 9))
        if dirs is None:
            dp = None
        else:
            d, dp = _f32(np.asarray(dirs).reshape(-1, 3))
            assert d.shape[0] == t.shape[0]
        _check(lib().orc_add_triangles(self._h, tp, dp, t.shape[0]), "add_triangles")

    def sample_splines(self, ctrl, radii, n: int):
        """§12: Catmull-Rom pieces (controls [S,4,3] world, radii [S]), n samples per piece."""
        cc, cp = _f32(np.asarray(ctrl).reshape(-1, 12))
        r, rp = _f32(np.asarray(radii).reshape(-1))
        assert cc.shape[0] == r.shape[0]
        _check(lib().orc_sample_splines(self._h, cp, rp, cc.shape[0], int(n)), "sample_splines")

    def sample_triangles(self, tris, dirs=None, budget: int = 64):
        """§12: triangles sampled with Heitz's map, budget samples for the largest one."""
        t, tp = _f32(np.asarray(tris).reshape(-1, 9))
        dp = None
        if dirs is not None:
            d, dp = _f32(np.asarray(dirs).reshape(-1, 3))
        _check(lib().orc_sample_triangles(self._h, tp, dp, t.shape[0], int(budget)), "sample_triangles")

    def density_fibers(self, segments, radii):
        """§13: OR the sub-voxel hits of fiber segments into the level-0 masks (after build)."""
        s, sp = _f32(np.asarray(segments).reshape(-1, 6))
        r, rp = _f32(np.asarray(radii).reshape(-1))
        _check(lib().orc_density_fibers(self._h, sp, rp, s.shape[0]), "density_fibers")

    def density_triangles(self, tris):
        t, tp = _f32(np.asarray(tris).reshape(-1, 9))
        _check(lib().orc_density_triangles(self._h, tp, t.shape[0]), "density_triangles")

    def density_level(self, l: int) -> dict:
        """§13 masks [n,8] uint64 (word z, bit x + 8 y), occupancy [n], axis [n,3] (YZ, XZ, XY)."""
        n = int(lib().orc_level_size(self._h, int(l)))
        out = dict(mask=np.zeros((n, 8), np.uint64), occ=np.zeros(n, np.float32), axis=np.zeros((n, 3), np.float32))
        P = lambda a, t: a.ctypes.data_as(C.POINTER(t))
        _check(lib().orc_density_level(self._h, int(l), P(out["mask"], C.c_uint64), P(out["occ"], C.c_float),
                                       P(out["axis"], C.c_float)), "density_level")
        return out

    def build(self, levels: int = 0):
        _check(lib().orc_build(self._h, int(levels)), "build")

    def build_from(self, l0: int, key, acc, ncl, cl_acc, levels: int):
        """Start the pyramid from given level-l0 records (sorted keys [n], exact acc [n,7],
        ncl [n], lobe accumulators [n,k,7]; ignored for l0 = 0) and build levels l0+1..levels
        with the same code as build() (test infrastructure: upper levels of workloads too large
        for the oracle's voxelization)."""
        key = np.ascontiguousarray(key, np.uint64)
        n = len(key)
        acc = np.ascontiguousarray(acc, np.int64).reshape(n, 7)
        ncl = np.ascontiguousarray(ncl if ncl is not None else np.zeros(n), np.uint8)
        cla = np.ascontiguousarray(cl_acc if cl_acc is not None else np.zeros((n, self.k, 7)), np.int64)
        P = lambda a, t: a.ctypes.data_as(C.POINTER(t))
        _check(lib().orc_build_from(self._h, int(l0), n, P(key, C.c_uint64), P(acc, C.c_int64), P(ncl, C.c_uint8),
                                    P(cla, C.c_int64), int(levels)), "build_from")

    def level(self, l: int) -> dict:
        n = int(lib().orc_level_size(self._h, int(l)))
        k = self.k
        out = dict(
            key=np.zeros(n, np.uint64), acc=np.zeros((n, 7), np.int64),
            mass=np.zeros(n, np.float32), m6=np.zeros((n, 6), np.float32),
            ncl=np.zeros(n, np.uint8), cl_acc=np.zeros((n, k, 7), np.int64),
            cl=np.zeros((n, k, 7), np.float32))
        P = lambda a, t: a.ctypes.data_as(C.POINTER(t))
        _check(lib().orc_level_copy(self._h, int(l), P(out["key"], C.c_uint64), P(out["acc"], C.c_int64),
                                    P(out["mass"], C.c_float), P(out["m6"], C.c_float),
                                    P(out["ncl"], C.c_uint8), P(out["cl_acc"], C.c_int64),
                                    P(out["cl"], C.c_float)), "level_copy")
        return out


# ----------------------------------------------------------------- unit entries

def morton(i, j, k) -> int:
    return int(lib().orc_morton(int(i), int(j), int(k)))


def unmorton(key):
    a, b, c = C.c_uint32(), C.c_uint32(), C.c_uint32()
    lib().orc_unmorton(int(key), C.byref(a), C.byref(b), C.byref(c))
    return a.value, b.value, c.value


def grid(bbox, n, p):
    bb, bp = _f32(np.asarray(bbox).reshape(6))
    pp, ppp = _f32(np.asarray(p).reshape(3))
    out = np.zeros(3, np.float32)
    lib().orc_grid(bp, int(n), ppp, out.ctypes.data_as(C.POINTER(C.c_float)))
    return out


def fiber_eval(a, b, rg, i, j, k):
    """Grid-space segment a->b, grid radius rg, voxel (i,j,k) -> (is_key, l_r)."""
    A, ap = _f32(np.asarray(a).reshape(3))
    B, bp = _f32(np.asarray(b).reshape(3))
    ell = C.c_float(0)
    key = lib().orc_fiber_eval(ap, bp, C.c_float(rg), int(i), int(j), int(k), C.byref(ell))
    return bool(key), float(np.float32(ell.value))


def tri_sat(g, i, j, k) -> bool:
    G, gp = _f32(np.asarray(g).reshape(9))
    return bool(lib().orc_tri_sat(gp, int(i), int(j), int(k)))


def tri_area(g, i, j, k) -> float:
    G, gp = _f32(np.asarray(g).reshape(9))
    return float(np.float32(lib().orc_tri_area(gp, int(i), int(j), int(k))))


def theta():
    t = np.zeros((32, 3), np.float32)
    c = np.zeros((32, 6), np.float32)
    lib().orc_theta(t.ctypes.data_as(C.POINTER(C.c_float)), c.ctypes.data_as(C.POINTER(C.c_float)))
    return t, c


def sggxh(acc, k=K_DEFAULT):
    """acc: (n,7) int64 cluster accumulators -> (m,7) kept clusters."""
    a, ap = _i64(np.asarray(acc).reshape(-1, 7))
    out = np.zeros((k, 7), np.int64)
    m = lib().orc_sggxh(a.shape[0], ap, int(k), out.ctypes.data_as(C.POINTER(C.c_int64)))
    if m < 0:
        raise OracleError(f"sggxh status {m}")
    return out[:m]


def sigma(acc7):
    a, ap = _i64(np.asarray(acc7).reshape(7))
    s = np.zeros(32, np.float32)
    lib().orc_sigma(ap, s.ctypes.data_as(C.POINTER(C.c_float)))
    return s


def distance(a7, b7) -> float:
    a, ap = _i64(np.asarray(a7).reshape(7))
    b, bp = _i64(np.asarray(b7).reshape(7))
    return float(np.float32(lib().orc_distance(ap, bp)))


# ----------------------------------------------------------------- §10 histogram distance

def sample_table(n=HIST_N_DEFAULT):
    """(n,3) fp32 whole-sphere spherical-Fibonacci sample points of §10."""
    u = np.zeros((n, 3), np.float32)
    lib().orc_sample_table(int(n), u.ctypes.data_as(C.POINTER(C.c_float)))
    return u


def sw_tables():
    """(perm [32][125] uint8, gap [32][124] int64) slice tables of §10."""
    perm = np.zeros((32, 125), np.uint8)
    gap = np.zeros((32, 124), np.int64)
    lib().orc_sw_tables(perm.ctypes.data_as(C.POINTER(C.c_uint8)), gap.ctypes.data_as(C.POINTER(C.c_int64)))
    return perm, gap


def hist(acc7, n=HIST_N_DEFAULT):
    """125-bin histogram (uint16, bin = b0 + 5 b1 + 25 b2) of one cluster's n samples."""
    a, ap = _i64(np.asarray(acc7).reshape(7))
    h = np.zeros(125, np.uint16)
    _check(lib().orc_hist(ap, int(n), h.ctypes.data_as(C.POINTER(C.c_uint16))), "hist")
    return h


def hist_distance(h1, h2) -> int:
    a = np.ascontiguousarray(h1, dtype=np.uint16)
    b = np.ascontiguousarray(h2, dtype=np.uint16)
    return int(lib().orc_hist_distance(a.ctypes.data_as(C.POINTER(C.c_uint16)),
                                       b.ctypes.data_as(C.POINTER(C.c_uint16))))


def sggxh_hist(acc, k=K_DEFAULT, n=HIST_N_DEFAULT):
    """SGGX-H with the histogram distance: (m,7) int64 -> kept clusters."""
    a, ap = _i64(np.asarray(acc).reshape(-1, 7))
    out = np.zeros((k, 7), np.int64)
    m = lib().orc_sggxh_hist(a.shape[0], ap, int(k), int(n), out.ctypes.data_as(C.POINTER(C.c_int64)))
    if m < 0:
        raise OracleError(f"sggxh_hist status {m}")
    return out[:m]


# ----------------------------------------------------------------- §12 sampling front end

def spline_eval(G, t):
    """Grid-space Catmull-Rom piece G [4,3] at t -> (position (3,), unit tangent (3,))."""
    g, gp = _f32(np.asarray(G).reshape(12))
    pos = np.zeros(3, np.float32)
    tan = np.zeros(3, np.float32)
    lib().orc_spline_eval(gp, C.c_float(t), pos.ctypes.data_as(C.POINTER(C.c_float)),
                          tan.ctypes.data_as(C.POINTER(C.c_float)))
    return pos, tan


def tri_samples(area, amax, budget) -> int:
    return int(lib().orc_tri_samples(C.c_float(area), C.c_float(amax), int(budget)))


def tri_sample_points(g9, n):
    g, gp = _f32(np.asarray(g9).reshape(9))
    out = np.zeros((n, 3), np.float32)
    lib().orc_tri_sample_points(gp, int(n), out.ctypes.data_as(C.POINTER(C.c_float)))
    return out


# ----------------------------------------------------------------- §11 compact form

def jacobi(S6):
    """Eigenvalues (fp32, unsorted) of the symmetric S given as (xx, yy, zz, xy, xz, yz)."""
    s, sp = _f32(np.asarray(S6).reshape(6))
    lam = np.zeros(3, np.float32)
    lib().orc_jacobi(sp, lam.ctypes.data_as(C.POINTER(C.c_float)))
    return lam


def finalize(acc7):
    """§11 up to the normalised matrix: (Sn (6,) fp32 as xx, yy, zz, xy, xz, yz, flag) with
    flag 1 = jittered, 0 = not, -1 = no SGGX (w = 0)."""
    a, ap = _i64(np.asarray(acc7).reshape(7))
    Sn = np.zeros(6, np.float32)
    f = lib().orc_finalize(ap, Sn.ctypes.data_as(C.POINTER(C.c_float)))
    return Sn, int(f)


def encode(acc):
    """(n,7) int64 (w, M6) records -> ((n,6) uint8 compact SGGX, (n,) uint8 jittered flags)."""
    a, ap = _i64(np.asarray(acc).reshape(-1, 7))
    out = np.zeros((a.shape[0], 6), np.uint8)
    jit = np.zeros(a.shape[0], np.uint8)
    lib().orc_encode(a.shape[0], ap, out.ctypes.data_as(C.POINTER(C.c_uint8)), jit.ctypes.data_as(C.POINTER(C.c_uint8)))
    return out, jit


def decode(b6):
    """Renderer-side decode of compact bytes (n,6) -> (n,3,3) fp64 S with negative eigenvalues
    clamped to 0. Not part of the path; used by the round-trip tests."""
    b = np.asarray(b6, np.float64).reshape(-1, 6)
    sg = b[:, :3] / 255.0
    r = b[:, 3:] / 127.5 - 1.0
    S = np.zeros((len(b), 3, 3))
    for a in range(3):
        S[:, a, a] = sg[:, a] ** 2
    for (i, j), c in zip(((0, 1), (0, 2), (1, 2)), range(3)):
        S[:, i, j] = S[:, j, i] = r[:, c] * sg[:, i] * sg[:, j]
    w, V = np.linalg.eigh(S)
    return np.einsum("nij,nj,nkj->nik", V, np.maximum(w, 0.0), V)


Q = 2.0 ** 32


def acc_from_float(w, m6):
    """Helper for tests: quantise (w, M6) floats to int64 accumulators exactly as §8."""
    v = np.concatenate([[w], m6]).astype(np.float32)
    return np.rint((v * np.float32(Q)).astype(np.float32).astype(np.float64)).astype(np.int64)
