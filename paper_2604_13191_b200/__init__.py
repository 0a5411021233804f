"""paper_2604_13191_b200 -- B200-native sparse voxelization with SGGX-H level of detail.

Thin Python binding (argument marshalling only) over the C ABI in ``include/vox.h``,
implemented by the sm_100a CUDA library ``libvox.so`` built in-tree by ``build.py``.
Every step of the hot path runs in that library's kernels; PyTorch only supplies device
memory, the CUDA stream and (in :mod:`.dist`) process groups. There is no CPU fallback: if
the library is missing, importing :data:`lib` raises.

Method: "Fast Voxelization and Level of Detail for Microgeometry Rendering" (arXiv
2604.13191); docs/PREDICATES.md pins the arithmetic, DESIGN.md lists the readings.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

__all__ = ["Vox", "VoxError", "lib", "plan_shards", "theta_table", "record_bytes", "STATUS"]

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libvox.so")
# VOX_DEBUG_LIB=1 loads the bounds-checked build libvox_dbg.so (tools/debug_checks.sh builds it)
if os.environ.get("VOX_DEBUG_LIB") == "1":
    LIB_PATH = os.path.join(os.path.dirname(LIB_PATH), "libvox_dbg.so")

STATUS = {0: "VOX_OK", 1: "VOX_ERR_INVALID_ARG", 2: "VOX_ERR_DEGENERATE_BBOX", 3: "VOX_ERR_STATE",
          4: "VOX_ERR_OOM", 5: "VOX_ERR_CAPACITY", 6: "VOX_ERR_CUDA", 7: "VOX_ERR_LEVEL", 8: "VOX_ERR_COMM"}


class VoxError(RuntimeError):
    def __init__(self, status: int, what: str, detail: str = ""):
        self.status = status
        self.name = STATUS.get(status, str(status))
        super().__init__(f"{what}: {self.name}" + (f" ({detail})" if detail else ""))


class _Options(C.Structure):
    _fields_ = [("stream", C.c_void_p), ("rank", C.c_int), ("world", C.c_int), ("top_depth", C.c_int),
                ("k", C.c_uint32), ("n_slices", C.c_uint32), ("max_bytes", C.c_uint64), ("profile", C.c_int),
                ("distance_mode", C.c_int), ("hist_samples", C.c_uint32),
                ("part_candidates", C.c_uint64)]


class _View(C.Structure):
    _fields_ = [("n", C.c_uint64), ("key", C.c_void_p), ("mass", C.c_void_p), ("m6", C.c_void_p),
                ("ncl", C.c_void_p), ("cl", C.c_void_p), ("acc", C.c_void_p)]


class _Stats(C.Structure):
    _fields_ = [("segments", C.c_uint64), ("candidates", C.c_uint64), ("pairs", C.c_uint64),
                ("voxels", C.c_uint64), ("top_depth", C.c_uint32), ("cell_lo", C.c_uint64), ("cell_hi", C.c_uint64),
                ("ms_bound", C.c_double), ("ms_emit", C.c_double), ("ms_sort", C.c_double),
                ("ms_reduce", C.c_double), ("ms_merge", C.c_double), ("ms_lod_scan", C.c_double),
                ("ms_lod", C.c_double), ("ms_total_vox", C.c_double), ("ms_total_lod", C.c_double),
                ("ms_lod_prep", C.c_double), ("ms_sggxh_quad", C.c_double),
                ("ms_sggxh_half", C.c_double), ("ms_sggxh_warp", C.c_double),
                ("launches", C.c_uint64), ("lod_sigma_evals", C.c_uint64), ("lod_dist_evals", C.c_uint64),
                ("lod_hard_parents", C.c_uint64), ("host_ms_alloc", C.c_double), ("host_ms_sync", C.c_double),
                ("ms_encode", C.c_double), ("ms_density", C.c_double)]


_lib = None


def lib():
    """Load libvox.so (fails loudly if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: build it with `python -m paper_2604_13191_b200.build` "
                           "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp, u64, u32, i32 = C.c_void_p, C.c_uint64, C.c_uint32, C.c_int
    L.vox_create.argtypes = [C.POINTER(vp), u32, C.POINTER(C.c_float), C.POINTER(_Options)]
    for name in ("vox_voxelize_fibers", "vox_voxelize_triangles", "vox_voxelize_fibers_host",
                 "vox_voxelize_triangles_host"):
        getattr(L, name).argtypes = [vp, vp, vp, u64]
    L.vox_build_lod.argtypes = [vp, u32]
    L.vox_built_levels.argtypes = [vp, C.POINTER(u32)]
    L.vox_level_size.argtypes = [vp, u32, C.POINTER(u64)]
    L.vox_debug_flags.argtypes = [C.POINTER(u32)]
    L.vox_read_level.argtypes = [vp, u32, C.POINTER(_View)]
    L.vox_copy_level.argtypes = [vp, u32, vp, vp, vp, vp, vp]
    L.vox_copy_level_acc.argtypes = [vp, u32, vp]
    L.vox_copy_level_async.argtypes = [vp, u32, vp, vp, vp, vp, vp, vp]
    L.vox_encode_level.argtypes = [vp, u32, vp, vp, vp]
    L.vox_sample_splines.argtypes = [vp, vp, vp, u64, u32]
    L.vox_density_fibers.argtypes = [vp, vp, vp, u64]
    L.vox_density_triangles.argtypes = [vp, vp, u64]
    L.vox_density_level.argtypes = [vp, u32, vp, vp, vp]
    L.vox_sample_triangles.argtypes = [vp, vp, vp, u64, u32]
    L.vox_export_level.argtypes = [vp, u32, vp, C.POINTER(u64)]
    L.vox_import_level.argtypes = [vp, u32, vp, u64]
    L.vox_plan_shards.argtypes = [C.POINTER(u64), u64, i32, C.POINTER(u64)]
    L.vox_theta_table.argtypes = [C.POINTER(C.c_float), C.POINTER(C.c_float)]
    L.vox_hist_tables.argtypes = [u32, vp, vp, vp]
    L.vox_stats_get.argtypes = [vp, C.POINTER(_Stats)]
    L.vox_stats_reset.argtypes = [vp]
    L.vox_sync.argtypes = [vp]
    L.vox_trim.argtypes = [vp]
    L.vox_status_str.restype = C.c_char_p
    L.vox_status_str.argtypes = [i32]
    L.vox_last_error.restype = C.c_char_p
    L.vox_last_error.argtypes = [vp]
    L.vox_destroy.argtypes = [vp]
    for name in ("vox_create", "vox_voxelize_fibers", "vox_voxelize_triangles", "vox_voxelize_fibers_host",
                 "vox_voxelize_triangles_host", "vox_build_lod", "vox_built_levels", "vox_level_size", "vox_debug_flags", "vox_read_level",
                 "vox_copy_level", "vox_copy_level_acc", "vox_copy_level_async", "vox_encode_level", "vox_sample_splines",
                 "vox_sample_triangles", "vox_density_fibers", "vox_density_triangles", "vox_density_level", "vox_export_level", "vox_import_level", "vox_plan_shards", "vox_theta_table",
                 "vox_hist_tables", "vox_stats_get", "vox_stats_reset", "vox_sync", "vox_trim"):
        getattr(L, name).restype = i32
    _lib = L
    return L


def record_bytes(k: int = 3) -> int:
    """Bytes of one exported level record (include/vox.h): key, acc[7], ncl, lobes[k][7]."""
    return 72 + 56 * int(k)


def plan_shards(weights, world: int) -> np.ndarray:
    """Host-only work-balanced Morton-range partition of the top cells (vox_plan_shards)."""
    w = np.ascontiguousarray(np.asarray(weights, dtype=np.uint64))
    b = np.zeros(world + 1, np.uint64)
    st = lib().vox_plan_shards(w.ctypes.data_as(C.POINTER(C.c_uint64)), w.size, int(world),
                               b.ctypes.data_as(C.POINTER(C.c_uint64)))
    if st:
        raise VoxError(st, "vox_plan_shards")
    return b


def theta_table():
    """The library's SGGX-H slice table (theta [32,3], coef [32,6])."""
    t = np.zeros((32, 3), np.float32)
    c = np.zeros((32, 6), np.float32)
    lib().vox_theta_table(t.ctypes.data_as(C.POINTER(C.c_float)), c.ctypes.data_as(C.POINTER(C.c_float)))
    return t, c


def hist_tables(n: int = 5000):
    """The library's histogram-distance tables (PREDICATES §10): u [3, n] (SoA sample table),
    perm [124, 32] and gap [124, 32] (transposed slice tables)."""
    u = np.zeros((3, n), np.float32)
    perm = np.zeros((124, 32), np.uint8)
    gap = np.zeros((124, 32), np.uint32)
    rc = lib().vox_hist_tables(int(n), C.c_void_p(u.ctypes.data), C.c_void_p(perm.ctypes.data),
                               C.c_void_p(gap.ctypes.data))
    if rc != 0:
        raise VoxError(rc, "vox_hist_tables")
    return u, perm, gap


def _dev_f32(t, name, shape_tail):
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA torch tensor (use the *_host methods for host arrays)")
    if t.dtype != torch.float32 or not t.is_contiguous():
        raise TypeError(f"{name} must be contiguous float32")
    if tuple(t.shape[1:]) != tuple(shape_tail):
        raise ValueError(f"{name} must have shape [n, {', '.join(map(str, shape_tail))}], got {tuple(t.shape)}")
    return t


class Vox:
    """One voxelization context (vox_ctx): an N^3 grid over the cubic extent of ``bbox``.

    >>> v = Vox(4096, bbox)                       # bbox = (xmin, ymin, zmin, xmax, ymax, zmax)
    >>> v.voxelize_fibers(segments, radii)        # cuda f32 [S,2,3], [S]
    >>> v.build_lod(12)
    >>> lv = v.level(3)                           # dict of cuda tensors
    """

    def __init__(self, grid_res: int, bbox, k: int = 3, rank: int = 0, world: int = 1, top_depth: int = 0,
                 max_bytes: int = 0, profile: bool = False, stream=None, distance: str = "sigma",
                 hist_samples: int = 5000, part_candidates: int = 0):
        import torch
        self.grid_res = int(grid_res)
        self.k = int(k)
        self.world = int(world)
        self.rank = int(rank)
        if stream is None:
            stream = torch.cuda.current_stream()
        self.stream = stream
        bb = (C.c_float * 6)(*[float(x) for x in np.asarray(bbox, np.float32).reshape(6)])
        if distance not in ("sigma", "hist"):
            raise ValueError(f"distance must be 'sigma' or 'hist', not {distance!r}")
        self.distance = distance
        opt = _Options(C.c_void_p(stream.cuda_stream), int(rank), int(world), int(top_depth), int(k), 32,
                       int(max_bytes), int(bool(profile)), 1 if distance == "hist" else 0, int(hist_samples),
                       int(part_candidates))
        h = C.c_void_p()
        st = lib().vox_create(C.byref(h), self.grid_res, bb, C.byref(opt))
        if st:
            raise VoxError(st, "vox_create")
        self._h = h
        self.levels_total = int(np.log2(self.grid_res))

    # ------------------------------------------------------------------ helpers
    def _check(self, st, what):
        if st:
            detail = lib().vox_last_error(self._h)
            raise VoxError(st, what, detail.decode() if detail else "")

    def close(self):
        if getattr(self, "_h", None):
            lib().vox_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------------ voxelize
    def voxelize_fibers(self, segments, radii):
        """segments: cuda f32 [S,2,3] world endpoints; radii: cuda f32 [S] (PREDICATES §4-§5)."""
        s = _dev_f32(segments.reshape(-1, 6), "segments", (6,))
        r = _dev_f32(radii.reshape(-1, 1), "radii", (1,))
        if s.shape[0] != r.shape[0]:
            raise ValueError("segments and radii differ in length")
        self._check(lib().vox_voxelize_fibers(self._h, s.data_ptr(), r.data_ptr(), s.shape[0]), "voxelize_fibers")

    def voxelize_triangles(self, tris, dirs=None):
        """tris: cuda f32 [T,3,3]; dirs: cuda f32 [T,3] or None for face normals (PREDICATES §6-§7)."""
        t = _dev_f32(tris.reshape(-1, 9), "tris", (9,))
        dp = 0
        if dirs is not None:
            d = _dev_f32(dirs.reshape(-1, 3), "dirs", (3,))
            if d.shape[0] != t.shape[0]:
                raise ValueError("tris and dirs differ in length")
            dp = d.data_ptr()
        self._check(lib().vox_voxelize_triangles(self._h, t.data_ptr(), dp, t.shape[0]), "voxelize_triangles")

    def voxelize_fibers_host(self, segments, radii):
        """Host (ideally pinned) arrays; the H2D copies run inside the library call."""
        s = _host_f32(segments, 6)
        r = _host_f32(radii, 1)
        self._check(lib().vox_voxelize_fibers_host(self._h, _hptr(s), _hptr(r), _hlen(s, 6)), "voxelize_fibers_host")

    def voxelize_triangles_host(self, tris, dirs=None):
        t = _host_f32(tris, 9)
        d = _host_f32(dirs, 3) if dirs is not None else None
        self._check(lib().vox_voxelize_triangles_host(self._h, _hptr(t), _hptr(d) if d is not None else 0,
                                                      _hlen(t, 9)), "voxelize_triangles_host")

    # ------------------------------------------------------------------ LoD
    def build_lod(self, levels: int, group=None):
        """Build levels 1..levels. With world > 1 and a process group,
        gathers level log2(N)-T across ranks (paper_2604_13191_b200.dist) and builds the top
        levels redundantly."""
        self._check(lib().vox_build_lod(self._h, int(levels)), "build_lod")
        if self.world > 1 and self.built_levels() < levels and _dist_ready(group):
            from . import dist
            dist.gather_top(self, group)
            self._check(lib().vox_build_lod(self._h, int(levels)), "build_lod")

    def built_levels(self) -> int:
        out = C.c_uint32()
        self._check(lib().vox_built_levels(self._h, C.byref(out)), "built_levels")
        return out.value

    def size(self, level: int) -> int:
        """vox_level_size: voxels of a built level (no device work)."""
        out = C.c_uint64()
        self._check(lib().vox_level_size(self._h, int(level), C.byref(out)), "level_size")
        return out.value

    def view(self, level: int) -> dict:
        """Borrowed device pointers of a level (valid until the next mutating call)."""
        v = _View()
        self._check(lib().vox_read_level(self._h, int(level), C.byref(v)), "read_level")
        return {f: getattr(v, f) for f, _ in _View._fields_}

    def level(self, level: int, device: str = "cuda") -> dict:
        """Copies of a level as torch tensors: key int64 [n], mass f32 [n], m6 f32 [n,6],
        ncl uint8 [n], cl f32 [n,k,7], acc int64 [n,7] (exact accumulators)."""
        import torch
        n = self.size(level)
        dev = torch.device(device)
        out = dict(key=torch.empty(n, dtype=torch.int64, device=dev),
                   mass=torch.empty(n, dtype=torch.float32, device=dev),
                   m6=torch.empty((n, 6), dtype=torch.float32, device=dev),
                   ncl=torch.empty(n, dtype=torch.uint8, device=dev),
                   cl=torch.empty((n, self.k, 7), dtype=torch.float32, device=dev),
                   acc=torch.empty((n, 7), dtype=torch.int64, device=dev))
        if n == 0:
            return out
        self._check(lib().vox_copy_level(self._h, int(level), out["key"].data_ptr(), out["mass"].data_ptr(),
                                         out["m6"].data_ptr(), out["ncl"].data_ptr(), out["cl"].data_ptr()),
                    "copy_level")
        self._check(lib().vox_copy_level_acc(self._h, int(level), out["acc"].data_ptr()), "copy_level_acc")
        return out

    def copy_level_to(self, level: int, out: dict):
        """vox_copy_level into caller tensors (device or pinned host): keys key/mass/m6/ncl/cl,
        each optional, each at least as large as the level."""
        ptr = lambda k: out[k].data_ptr() if k in out and out[k] is not None else None
        self._check(lib().vox_copy_level(self._h, int(level), ptr("key"), ptr("mass"), ptr("m6"), ptr("ncl"),
                                         ptr("cl")), "copy_level")

    def sample_splines(self, ctrl, radii, n: int):
        """vox_sample_splines (PREDICATES §12): Catmull-Rom pieces ctrl [S,4,3] and radii [S]
        (cuda float32), n samples per piece."""
        c = _dev_f32(ctrl, "ctrl", (4, 3))
        r = _dev_f32(radii, "radii", ())
        if r.shape[0] != c.shape[0]:
            raise ValueError("ctrl and radii disagree on S")
        self._check(lib().vox_sample_splines(self._h, c.data_ptr(), r.data_ptr(), c.shape[0], int(n)),
                    "sample_splines")

    def sample_triangles(self, tris, dirs=None, budget: int = 64):
        """vox_sample_triangles (PREDICATES §12): tris [T,3,3] (+ dirs [T,3]) cuda float32,
        `budget` samples for the largest triangle."""
        t = _dev_f32(tris, "tris", (3, 3))
        d = None if dirs is None else _dev_f32(dirs, "dirs", (3,))
        self._check(lib().vox_sample_triangles(self._h, t.data_ptr(), None if d is None else d.data_ptr(),
                                               t.shape[0], int(budget)), "sample_triangles")

    def density_fibers(self, segments, radii):
        """vox_density_fibers (PREDICATES §13): OR the sub-voxel hits of fiber segments into the
        level-0 masks (after the last voxelize call)."""
        s = _dev_f32(segments, "segments", (2, 3))
        r = _dev_f32(radii, "radii", ())
        self._check(lib().vox_density_fibers(self._h, s.data_ptr(), r.data_ptr(), s.shape[0]), "density_fibers")

    def density_triangles(self, tris):
        t = _dev_f32(tris, "tris", (3, 3))
        self._check(lib().vox_density_triangles(self._h, t.data_ptr(), t.shape[0]), "density_triangles")

    def density_level(self, level: int, masks: bool = False) -> dict:
        """vox_density_level: occupancy [n] and axis densities [n,3] (YZ, XZ, XY) as cuda
        tensors, plus the 512-bit masks [n,8] (int64 bit patterns) when masks=True."""
        import torch
        n = self.size(level)
        out = {"occ": torch.empty(max(n, 1), dtype=torch.float32, device="cuda"),
               "axis": torch.empty((max(n, 1), 3), dtype=torch.float32, device="cuda")}
        if masks:
            out["mask"] = torch.empty((max(n, 1), 8), dtype=torch.int64, device="cuda")
        self._check(lib().vox_density_level(self._h, int(level), out["occ"].data_ptr(), out["axis"].data_ptr(),
                                            out["mask"].data_ptr() if masks else None), "density_level")
        return {k: t[:n] for k, t in out.items()}

    def encode_level(self, level: int, lobes: bool = True, flags: bool = True) -> dict:
        """vox_encode_level (PREDICATES §11): the 6-byte compact SGGX of every voxel
        (sggx6 uint8 [n,6]) and, optionally, of its lobes (cl6 uint8 [n,k,6]) and the jitter
        flags (uint8 [n]) as cuda tensors."""
        import torch
        n = self.size(level)
        out = {"sggx6": torch.empty((max(n, 1), 6), dtype=torch.uint8, device="cuda")}
        if lobes:
            out["cl6"] = torch.empty((max(n, 1), self.k, 6), dtype=torch.uint8, device="cuda")
        if flags:
            out["flags"] = torch.empty(max(n, 1), dtype=torch.uint8, device="cuda")
        ptr = lambda k: out[k].data_ptr() if k in out else None
        self._check(lib().vox_encode_level(self._h, int(level), ptr("sggx6"), ptr("cl6"), ptr("flags")),
                    "encode_level")
        return {k: t[:n] for k, t in out.items()}

    def copy_level_async(self, level: int, out: dict, stream):
        """vox_copy_level_async: enqueue the copy of a level into caller tensors (pinned host or
        device; keys key/mass/m6/ncl/cl, each optional) on `stream` (torch.cuda.Stream), ordered
        after the ctx's work so far; no synchronisation."""
        ptr = lambda k: out[k].data_ptr() if k in out and out[k] is not None else None
        self._check(lib().vox_copy_level_async(self._h, int(level), ptr("key"), ptr("mass"), ptr("m6"),
                                               ptr("ncl"), ptr("cl"), C.c_void_p(stream.cuda_stream)),
                    "copy_level_async")

    # ------------------------------------------------------------------ multi-GPU records
    def export_level(self, level: int):
        """This rank's records of `level` as a cuda uint8 tensor (include/vox.h layout)."""
        import torch
        nb = C.c_uint64(0)
        self._check(lib().vox_export_level(self._h, int(level), None, C.byref(nb)), "export_level")
        buf = torch.empty(max(int(nb.value), 1), dtype=torch.uint8, device="cuda")
        if nb.value:
            self._check(lib().vox_export_level(self._h, int(level), buf.data_ptr(), C.byref(nb)), "export_level")
        return buf[: int(nb.value)]

    def import_level(self, level: int, buf):
        """Replace `level` with the concatenated records of all ranks (cuda uint8 tensor)."""
        ptr = buf.data_ptr() if buf.numel() else None
        self._check(lib().vox_import_level(self._h, int(level), ptr, int(buf.numel())), "import_level")

    # ------------------------------------------------------------------ misc
    def stats(self) -> dict:
        s = _Stats()
        self._check(lib().vox_stats_get(self._h, C.byref(s)), "stats")
        return {f: getattr(s, f) for f, _ in _Stats._fields_}

    def stats_reset(self):
        self._check(lib().vox_stats_reset(self._h), "stats_reset")

    def sync(self):
        self._check(lib().vox_sync(self._h), "sync")

    def trim(self):
        """Release the library's cached device blocks of this stream."""
        self._check(lib().vox_trim(self._h), "trim")


def _dist_ready(group) -> bool:
    """The top-level gather runs when a process group exists; without one (e.g. a fake world
    of shards on one device) build_lod stops at level log2(N) - T and the caller exchanges
    export_level / import_level itself."""
    if group is not None:
        return True
    import torch.distributed as dist
    return dist.is_available() and dist.is_initialized()


def _host_f32(a, width):
    import torch
    if isinstance(a, torch.Tensor):
        if a.is_cuda or a.dtype != torch.float32 or not a.is_contiguous():
            raise TypeError("host arrays must be contiguous float32 CPU tensors or numpy arrays")
        return a
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float32).reshape(-1, width))
    return a


def _hptr(a):
    import torch
    return a.data_ptr() if isinstance(a, torch.Tensor) else a.ctypes.data


def _hlen(a, width):
    return (a.numel() if hasattr(a, "numel") else a.size) // width
