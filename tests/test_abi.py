"""CPU-side checks of the C ABI: the library loads, exports every symbol include/vox.h
declares, and its host-only entry points behave (no GPU needed)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def P():
    from paper_2604_13191_b200 import build
    build.build()
    import paper_2604_13191_b200 as P
    P.lib()
    return P


def test_exports_every_declared_symbol(P):
    hdr = open(os.path.join(ROOT, "include", "vox.h")).read()
    names = set(re.findall(r"^(?:vox_status|const char\*|void)\s+(vox_\w+)\s*\(", hdr, re.M))
    assert len(names) >= 20
    L = C.CDLL(P.LIB_PATH)
    for n in sorted(names):
        assert hasattr(L, n), n


def test_hist_tables_bit_identical_to_oracle(P):
    for n in (32, 5000, 8160):
        u1, perm1, gap1 = P.hist_tables(n)
        assert np.array_equal(u1.T.view(np.uint32), oracle.sample_table(n).view(np.uint32))
    perm2, gap2 = oracle.sw_tables()
    assert np.array_equal(perm1.T, perm2[:, :124])
    assert np.array_equal(gap1.T.astype(np.int64), gap2)
    with pytest.raises(P.VoxError):
        P.hist_tables(31)


def test_theta_table_bit_identical_to_oracle(P):
    t1, c1 = P.theta_table()
    t2, c2 = oracle.theta()
    assert t1.tobytes() == t2.tobytes() and c1.tobytes() == c2.tobytes()


def test_create_validation_without_gpu(P):
    L = P.lib()
    h = C.c_void_p()
    bb = (C.c_float * 6)(0, 0, 0, 1, 1, 1)
    assert L.vox_create(C.byref(h), 100, bb, None) == 1          # not a power of two
    assert L.vox_create(C.byref(h), 16384, bb, None) == 1        # > 8192
    bad = (C.c_float * 6)(0, 0, 0, 1, 0, 1)
    assert L.vox_create(C.byref(h), 64, bad, None) == 2          # degenerate bbox
    nan = (C.c_float * 6)(0, 0, float("nan"), 1, 1, 1)
    assert L.vox_create(C.byref(h), 64, nan, None) == 2
    opt = P._Options(None, 2, 2, 0, 3, 32, 0, 0)                 # rank >= world
    assert L.vox_create(C.byref(h), 64, bb, C.byref(opt)) == 1
    opt = P._Options(None, 0, 1, 0, 9, 32, 0, 0)                 # k > 8
    assert L.vox_create(C.byref(h), 64, bb, C.byref(opt)) == 1
    opt = P._Options(None, 0, 1, 0, 3, 16, 0, 0)                 # only 32 slices
    assert L.vox_create(C.byref(h), 64, bb, C.byref(opt)) == 1
    opt = P._Options(None, 0, 1, 0, 3, 32, 0, 0, 0, 0, (3 << 30) + 1)   # part_candidates > 3*2^30
    assert L.vox_create(C.byref(h), 64, bb, C.byref(opt)) == 1
    opt = P._Options(None, 0, 1, 0, 3, 32, 0, 0, 0, 0, 1)       # one top cell per part: allowed
    assert L.vox_create(C.byref(h), 64, bb, C.byref(opt)) == 0
    L.vox_destroy(h)
    assert L.vox_create(C.byref(h), 64, bb, None) == 0           # no device work at create
    L.vox_destroy(h)
    assert P.lib().vox_status_str(5) == b"VOX_ERR_CAPACITY"


def test_plan_shards_properties(P):
    rng = np.random.default_rng(0)
    for world in (1, 2, 3, 8):
        w = rng.integers(0, 1000, 4096).astype(np.uint64)
        w[rng.random(4096) < 0.7] = 0
        b = P.plan_shards(w, world)
        assert b[0] == 0 and b[-1] == 4096 and np.all(np.diff(b.astype(np.int64)) >= 0)
        loads = [int(w[b[r]:b[r + 1]].sum()) for r in range(world)]
        assert sum(loads) == int(w.sum())
        assert max(loads) <= w.sum() / world + w.max() + 1          # balanced up to one cell
        assert np.array_equal(b, P.plan_shards(w, world))           # deterministic
    b = P.plan_shards(np.zeros(64, np.uint64), 4)
    assert list(b) == [0, 16, 32, 48, 64]


def test_release_debug_flags_zero(P):
    # the bounds checks exist only in the -DVOX_DEBUG build; the release library reports none
    f = C.c_uint32(7)
    assert P.lib().vox_debug_flags(C.byref(f)) == 0 and f.value == 0


def test_no_contracted_packed_fma_in_sass(P):
    """The pinned sequences forbid FMA contraction (-fmad=false). ptxas contracts packed
    mul.f32x2 + add.f32x2 into FFMA2 even then, so the shipped SASS must hold no
    FFMA2 at all."""
    import shutil
    import subprocess
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump not available")
    sass = subprocess.run([exe, "-sass", P.LIB_PATH], capture_output=True, text=True).stdout
    assert "Function :" in sass
    assert "FFMA2" not in sass
