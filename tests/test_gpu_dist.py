"""Multi-process runs of the sharded path, compared with the oracle.

* world 2 and 3, one process per rank, all on cuda:0, process group over gloo (the box has one
  GPU; the ranks' kernels never wait on one another -- the one exchange, the all-gather of the
  level log2(N) - T records, is staged through host memory by `dist.gather_varlen`). Each rank
  runs `Vox.build_lod(L, group)` end to end: local levels, `dist.gather_top`, import, the
  redundant top levels. The union of the ranks' local levels and every rank's top levels must
  equal the oracle's levels bit for bit.
* world 1 over NCCL: the device path of `gather_varlen` (`all_gather_into_tensor`) and
  `gather_top` (export -> gather -> import -> rebuild of the top levels) leave the levels
  unchanged.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import gen
import oracle

pytestmark = pytest.mark.gpu

N, L = 128, 7
BBOX = [0, 0, 0, 1, 1, 1]
FIELDS = ("key", "acc", "mass", "m6", "ncl", "cl")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _weave():
    return gen.plain_weave(n_warp=16, n_weft=16, n_seg=64, pitch=1 / 16)


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_2604_13191_b200 as P
        s, r = _weave()
        v = P.Vox(N, BBOX, rank=rank, world=world)
        v.voxelize_fibers(torch.from_numpy(s).cuda(), torch.from_numpy(r).cuda())
        v.build_lod(L, dist.group.WORLD)
        st = v.stats()
        out = {l: {k: t.cpu().numpy() for k, t in v.level(l).items()} for l in range(L + 1)}
        q.put((rank, int(st["cell_lo"]), int(st["cell_hi"]), int(st["top_depth"]), out, None))
        dist.destroy_process_group()
    except Exception as e:   # reported to the parent, which fails the test
        import traceback
        q.put((rank, 0, 0, 0, None, traceback.format_exc()))


def _spawn(world, target):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, *_, err in res:
        assert err is None, f"rank {rank} failed:\n{err}"
    for p in procs:
        assert p.exitcode == 0
    return sorted(res, key=lambda x: x[0])


def _same(got, ref, l, tag):
    assert np.array_equal(got["key"].astype(np.uint64), ref["key"]), f"{tag} level {l} keys"
    assert np.array_equal(got["acc"], ref["acc"]), f"{tag} level {l} acc"
    assert np.array_equal(got["mass"], ref["mass"]) and np.array_equal(got["m6"], ref["m6"]), f"{tag} level {l} fp32"
    if l > 0:
        assert np.array_equal(got["ncl"], ref["ncl"]), f"{tag} level {l} ncl"
        assert np.array_equal(got["cl"], ref["cl"]), f"{tag} level {l} lobes"


@pytest.mark.parametrize("world", [2, 3])
def test_multiprocess_shards_equal_oracle(world):
    from paper_2604_13191_b200 import build
    build.build()
    res = _spawn(world, _worker)
    s, r = _weave()
    o = oracle.Oracle(N, np.array(BBOX, np.float32))
    o.add_fibers(s, r)
    o.build(L)
    T = res[0][3]
    lt = L - T
    # the plan: disjoint, ordered top-cell ranges covering [0, 8^T)
    assert res[0][1] == 0 and res[-1][2] == 8 ** T
    assert all(res[q][2] == res[q + 1][1] for q in range(world - 1))
    for l in range(L + 1):
        ref = o.level(l)
        if l < lt:   # local levels: each rank holds exactly its cells' voxels, the union is the oracle's
            shift = 3 * (lt - l)
            for rank, lo, hi, _, out, _ in res:
                cells = out[l]["key"].astype(np.uint64) >> np.uint64(shift)
                assert np.all((cells >= lo) & (cells < hi)), (rank, l)
            got = {k: np.concatenate([x[4][l][k] for x in res]) for k in FIELDS}
            _same(got, ref, l, f"world {world} union")
        else:        # gathered level and the top levels: identical on every rank
            for rank, *_, out, _ in res:
                _same(out[l], ref, l, f"world {world} rank {rank}")


def _nccl_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        torch.cuda.set_device(0)
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
        import paper_2604_13191_b200 as P
        from paper_2604_13191_b200 import dist as vdist
        buf = torch.arange(1000, device="cuda", dtype=torch.int64).to(torch.uint8)
        ok_gather = bool(torch.equal(vdist.gather_varlen(buf), buf))
        s, r = _weave()
        v = P.Vox(N, BBOX)
        v.voxelize_fibers(torch.from_numpy(s).cuda(), torch.from_numpy(r).cuda())
        v.build_lod(L)
        before = {l: {k: t.cpu().numpy() for k, t in v.level(l).items()} for l in range(L + 1)}
        lt = vdist.gather_top(v)     # export -> all_gather_into_tensor -> import (replaces levels >= lt)
        v.build_lod(L)
        after = {l: {k: t.cpu().numpy() for k, t in v.level(l).items()} for l in range(L + 1)}
        q.put((rank, lt, ok_gather, before, after, None))
        dist.destroy_process_group()
    except Exception:
        import traceback
        q.put((rank, 0, False, None, None, traceback.format_exc()))


def test_nccl_world1_gather_top():
    from paper_2604_13191_b200 import build
    build.build()
    (_, lt, ok_gather, before, after, _), = _spawn(1, _nccl_worker)
    assert ok_gather
    assert lt == L - 4
    for l in range(L + 1):
        _same(after[l], {k: (v.astype(np.uint64) if k == "key" else v) for k, v in before[l].items()}, l, "nccl")
