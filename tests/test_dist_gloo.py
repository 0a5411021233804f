"""World-size-2 tests of the multi-GPU host logic on CPU (gloo): the variable-length gather
used for the top-level exchange, and that every rank derives the identical shard plan."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2604_13191_b200 import dist as vdist
        import paper_2604_13191_b200 as P
        # variable-length byte buffers (rank r sends r*5+3 bytes, one rank may send none)
        n = 0 if (rank == 1 and world > 2) else rank * 5 + 3
        buf = torch.arange(n, dtype=torch.int64).add(100 * rank).to(torch.uint8)
        out = vdist.gather_varlen(buf)
        # identical plan on every rank from the (replicated) per-cell candidate counts
        rng = np.random.default_rng(42)
        w = rng.integers(0, 50, 512).astype(np.uint64)
        b = P.plan_shards(w, world)
        bt = torch.from_numpy(b.astype(np.int64))
        allb = [torch.zeros_like(bt) for _ in range(world)]
        dist.all_gather(allb, bt)
        # synthetic sorted records: each rank owns keys of its cell range -> the rank-order
        # concatenation must be globally sorted
        keys = torch.arange(int(b[rank]), int(b[rank + 1]), dtype=torch.int64)
        kb = keys.view(torch.uint8)
        allk = vdist.gather_varlen(kb).view(torch.int64)
        q.put((rank, out.tolist(), [x.tolist() for x in allb], allk.tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_gather_and_plan(world):
    from paper_2604_13191_b200 import build
    build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = []
    for r in range(world):
        n = 0 if (r == 1 and world > 2) else r * 5 + 3
        want += [(i + 100 * r) % 256 for i in range(n)]
    for rank, out, allb, allk in res:
        assert out == want
        assert all(b == allb[0] for b in allb)               # same plan everywhere
        assert allk == list(range(allb[0][-1]))              # rank-order concat = sorted cells
