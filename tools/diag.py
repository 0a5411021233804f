"""Diagnostics on a GPU box (not part of the product or the tests).

    python tools/diag.py stages  [segments]        per-stage device times of config 4 (profile mode)
    python tools/diag.py nhist                     per-level histogram of SGGX-H lobe counts n > K, kernel times
    python tools/diag.py shard   [world ...]       per-rank device time of config-4 Morton shards, one GPU
    python tools/diag.py maxsize [segments] [N]    config 5 point: device time, counts, memory
    python tools/diag.py density [segments]        device time of the sub-voxel density pass (NEXT-2)
    python tools/diag.py overlap [parts]           config 4 as Morton parts on concurrent streams (host threads)
    python tools/diag.py copies  [priority]        e2e step timeline: when each level's D2H starts / ends on the copy stream
    python tools/diag.py e2e     [steps]           e2e loop of config 4, steps synchronised vs pipelined, copy-stream priority 0 / -1
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import gen  # noqa: E402
from paper_2604_13191_b200 import Vox  # noqa: E402


def _dev(c):
    return torch.from_numpy(c["segments"]).cuda(), torch.from_numpy(c["radii"]).cuda()


def stages(n=10_000_000):
    c = gen.config(4, n_segments=int(n))
    S, R = _dev(c)
    acc = {}
    for it in range(5):
        v = Vox(c["grid_res"], c["bbox"], profile=True)
        v.voxelize_fibers(S, R)
        v.build_lod(c["levels"])
        st = v.stats()
        v.close()
        if it >= 2:
            for k, x in st.items():
                if k.startswith("ms_"):
                    acc[k] = acc.get(k, 0) + x / 3
    print({k: round(x, 3) for k, x in acc.items()})


def nhist():
    c = gen.config(4)
    S, R = _dev(c)
    v = Vox(c["grid_res"], c["bbox"], profile=True)
    v.voxelize_fibers(S, R)
    prev = v.level(0)
    for l in range(1, c["levels"] + 1):
        v.stats_reset()
        v.build_lod(l)
        st = v.stats()
        cur = v.level(l)
        pk = prev["key"] >> 3
        lob = prev["ncl"].long() if l > 1 else (prev["acc"][:, 0] > 0).long()
        idx = torch.searchsorted(cur["key"], pk)
        n = torch.zeros(len(cur["key"]), dtype=torch.long, device="cuda").index_add_(0, idx, lob)
        h = torch.bincount(n[n > v.k], minlength=25).cpu().tolist()
        print(l, "parents", len(n), "hard", int((n > v.k).sum()),
              {k: round(st[k], 2) for k in ("ms_lod_scan", "ms_lod_prep", "ms_sggxh_quad", "ms_sggxh_half", "ms_sggxh_warp")},
              {k: x for k, x in enumerate(h) if x}, flush=True)
        prev = cur


def shard(*worlds):
    c = gen.config(4)
    S, R = _dev(c)
    for world in [int(x) for x in (worlds or (1, 2, 4, 8))]:
        worst = 0.0
        for rank in range(world):
            for _ in range(2):
                v = Vox(c["grid_res"], c["bbox"], rank=rank, world=world, profile=True)
                v.voxelize_fibers(S, R)
                v.build_lod(c["levels"])
                st = v.stats()
                v.close()
            t = st["ms_total_vox"] + st["ms_total_lod"]
            worst = max(worst, t)
            print(world, "rank", rank, "cells", st["cell_lo"], st["cell_hi"], "emit", round(st["ms_emit"], 2),
                  "vox", round(st["ms_total_vox"], 2), "lod", round(st["ms_total_lod"], 2), flush=True)
        print(world, "max over ranks", round(worst, 2), "ms", flush=True)


def maxsize(n=15_000_000, N=8192):
    t0 = time.time()
    c = gen.config(5, n_segments=int(n), grid_res=int(N))
    print("generated", len(c["segments"]), "segments in", round(time.time() - t0, 1), "s", flush=True)
    S, R = _dev(c)
    for _ in range(2):
        v = Vox(c["grid_res"], c["bbox"], profile=True)
        v.voxelize_fibers(S, R)
        v.build_lod(c["levels"])
        st = v.stats()
        print({k: round(st[k], 1) for k in ("ms_total_vox", "ms_total_lod")}, "pairs", st["pairs"],
              "cand", st["candidates"], "leaves", st["voxels"],
              "peak GB", round(torch.cuda.max_memory_allocated() / 1e9, 1),
              "free GB", round(torch.cuda.mem_get_info()[0] / 1e9, 1), flush=True)
        v.close()


def density(n=10_000_000):
    c = gen.config(4, n_segments=int(n))
    S, R = _dev(c)
    for _ in range(3):
        v = Vox(c["grid_res"], c["bbox"], profile=True)
        v.voxelize_fibers(S, R)
        v.build_lod(c["levels"])
        v.stats_reset()
        v.density_fibers(S, R)
        for l in range(c["levels"] + 1):
            v.density_level(l)
        st = v.stats()
        print("density ms", round(st["ms_density"], 2), "alloc ms", round(st["host_ms_alloc"], 2), flush=True)
        v.close()


def overlap(parts=2):
    """Wall time of config 4 (voxelize + local levels) as `parts` Morton shards of one GPU, run
    one after the other on one stream vs concurrently (one host thread + stream per shard)."""
    import threading
    parts = int(parts)
    c = gen.config(4)
    S, R = _dev(c)
    Lt = c["levels"] - 4

    def one(rank, world, stream):
        with torch.cuda.stream(stream):
            v = Vox(c["grid_res"], c["bbox"], rank=rank, world=world, stream=stream)
            v.voxelize_fibers(S, R)
            v.build_lod(Lt if world > 1 else c["levels"])
            stream.synchronize()
            v.close()

    streams = [torch.cuda.Stream() for _ in range(parts)]
    for it in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        one(0, 1, streams[0])
        t1 = time.perf_counter()
        for r in range(parts):
            one(r, parts, streams[0])
        t2 = time.perf_counter()
        th = [threading.Thread(target=one, args=(r, parts, streams[r])) for r in range(parts)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        t3 = time.perf_counter()
        print(f"whole {1e3 * (t1 - t0):.1f} ms | {parts} shards sequential {1e3 * (t2 - t1):.1f} ms | "
              f"concurrent {1e3 * (t3 - t2):.1f} ms", flush=True)


def copies(priority=-1):
    """One e2e step of config 4 (host buffers, all 13 levels copied back as bench.py does), with
    events on the main and the copy stream: when each level is built and when its D2H starts and
    lands, in ms from the step's start."""
    c = gen.config(4)
    pa = torch.from_numpy(c["segments"]).pin_memory()
    pb = torch.from_numpy(c["radii"]).pin_memory()
    cs = torch.cuda.Stream(priority=int(priority))
    main = torch.cuda.current_stream()
    host = {}

    def ev(s):
        e = torch.cuda.Event(enable_timing=True)
        e.record(s)
        return e

    for it in range(3):
        marks = []
        t0 = ev(main)
        v = Vox(c["grid_res"], c["bbox"])
        v.voxelize_fibers_host(pa, pb)
        for l in range(0, c["levels"] + 1):
            if l > 0:
                v.build_lod(l)
            n = v.size(l)
            if l not in host:
                host[l] = {"key": torch.empty(n, dtype=torch.int64).pin_memory(),
                           "mass": torch.empty(n, dtype=torch.float32).pin_memory(),
                           "m6": torch.empty(6 * n, dtype=torch.float32).pin_memory()}
                if l > 0:
                    host[l]["ncl"] = torch.empty(n, dtype=torch.uint8).pin_memory()
                    host[l]["cl"] = torch.empty(n * 21, dtype=torch.float32).pin_memory()
            built = ev(main)
            b = ev(cs)
            v.copy_level_async(l, host[l], cs)
            e = ev(cs)
            marks.append((l, n, built, b, e))
        cs.synchronize()
        torch.cuda.synchronize()
        v.close()
        if it == 2:
            for l, n, built, b, e in marks:
                byt = n * (36 + (85 if l > 0 else 0))
                print(f"level {l:2d} n={n:10d} built {t0.elapsed_time(built):7.1f}  d2h queued-after "
                      f"{t0.elapsed_time(b):7.1f} .. landed {t0.elapsed_time(e):7.1f} ms  "
                      f"({byt / 1e9:.2f} GB, {byt / 1e6 / max(b.elapsed_time(e), 1e-3):.1f} GB/s)", flush=True)


def e2e(steps=5):
    c = gen.config(4)
    pa = torch.from_numpy(c["segments"]).pin_memory()
    pb = torch.from_numpy(c["radii"]).pin_memory()
    main = torch.cuda.current_stream()
    host = {}
    L = c["levels"]

    def run(pipelined, prio):
        cs = torch.cuda.Stream(priority=prio)
        pend = []

        def step():
            v = Vox(c["grid_res"], c["bbox"])
            v.voxelize_fibers_host(pa, pb)
            for l in range(0, L + 1):
                if l > 0:
                    v.build_lod(l)
                n = v.size(l)
                if l not in host:
                    host[l] = {"key": torch.empty(n, dtype=torch.int64).pin_memory(),
                               "mass": torch.empty(n, dtype=torch.float32).pin_memory(),
                               "m6": torch.empty(6 * n, dtype=torch.float32).pin_memory()}
                    if l > 0:
                        host[l]["ncl"] = torch.empty(n, dtype=torch.uint8).pin_memory()
                        host[l]["cl"] = torch.empty(n * 21, dtype=torch.float32).pin_memory()
                v.copy_level_async(l, host[l], cs)
            if pipelined:
                e = torch.cuda.Event()
                e.record(cs)
                while pend:
                    pv, pe = pend.pop(0)
                    pe.synchronize()
                    pv.close()
                pend.append((v, e))
            else:
                cs.synchronize()
                v.close()

        step()
        while pend:
            pv, pe = pend.pop(0)
            pe.synchronize()
            pv.close()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(main)
        for _ in range(int(steps)):
            step()
        if pend:
            last = pend[-1][1]
            while pend:
                pv, pe = pend.pop(0)
                pe.synchronize()
                pv.close()
            main.wait_event(last)
        e1.record(main)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / int(steps)
        print(f"pipelined={pipelined} priority={prio}: {ms:.1f} ms/step (events), "
              f"{1e3 * (time.perf_counter() - t0) / int(steps):.1f} ms/step (wall), "
              f"{c['segments'].shape[0] / ms / 1e3:.1f} M segments/s", flush=True)

    for pipelined in (False, True):
        for prio in (0, -1):
            run(pipelined, prio)


if __name__ == "__main__":
    cmd = sys.argv[1] if len(sys.argv) > 1 else "stages"
    globals()[cmd](*sys.argv[2:])
