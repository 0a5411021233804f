#!/usr/bin/env python
"""Benchmark of the hot path: voxelize + full LoD build (one "step") on the BASELINE.json
workload, printed as ONE JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...        (N > 1: Morton-range shards)

Workload (default): config 4 -- explicit-fiber knit, ~10M segments at 4096^3, 12 levels
(synthetic, seeded; gen.knit). Inputs are resident in HBM before the timed region; they are
larger than L2 (280 MB > 126 MB), so no L2 flush is needed between steps.
`--impl reference` times the CPU oracle (the reference arm of this tier) on bounded samples.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "fiber segments voxelized/s + full LoD build ms; achieved HBM GB/s vs 8 TB/s"


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "_fallback": True}


class ClockSampler:
    """nvidia-smi SM clocks + throttle reasons sampled every 200 ms during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._p = None

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self._p = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                                        "--format=csv,noheader,nounits", "-lms", "200"],
                                       stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except Exception:
            self._p = None
        return self

    def _read(self):
        for line in self._p.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self._p:
            time.sleep(0.25)
            self._p.terminate()
            try:
                self._p.wait(timeout=2)
            except Exception:
                self._p.kill()

    def summary(self):
        sm = [float(r[1]) for r in self.rows if len(r) > 8 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) > 8 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows if len(r) > 8 for i in range(4) if r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm)}


def _workload(cfg: int, n_segments: int | None, grid_res: int | None = None):
    import gen
    kw = {}
    if n_segments:
        kw["n_segments"] = n_segments
    if grid_res and cfg == 5:
        kw["grid_res"] = grid_res
    c = gen.config(cfg, **kw)
    return c


def _cells_by_count(seg, bbox, N, level):
    """Morton cells at `level` with their segment counts (by segment midpoint), largest first."""
    E = float(np.max(bbox[3:] - bbox[:3]))
    mid = 0.5 * (seg[:, 0].astype(np.float64) + seg[:, 1])
    g = np.floor((mid - bbox[:3]) / E * N).astype(np.int64) >> level
    g = np.clip(g, 0, (N >> level) - 1)
    cells = np.zeros(len(g), np.uint64)
    for b in range(13):
        for a in range(3):
            cells |= ((g[:, a].astype(np.uint64) >> np.uint64(b)) & np.uint64(1)) << np.uint64(3 * b + a)
    u, cnt = np.unique(cells, return_counts=True)
    order = np.argsort(-cnt, kind="stable")
    return u[order], cnt[order]


def _cell_inputs(c, level):
    """Morton cells at `level`, largest first, each with every segment whose box touches it."""
    seg, rad, bbox, N = c["segments"], c["radii"], c["bbox"], c["grid_res"]
    E = float(np.max(bbox[3:] - bbox[:3]))
    lo = np.minimum(seg[:, 0], seg[:, 1]) - rad[:, None]
    hi = np.maximum(seg[:, 0], seg[:, 1]) + rad[:, None]
    cells, _ = _cells_by_count(seg, bbox, N, level)
    import oracle
    for cell in cells:
        i, j, k = oracle.unmorton(int(cell))
        box_lo = np.array([i, j, k], np.float64) * (1 << level) * E / N + bbox[:3] - 2 * E / N
        box_hi = box_lo + ((1 << level) + 4) * E / N
        sel = np.all((hi >= box_lo) & (lo <= box_hi), axis=1)
        yield int(cell), np.ascontiguousarray(seg[sel]), np.ascontiguousarray(rad[sel])


def _oracle_cell(N, bbox, level, cell, s, r, distance, hist_samples):
    """One oracle run (voxelize + LoD inside one Morton cell); returns (segments, seconds,
    digest of every level's keys, accumulators and lobes). Module level: it runs in worker
    processes for the all-cores sample."""
    import hashlib
    sys.path.insert(0, ROOT)
    import oracle
    o = oracle.Oracle(N, bbox, distance=distance, hist_samples=hist_samples)
    o.set_window(level, cell)
    t0 = time.perf_counter()
    o.add_fibers(s, r)
    o.build(level)
    dt = time.perf_counter() - t0
    h = hashlib.sha256()
    for l in range(level + 1):
        L = o.level(l)
        h.update(L["key"].tobytes())
        h.update(L["acc"].tobytes())
        if l > 0:
            h.update(L["cl"].tobytes())
    o.close()
    return len(s), dt, h.hexdigest()


def _oracle_job(a):
    return _oracle_cell(*a)


def _warm(_):
    sys.path.insert(0, ROOT)
    import oracle
    oracle.lib()
    return 0


def oracle_sample(c, target_segments: int, level: int, distance: str = "sigma", hist_samples: int = 5000,
                  threads: int = 1, n_cells: int = 0):
    """Time the oracle (as it stands: plain C, no tuning) on whole Morton cells at `level`,
    largest first: every segment touching a cell is voxelized (its S_p needs all its keys) and
    the LoD is built inside the cell up to `level`. threads == 1: cells one after another until
    `target_segments` segments; threads > 1: the first `n_cells` cells, one oracle per cell on a
    pool of `threads` host threads (wall time). Returns (segments, seconds, description, digests
    per cell)."""
    import concurrent.futures as cf
    done, secs, used, digests = 0, 0.0, [], []
    N, bbox = c["grid_res"], c["bbox"]
    if threads <= 1:
        for cell, s, r in _cell_inputs(c, level):
            n, dt, dg = _oracle_cell(N, bbox, level, cell, s, r, distance, hist_samples)
            done += n
            secs += dt
            used.append(cell)
            digests.append(dg)
            if done >= target_segments:
                break
    else:
        jobs = []
        for cell, s, r in _cell_inputs(c, level):
            jobs.append((cell, s, r))
            if len(jobs) >= n_cells:
                break
        threads = min(threads, len(jobs))
        import multiprocessing as mp
        # one process per host core (the C oracle is single-threaded; processes avoid the
        # allocator contention threads showed); workers are started before the clock
        with cf.ProcessPoolExecutor(threads, mp_context=mp.get_context("spawn")) as ex:
            list(ex.map(_warm, range(threads)))
            t0 = time.perf_counter()
            res = list(ex.map(_oracle_job, [(N, bbox, level, j[0], j[1], j[2], distance, hist_samples)
                                            for j in jobs]))
            secs = time.perf_counter() - t0
        done = sum(x[0] for x in res)
        used = [j[0] for j in jobs]
        digests = [x[2] for x in res]
    desc = (f"oracle (plain C, {threads} host process{'es' if threads > 1 else ''}, {distance} distance) on "
            f"{len(used)} Morton cell(s) at level {level} ({1 << level}^3 voxels each): {done} segments touching "
            f"them voxelized + LoD levels 1..{level} inside them")
    return done, secs, desc, digests


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def _config_of(args, n_prims, N, levels, world, fib=True):
    """The bench line's `config` (shared by both arms, so the driver compares like with like)."""
    return {"workload": f"config {args.config}: " + __import__("gen").CONFIGS[args.config]
                        + (f" [point: {n_prims} segments at {N}^3]" if args.config == 5 else ""),
            "prims": n_prims, "grid_res": N, "levels": levels, "parallelism": f"morton{world}",
            "front_end": (f"sampled ({args.sampled} samples per Catmull-Rom piece)" if fib else
                          f"sampled (budget {args.sampled} per largest triangle)") if args.sampled
            else "exact overlap",
            "sggxh_distance": args.distance if args.distance == "sigma"
            else f"hist (N={args.hist_samples} samples, 5x5x5 bins, sliced W1)",
            "l2": "inputs (28 B x prims) larger than L2; no flush"}


def run_reference(args):
    """--impl reference: the oracle as it stands on the host cores, bounded samples."""
    c = _workload(args.config, args.segments)
    lvl = 7 if c["grid_res"] >= 2048 else max(1, int(math.log2(c["grid_res"])) - 2)
    times, counts, desc = [], [], ""   # each step: one bounded oracle sample, every host core
    ncpu = os.cpu_count() or 1
    thr = 1
    for it in range(args.warmup + args.steps):
        if ncpu > 1:
            n, dt, desc, dg = oracle_sample(c, 0, lvl, threads=ncpu, n_cells=min(ncpu, args.cpu_cells))
            thr = min(ncpu, len(dg))
        else:
            n, dt, desc, _ = oracle_sample(c, args.ref_segments, lvl)
        if it >= args.warmup:
            times.append(dt)
            counts.append(n)
    value = sum(counts) / sum(times)
    # the same `config` as our arm (the workload the value is quoted on); the sample each step
    # actually ran is in cpu_baseline.sample
    world = int(os.environ.get("WORLD_SIZE", "1"))
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "segments/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": _config_of(args, int(c["segments"].shape[0]), c["grid_res"], c["levels"], world),
            "cpu_baseline": {"value": value, "unit": "segments/s", "cores": thr, "kind": "oracle", "sample": desc,
                             "host_cpus": ncpu, "cpu_model": _cpu_model()},
            "e2e": {"value": value, "unit": "segments/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--segments", type=int, default=None, help="override the segment count (config 4/5)")
    ap.add_argument("--grid", type=int, default=None, help="grid resolution of a config-5 sweep point")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--distance", default="sigma", choices=["sigma", "hist"],
                    help="SGGX-H distance: sigma (PREDICATES §9) or the paper's histogram distance (§10)")
    ap.add_argument("--hist-samples", type=int, default=5000, help="N samples per SGGX histogram (P:389)")
    ap.add_argument("--sampled", type=int, default=0,
                    help="N > 0: the paper's sampling front end (PREDICATES §12), N samples per Catmull-Rom "
                         "piece (fibers) or N samples for the largest triangle, instead of exact overlap")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-finalize", action="store_true", help="skip the compact-form (NEXT-3) measurement")
    ap.add_argument("--cpu-segments", type=int, default=200_000, help="oracle sample size, 1 thread (cpu_baseline)")
    ap.add_argument("--cpu-cells", type=int, default=64, help="cells of the all-cores oracle sample (cpu_baseline)")
    ap.add_argument("--ref-segments", type=int, default=40_000, help="oracle sample size per reference step")
    args = ap.parse_args()

    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # one process per GPU: re-launch this command under torchrun with N ranks
        import socket
        sk = socket.socket()
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
        sk.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU")
    if args.impl == "reference":
        if rank == 0:
            run_reference(args)
        return

    import torch
    import torch.distributed as dist

    from paper_2604_13191_b200 import Vox, build as vbuild
    vbuild.build()
    if torch.cuda.device_count() < world:
        sys.exit(f"bench.py: {world} ranks but {torch.cuda.device_count()} visible GPU(s)")
    torch.cuda.set_device(local)
    group = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    c = _workload(args.config, args.segments, args.grid)
    N, levels, bbox = c["grid_res"], c["levels"], c["bbox"]
    fib = c["kind"] == "fiber"
    if fib:
        h_a, h_b = c["segments"], c["radii"]
    else:
        h_a, h_b = c["tris"], c["dirs"]
    if args.sampled and fib:
        import gen as _gen
        h_a = _gen.splines_from_segments(h_a)      # Catmull-Rom controls [S,4,3] of the same fibers
    n_prims = len(h_a)
    d_a = torch.from_numpy(h_a).cuda()
    d_b = torch.from_numpy(h_b).cuda() if h_b is not None else None
    stream = torch.cuda.current_stream()

    def step(profile=False):
        v = Vox(N, bbox, rank=rank, world=world, profile=profile, distance=args.distance,
                hist_samples=args.hist_samples)
        if args.sampled:
            if fib:
                v.sample_splines(d_a, d_b, args.sampled)
            else:
                v.sample_triangles(d_a, d_b, args.sampled)
        elif fib:
            v.voxelize_fibers(d_a, d_b)
        else:
            v.voxelize_triangles(d_a, d_b)
        v.build_lod(levels, group)
        return v

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        step().close()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    # ---------------------------------------------------------------- timed region (device time)
    stage = {}
    counts = {}
    launches = 0
    lodwork = {"sigma": 0, "dist": 0, "hard": 0}
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            v = step(profile=True)
            st = v.stats()
            for k2 in ("ms_bound", "ms_emit", "ms_sort", "ms_reduce", "ms_merge", "ms_lod_scan", "ms_lod",
                       "ms_total_vox", "ms_total_lod", "ms_lod_prep", "ms_sggxh_quad", "ms_sggxh_half",
                       "ms_sggxh_warp"):
                stage[k2] = stage.get(k2, 0.0) + st[k2]
            launches += st["launches"]
            lodwork["sigma"] += st["lod_sigma_evals"]
            lodwork["dist"] += st["lod_dist_evals"]
            lodwork["hard"] += st["lod_hard_parents"]
            counts = {"pairs": st["pairs"], "candidates": st["candidates"], "voxels": st["voxels"]}
            if _ + 1 < args.steps:
                v.close()
        ev1.record(stream)
        torch.cuda.synchronize()
    counts["levels"] = [v.size(l) for l in range(levels + 1)]
    v.close()
    barrier()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    value = n_prims * args.steps / (ms / 1e3)
    for k2 in stage:
        stage[k2] /= args.steps

    # ---------------------------------------------------------------- roofline of the dominant kernel
    peaks = _peaks()
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    sm_mhz = float(peaks.get("sm_max_mhz", 1965.0))
    nsm = torch.cuda.get_device_properties(local).multi_processor_count
    # fp32 lane-op ceiling: SMs x 128 FP32 lanes x clock (no FMA on the pinned path: 1 op per lane-cycle)
    alu_peak_tflops = nsm * 128 * sm_mhz * 1e6 / 1e12
    V = counts["levels"]
    P = counts["pairs"]
    bytes_vox = 28 * n_prims + 32 * P + 36 * V[0]
    bytes_lod = sum((36 * V[0] if l == 1 else 121 * V[l - 1]) + 121 * V[l] for l in range(1, levels + 1))
    sig_ev, dist_ev = lodwork["sigma"] / args.steps, lodwork["dist"] / args.steps
    # SURVEY §8(d) op model: 15 fp32 ops per sigma slice (6 mul, 5 add, max, sqrt counted as 3),
    # 2 per slice of a distance (subtract, accumulate the absolute value); 32 slices
    flops_sggxh = 32 * 15.0 * sig_ev + 32 * 2.0 * dist_ev
    emit_name = ("k_spline_emit" if fib else "k_tris_emit") if args.sampled else ("k_fiber_emit" if fib else "k_tri_emit")
    emit_bytes = (52 * n_prims + 32 * P) if (args.sampled and fib) else (28 * n_prims + 16 * P + 16 * n_prims)
    # emit is issue-bound on the pinned predicate (ALU): its algorithmic bytes are reported, its
    # fraction is not a bandwidth fraction (profiles/ carry the issue-slot utilisation)
    kern = {
        emit_name: (stage["ms_emit"], "alu-issue", emit_bytes),
        "k_bin_count": (stage["ms_sort"], "hbm", 8 * P),
        "k_bin_reduce": (stage["ms_reduce"], "hbm", 16 * P + 16 * n_prims + 64 * V[0]),
        "k_lod_prep": (stage["ms_lod_prep"], "hbm", bytes_lod),
    }
    if args.distance == "hist":
        # PREDICATES §10: ~25 fp32 ops per sample (L u, |v|^2, sqrt, 1/r, 3 x (scale, +1, x2.5)), 4 integer
        # ops per slice step of a distance (sub/add, abs, multiply, add), 32 x 124 steps per distance
        flops_hist = 25.0 * sig_ev * args.hist_samples + 4.0 * 32 * 124 * dist_ev
        kern["k_sggxh_hist"] = (stage["ms_sggxh_warp"], "alu", flops_hist)
    else:
        kern["k_sggxh_quad+half+warp"] = (stage["ms_sggxh_quad"] + stage["ms_sggxh_half"] + stage["ms_sggxh_warp"],
                                          "alu", flops_sggxh)
    dom = max(kern, key=lambda k: kern[k][0])
    def roof_of(name):
        ms_k, bound, work = kern[name]
        dur = ms_k / 1e3
        if bound == "hbm":
            ach = work / dur / 1e9 if dur > 0 else None
            r = {"kernel": name, "bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s",
                 "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy, burst)", "alg_bytes_per_launch": work}
        elif bound == "alu-issue":
            r = {"kernel": name, "bound": "alu", "achieved": None, "peak": None, "unit": "GB/s",
                 "note": "issue-bound on the pinned predicate; algorithmic GB/s given, no lane-op count",
                 "alg_gbs": work / dur / 1e9 if dur > 0 else None, "alg_bytes_per_launch": work}
        else:
            ach = work / dur / 1e12 if dur > 0 else None
            r = {"kernel": name, "bound": "alu", "achieved": ach, "peak": alu_peak_tflops, "unit": "TFLOP/s",
                 "peak_source": f"{nsm} SMs x 128 fp32 lanes x {sm_mhz:.0f} MHz (MEASURED_PEAKS sm_max_mhz; no FMA)",
                 "alg_flops_per_launch": work,
                 "op_model": "SURVEY 8(d): 32 x 15 per sigma evaluation, 32 x 2 per distance evaluation"}
        r["frac"] = (r["achieved"] / r["peak"]) if r["achieved"] and r["peak"] else None
        r["ms_per_launch"] = ms_k
        r["traffic"] = traffic.get(name)
        if r["traffic"] is not None:
            r["traffic_source"] = f"{traffic_src}: dram__bytes_read.sum + dram__bytes_write.sum, all launches of one step"
        return r
    # traffic: DRAM bytes per step of the same kernels from the committed ncu launch list of this
    # workload (profiles/rNN_traffic.json, tools/profile_round.sh); null for other workloads
    groups = {"k_sggxh_quad+half+warp": ["k_sggxh_quad", "k_sggxh_half", "k_sggxh_warp"],
              "k_fiber_emit": ["k_fiber_emit"], "k_bin_count": ["k_bin_count"],
              "k_bin_reduce": ["k_bin_reduce", "k_bin_reduce_warp"],
              "k_lod_prep": ["k_lod_prep", "k_lod_prep_leaf"]}
    traffic, traffic_src = {}, None
    if args.config == 4 and not args.segments and not args.sampled and args.distance == "sigma":
        import glob
        tf = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_traffic.json")))
        if tf:
            tj = json.load(open(tf[-1]))
            traffic_src = os.path.relpath(tf[-1], ROOT)
            for g, ks in groups.items():
                if all(k in tj for k in ks):
                    traffic[g] = sum(tj[k]["dram_bytes"] for k in ks)
    roof = roof_of(dom)
    others = {k: {kk: roof_of(k)[kk] for kk in ("bound", "achieved", "unit", "frac", "ms_per_launch", "traffic")}
              for k in kern}

    line = {"metric": METRIC, "value": value, "unit": "segments/s" if fib else "triangles/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": _config_of(args, n_prims, N, levels, world, fib),
            "lod_ms": stage["ms_total_lod"], "vox_ms": stage["ms_total_vox"],
            "hbm_alg_gbs_full_build": (bytes_vox + bytes_lod) / (ms_step / 1e3) / 1e9,
            "stages_ms": {k2: round(v2, 4) for k2, v2 in stage.items()},
            "counts": {"pairs": P, "candidates": counts["candidates"], "voxels_per_level": V},
            "roofline": roof, "kernels": others, "gpu_launches": launches,
            "sggxh_work": {"sigma_evals": sig_ev, "dist_evals": dist_ev, "hard_parents": lodwork["hard"] / args.steps}}

    # ---------------------------------------------------------------- e2e through the C ABI, host buffers
    if not args.no_e2e and not args.sampled:
        pa = torch.from_numpy(h_a).pin_memory()
        pb = torch.from_numpy(h_b).pin_memory() if h_b is not None else None
        outs = {}
        host = {}

        # high priority: the copy stream's fp32-view kernels (vox_copy_level_async forms mass /
        # m6 / lobes on it right before their D2H) get SMs ahead of the build's blocks, so the
        # copy engine is not left waiting behind them (tools/diag.py e2e: 243 -> 222 ms per step)
        copy_stream = torch.cuda.Stream(priority=-1)

        lt = int(math.log2(N)) - 4 if world > 1 else -1   # the gathered level (top_depth 4)

        def copy_out(v, l):
            """vox_copy_level_async of level l into pinned host buffers; returns its bytes."""
            n_l = v.size(l)
            if l not in host or host[l]["key"].numel() < n_l:
                host[l] = {"key": torch.empty(n_l, dtype=torch.int64).pin_memory(),
                           "mass": torch.empty(n_l, dtype=torch.float32).pin_memory(),
                           "m6": torch.empty(n_l * 6, dtype=torch.float32).pin_memory()}
                if l > 0:
                    host[l]["ncl"] = torch.empty(n_l, dtype=torch.uint8).pin_memory()
                    host[l]["cl"] = torch.empty(n_l * v.k * 7, dtype=torch.float32).pin_memory()
            v.copy_level_async(l, host[l], copy_stream)
            return n_l * (8 + 4 + 24 + ((1 + 28 * v.k) if l > 0 else 0))

        # Consecutive steps are pipelined as a stream of jobs would be: a step's context is
        # released once its D2H has landed, so the next step's H2D, voxelize and build overlap
        # the previous step's trailing copies (one copy stream: copies stay in step order, and
        # every step still moves all of its input and all of its result over PCIe).
        pend = []

        def e2e_release():
            while pend:
                pv, pe = pend.pop(0)
                pe.synchronize()
                pv.close()

        def e2e_step():
            v = Vox(N, bbox, rank=rank, world=world, distance=args.distance, hist_samples=args.hist_samples)
            if fib:
                v.voxelize_fibers_host(pa, pb)
            else:
                v.voxelize_triangles_host(pa, pb)
            # the leaf level (the voxelization itself) first, then level by level;
            # each finished level's D2H runs on a second stream while the next levels are built
            # (vox_copy_level_async: event-ordered, no sync)
            d2h = copy_out(v, 0)
            for l in range(1, levels + 1):
                v.build_lod(l, group)
                if l != lt:          # sharded: level lt is copied once gathered (below)
                    d2h += copy_out(v, l)
            if 0 < lt <= levels:
                d2h += copy_out(v, lt)
            ev = torch.cuda.Event()
            ev.record(copy_stream)
            e2e_release()            # the previous step's copies have had this whole step to land
            pend.append((v, ev))
            outs["d2h"] = d2h

        # warm-up: two overlapped steps, so that the allocation cache already holds two
        # contexts' blocks (the first overlapped step would otherwise grow the device pool)
        e2e_step()
        e2e_step()
        e2e_release()
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            e2e_step()
        last_copy = pend[-1][1]
        e2e_release()
        stream.wait_event(last_copy)   # e1 after the last step's D2H has landed
        e1.record(stream)
        torch.cuda.synchronize()
        ems = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([ems], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        line["e2e"] = {"value": n_prims * args.steps / (ems / 1e3), "unit": line["unit"],
                       "h2d_bytes_per_step": int(h_a.nbytes + (h_b.nbytes if h_b is not None else 0)),
                       "d2h_bytes_per_step": int(outs["d2h"]), "pipelined": True,
                       "wall_s": time.perf_counter() - t0}
    line["clocks"] = clk.summary()

    # ---------------------------------------------------------------- NEXT-3: compact form of every level
    # (not part of the timed step: one extra build, then vox_encode_level on levels 0..L, device time
    # from the library's events)
    if not args.no_finalize:
        v = step(profile=True)
        v.stats_reset()
        bufs = []
        for l in range(levels + 1):
            bufs.append(v.encode_level(l))
        st = v.stats()
        recs = V[0] + sum(V[l] * (1 + v.k) for l in range(1, levels + 1))
        byts = V[0] * (56 + 6 + 6 * v.k + 1) + sum(V[l] * (56 + 1 + 56 * v.k + 6 + 6 * v.k + 1)
                                                    for l in range(1, levels + 1))
        line["finalize"] = {"ms": st["ms_encode"], "records": recs, "records_per_s": recs / (st["ms_encode"] / 1e3),
                            "alg_bytes": byts, "achieved_gbs": byts / (st["ms_encode"] / 1e3) / 1e9,
                            "bound": "alu (pinned Jacobi, 2-3 sweeps of IEEE div/sqrt rotations per record)"}
        # NEXT-2: sub-voxel occupancy and axis densities of every level (same ctx, after the build)
        if fib and not args.sampled:
            v.stats_reset()
            v.density_fibers(d_a, d_b)
            top = levels if world == 1 else min(levels, int(math.log2(N)) - int(v.stats()["top_depth"]))
            dens = [v.density_level(l) for l in range(top + 1)]   # sharded: masks are per shard
            st = v.stats()
            line["density"] = {"ms": st["ms_density"], "host_ms_alloc": st["host_ms_alloc"],
                               "host_ms_sync": st["host_ms_sync"], "leaf_voxels": V[0],
                               "sub_voxel_tests_per_leaf": 512,
                               "leaf_voxels_per_s": V[0] / (st["ms_density"] / 1e3),
                               "bound": "alu (pinned capsule-box predicate on the 8N grid for boundary sub-voxels)"}
            del dens
        v.close()
        del bufs

    # ---------------------------------------------------------------- CPU baseline (oracle), rank 0, N = 1
    # the oracle as it stands, on the box's host cores: one thread on the densest cell(s), then
    # one oracle per cell on every core (ctypes releases the GIL); the cells both runs share
    # must give bit-identical levels
    if rank == 0 and world == 1 and not args.no_cpu_baseline and fib and not args.sampled:
        lvl = 9 if N >= 4096 else max(1, int(math.log2(N)) - 3)
        target = args.cpu_segments if args.distance == "sigma" else max(1000, args.cpu_segments // 100)
        n1, dt1, desc1, dg1 = oracle_sample(c, target, lvl, args.distance, args.hist_samples)
        ncpu = os.cpu_count() or 1
        cb = {"value": n1 / dt1, "unit": "segments/s", "cores": 1, "kind": "oracle", "sample": desc1,
              "seconds": dt1, "host_cpus": ncpu, "cpu_model": _cpu_model()}
        if ncpu > 1 and args.distance == "sigma":
            ncell = max(len(dg1), min(ncpu, args.cpu_cells))
            nm, dtm, descm, dgm = oracle_sample(c, 0, lvl, args.distance, args.hist_samples, threads=ncpu,
                                                n_cells=ncell)
            thr = min(ncpu, len(dgm))
            cb = {"value": nm / dtm, "unit": "segments/s", "cores": thr, "kind": "oracle", "sample": descm,
                  "seconds": dtm, "host_cpus": ncpu, "cpu_model": _cpu_model(),
                  "bit_identical_to_1_thread": dgm[:len(dg1)] == dg1,
                  "one_thread": {"value": n1 / dt1, "cores": 1, "sample": desc1, "seconds": dt1}}
        line["cpu_baseline"] = cb
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
