"""Multi-GPU plumbing: Morton-range shards, one process per GPU.

Every rank holds all primitives and emits only the keys of its own top cells (the plan is
computed identically on every rank from the per-cell candidate counts, no communication).
Leaf and local levels (<= log2(N) - T) are independent per rank. The one exchange step is
here: the records of level log2(N) - T are all-gathered (NCCL over NVLink on GPUs, gloo on
CPU tests) and imported, after which every rank builds the top T levels redundantly and
bit-identically.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def gather_varlen(buf: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather 1-D uint8 buffers of different lengths; returns their concatenation in rank order.

    Two collectives: an all_gather of the lengths, then one all_gather_into_tensor of the
    buffers padded to the longest one.
    """
    world = dist.get_world_size(group)
    dev = buf.device
    if dev.type == "cuda" and dist.get_backend(group) == "gloo":
        # gloo collectives run on host memory: stage the records through the CPU (used by the
        # multi-process tests on one GPU; NCCL moves device buffers directly over NVLink)
        return gather_varlen(buf.cpu(), group).to(dev)
    n = torch.tensor([buf.numel()], dtype=torch.int64, device=buf.device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(s.item()) for s in sizes]
    m = max(max(sizes), 1)
    pad = torch.zeros(m, dtype=torch.uint8, device=buf.device)
    pad[: buf.numel()] = buf
    out = torch.empty(world * m, dtype=torch.uint8, device=buf.device)
    if hasattr(dist, "all_gather_into_tensor") and buf.device.type == "cuda":
        dist.all_gather_into_tensor(out, pad, group=group)
    else:
        parts = list(out.chunk(world))
        dist.all_gather(parts, pad, group=group)
        out = torch.cat(parts)
    return torch.cat([out[r * m: r * m + sizes[r]] for r in range(world)])


def gather_top(vox, group=None) -> int:
    """Export this rank's level log2(N) - T, gather all ranks' records, import them.

    Returns the gathered level. Ranks' top-cell ranges are disjoint and ordered, so the
    rank-order concatenation is sorted by key (vox_import_level checks it).
    """
    T = int(vox.stats()["top_depth"])
    lt = vox.levels_total - T
    if vox.built_levels() < lt:
        raise RuntimeError("build the local levels first (vox_build_lod stops at log2(N) - T)")
    mine = vox.export_level(lt)
    allrec = gather_varlen(mine, group)
    vox.import_level(lt, allrec)
    return lt
