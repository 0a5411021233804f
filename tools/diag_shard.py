"""Per-rank device time of a Morton shard of config 4 (strong-scaling estimate on one GPU: each
shard voxelizes its range and builds its local levels; the top levels and the all-gather are
not included). Diagnostics only: ranks run one after another, not concurrently."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, gen
from paper_2604_13191_b200 import Vox
c = gen.config(4)
S = torch.from_numpy(c["segments"]).cuda(); R = torch.from_numpy(c["radii"]).cuda()
for world in [int(x) for x in (sys.argv[1:] or ['1', '2', '4', '8'])]:
    worst = 0.0
    for rank in range(world):
        for it in range(2):
            v = Vox(4096, c["bbox"], rank=rank, world=world, profile=True)
            v.voxelize_fibers(S, R); v.build_lod(12)
            st = v.stats(); v.close()
        t = st["ms_total_vox"] + st["ms_total_lod"]
        worst = max(worst, t)
        print(world, "rank", rank, "cells", st["cell_lo"], st["cell_hi"], "emit", round(st["ms_emit"], 2), "vox",
              round(st["ms_total_vox"], 2), "lod", round(st["ms_total_lod"], 2), "pairs", st["pairs"],
              "hard", st["lod_hard_parents"], flush=True)
    print(world, "max over ranks", round(worst, 2), "ms", flush=True)
