"""Per-level histogram of lobe counts n of the parents SGGX-H must cluster (n > K), with
per-level SGGX-H kernel times (diagnostics)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, gen
from paper_2604_13191_b200 import Vox
c = gen.config(4)
S = torch.from_numpy(c["segments"]).cuda(); R = torch.from_numpy(c["radii"]).cuda()
v = Vox(4096, c["bbox"], profile=True)
v.voxelize_fibers(S, R)
prev = v.level(0)
for l in range(1, 13):
    v.stats_reset(); v.build_lod(l); st = v.stats()
    cur = v.level(l)
    pk = prev["key"] >> 3
    lob = prev["ncl"].long() if l > 1 else (prev["acc"][:, 0] > 0).long()
    idx = torch.searchsorted(cur["key"], pk)
    n = torch.zeros(len(cur["key"]), dtype=torch.long, device="cuda").index_add_(0, idx, lob)
    h = torch.bincount(n[n > 3], minlength=25).cpu().tolist()
    print(l, "parents", len(n), "hard", int((n > 3).sum()), "quad", round(st["ms_sggxh_quad"], 2), "half", round(st["ms_sggxh_half"], 2), "warp",
          round(st["ms_sggxh_warp"], 2), "prep", round(st["ms_lod_prep"], 2),
          {k: x for k, x in enumerate(h) if x}, flush=True)
    prev = cur
