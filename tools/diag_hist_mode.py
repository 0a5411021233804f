"""Device time of the LoD build with the histogram distance vs the sigma distance (diagnostics)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, gen
from paper_2604_13191_b200 import Vox
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
c = gen.config(cfg)
fib = c["kind"] == "fiber"
A = torch.from_numpy(c["segments"] if fib else c["tris"]).cuda()
B = torch.from_numpy(c["radii"]).cuda() if fib else (None if c["dirs"] is None else torch.from_numpy(c["dirs"]).cuda())
for mode in ("sigma", "hist", "hist"):
    v = Vox(c["grid_res"], c["bbox"], profile=True, distance=mode)
    (v.voxelize_fibers if fib else v.voxelize_triangles)(A, B)
    v.build_lod(c["levels"])
    st = v.stats()
    print(cfg, mode, {k: round(st[k], 2) for k in ("ms_total_vox", "ms_total_lod", "ms_lod_prep", "ms_sggxh_quad",
                                                   "ms_sggxh_half", "ms_sggxh_warp")},
          "sigma_evals", st["lod_sigma_evals"], "dist_evals", st["lod_dist_evals"], flush=True)
    v.close()
