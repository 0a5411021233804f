"""vox_density_fibers device time on config 4: fresh context vs after a build + encode (diagnostics)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, gen
from paper_2604_13191_b200 import Vox
c = gen.config(4)
S = torch.from_numpy(c["segments"]).cuda(); R = torch.from_numpy(c["radii"]).cuda()
for it in range(3):
    v = Vox(4096, c["bbox"], profile=True)
    v.voxelize_fibers(S, R); v.build_lod(12)
    bufs = [v.encode_level(l) for l in range(13)] if it == 2 else []
    v.stats_reset()
    v.density_fibers(S, R)
    a = v.stats()["ms_density"]
    d = [v.density_level(l) for l in range(13)]
    print(it, "density_fibers", round(a, 1), "ms; with all levels", round(v.stats()["ms_density"], 1), flush=True)
    del d, bufs
    v.close()
