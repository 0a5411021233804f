"""Device time of vox_density_fibers on config 4 (diagnostics)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, gen
from paper_2604_13191_b200 import Vox
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
c = gen.config(4, n_segments=n)
S = torch.from_numpy(c["segments"]).cuda(); R = torch.from_numpy(c["radii"]).cuda()
for it in range(2):
    v = Vox(4096, c["bbox"], profile=True)
    v.voxelize_fibers(S, R); v.build_lod(12)
    v.stats_reset()
    v.density_fibers(S, R)
    d = v.density_level(0)
    st = v.stats()
    print(len(S), "segments: density", round(st["ms_density"], 1), "ms; mean occupancy", float(d["occ"].mean()), flush=True)
    v.close()
