"""build_lod(12) in one call vs per-level calls, profile on/off (diagnostics)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, gen
from paper_2604_13191_b200 import Vox
c = gen.config(4)
S = torch.from_numpy(c["segments"]).cuda(); R = torch.from_numpy(c["radii"]).cuda()
for prof in (False, True):
    for mode in ("one", "per", "one"):
        v = Vox(4096, c["bbox"], profile=prof)
        v.voxelize_fibers(S, R); torch.cuda.synchronize()
        t0 = time.perf_counter()
        if mode == "one":
            v.build_lod(12)
        else:
            for l in range(1, 13): v.build_lod(l)
        torch.cuda.synchronize()
        print(prof, mode, round(1e3 * (time.perf_counter() - t0), 1), flush=True)
        v.close()
