"""Host-side timing of each LoD level (diagnostics): where does build_lod's wall time go?"""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, gen
from paper_2604_13191_b200 import Vox
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
c = gen.config(4, n_segments=n)
S = torch.from_numpy(c["segments"]).cuda(); R = torch.from_numpy(c["radii"]).cuda()
for it in range(3):
    v = Vox(4096, c["bbox"], profile=True)
    v.voxelize_fibers(S, R); torch.cuda.synchronize()
    t = [time.perf_counter()]
    for l in range(1, 13):
        v.build_lod(l); torch.cuda.synchronize(); t.append(time.perf_counter())
    st = v.stats()
    print("per-level ms:", [round(1e3 * (b - a), 2) for a, b in zip(t, t[1:])], "sum", round(1e3 * (t[-1] - t[0]), 1),
          "lod kernels", round(st["ms_lod"], 1), flush=True)
    v.close()
