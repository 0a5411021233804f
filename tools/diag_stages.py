"""Per-stage device times of one config-4 step (profile mode), averaged over 3 steps."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, gen
from paper_2604_13191_b200 import Vox
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
c = gen.config(4, n_segments=n)
S = torch.from_numpy(c["segments"]).cuda(); R = torch.from_numpy(c["radii"]).cuda()
acc = {}
for it in range(5):
    v = Vox(4096, c["bbox"], profile=True)
    v.voxelize_fibers(S, R); v.build_lod(12)
    st = v.stats(); v.close()
    if it >= 2:
        for k, x in st.items():
            if k.startswith("ms_"): acc[k] = acc.get(k, 0) + x / 3
print({k: round(x, 2) for k, x in acc.items()})
