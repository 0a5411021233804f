"""Host-side phase timing of one bench step (diagnostics only)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, gen
from paper_2604_13191_b200 import Vox
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
c = gen.config(4, n_segments=n)
S = torch.from_numpy(c["segments"]).cuda(); R = torch.from_numpy(c["radii"]).cuda()
for it in range(4):
    torch.cuda.synchronize(); t = [time.perf_counter()]
    v = Vox(4096, c["bbox"], profile=True); torch.cuda.synchronize(); t.append(time.perf_counter())
    v.voxelize_fibers(S, R); torch.cuda.synchronize(); t.append(time.perf_counter())
    v.build_lod(12); torch.cuda.synchronize(); t.append(time.perf_counter())
    st = v.stats(); t.append(time.perf_counter())
    v.close(); torch.cuda.synchronize(); t.append(time.perf_counter())
    d = [round(1e3 * (b - a), 2) for a, b in zip(t, t[1:])]
    print("create/vox/lod/stats/close ms:", d, "stage:", {k: round(v_, 2) for k, v_ in st.items() if k.startswith("ms_")}, flush=True)
