"""Config 5 at 8192^3: device time, counts, memory for N segments (diagnostics; default 15M, the largest that fits one B200)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, gen
from paper_2604_13191_b200 import Vox
n = int(sys.argv[1]) if len(sys.argv) > 1 else 15_000_000
t0 = time.time()
c = gen.config(5, n_segments=n, grid_res=8192)
print("generated", len(c["segments"]), "segments in", round(time.time() - t0, 1), "s", flush=True)
S = torch.from_numpy(c["segments"]).cuda(); R = torch.from_numpy(c["radii"]).cuda()
for it in range(2):
    v = Vox(8192, c["bbox"], profile=True)
    v.voxelize_fibers(S, R); v.build_lod(13)
    st = v.stats()
    print({k: round(st[k], 1) for k in ("ms_total_vox", "ms_total_lod")}, "pairs", st["pairs"], "cand", st["candidates"],
          "leaves", st["voxels"], "peak GB", round(torch.cuda.max_memory_allocated() / 1e9, 1),
          "free GB", round(torch.cuda.mem_get_info()[0] / 1e9, 1), flush=True)
    v.close()
