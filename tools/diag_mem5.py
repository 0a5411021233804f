"""Device memory after each bench-like step and around encode/density (diagnostics)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, gen
from paper_2604_13191_b200 import Vox
c = gen.config(4)
S = torch.from_numpy(c["segments"]).cuda(); R = torch.from_numpy(c["radii"]).cuda()
def free(): return round(torch.cuda.mem_get_info()[0] / 1e9, 1)
for i in range(5):
    v = Vox(4096, c["bbox"], profile=True); v.voxelize_fibers(S, R); v.build_lod(12)
    n = [int(v.view(l)["n"]) for l in range(13)]
    v.close(); torch.cuda.synchronize(); print("step", i, "free", free(), "torch reserved", torch.cuda.memory_reserved() / 1e9, flush=True)
v = Vox(4096, c["bbox"], profile=True); v.voxelize_fibers(S, R); v.build_lod(12)
print("built free", free(), flush=True)
bufs = [v.encode_level(l) for l in range(13)]
torch.cuda.synchronize(); print("encoded free", free(), "torch reserved", torch.cuda.memory_reserved() / 1e9, flush=True)
v.stats_reset(); v.density_fibers(S, R); torch.cuda.synchronize(); print("density free", free(), v.stats()["host_ms_alloc"], flush=True)
d = [v.density_level(l) for l in range(13)]; st = v.stats()
print("levels free", free(), "ms", st["ms_density"], "alloc", st["host_ms_alloc"], flush=True)
