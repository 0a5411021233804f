"""Bench-like loop with host phase timing and the CUDA default mem-pool reserved size."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, gen
from cuda.bindings import runtime as rt
from paper_2604_13191_b200 import Vox
c = gen.config(4)
S = torch.from_numpy(c["segments"]).cuda(); R = torch.from_numpy(c["radii"]).cuda()
def reserved():
    err, pool = rt.cudaDeviceGetDefaultMemPool(0)
    err, v = rt.cudaMemPoolGetAttribute(pool, rt.cudaMemPoolAttr.cudaMemPoolAttrReservedMemCurrent)
    return int(v) / 2**30
prof = len(sys.argv) > 1
for it in range(6):
    torch.cuda.synchronize(); t = [time.perf_counter()]
    v = Vox(4096, c["bbox"], profile=prof)
    v.voxelize_fibers(S, R); torch.cuda.synchronize(); t.append(time.perf_counter())
    v.build_lod(12); torch.cuda.synchronize(); t.append(time.perf_counter())
    st = v.stats(); v.close(); torch.cuda.synchronize(); t.append(time.perf_counter())
    print(it, "vox/lod/close ms", [round(1e3 * (b - a), 1) for a, b in zip(t, t[1:])], "pool GiB %.1f" % reserved(),
          {k: round(x, 1) for k, x in st.items() if k in ("ms_lod", "ms_total_lod", "ms_lod_scan", "host_ms_alloc", "host_ms_sync", "ms_total_vox")}, flush=True)
