"""Where does the end-to-end step time go? H2D + build, + serial D2H, + overlapped D2H (diagnostics)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, gen
from paper_2604_13191_b200 import Vox
c = gen.config(4)
pa = torch.from_numpy(c["segments"]).pin_memory(); pb = torch.from_numpy(c["radii"]).pin_memory()
side = torch.cuda.Stream()
host = {}
def buf(l, n, k):
    if l not in host or host[l]["key"].numel() < n:
        host[l] = {"key": torch.empty(n, dtype=torch.int64).pin_memory(), "mass": torch.empty(n).pin_memory(),
                   "m6": torch.empty(n * 6).pin_memory(), "ncl": torch.empty(n, dtype=torch.uint8).pin_memory(),
                   "cl": torch.empty(n * k * 7).pin_memory()}
    return host[l]
main = torch.cuda.Stream()
def step(mode):
    v = Vox(4096, c["bbox"], stream=main if mode.endswith("own") else None)
    v.voxelize_fibers_host(pa, pb)
    for l in range(1, 13):
        v.build_lod(l)
        if mode.startswith("async"):
            v.copy_level_async(l, buf(l, int(v.view(l)["n"]), v.k), side)
    if mode == "serial":
        for l in range(1, 13):
            v.copy_level_to(l, buf(l, int(v.view(l)["n"]), v.k))
    side.synchronize()
    torch.cuda.synchronize()
    v.close()
import ctypes
rt = ctypes.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None
for st, nm in ((side, "side"), (main, "main")):
    f = ctypes.c_uint(99)
    try:
        r = ctypes.CDLL("/usr/local/cuda/lib64/libcudart.so").cudaStreamGetFlags(ctypes.c_void_p(st.cuda_stream), ctypes.byref(f))
        print(nm, "stream flags", f.value, "rc", r)
    except Exception as e:
        print("flags?", e)
for mode in ("none", "serial", "async", "async_own", "none", "serial", "async", "async_own"):
    torch.cuda.synchronize(); t = time.perf_counter(); step(mode); torch.cuda.synchronize()
    print(mode, round(1e3 * (time.perf_counter() - t), 1), "ms", flush=True)
x = torch.empty(4_500_000_000 // 4, device="cuda"); h = torch.empty(x.numel()).pin_memory()
for _ in range(2):
    torch.cuda.synchronize(); t = time.perf_counter(); h.copy_(x, non_blocking=True); torch.cuda.synchronize()
    print("D2H 4.5 GB", round(1e3 * (time.perf_counter() - t), 1), "ms", round(4.5 / (time.perf_counter() - t), 1), "GB/s")
