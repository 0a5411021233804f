"""Density device time after N full bench steps, with SM clock and throttle reasons (diagnostics)."""
import sys, os, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, gen, pynvml
from paper_2604_13191_b200 import Vox
pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(0)
def clk(): return pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM), pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h), pynvml.nvmlDeviceGetPowerUsage(h) // 1000
c = gen.config(4)
S = torch.from_numpy(c["segments"]).cuda(); R = torch.from_numpy(c["radii"]).cuda()
nsteps = int(sys.argv[1]) if len(sys.argv) > 1 else 8
for i in range(nsteps):
    v = Vox(4096, c["bbox"]); v.voxelize_fibers(S, R); v.build_lod(12); v.close()
torch.cuda.synchronize()
for rep in range(3):
    v = Vox(4096, c["bbox"], profile=True); v.voxelize_fibers(S, R); v.build_lod(12)
    bufs = [v.encode_level(l) for l in range(13)]
    v.stats_reset()
    samples = []
    stop = False
    def mon():
        while not stop:
            samples.append(clk()); time.sleep(0.05)
    t = threading.Thread(target=mon); t.start()
    v.density_fibers(S, R); torch.cuda.synchronize()
    stop = True; t.join()
    print(nsteps, rep, "density", round(v.stats()["ms_density"], 1), "clk/reasons/W", samples[::4][:8], flush=True)
    del bufs; v.close()
