import sys, time, os
sys.path.insert(0, os.getcwd())
import bench, torch
c = bench.ClockSampler(0)
print("nvml", c._nvml is not None)
orig = c._sample_nvml
ts = []
def wrapped():
    ts.append(time.time()); orig()
c._sample_nvml = wrapped
x = torch.randn(4096, 4096, device="cuda")
with c:
    t = time.time()
    while time.time() - t < 0.3:
        y = x @ x
        torch.cuda.synchronize()
print(len(c.rows), [round(b - a, 4) for a, b in zip(ts, ts[1:])][:10], c.summary())
