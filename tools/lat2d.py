"""Single-frame 2D denoise latency (sl_denoise_dev, one stream) and a short inpaint."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1402_5670_b200 as P  # noqa: E402

n = 512
s = P.build_system_2d(n, n, P.ScaleProfile.from_levels([1, 1, 2, 2]))
sch = P.ThresholdSchedule.defaults_2d(40.0)
f = torch.from_numpy(P.add_gaussian_noise(P.cartoon(n), 40.0, 7)).cuda()
for _ in range(5):
    P.denoise(f, s, sch)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(50):
    P.denoise(f, s, sch)
e1.record()
torch.cuda.synchronize()
print(f"single-frame denoise {e0.elapsed_time(e1) / 50 * 1000:.1f} us", flush=True)
mask = (torch.rand((n, n), dtype=torch.float64, device="cuda") < 0.3).double()
cfg = P.InpaintConfig(iterations=50)
P.inpaint(f * mask, mask, s, cfg)
torch.cuda.synchronize()
t0 = time.perf_counter()
P.inpaint(f * mask, mask, s, cfg)
torch.cuda.synchronize()
print(f"inpaint 50 iterations {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
