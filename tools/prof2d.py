"""Small driver for ncu: a few 2D dec+thr+rec calls at 512^2 (R=49)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1402_5670_b200 as P
mode = sys.argv[1] if len(sys.argv) > 1 else "decrec"   # "denoise" = fused path
n = 512
dev = torch.device("cuda:0")
s = P.build_system_2d(n, n, P.ScaleProfile.from_levels([1, 1, 2, 2]))
f = torch.from_numpy(P.add_gaussian_noise(P.cartoon(n), 40.0, 7)).to(dev)
sch = P.ThresholdSchedule.defaults_2d(40.0)
for _ in range(3):
    if mode == "denoise":
        r = P.denoise(f, s, sch)
    else:
        b = P.forward_thresholded(f, s, sch)
        r = P.inverse(b, s)
torch.cuda.synchronize()
print("ok", float(r.abs().sum()))
