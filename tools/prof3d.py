"""Small driver for ncu: 3D 192^3 SL3D_2 denoise (a few bands only via shard)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1402_5670_b200 as P
n = int(sys.argv[1]) if len(sys.argv) > 1 else 192
dev = torch.device("cuda:0")
s = P.build_system_3d((n, n, n), P.ScaleProfile.from_levels([1, 1, 2]), shard=(100, 112))
f = torch.from_numpy(P.add_gaussian_noise(P.cartoon_volume(n), 40.0, 3)).to(dev)
sch = P.ThresholdSchedule.defaults_3d(40.0)
for _ in range(3):
    r = P.denoise(f, s, sch)
torch.cuda.synchronize()
print("ok", float(r.abs().sum()))
