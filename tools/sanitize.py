"""Small end-to-end run of every hot entry point for compute-sanitizer
(memcheck / racecheck): 2D fast + generic + fp32 + asymmetric fan, 3D split +
fp32 + sharded, batches, the in-library NCCL path on one rank."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1402_5670_b200 as P
dev = torch.device("cuda:0")
sch2 = P.ThresholdSchedule.defaults_2d(0.3, 2)
for n, lv, dt in ((64, [0, 1], "f64"), (48, [0, 1], "f64"), (64, [0, 1], "f32")):
    s = P.build_system_2d(n, n, P.ScaleProfile.from_levels(lv), dtype=dt)
    x = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, (3, n, n))).to(dev)
    if dt == "f32":
        x = x.float()
    d = P.denoise_batch(x, s, sch2)
    d1, st = P.denoise(x[0], s, sch2, return_stack=True)
    b = P.forward(x[0], s)
    r = P.inverse(b, s)
    if dt == "f64":
        P.denoise_batch(x.cpu().numpy(), s, sch2)
fan = P.FanFilter(np.array([[0.0, 1.0, 0.5]]), 0, 0, "asym")
sa = P.build_system_2d(32, 32, P.ScaleProfile.from_levels([0, 1]), fan=fan)
P.denoise(np.random.default_rng(2).uniform(-1, 1, (32, 32)), sa, sch2)
sch3 = P.ThresholdSchedule.defaults_3d(0.3, 2)
s3 = P.build_system_3d((64, 64, 64), P.ScaleProfile.from_levels([0, 1]), dtype="f32")
v = torch.from_numpy(np.random.default_rng(3).uniform(-1, 1, (64, 64, 64))).to(dev)
P.denoise(v, s3, sch3, return_stack=True)
P.denoise(v.float(), s3, sch3, return_stack=True)
P.inverse(P.forward(v, s3), s3)
sh = P.build_system_3d((64, 64, 64), P.ScaleProfile.from_levels([0, 1]), shard=(10, 40))
P.denoise(v, sh, sch3)
comm = P.Comm(P.Comm.unique_id(), 1, 0, 0)
s3.set_comm(comm)
P.denoise_dist(v.clone(), s3, sch3)
s3.set_comm(None)
torch.cuda.synchronize()
print("sanitize driver ok")
