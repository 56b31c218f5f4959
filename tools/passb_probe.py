"""Pass-B probe: 3D 192^3 SL3D_2 fused denoise with and without the
materialised stack (the stack is a third of pass B's HBM bytes), per-pass
times from sl_profile. Tells a bandwidth-bound pass B (time drops with the
bytes) from a latency / issue-bound one (time stays)."""
import sys, torch, numpy as np
sys.path.insert(0, '.')
import paper_1402_5670_b200 as P
dev = torch.device('cuda:0')
s = P.build_system_3d((192, 192, 192), P.ScaleProfile.from_levels([1, 1, 2]))
x = torch.from_numpy(P.add_gaussian_noise(P.cartoon_volume(192), 40.0, 3)).to(dev)
sch = P.ThresholdSchedule.defaults_3d(40.0)
for stack in (True, False, True, False):
    s.set_stack_output(stack)
    P.denoise(x, s, sch); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        P.denoise(x, s, sch)
    e1.record(); torch.cuda.synchronize()
    print(f"stack={stack}: {e0.elapsed_time(e1) / 5:.2f} ms / volume", flush=True)
