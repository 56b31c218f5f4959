import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_1402_5670_b200 as P
for shape, lv in [((2048, 2048), [0, 1, 1]), ((256, 256, 256), [0, 1]), ((1000, 600), [0, 1])]:
    s = P.build_system_2d(*shape, P.ScaleProfile.from_levels(lv)) if len(shape) == 2 else P.build_system_3d(shape, P.ScaleProfile.from_levels(lv))
    f = torch.rand(shape, dtype=torch.float64, device='cuda')
    r = P.inverse(P.forward(f, s), s)
    sch = P.ThresholdSchedule.defaults_2d(0.0, len(lv)) if len(shape) == 2 else P.ThresholdSchedule.defaults_3d(0.0, len(lv))
    d = P.denoise(f, s, sch)
    print(shape, s.redundancy(), float(torch.linalg.norm(r - f) / torch.linalg.norm(f)), float(torch.linalg.norm(d - f) / torch.linalg.norm(f)), flush=True)
    del s, r, d
    torch.cuda.empty_cache()
