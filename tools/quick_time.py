import sys, time, torch, numpy as np
sys.path.insert(0, '.')
import paper_1402_5670_b200 as P
dev = torch.device('cuda:0')
for (shape, lv) in [((512, 512), [1, 1, 2, 2]), ((1024, 1024), [1, 1, 2, 2]), ((128, 128, 128), [1, 1]), ((192, 192, 192), [1, 1, 2])]:
    t = time.time()
    s = P.build_system_2d(*shape, P.ScaleProfile.from_levels(lv)) if len(shape) == 2 else P.build_system_3d(shape, P.ScaleProfile.from_levels(lv))
    tb = time.time() - t
    f = torch.rand(shape, dtype=torch.float64, device=dev)
    b = P.forward(f, s); r = P.inverse(b, s); torch.cuda.synchronize()
    e0, e1, e2 = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    n = 5
    e0.record()
    for _ in range(n):
        b = P.forward(f, s)
    e1.record()
    for _ in range(n):
        r = P.inverse(b, s)
    e2.record(); torch.cuda.synchronize()
    err = (torch.linalg.norm(r - f) / torch.linalg.norm(f)).item()
    print(f"{shape} R={s.redundancy()} build {tb:.2f}s dec {e0.elapsed_time(e1)/n:.3f} ms rec {e1.elapsed_time(e2)/n:.3f} ms err {err:.2e}", flush=True)
    del b, r, s
    torch.cuda.empty_cache()
