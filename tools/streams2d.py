"""Experiment: frames spread over S streams (one system handle each)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1402_5670_b200 as P
n = 512
S = int(sys.argv[1]) if len(sys.argv) > 1 else 2
B = 8
dev = torch.device("cuda:0")
prof = P.ScaleProfile.from_levels([1, 1, 2, 2])
systems = [P.build_system_2d(n, n, prof) for _ in range(S)]
streams = [torch.cuda.Stream() for _ in range(S)]
sch = P.ThresholdSchedule.defaults_2d(40.0)
fs = [torch.from_numpy(P.add_gaussian_noise(P.cartoon(n), 40.0, i)).to(dev) for i in range(B)]
stacks = [torch.empty((49, n, n), dtype=torch.float64, device=dev) for _ in range(S)]
outs = [torch.empty_like(f) for f in fs]
import ctypes as C
L = P.lib()
K = np.ascontiguousarray(sch.per_scale_factors); Kp = K.ctypes.data_as(C.POINTER(C.c_double))
def step():
    for i, f in enumerate(fs):
        k = i % S
        st = C.c_void_p(streams[k].cuda_stream)
        P._check(L.sl_sheardec_threshold_dev(systems[k].handle, C.c_void_p(f.data_ptr()), C.c_void_p(stacks[k].data_ptr()), Kp, 4, 40.0, 1, st))
        P._check(L.sl_shearrec_dev(systems[k].handle, C.c_void_p(stacks[k].data_ptr()), 49, C.c_void_p(outs[i].data_ptr()), st))
for _ in range(3): step()
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(10): step()
torch.cuda.synchronize()
dt = time.perf_counter() - t
print(f"S={S}: {10 * B / dt:.0f} frames/s")
