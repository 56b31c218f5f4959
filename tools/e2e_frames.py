"""e2e vs device throughput of the 2D 512^2 batch as the frame count grows
(separates the fixed first-H2D / last-D2H tails from per-frame costs)."""
import ctypes as C, json, os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1402_5670_b200 as P
dev = torch.device("cuda:0")
s = P.build_system_2d(512, 512, P.ScaleProfile.from_levels([1, 1, 2, 2]))
sch = P.ThresholdSchedule.defaults_2d(40.0)
K = np.ascontiguousarray(sch.per_scale_factors); Kp = K.ctypes.data_as(C.POINTER(C.c_double))
def med(fn, n=15):
    ts = []
    for _ in range(n + 2):
        torch.cuda.synchronize(); t0 = time.perf_counter(); fn(); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    return float(np.median(ts[2:])) * 1e3
for nf in (8, 16, 32):
    fr = np.stack([P.add_gaussian_noise(P.cartoon(512), 40.0, i) for i in range(nf)])
    pin_in = torch.from_numpy(fr).pin_memory(); pin_out = torch.empty_like(pin_in).pin_memory()
    d_in = pin_in.to(dev); d_out = torch.empty_like(d_in)
    dv = med(lambda: P._check(P.lib().sl_denoise_batch_dev(s.handle, C.c_void_p(d_in.data_ptr()), nf, C.c_void_p(d_out.data_ptr()), Kp, 4, 40.0, 1, P._stream_ptr(0))))
    hb = med(lambda: P._check(P.lib().sl_denoise_batch_host(s.handle, P._dp(pin_in.numpy()), nf, P._dp(pin_out.numpy()), Kp, 4, 40.0, 1)))
    t0 = time.perf_counter(); P._check(P.lib().sl_denoise_batch_host(s.handle, P._dp(pin_in.numpy()), nf, P._dp(pin_out.numpy()), Kp, 4, 40.0, 1)); 
    print(json.dumps({"frames": nf, "device_ms": dv, "host_ms": hb, "device_fps": nf / dv * 1e3, "e2e_fps": nf / hb * 1e3, "ratio": dv / hb}))
