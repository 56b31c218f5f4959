"""e2e decomposition at 2D 512^2 x 8: pinned H2D + D2H alone, device batch alone,
and the host-batch entry point under its schedule knobs (run per env)."""
import ctypes as C, json, os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1402_5670_b200 as P
dev = torch.device("cuda:0")
s = P.build_system_2d(512, 512, P.ScaleProfile.from_levels([1, 1, 2, 2]))
sch = P.ThresholdSchedule.defaults_2d(40.0)
fr = np.stack([P.add_gaussian_noise(P.cartoon(512), 40.0, i) for i in range(8)])
pin_in = torch.from_numpy(fr).pin_memory(); pin_out = torch.empty_like(pin_in).pin_memory()
d_in = pin_in.to(dev); d_out = torch.empty_like(d_in)
K = np.ascontiguousarray(sch.per_scale_factors); Kp = K.ctypes.data_as(C.POINTER(C.c_double))
def med(fn, n=30):
    ts = []
    for _ in range(n + 2):
        torch.cuda.synchronize(); t0 = time.perf_counter(); fn(); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    return float(np.median(ts[2:])) * 1e3
copies = med(lambda: (d_in.copy_(pin_in, non_blocking=True), pin_out.copy_(d_out, non_blocking=True)))
dev_b = med(lambda: P._check(P.lib().sl_denoise_batch_dev(s.handle, C.c_void_p(d_in.data_ptr()), 8, C.c_void_p(d_out.data_ptr()), Kp, 4, 40.0, 1, P._stream_ptr(0))))
host_b = med(lambda: P._check(P.lib().sl_denoise_batch_host(s.handle, P._dp(pin_in.numpy()), 8, P._dp(pin_out.numpy()), Kp, 4, 40.0, 1)))
print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("SLB_")}, "copies_ms": copies, "device_batch_ms": dev_b, "host_batch_ms": host_b, "host_frames_per_s": 8 / host_b * 1e3}))
