"""Where does the 2D e2e time go? Wall-clock per batch call for: the host API
(pinned in/out), the device API (inputs resident, synchronised), and the
device API on already-resident data without the final sync (enqueue cost)."""
import ctypes as C
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1402_5670_b200 as P  # noqa: E402

n, frames = 512, int(sys.argv[1]) if len(sys.argv) > 1 else 8
s = P.build_system_2d(n, n, P.ScaleProfile.from_levels([1, 1, 2, 2]))
s.set_streams(int(os.environ.get("SLB_STREAMS", "6")))
sch = P.ThresholdSchedule.defaults_2d(40.0)
K = np.ascontiguousarray(sch.per_scale_factors, dtype=np.float64)
Kp = K.ctypes.data_as(C.POINTER(C.c_double))
L = P.lib()
x = np.stack([P.add_gaussian_noise(P.cartoon(n), 40.0, i) for i in range(frames)])
pin_in = torch.from_numpy(x).pin_memory()
pin_out = torch.empty_like(pin_in).pin_memory()
d_in = pin_in.cuda()
d_out = torch.empty_like(d_in)


def host():
    P._check(L.sl_denoise_batch_host(s.handle, P._dp(pin_in.numpy()), frames, P._dp(pin_out.numpy()), Kp, len(K),
                                     40.0, 1))


def dev(sync=True):
    P._check(L.sl_denoise_batch_dev(s.handle, C.c_void_p(d_in.data_ptr()), frames, C.c_void_p(d_out.data_ptr()), Kp,
                                    len(K), 40.0, 1, P._stream_ptr(0)))
    if sync:
        torch.cuda.synchronize()


for name, fn in (("host", host), ("dev+sync", dev)):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(30):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    print(f"{name:10s} median {1e3 * np.median(ts):.3f} ms/call -> {frames / np.median(ts):.0f} frames/s", flush=True)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(30):
    dev(sync=False)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"enqueue only {1e3 * (t1 - t0) / 30:.3f} ms/call; pipelined {frames * 30 / (t2 - t0):.0f} frames/s")
