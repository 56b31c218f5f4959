"""Bench-only FFT-stage yardstick (cuFFT is a yardstick, never on
the product path): fp64 cuFFT D2Z + Z2D (torch.fft.rfftn / irfftn) of one
band-sized grid at 512^2 and 192^3, batched like our band chunks, against
the per-band time of our fused dec -> threshold -> rec passes (which do the
same two real FFTs per band plus the filter multiplies, the threshold, the
band store and the accumulation). Prints one JSON line."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def time_ms(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


out = {}
dev = torch.device("cuda:0")
for name, dims, batch in (("2d512", (512, 512), 49), ("3d192", (192, 192, 192), 8)):
    x = torch.randn((batch,) + dims, dtype=torch.float64, device=dev)
    axes = tuple(range(1, len(dims) + 1))
    X = torch.fft.rfftn(x, dim=axes)
    fwd = time_ms(lambda: torch.fft.rfftn(x, dim=axes))
    inv = time_ms(lambda: torch.fft.irfftn(X, s=dims, dim=axes))
    per_band_us = (fwd + inv) / batch * 1000.0
    nbytes = 8 * x[0].numel() + 16 * X[0].numel()  # one D2Z and one Z2D: real in + half out, and back
    out[name] = {"cufft_d2z_plus_z2d_us_per_band": per_band_us, "batch": batch,
                 "d2z_ms": fwd, "z2d_ms": inv,
                 "hbm_gbs_cufft": 2 * nbytes / (per_band_us * 1e-6) / 1e9}
print(json.dumps({"cufft_yardstick": out, "torch": torch.__version__,
                  "note": "cuFFT via torch.fft (bench-only yardstick); compare with bench.py per-band kernel sums"}))
