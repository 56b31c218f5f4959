"""Time the fp32-mode 2D 512^2 lock-step batch (sl_denoise_batch_f32_dev) for A/B runs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

r = bench.run_fp32("2d512", int(sys.argv[1]) if len(sys.argv) > 1 else 20, 3, 0)
print(round(r["value"], 1), round(r["ms_per_step"], 4))
