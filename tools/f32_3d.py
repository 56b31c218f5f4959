"""Time the fp32-mode 3D 192^3 fused denoise (sl_denoise_f32_dev) for A/B runs:
python tools/f32_3d.py [steps]  (SLB_LIB selects a library variant)."""
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
r = bench.run_fp32("3d192", steps, 3, 0)
print(round(r["value"], 2), round(r["ms_per_step"], 3))
