"""Single-frame (no cross-stream concurrency) 2D denoise latency vs the
lone-frame knobs SLB_GROUP1 / SLB_CHUNK1 (read by the library per call)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1402_5670_b200 as P  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
groups = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "1,2,4,7").split(",")]
chunks = [int(x) for x in (sys.argv[3] if len(sys.argv) > 3 else "7,14,28").split(",")]
s = P.build_system_2d(n, n, P.ScaleProfile.from_levels([1, 1, 2, 2]))
sch = P.ThresholdSchedule.defaults_2d(40.0)
f = torch.rand((n, n), dtype=torch.float64, device="cuda") * 255
for g in groups:
    for c in chunks:
        os.environ["SLB_GROUP1"], os.environ["SLB_CHUNK1"] = str(g), str(c)
        for _ in range(3):
            P.denoise(f, s, sch)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            P.denoise(f, s, sch)
        e1.record()
        torch.cuda.synchronize()
        print(f"n={n} G1={g} C1={c}: {e0.elapsed_time(e1) / 20 * 1000:.1f} us/frame", flush=True)
