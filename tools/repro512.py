import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1402_5670_b200 as P
n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
s = P.build_system_2d(n, n, P.ScaleProfile.from_levels([1, 1, 2, 2]))
f = P.add_gaussian_noise(P.cartoon(n), 40.0, 7)
try:
    b = P.forward(f, s); print("forward ok")
    r = P.inverse(b, s); print("inverse ok", np.abs(r - f).max())
except Exception as e:
    print("ERR", e)
