import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from gpu_util import Case
for (M, N, K, al, be) in [(256, 256, 256, 1.0, 0.0), (256, 256, 256, 1.5, -0.5), (500, 1024, 256, 1.0, 0.0), (4096, 4096, 256, 1.5, -0.5)]:
    c = Case("bf16", M, N, K, alpha=al, beta=be)
    err = np.abs(c.C - c.ref.C) > 0.05 * (np.abs(c.ref.C) + 1)
    print(M, N, K, al, be, "fro", c.fro(), "bad", err.sum(), "tile", c.plan.check_tile_m, c.plan.check_tile_n)
    bc = np.where(err.any(axis=0))[0]; br = np.where(err.any(axis=1))[0]
    print("  bad cols", bc[:40], "... n", len(bc)); print("  bad rows", br[:40], "... n", len(br))
