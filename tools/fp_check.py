import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from gpu_util import Case
for dt in ["bf16", "tf32", "f32_simt"]:
    for (M, N, K) in [(2048, 2048, 128), (2048, 2048, 64), (2048, 2048, 8), (1024, 1024, 16), (4096, 4096, 128)]:
        for dist in ["signed", "unit"]:
            c = Case(dt, M, N, K, dist=dist, run_oracle=(M <= 2048))
            msg = f"{dt} {M}x{N}x{K} {dist}: gpu {dict((k,v) for k,v in c.counts.items() if v)}"
            if c.ref is not None:
                msg += f" oracle {dict((k,v) for k,v in c.ref.counts.items() if v)} fro {c.fro():.2e}"
            print(msg, flush=True)
            if c.events[:2]: print("   ", c.events[:2])
