"""smg_vmult_host wall time per call vs the number of z-chunks (SMG_HOST_CHUNKS is read per call)."""
import os
import time

import numpy as np
import torch

import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_09497_b200 as smg  # noqa: E402

k, level = 2, 5
ctx = smg.Context(k, level)
s = ctx.sizes(level)
xb = [torch.empty(s[i], dtype=torch.float64, pin_memory=True).numpy() for i in range(4)]
yb = [torch.empty(s[i], dtype=torch.float64, pin_memory=True).numpy() for i in range(4)]
for a in xb:
    a[:] = np.random.default_rng(0).standard_normal(a.size)
for n in (16, 32, 24, 8, 16, 32):
    os.environ["SMG_HOST_CHUNKS"] = str(n)
    for _ in range(3):
        ctx.vmult_host(level, xb, smg.F64, out=yb)
    t0 = time.perf_counter()
    for _ in range(20):
        ctx.vmult_host(level, xb, smg.F64, out=yb)
    t = (time.perf_counter() - t0) / 20
    print(n, f"{t*1e3:.3f} ms", f"{s[4]/t/1e9:.2f} GDoF/s", flush=True)
