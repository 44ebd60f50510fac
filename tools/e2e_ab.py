"""smg_vmult_host wall time per call: one vs two copy streams per direction, alternating in one process."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_09497_b200 as smg  # noqa: E402
import subprocess  # noqa: E402

if len(sys.argv) > 1 and sys.argv[1] == "--run":
    k, level = 2, 5
    ctx = smg.Context(k, level)
    s = ctx.sizes(level)
    xb = [torch.empty(s[i], dtype=torch.float64, pin_memory=True).numpy() for i in range(4)]
    yb = [torch.empty(s[i], dtype=torch.float64, pin_memory=True).numpy() for i in range(4)]
    for a in xb:
        a[:] = np.random.default_rng(0).standard_normal(a.size)
    for _ in range(5):
        ctx.vmult_host(level, xb, smg.F64, out=yb)
    best = []
    for rep in range(3):
        t0 = time.perf_counter()
        for _ in range(20):
            ctx.vmult_host(level, xb, smg.F64, out=yb)
        best.append((time.perf_counter() - t0) / 20)
    t = min(best)
    print(f"{t*1e3:.3f} ms {s[4]/t/1e9:.2f} GDoF/s")
else:
    for r in range(2):
        for n in ("1", "2"):
            env = dict(os.environ, SMG_HOST_COPY_STREAMS=n)
            o = subprocess.run([sys.executable, __file__, "--run"], capture_output=True, text=True, env=env)
            print("copy streams", n, o.stdout.strip() or o.stderr[-300:], flush=True)
