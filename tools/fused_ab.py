"""fp32 smoothing step at C2 (k=2, level 5): unfused (residual launch per colour) vs fused halo residual."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_09497_b200 as smg  # noqa: E402

k, level = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (2, 5)
res = {}
for fused in (False, True):
    ctx = smg.Context(k, level, cg_max_iter=30, cg_tol=1e-5, smoother_fused=fused)
    n = ctx.sizes(level)[4]
    x = torch.rand(n, dtype=torch.float64, device="cuda") * 2 - 1
    b = ctx.apply_stokes(level, x).float()
    xs = torch.zeros_like(b)
    for _ in range(3):
        ctx.smooth(level, xs, b, zero_init=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        ctx.smooth(level, xs, b, zero_init=True)
    e1.record()
    torch.cuda.synchronize()
    bb = b.double()
    t0 = torch.cuda.Event(enable_timing=True)
    res["fused" if fused else "unfused"] = {"ms_per_step": e0.elapsed_time(e1) / 10,
                                            "x_norm": float(xs.double().norm())}
print(json.dumps(res))
