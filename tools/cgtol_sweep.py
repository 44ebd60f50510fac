"""MG-FGMRES at C2 (k=2, level 5, tol 1e-8, fp32 V-cycle) against the inner patch-CG tolerance."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_09497_b200 as smg  # noqa: E402

k, level = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (2, 5)
for tol in (1e-5, 1e-4, 1e-3, 1e-2):
    ctx = smg.Context(k, level, cg_max_iter=30, cg_tol=tol)
    n = ctx.sizes(level)[4]
    g = torch.Generator(device="cuda").manual_seed(1234)
    x = torch.rand(n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    b = ctx.apply_stokes(level, x)
    ctx.solve(level, b, 1e-8, 30, smg.F32, allow_not_converged=True)
    torch.cuda.synchronize()
    ctx.smoother_stats(reset=True)
    t0 = time.perf_counter()
    xs, it, hist = ctx.solve(level, b, 1e-8, 30, smg.F32, allow_not_converged=True)
    torch.cuda.synchronize()
    t = time.perf_counter() - t0
    p, c = ctx.smoother_stats(reset=True)
    print(json.dumps({"cg_tol": tol, "time_s": t, "iterations": it, "rel_res": float(hist[-1] / hist[0]),
                      "mean_inner_cg": c / max(p, 1)}), flush=True)
    del ctx
    torch.cuda.empty_cache()
