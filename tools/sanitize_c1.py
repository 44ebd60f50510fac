"""Workload for compute-sanitizer (racecheck / memcheck / synccheck) at C1 (k=1, L=3) plus the
warp-per-patch smoother variant (level 4): vmult, residual, smoothing step, transfers, V-cycle and
FGMRES through the C ABI. Usage: compute-sanitizer --tool racecheck python tools/sanitize_c1.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_09497_b200 as smg  # noqa: E402


def main():
    for k, level in ((1, 3), (1, 4), (2, 2)):
        ctx = smg.Context(k, level, cg_max_iter=4, cg_fixed=True)
        n = ctx.sizes(level)[4]
        g = torch.Generator(device="cpu").manual_seed(0)
        for dt in (torch.float64, torch.float32):
            x = (torch.rand(n, generator=g, dtype=torch.float64) * 2 - 1).to("cuda", dt)
            b = (torch.rand(n, generator=g, dtype=torch.float64) * 2 - 1).to("cuda", dt)
            y = ctx.apply_stokes(level, x)
            r = ctx.residual(level, b, x)
            ctx.smooth(level, x, b)
            rc = ctx.restrict(level - 1, r)
            ctx.prolongate_add(level - 1, x, rc)
            if level <= 3:
                ctx.vcycle(level, b)
            torch.cuda.synchronize()
            print(k, level, dt, float(y.norm()), float(x.norm()))
        if level == 3:
            bb = ctx.apply_stokes(level, (torch.rand(n, generator=g, dtype=torch.float64) * 2 - 1).cuda())
            _, it, _ = ctx.solve(level, bb, 1e-8, 30, smg.F32, allow_not_converged=True)
            print("solve iterations", it)
    print("sanitize workload done")


if __name__ == "__main__":
    main()
