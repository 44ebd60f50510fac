"""Worker of the multi-process test of the C-ABI multi-GPU driver (tests/test_gpu_configs.py): RANK /
WORLD_SIZE ranks on one GPU, torch.distributed gloo transport callbacks (NCCL cannot run two ranks on
one device). Every rank solves its slabs with smg_dist_solve; the owned rows are summed on the host and
rank 0 compares with the single-GPU smg_solve. Prints one JSON line on rank 0."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_09497_b200 as smg  # noqa: E402
from paper_2410_09497_b200 import dist as sd  # noqa: E402


def main():
    k, level = int(sys.argv[1]), int(sys.argv[2])
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo")
    ctx = smg.Context(k, level, cg_max_iter=10, cg_fixed=True)
    D = sd.DistContext(ctx, world, rank).init_torch_transport()
    n = ctx.sizes(level)[4]
    g = torch.Generator().manual_seed(5)
    xr = (torch.rand(n, generator=g, dtype=torch.float64) * 2 - 1).cuda()
    b = ctx.apply_stokes(level, xr)
    out = {}
    # operator on the slabs
    xh = D.extract(level, xr)
    yh = torch.zeros_like(xh)
    D.vmult(level, yh, xh)
    yfull = torch.zeros(n, dtype=torch.float64, device="cuda")
    D.insert_owned(level, yfull, yh)
    yc = yfull.cpu()
    dist.all_reduce(yc)
    # solve, fp64 and mixed-precision V-cycles
    res = {}
    for vp in (smg.F64, smg.F32):
        bh = D.extract(level, b)
        x, it, hist = D.solve(bh, 1e-8, 30, vp)
        xf = torch.zeros(n, dtype=torch.float64, device="cuda")
        D.insert_owned(level, xf, x)
        xc = xf.cpu()
        dist.all_reduce(xc)
        res[vp] = (xc, it)
    if rank == 0:
        ref_y = ctx.apply_stokes(level, xr).cpu()
        out["vmult_rel"] = float((yc - ref_y).abs().max() / ref_y.abs().max())
        for vp, name in ((smg.F64, "f64"), (smg.F32, "f32")):
            xs, its, _ = ctx.solve(level, b, 1e-8, 30, vp)
            xc, it = res[vp]
            out[name] = {"iters": it, "iters_single": its,
                         "x_rel": float((xc - xs.cpu()).abs().max() / xs.cpu().abs().max())}
        print(json.dumps(out))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
