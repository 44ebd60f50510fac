"""Tiny driver for ncu: a few fp64 (and fp32) vmults at the bench workload, plus one smoothing step."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2410_09497_b200 as smg

k = int(sys.argv[1]) if len(sys.argv) > 1 else 2
level = int(sys.argv[2]) if len(sys.argv) > 2 else 5
what = sys.argv[3] if len(sys.argv) > 3 else "vmult"
ctx = smg.Context(k, level, cg_max_iter=30, cg_tol=1e-5)
n = ctx.sizes(level)[4]
x = torch.rand(n, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
for _ in range(3):
    ctx.apply_stokes(level, x, out=y)
if what in ("all", "smooth"):
    x32 = x.float()
    b32 = ctx.apply_stokes(level, x32)
    xs = torch.zeros_like(b32)
    ctx.smooth(level, xs, b32)
if what in ("all", "vmult32"):
    x32 = x.float()
    for _ in range(3):
        ctx.apply_stokes(level, x32)
torch.cuda.synchronize()
print("done", ctx.launch_count)
