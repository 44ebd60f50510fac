"""Deterministic smoother timing (fixed inner CG iterations): python tools/smooth_ab.py [k] [L] [its]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2410_09497_b200 as smg
k = int(sys.argv[1]) if len(sys.argv) > 1 else 2
L = int(sys.argv[2]) if len(sys.argv) > 2 else 5
its = int(sys.argv[3]) if len(sys.argv) > 3 else 15
ctx = smg.Context(k, L, cg_max_iter=its, cg_fixed=True)
b = torch.rand(ctx.sizes(L)[4], dtype=torch.float32, device="cuda")
x = torch.zeros_like(b)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name, fn in (("smooth", lambda: ctx.smooth(L, x, b, zero_init=True)), ("vcycle", lambda: ctx.vcycle(L, b))):
    fn(); torch.cuda.synchronize()
    e0.record()
    for _ in range(5):
        fn()
    e1.record(); torch.cuda.synchronize()
    print(f"{name} {e0.elapsed_time(e1) / 5:.3f} ms (k={k}, level {L}, {its} fixed CG its)")
