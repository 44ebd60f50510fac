"""Time the V-cycle and its pieces per level (CUDA events): python tools/vcycle_time.py [k] [L]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2410_09497_b200 as smg

k = int(sys.argv[1]) if len(sys.argv) > 1 else 2
L = int(sys.argv[2]) if len(sys.argv) > 2 else 5
ctx = smg.Context(k, L, cg_max_iter=30, cg_tol=1e-5)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

def t(fn, reps=3):
    fn(); torch.cuda.synchronize()
    e0.record()
    w0 = time.perf_counter()
    for _ in range(reps):
        fn()
    w1 = time.perf_counter()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, (w1 - w0) / reps * 1e3

for lvl in range(L, 0, -1):
    n = ctx.sizes(lvl)[4]
    b = torch.rand(n, dtype=torch.float32, device="cuda")
    x = torch.zeros_like(b)
    l0 = ctx.launch_count
    ms_s, wall_s = t(lambda: ctx.smooth(lvl, x, b))
    nl_s = (ctx.launch_count - l0) // 4
    l0 = ctx.launch_count
    ms_v, wall_v = t(lambda: ctx.vcycle(lvl, b))
    nl_v = (ctx.launch_count - l0) // 4
    print(f"level {lvl}: smooth {ms_s:8.3f} ms ({nl_s} launches, host {wall_s:.3f} ms)   vcycle {ms_v:8.3f} ms ({nl_v} launches, host {wall_v:.3f} ms)")
b0 = torch.rand(ctx.sizes(0)[4], dtype=torch.float32, device="cuda")
print("coarse solve ms", t(lambda: ctx.coarse_solve(b0)))
bb = ctx.apply_stokes(L, torch.rand(ctx.sizes(L)[4], dtype=torch.float64, device="cuda"))
ctx.solve(L, bb, 1e-8, 30, smg.F32)
torch.cuda.synchronize()
w = time.perf_counter(); l0 = ctx.launch_count
x, it, hist = ctx.solve(L, bb, 1e-8, 30, smg.F32)
torch.cuda.synchronize()
print(f"solve {time.perf_counter() - w:.4f} s, {it} its, {ctx.launch_count - l0} launches")
