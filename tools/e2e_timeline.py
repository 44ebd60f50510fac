"""Timeline of one smg_vmult_host call (torch profiler / CUPTI): copies and kernels per stream."""
import json
import time

import numpy as np
import torch

import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_09497_b200 as smg  # noqa: E402

k, level = 2, 5
ctx = smg.Context(k, level)
s = ctx.sizes(level)
xb = [torch.empty(s[i], dtype=torch.float64, pin_memory=True).numpy() for i in range(4)]
yb = [torch.empty(s[i], dtype=torch.float64, pin_memory=True).numpy() for i in range(4)]
rng = np.random.default_rng(0)
for a in xb:
    a[:] = rng.standard_normal(a.size)
for _ in range(3):
    ctx.vmult_host(level, xb, smg.F64, out=yb)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    ctx.vmult_host(level, xb, smg.F64, out=yb)
print("wall ms per call", (time.perf_counter() - t0) / 10 * 1e3)
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA, torch.profiler.ProfilerActivity.CPU]) as prof:
    ctx.vmult_host(level, xb, smg.F64, out=yb)
    torch.cuda.synchronize()
prof.export_chrome_trace("gpurun_out/e2e_trace.json")
ev = json.load(open("gpurun_out/e2e_trace.json"))["traceEvents"]
g = [e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset") and "ts" in e]
t0 = min(e["ts"] for e in g)
for e in sorted(g, key=lambda e: e["ts"]):
    print(f'{e["ts"]-t0:9.1f} {e["dur"]:8.1f} s{e["args"].get("stream")} {e["cat"]:10s} {e["name"][:60]}')
print("span us", max(e["ts"] + e["dur"] for e in g) - t0)
