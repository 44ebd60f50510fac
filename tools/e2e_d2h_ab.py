"""Host BlockVector apply: copy-engine D2H vs SM-store D2H (SMG_HOST_D2H_KERNEL=1), alternating processes."""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import json, sys, time, torch, numpy as np
sys.path.insert(0, %r)
import paper_2410_09497_b200 as smg
k, level = 2, 5
ctx = smg.Context(k, level)
s = ctx.sizes(level)
xb = [torch.empty(s[i], dtype=torch.float64, pin_memory=True).numpy() for i in range(4)]
yb = [torch.empty(s[i], dtype=torch.float64, pin_memory=True).numpy() for i in range(4)]
for a in xb: a[:] = np.random.default_rng(0).standard_normal(a.size)
for _ in range(3): ctx.vmult_host(level, xb, smg.F64, out=yb)
ref = [y.copy() for y in yb]
t0 = time.perf_counter()
for _ in range(30): ctx.vmult_host(level, xb, smg.F64, out=yb)
t = (time.perf_counter() - t0) / 30
err = max(float(np.abs(a - b).max()) for a, b in zip(yb, ref))
print(json.dumps({"ms": round(t * 1e3, 3), "gdofs": round(s[4] / t / 1e9, 3), "max_diff": err}))
""" % ROOT
for rep in range(3):
    for mode in ("0", "1"):
        env = dict(os.environ, SMG_HOST_D2H_KERNEL=mode)
        r = subprocess.run([sys.executable, "-c", CHILD], capture_output=True, text=True, env=env)
        print(mode, r.stdout.strip().splitlines()[-1] if r.returncode == 0 else r.stderr[-300:], flush=True)
