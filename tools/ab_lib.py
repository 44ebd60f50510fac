"""A/B timing of two builds of libsmg_b200.so on the same box: the candidate (in-tree) and a baseline copy
(ab/base.so, git-ignored scratch). Each measurement runs in a fresh process with the chosen library copied
in place; the in-tree candidate is restored at the end.
Usage: python tools/ab_lib.py [vmult|smooth|e2e] [k:level ...]   (default: vmult 2:5 1:5 3:5 4:4)"""
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2410_09497_b200", "libsmg_b200.so")
BASE = os.path.join(ROOT, "ab", "base.so")
CAND = os.path.join(ROOT, "ab", "cand.so")

CHILD = r"""
import json, sys, time, torch
sys.path.insert(0, %r)
import paper_2410_09497_b200 as smg
what, k, level = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
out = {}
if what == "e2e":  # host BlockVector apply (pinned), wall time per call
    import numpy as np
    ctx = smg.Context(k, level)
    s = ctx.sizes(level)
    xb = [torch.empty(s[i], dtype=torch.float64, pin_memory=True).numpy() for i in range(4)]
    yb = [torch.empty(s[i], dtype=torch.float64, pin_memory=True).numpy() for i in range(4)]
    for a in xb:
        a[:] = np.random.default_rng(0).standard_normal(a.size)
    for _ in range(3):
        ctx.vmult_host(level, xb, smg.F64, out=yb)
    t0 = time.perf_counter()
    for _ in range(30):
        ctx.vmult_host(level, xb, smg.F64, out=yb)
    t = (time.perf_counter() - t0) / 30
    print(json.dumps({"f64": {"ms": round(t * 1e3, 3), "gdofs": round(s[4] / t / 1e9, 3)}}))
    sys.exit(0)
for name, dt in (("f64", torch.float64), ("f32", torch.float32)):
    if what == "smooth" and name == "f64":
        continue
    ctx = smg.Context(k, level, cg_max_iter=30, cg_tol=1e-5)
    n = ctx.sizes(level)[4]
    x = (torch.rand(n, dtype=torch.float64, device="cuda") * 2 - 1).to(dt)
    y = torch.empty_like(x)
    reps = 200 if what == "vmult" else 5
    def step():
        if what == "vmult":
            ctx.apply_stokes(level, x, out=y)
        else:
            y.zero_()
            ctx.smooth(level, y, x)
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        step()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    out[name] = {"ms": round(ms, 4), "gdofs": round(n / ms / 1e6, 2)}
print(json.dumps(out))
""" % ROOT


def run(lib, what, k, level):
    shutil.copyfile(lib, LIB)
    r = subprocess.run([sys.executable, "-c", CHILD, what, str(k), str(level)], capture_output=True, text=True, cwd=ROOT)
    if r.returncode != 0:
        return {"error": r.stderr[-400:]}
    return json.loads(r.stdout.strip().splitlines()[-1])


def main():
    what = sys.argv[1] if len(sys.argv) > 1 and sys.argv[1] in ("vmult", "smooth", "e2e") else "vmult"
    cases = [a for a in sys.argv[1:] if ":" in a] or ["2:5", "1:5", "3:5", "4:4"]
    shutil.copyfile(LIB, CAND)
    try:
        for c in cases:
            k, level = map(int, c.split(":"))
            for rep in range(2):  # interleaved: base, cand, base, cand
                rb = run(BASE, what, k, level)
                rc = run(CAND, what, k, level)
                print(json.dumps({"what": what, "k": k, "level": level, "rep": rep, "base": rb, "cand": rc}), flush=True)
    finally:
        shutil.copyfile(CAND, LIB)


if __name__ == "__main__":
    main()
