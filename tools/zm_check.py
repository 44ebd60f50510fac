"""z-march operator (vmult_zm.cuh, opt-in with SMG_ZMARCH=1) check + timing: parity against the oracle for k = 1, 2 (fp64 / fp32,
apply / residual, whole level / slab rows) and the C2 apply time next to the brick kernel
(the default). Usage: python tools/zm_check.py [--time-only]"""
import json
import os
import subprocess
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import paper_2410_09497_b200 as smg  # noqa: E402


def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def timing(k, level, dt, reps=200):
    ctx = smg.Context(k, level)
    n = ctx.sizes(level)[4]
    x = (torch.rand(n, dtype=torch.float64, device="cuda") * 2 - 1).to(dt)
    y = torch.empty_like(x)
    for _ in range(5):
        ctx.apply_stokes(level, x, out=y)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        ctx.apply_stokes(level, x, out=y)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    if "--time" not in sys.argv:
        os.environ["SMG_ZMARCH"] = "1"  # parity of the opt-in kernel (read once per process)
    if "--time" in sys.argv:
        k, level = int(sys.argv[2]), int(sys.argv[3])
        out = {}
        for name, dt in (("f64", torch.float64), ("f32", torch.float32)):
            ms = timing(k, level, dt)
            n = smg.level_sizes(k, level)[4]
            out[name] = {"ms": ms, "gdofs": n / ms / 1e6}
        print(json.dumps(out))
        return
    worst = {}
    for k, levels in ((1, (2, 3, 4)), (2, (2, 3, 4))):
        for level in levels:
            ctx = smg.Context(k, level)
            rng = np.random.default_rng(k * 10 + level)
            x = rng.uniform(-1, 1, oracle.sizes(k, level)[4])
            b = rng.uniform(-1, 1, x.size)
            y_ref = oracle.apply_stokes(k, level, x)
            r_ref = b - y_ref
            r_ref[oracle.constrained_mask(k, level)] = 0.0
            for dt, tol in ((torch.float64, 1e-12), (torch.float32, 1e-5)):
                xd = torch.from_numpy(x).to("cuda", dt)
                y = ctx.apply_stokes(level, xd).double().cpu().numpy()
                e1 = rel(y, y_ref)
                r = ctx.residual(level, torch.from_numpy(b).to("cuda", dt), xd).double().cpu().numpy()
                e2 = rel(r, r_ref)
                key = f"k{k}_l{level}_{'f64' if dt == torch.float64 else 'f32'}"
                worst[key] = (e1, e2)
                print(key, "vmult", e1, "resid", e2, "OK" if max(e1, e2) <= tol else "FAIL", flush=True)
    # timing: z-march vs brick kernel at C2 and C1-size k=1 level 5
    res = {}
    for k, level in ((2, 5), (1, 5), (2, 4)):
        env = dict(os.environ, SMG_ZMARCH="1")
        zm = json.loads(subprocess.run([sys.executable, __file__, "--time", str(k), str(level)], capture_output=True,
                                       text=True, cwd=ROOT, env=env).stdout.strip().splitlines()[-1])
        br = json.loads(subprocess.run([sys.executable, __file__, "--time", str(k), str(level)], capture_output=True,
                                       text=True, cwd=ROOT).stdout.strip().splitlines()[-1])
        res[f"k{k}_l{level}"] = {"zmarch": zm, "brick": br}
        print(f"k{k}_l{level}", json.dumps(res[f"k{k}_l{level}"]), flush=True)


if __name__ == "__main__":
    main()
