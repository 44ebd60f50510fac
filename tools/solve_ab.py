"""C2 MG-FGMRES solve: time / iterations / host syncs with the batched CGS2 + graph-captured V-cycle
(default) against SMG_KRYLOV_MGS=1 SMG_NO_GRAPH=1 (round-1 behaviour), each in a fresh process."""
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run():
    sys.path.insert(0, ROOT)
    import torch
    import paper_2410_09497_b200 as smg
    k, level = int(sys.argv[2]), int(sys.argv[3])
    ctx = smg.Context(k, level, cg_max_iter=30, cg_tol=1e-5)
    n = ctx.sizes(level)[4]
    g = torch.Generator(device="cuda").manual_seed(1234)
    x = torch.rand(n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    b = ctx.apply_stokes(level, x)
    ctx.solve(level, b, 1e-8, 30, smg.F32, allow_not_converged=True)
    torch.cuda.synchronize()
    l0 = ctx.launch_count
    t0 = time.perf_counter()
    xs, it, hist = ctx.solve(level, b, 1e-8, 30, smg.F32, allow_not_converged=True)
    torch.cuda.synchronize()
    t = time.perf_counter() - t0
    print(json.dumps({"time_s": t, "iterations": it, "rel_res": float(hist[-1] / hist[0]),
                      "launches": ctx.launch_count - l0, "x_norm": float(xs.norm())}))


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--run":
        run()
    else:
        k, level = (sys.argv[1], sys.argv[2]) if len(sys.argv) > 2 else ("2", "5")
        res = {}
        for name, env in (("graph_cgs2", {}), ("plain_mgs", {"SMG_KRYLOV_MGS": "1", "SMG_NO_GRAPH": "1"})):
            out = subprocess.run([sys.executable, __file__, "--run", k, level], capture_output=True, text=True,
                                 env=dict(os.environ, **env), cwd=ROOT)
            res[name] = json.loads(out.stdout.strip().splitlines()[-1]) if out.returncode == 0 else out.stderr[-500:]
        print(json.dumps(res))
