"""C2 fp32 transfer times: round-2 row kernels (default) vs the round-1 per-DoF kernels
(SMG_LEGACY_TRANSFER=1), each in a fresh process."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run():
    sys.path.insert(0, ROOT)
    import torch
    import paper_2410_09497_b200 as smg
    k, level = int(sys.argv[2]), int(sys.argv[3])
    ctx = smg.Context(k, level)
    nf, nc = ctx.sizes(level)[4], ctx.sizes(level - 1)[4]
    out = {}
    for dt in (torch.float32, torch.float64):
        f = torch.rand(nf, dtype=dt, device="cuda")
        c = torch.rand(nc, dtype=dt, device="cuda")
        rc = torch.zeros_like(c)
        for name, fn in (("restrict", lambda: ctx.restrict(level - 1, f, out=rc)),
                         ("prolongate_add", lambda: ctx.prolongate_add(level - 1, f, c))):
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(50):
                fn()
            b.record()
            torch.cuda.synchronize()
            out[f"{name}_{str(dt)[-7:]}_ms"] = a.elapsed_time(b) / 50
    print(json.dumps(out))


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--run":
        run()
    else:
        k, level = (sys.argv[1], sys.argv[2]) if len(sys.argv) > 2 else ("2", "5")
        res = {}
        for name, env in (("row_kernels", {}), ("legacy", {"SMG_LEGACY_TRANSFER": "1"})):
            o = subprocess.run([sys.executable, __file__, "--run", k, level], capture_output=True, text=True,
                               env=dict(os.environ, **env), cwd=ROOT)
            res[name] = json.loads(o.stdout.strip().splitlines()[-1]) if o.returncode == 0 else o.stderr[-400:]
        print(json.dumps(res))
