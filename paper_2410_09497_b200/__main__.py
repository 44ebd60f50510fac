"""Command line of the harness, 3D only, on the B200 solver:

  python -m paper_2410_09497_b200 solve --degree K --level L [--precision double|mixed] [--tol 1e-8]
                                      [--sigma 0.1] [--mu 0.5] [--out PATH.json]
  python -m paper_2410_09497_b200 convergence --degree-range A..B --level-range A..B [--precision ...] --out PATH.csv
  python -m paper_2410_09497_b200 perf --degree K --level L [--reps R] [--warmup W] [--out PATH.json]

Exit code 0 on success, nonzero on solver failure."""
import argparse
import csv
import json
import sys


def _range(s):
    a, b = s.split("..")
    return list(range(int(a), int(b) + 1))


def main(argv=None):
    ap = argparse.ArgumentParser(prog="python -m paper_2410_09497_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    for name in ("solve", "convergence", "perf"):
        p = sub.add_parser(name)
        p.add_argument("--dim", type=int, default=3, choices=[3])
        p.add_argument("--precision", default="mixed", choices=["double", "mixed"])
        p.add_argument("--tol", type=float, default=1e-8)
        p.add_argument("--sigma", type=float, default=0.1)
        p.add_argument("--mu", type=float, default=0.5)
        p.add_argument("--device", type=int, default=0)
        p.add_argument("--out")
        if name == "convergence":
            p.add_argument("--degree-range", required=True)
            p.add_argument("--level-range", required=True)
        else:
            p.add_argument("--degree", type=int, required=True)
            p.add_argument("--level", type=int, required=True)
        if name == "perf":
            p.add_argument("--reps", type=int, default=10)
            p.add_argument("--warmup", type=int, default=3)
    a = ap.parse_args(argv)

    import paper_2410_09497_b200 as smg
    from paper_2410_09497_b200 import harness
    vp = smg.F32 if a.precision == "mixed" else smg.F64
    ms = harness.Manufactured(a.sigma, a.mu)
    if a.cmd == "solve":
        ctx = smg.Context(a.degree, a.level, device=a.device, cg_max_iter=30, cg_tol=1e-5 if vp == smg.F32 else 1e-8)
        rep = harness.solve_manufactured(ctx, a.level, a.tol, 100, vp, ms)
        rep.update({"sigma": a.sigma, "mu": a.mu})
        txt = json.dumps(rep)
        if a.out:
            open(a.out, "w").write(txt + "\n")
        print(txt)
    elif a.cmd == "convergence":
        rows = harness.convergence_study(_range(a.degree_range), _range(a.level_range), a.tol, vp, a.device)
        cols = ["dim", "degree", "level", "dofs", "iterations", "nu", "err_u", "err_p", "time_total_s", "dofs_per_s",
                "precision", "local_solver", "order_u", "order_p", "div_l2"]
        w = csv.DictWriter(open(a.out, "w", newline="") if a.out else sys.stdout, fieldnames=cols, extrasaction="ignore")
        w.writeheader()
        for r in rows:
            w.writerow(r)
    else:
        import torch
        ctx = smg.Context(a.degree, a.level, device=a.device)
        n = ctx.sizes(a.level)[4]
        res = {}
        for name, dt in (("vmult_f64", torch.float64), ("vmult_f32", torch.float32)):
            x = torch.rand(n, dtype=dt, device=f"cuda:{a.device}")
            y = torch.empty_like(x)
            for _ in range(a.warmup):
                ctx.apply_stokes(a.level, x, out=y)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.reps):
                ctx.apply_stokes(a.level, x, out=y)
            e1.record()
            torch.cuda.synchronize()
            res[name] = n * a.reps / (e0.elapsed_time(e1) * 1e-3)
        b = torch.rand(n, dtype=torch.float32, device=f"cuda:{a.device}")
        xs = torch.zeros_like(b)
        ctx.smooth(a.level, xs, b)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(max(1, a.reps // 3)):
            ctx.smooth(a.level, xs, b)
        e1.record()
        torch.cuda.synchronize()
        res["smooth_f32"] = n * max(1, a.reps // 3) / (e0.elapsed_time(e1) * 1e-3)
        rep = {"degree": a.degree, "level": a.level, "dofs": n, "dofs_per_s": res}
        if a.out:
            open(a.out, "w").write(json.dumps(rep) + "\n")
        print(json.dumps(rep))
    return 0


if __name__ == "__main__":
    sys.exit(main())
