"""Reproduction of the paper's Table 2 setting on one B200: RT_2 and RT_4 on 32^3
cells (level 4), MG-FGMRES to a relative tolerance of 1e-6. Reports, like the paper's
rows: DoF, mat-vec (fp64 operator apply) ns/DoF, one smoothing step (fp32) ns/DoF, GMRES iterations,
time to solution ns/DoF (fp64 FGMRES + fp32 V-cycle), next to the paper's A100 numbers.
Usage: python tools/table2.py [out.json]"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_09497_b200 as smg  # noqa: E402

PAPER_A100 = {2: {"dofs": "3.57 M", "matvec_ns": 0.535, "smooth_ns": 7.576, "iterations": 3, "solve_ns": 63.694},
              4: {"dofs": "16.5 M", "matvec_ns": 0.813, "smooth_ns": 10.582, "iterations": 3, "solve_ns": 79.365}}


def ev_time(fn, reps):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e-3


def main():
    rows = []
    level = 4
    for k in (2, 4):
        t0 = time.perf_counter()
        ctx = smg.Context(k, level, cg_max_iter=30, cg_tol=1e-5, cg_fixed=False, cg_precond=1)
        n = ctx.sizes(level)[4]
        g = torch.Generator(device="cuda").manual_seed(7)
        x = torch.rand(n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
        y = torch.empty_like(x)
        t_mv = ev_time(lambda: ctx.apply_stokes(level, x, out=y), 50)
        b32 = ctx.apply_stokes(level, x).float()
        xs = torch.zeros_like(b32)
        ctx.smoother_stats(reset=True)
        t_sm = ev_time(lambda: ctx.smooth(level, xs, b32, zero_init=True), 10)
        npatch, cgit = ctx.smoother_stats(reset=True)
        b = ctx.apply_stokes(level, x)
        ctx.solve(level, b, 1e-6, 30, smg.F32, allow_not_converged=True)  # warm-up incl. coarse setup
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        _, it, hist = ctx.solve(level, b, 1e-6, 30, smg.F32, allow_not_converged=True)
        torch.cuda.synchronize()
        t_solve = time.perf_counter() - t1
        rows.append({"k": k, "level": level, "cells": "32^3", "dofs": n, "matvec_ns_per_dof": t_mv / n * 1e9,
                     "smooth_ns_per_dof": t_sm / n * 1e9, "mean_inner_cg_iterations": cgit / max(npatch, 1),
                     "gmres_iterations": it, "rel_residual": float(hist[-1] / hist[0]),
                     "solve_ns_per_dof": t_solve / n * 1e9, "setup_s": time.perf_counter() - t0 - t_solve,
                     "paper_a100": PAPER_A100[k]})
        print(json.dumps(rows[-1]), flush=True)
        del ctx
        torch.cuda.empty_cache()
    if len(sys.argv) > 1:
        with open(sys.argv[1], "w") as f:
            json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()
