# slow-marked parity tests (C2 FGMRES vs oracle, k=5 FGMRES vs oracle) and the high-degree MG at level 4
mkdir -p gpurun_out
SMG_SLOW=1 timeout 1500 python -m pytest tests/test_gpu_configs.py -m gpu -q -k "c2_fgmres or k5_iterations" > gpurun_out/pytest_slow.log 2>&1; echo "rc $?" >> gpurun_out/pytest_slow.log
tail -3 gpurun_out/pytest_slow.log
python - <<'PY' > gpurun_out/high_degree_l4.jsonl 2>&1
import json, time, torch, sys, os
sys.path.insert(0, os.getcwd())
import paper_2410_09497_b200 as smg
for k in (5, 6, 7):
    L = 4
    t0 = time.perf_counter()
    ctx = smg.Context(k, L, cg_max_iter=30, cg_tol=1e-5)
    n = ctx.sizes(L)[4]
    x = torch.rand(n, dtype=torch.float64, device="cuda") * 2 - 1
    b = ctx.apply_stokes(L, x)
    ctx.solve(L, b, 1e-8, 30, smg.F32, allow_not_converged=True)
    torch.cuda.synchronize()
    setup = time.perf_counter() - t0
    t0 = time.perf_counter()
    xs, it, hist = ctx.solve(L, b, 1e-8, 30, smg.F32, allow_not_converged=True)
    torch.cuda.synchronize()
    ts = time.perf_counter() - t0
    r = ctx.residual(L, b, xs)
    print(json.dumps({"k": k, "level": L, "dofs": n, "iterations": it, "rel_res_fgmres": float(hist[-1] / hist[0]),
                      "rel_res_true": float(r.norm() / b.norm()), "solve_s": ts, "setup_plus_first_solve_s": setup}), flush=True)
    del ctx; torch.cuda.empty_cache()
PY
cat gpurun_out/high_degree_l4.jsonl
