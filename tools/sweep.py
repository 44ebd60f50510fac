"""vmult timing sweep: python tools/sweep.py [level] [k,...] -> ms, GDoF/s and HBM fraction per (k, precision)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2410_09497_b200 as smg

level = int(sys.argv[1]) if len(sys.argv) > 1 else 5
ks = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1, 2, 3, 4, 5, 6, 7]
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]
for k in ks:
    ctx = smg.Context(k, level)
    n = ctx.sizes(level)[4]
    for dt in (torch.float64, torch.float32):
        x = torch.rand(n, dtype=dt, device="cuda")
        y = torch.empty_like(x)
        for _ in range(3):
            ctx.apply_stokes(level, x, out=y)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10
        e0.record()
        for _ in range(reps):
            ctx.apply_stokes(level, x, out=y)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        gb = 2 * x.element_size() * n / (ms * 1e-3) / 1e9
        print(json.dumps({"k": k, "level": level, "dtype": str(dt)[6:], "dofs": n, "ms": round(ms, 4),
                          "GDoF/s": round(n / ms / 1e6, 2), "GB/s": round(gb, 1), "hbm_frac": round(gb / peak, 4)}), flush=True)
    del ctx
    torch.cuda.empty_cache()
