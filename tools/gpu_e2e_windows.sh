# host pipeline (shifted output windows, tapered chunks): parity tests, then wall time per call vs chunking
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "host" > gpurun_out/e2ew_tests.log 2>&1; echo "rc $?" >> gpurun_out/e2ew_tests.log
tail -3 gpurun_out/e2ew_tests.log
python - <<'PY' 2>&1 | tee gpurun_out/e2e_windows.txt
import os, sys, time, numpy as np, torch
sys.path.insert(0, ".")
import paper_2410_09497_b200 as smg
k, level = 2, 5
ctx = smg.Context(k, level)
s = ctx.sizes(level)
xb = [torch.empty(s[i], dtype=torch.float64, pin_memory=True).numpy() for i in range(4)]
yb = [torch.empty(s[i], dtype=torch.float64, pin_memory=True).numpy() for i in range(4)]
for a in xb:
    a[:] = np.random.default_rng(0).standard_normal(a.size)
for rep in range(2):
    for taper in ("0", "1"):
        for n in ("8", "16", "32"):
            os.environ["SMG_HOST_CHUNKS"] = n
            os.environ["SMG_HOST_TAPER"] = taper
            for _ in range(3):
                ctx.vmult_host(level, xb, smg.F64, out=yb)
            t0 = time.perf_counter()
            for _ in range(20):
                ctx.vmult_host(level, xb, smg.F64, out=yb)
            t = (time.perf_counter() - t0) / 20
            print(f"rep {rep} taper {taper} chunks {n}: {t*1e3:.3f} ms {s[4]/t/1e9:.3f} GDoF/s", flush=True)
PY
