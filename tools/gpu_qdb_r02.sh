# QDB (barrier-free pass-3 release) candidate: vmult parity tests, racecheck / synccheck of the vmult at
# TMA-staged levels, then A/B timing against ab/base.so
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -q -x -k "vmult or residual or slab or dist or staging or operator" > gpurun_out/qdb_tests.log 2>&1; echo "rc $?" >> gpurun_out/qdb_tests.log
tail -3 gpurun_out/qdb_tests.log
cat > /tmp/race_vmult.py <<'PY'
import sys, torch
sys.path.insert(0, ".")
import paper_2410_09497_b200 as smg
for k, level in ((2, 3), (1, 4), (3, 3), (4, 3)):
    ctx = smg.Context(k, level)
    n = ctx.sizes(level)[4]
    for dt in (torch.float64, torch.float32):
        x = (torch.rand(n, dtype=torch.float64) * 2 - 1).to("cuda", dt)
        y = ctx.apply_stokes(level, x)
        r = ctx.residual(level, x, y)
        torch.cuda.synchronize()
        print(k, level, dt, float(y.norm()), float(r.norm()))
print("race workload done")
PY
for tool in racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool python /tmp/race_vmult.py > gpurun_out/qdb_$tool.log 2>&1; echo "rc $?" >> gpurun_out/qdb_$tool.log
  tail -3 gpurun_out/qdb_$tool.log
done
python tools/ab_lib.py vmult ${AB_CASES:-2:5 1:5 3:5 4:4} | tee gpurun_out/ab_qdb.jsonl
