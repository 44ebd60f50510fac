#!/bin/bash
# TMA probe variants + the cp.async (SMG_NO_TMA) path through the GPU parity tests and the bench.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
for v in 0 1 8 9 11 12 13 14 15 16 17; do timeout 20 ./tools/tma_test $v; done > gpurun_out/tma_probe.txt 2>&1
SMG_NO_TMA=1 timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_notma.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_notma.log
SMG_NO_TMA=1 timeout 600 python bench.py --no-cpu > gpurun_out/bench_notma.json 2> gpurun_out/bench_notma.err
