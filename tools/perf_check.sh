#!/bin/bash
# GPU parity tests + k=2 brick variants + default sweep over degrees
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu --maxfail=5 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
VARIANTS="${VARIANTS:-0 1 4 5}" bash tools/tune.sh
timeout 600 python tools/sweep.py 5 1,2,3,4 > gpurun_out/sweep.txt 2>&1
