#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
: > gpurun_out/tune3.txt
for v in 0 1 2 3 4 5; do
  echo "k 2 variant $v" >> gpurun_out/tune3.txt
  SMG_VMULT_VARIANT=$v timeout 120 python tools/sweep.py 5 2 >> gpurun_out/tune3.txt 2>&1
  SMG_VMULT_VARIANT=$v timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "vmult and (2-" 2>&1 | tail -1 >> gpurun_out/tune3.txt
done
