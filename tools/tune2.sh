#!/bin/bash
# brick-shape variants for k=1,2,3 (fp64 + fp32, TMA) at level 5
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
: > gpurun_out/tune2.txt
for k in 1 2 3; do
  for v in 0 1 2 3 4 5; do
    echo "k $k variant $v" >> gpurun_out/tune2.txt
    SMG_VMULT_VARIANT=$v timeout 120 python tools/sweep.py 5 $k >> gpurun_out/tune2.txt 2>&1
  done
done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "vmult or slab" > gpurun_out/pytest_vmult.log 2>&1
