#!/bin/bash
# vmult brick-shape tuning (k=2): each SMG_VMULT_VARIANT, TMA and cp.async staging, plus parity of each variant
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
: > gpurun_out/tune.txt
for v in ${VARIANTS:-0 1 2 3 4 5 6}; do
  echo "variant $v" >> gpurun_out/tune.txt
  SMG_VMULT_VARIANT=$v timeout 120 python tools/sweep.py 5 2 >> gpurun_out/tune.txt 2>&1
  SMG_NO_TMA=1 SMG_VMULT_VARIANT=$v timeout 120 python tools/sweep.py 5 2 | sed 's/^/notma /' >> gpurun_out/tune.txt 2>&1
  SMG_VMULT_VARIANT=$v timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "vmult and (2-" 2>&1 | tail -1 >> gpurun_out/tune.txt
done
