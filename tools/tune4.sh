#!/bin/bash
# brick-shape variants (build with `make -C paper_2410_09497_b200 TUNE=1` first): KS="2 3" bash tools/tune4.sh
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
: > gpurun_out/tune4.txt
for k in ${KS:-1 3 4}; do
  for v in 0 1 2 3 4; do
    echo "k $k variant $v" >> gpurun_out/tune4.txt
    SMG_VMULT_VARIANT=$v timeout 200 python tools/sweep.py 5 $k >> gpurun_out/tune4.txt 2>&1
  done
done
