#!/bin/bash
# quick perf check: sweep (TMA and cp.async paths) + optional ncu capture of the k=2 fp64 vmult
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 300 python tools/sweep.py ${LEVEL:-5} ${KS:-1,2,3,4} > gpurun_out/sweep.txt 2>&1
SMG_NO_TMA=1 timeout 300 python tools/sweep.py ${LEVEL:-5} ${KS:-1,2,3,4} > gpurun_out/sweep_notma.txt 2>&1
if [ -n "$NCU" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:stokes_vmult -s 2 -c 1 -o gpurun_out/prof -f python tools/prof_vmult.py 2 5 vmult > gpurun_out/ncu_full.log 2>&1
fi
