#!/bin/bash
# ncu --set full of the fp64 vmult (k=2, level 5) and of one smoother colour kernel (fp32)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stokes_vmult -s 2 -c 1 -o gpurun_out/prof -f python tools/prof_vmult.py 2 5 vmult > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:patch_smooth -s 1 -c 1 -o gpurun_out/prof_smooth -f python tools/prof_vmult.py 2 5 smooth > gpurun_out/ncu_smooth.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/prof_vmult.py 2 5 all > gpurun_out/launches.log 2>&1
