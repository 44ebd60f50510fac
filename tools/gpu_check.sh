#!/bin/bash
# One gpurun call: GPU tests, smoke, bench, launch list, optional ncu full capture.
#   KEXPR  pytest -k expression (default: all GPU tests)
#   NCU    regex of the kernel to capture with ncu --set full (default stokes_vmult; "none" to skip)
#   NCUARGS args of tools/prof_vmult.py for the ncu runs (default "2 5 vmult")
#   BENCH  extra bench.py args
set -x
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
nproc > gpurun_out/nproc.txt; lscpu | grep "Model name" >> gpurun_out/nproc.txt
if [ -n "$KEXPR" ]; then K="-k $KEXPR"; else K=""; fi
timeout 900 python -m pytest tests -q -m gpu --maxfail=8 $K > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py $BENCH > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/prof_vmult.py 2 5 all > gpurun_out/launches.log 2>&1
NCU=${NCU:-stokes_vmult}
NCUARGS=${NCUARGS:-"2 5 vmult"}
if [ "$NCU" != "none" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$NCU -s 2 -c 1 -o gpurun_out/prof -f python tools/prof_vmult.py $NCUARGS > gpurun_out/ncu_full.log 2>&1
fi
ls -la gpurun_out
