#!/bin/bash
# full check: GPU tests, smoke, bench (N=1), multi-rank logic check, launch list, ncu full of the vmult
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu --maxfail=8 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
bash tools/multi_rank_check.sh
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/prof_vmult.py 2 5 all > gpurun_out/launches.log 2>&1
if [ "${NCU:-1}" != "0" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:stokes_vmult -s 2 -c 1 -o gpurun_out/prof -f python tools/prof_vmult.py 2 5 vmult > gpurun_out/ncu_full.log 2>&1
fi
