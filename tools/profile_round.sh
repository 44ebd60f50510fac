#!/bin/bash
# Evidence for profiles/: GPU tests, smoke, bench (N=1, reference arm), degree sweep (C4) and C3 size,
# launch list of a bench-like run, ncu --set full of the vmult and of one smoother colour.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt 2>&1
(nproc; lscpu | grep "Model name") > gpurun_out/host.txt
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 python tools/sweep.py 5 1,2,3,4,5,6,7 > gpurun_out/sweep_l5.txt 2>&1
timeout 600 python tools/sweep.py 6 3 > gpurun_out/sweep_c3.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/prof_vmult.py 2 5 all > gpurun_out/launches.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stokes_vmult -s 2 -c 1 -o gpurun_out/prof -f python tools/prof_vmult.py 2 5 vmult > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:patch_smooth -s 1 -c 1 -o gpurun_out/prof_smooth -f python tools/prof_vmult.py 2 5 smooth > gpurun_out/ncu_smooth.log 2>&1
