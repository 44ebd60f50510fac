# ncu sections of the z-march vmult at C2 (k=2, level 5, fp64): stall reasons, instruction mix, occupancy
mkdir -p gpurun_out
python - <<'PY' > /dev/null
PY
ncu --kernel-name regex:zm_vmult_kernel --launch-skip 2 --launch-count 1 --clock-control none \
    --section WarpStateStats --section SchedulerStats --section Occupancy --section LaunchStats \
    --section MemoryWorkloadAnalysis --section ComputeWorkloadAnalysis --section InstructionStats \
    --csv --page details python tools/prof_vmult.py 2 5 vmult > gpurun_out/ncu_zm_details.csv 2> gpurun_out/ncu_zm.err
tail -3 gpurun_out/ncu_zm.err
