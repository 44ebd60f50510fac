# per-launch durations of one C2 fp32 smoothing step (per-patch modes 1/2 + batched CG) + ncu of one batched launch
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'patch_' --csv \
    python tools/prof_vmult.py 2 5 smooth > gpurun_out/batched_launches.csv 2>&1
ncu --set full --clock-control none --import-source on -k regex:patch_cg_batched -s 2 -c 1 \
    -o gpurun_out/prof_batched -f python tools/prof_vmult.py 2 5 smooth > gpurun_out/prof_batched.log 2>&1
ls -la gpurun_out/prof_batched*
