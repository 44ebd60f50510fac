# closing ncu evidence: brick operator (C2 fp64) and warp-per-patch smoother (C2 fp32), --set full with source
mkdir -p gpurun_out
bash tools/prof_brick.sh
ncu --set full --clock-control none --import-source on -k regex:patch_smooth_kernel -s 4 -c 1 \
    -o gpurun_out/prof_smoother_k2 -f python tools/prof_vmult.py 2 5 smooth > gpurun_out/prof_smoother.log 2>&1
ls -la gpurun_out/prof_*k2*
