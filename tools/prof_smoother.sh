# ncu --set full + source of the fp32 patch smoother (warp-per-patch variant) at C2, one launch
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:patch_smooth_kernel -s 4 -c 1 \
    -o gpurun_out/prof_smoother_k2 -f python tools/prof_vmult.py 2 5 smooth > gpurun_out/prof_smoother.log 2>&1
ncu -i gpurun_out/prof_smoother_k2.ncu-rep --page source --csv > gpurun_out/prof_smoother_source.csv 2>&1
ncu -i gpurun_out/prof_smoother_k2.ncu-rep --page details --csv > gpurun_out/prof_smoother_details.csv 2>&1
ls -la gpurun_out/prof_smoother*
