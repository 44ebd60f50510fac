# ncu --set full + source of the brick vmult kernel at C2 (k=2, level 5, fp64), one launch
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:stokes_vmult_kernel -s 2 -c 1 \
    -o gpurun_out/prof_brick_k2 -f python tools/prof_vmult.py 2 5 vmult > gpurun_out/prof_brick.log 2>&1
ncu -i gpurun_out/prof_brick_k2.ncu-rep --page source --csv > gpurun_out/prof_brick_source.csv 2>&1
ncu -i gpurun_out/prof_brick_k2.ncu-rep --page details --csv > gpurun_out/prof_brick_details.csv 2>&1
ls -la gpurun_out/prof_brick*
