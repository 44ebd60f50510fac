# ncu --set full of the fp64 brick operator at k = 5, 6, 7 (level 4), one launch each, + timing
mkdir -p gpurun_out
for k in 5 6 7; do
  ncu --set full --clock-control none --import-source on -k regex:stokes_vmult_kernel -s 2 -c 1 \
      -o gpurun_out/prof_vmult_k$k -f python tools/prof_vmult.py $k 4 vmult > gpurun_out/prof_vmult_k$k.log 2>&1
done
python tools/ab_lib.py vmult 5:4 6:4 7:4 > gpurun_out/high_degree_timing.jsonl 2>&1
ls -la gpurun_out/prof_vmult_k*
