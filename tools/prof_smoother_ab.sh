# ncu --set full of one C2 fp32 smoother colour launch for ab/base.so and the in-tree candidate
mkdir -p gpurun_out
cp paper_2410_09497_b200/libsmg_b200.so ab/cand.so
for v in base cand; do
  cp ab/$v.so paper_2410_09497_b200/libsmg_b200.so
  ncu --set full --clock-control none --import-source on -k regex:patch_smooth_kernel -s 4 -c 1 \
      -o gpurun_out/prof_smoother_$v -f python tools/prof_vmult.py 2 5 smooth > gpurun_out/prof_smoother_$v.log 2>&1
done
cp ab/cand.so paper_2410_09497_b200/libsmg_b200.so
ls -la gpurun_out/prof_smoother_*
