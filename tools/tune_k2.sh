# k=2 brick-shape variants at C2 (library built with TUNE=1): fp64 / fp32 apply time per variant
mkdir -p gpurun_out
: > gpurun_out/tune_k2.txt
for v in ${VARS:-0 1 2 3 4 5 6 7 8 9 0}; do
  echo "variant $v $(SMG_VMULT_VARIANT=$v timeout 300 python tools/zm_check.py --time 2 5 2>&1 | tail -1)" >> gpurun_out/tune_k2.txt
done
cat gpurun_out/tune_k2.txt
