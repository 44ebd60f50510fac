set -x
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt
python -m pytest tests -m gpu -x -q -rs > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
SMG_SLOW=1 timeout 900 python -m pytest tests/test_gpu_configs.py -m gpu -q -k c2_fgmres > gpurun_out/pytest_c2_solve.log 2>&1; echo "rc $?" >> gpurun_out/pytest_c2_solve.log
for t in racecheck memcheck synccheck; do
  timeout 600 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_c1.py > gpurun_out/sanitizer_$t.log 2>&1; echo "rc $?" >> gpurun_out/sanitizer_$t.log
done
tail -3 gpurun_out/pytest_gpu.log
