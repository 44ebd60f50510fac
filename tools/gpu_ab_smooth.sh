# candidate build: smoother GPU parity tests, then A/B timing of one smoothing step against ab/base.so
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -q -x -k "smooth or vcycle or fgmres or solve or fused or patch" > gpurun_out/ab_tests.log 2>&1; echo "rc $?" >> gpurun_out/ab_tests.log
tail -3 gpurun_out/ab_tests.log
python tools/ab_lib.py smooth ${AB_CASES:-2:5 2:4 1:5 3:4} | tee gpurun_out/ab_smooth.jsonl
