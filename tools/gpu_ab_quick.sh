# candidate build (in-tree): vmult parity tests, then A/B timing against ab/base.so -> gpurun_out/ab_$TAG.jsonl
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -q -x -k "vmult or residual or slab or dist or staging or operator" > gpurun_out/${TAG}_tests.log 2>&1; echo "rc $?" >> gpurun_out/${TAG}_tests.log
tail -3 gpurun_out/${TAG}_tests.log
python tools/ab_lib.py vmult ${AB_CASES:-2:5 1:5 3:5 4:4} | tee gpurun_out/ab_$TAG.jsonl
