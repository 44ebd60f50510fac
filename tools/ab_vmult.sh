# vmult parity tests + C2 timing (fp64/fp32) of the default kernel
python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -q -x -k "vmult or residual" 2>&1 | tail -2
python tools/zm_check.py --time 2 5
python tools/zm_check.py --time 2 5
