#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
SMG_NO_TMA=1 timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "slab" > gpurun_out/slab_notma.log 2>&1
timeout 600 compute-sanitizer --tool memcheck --print-limit 5 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "slab and 3-3-4" > gpurun_out/slab_memcheck.log 2>&1
