#!/bin/bash
# multi-rank bench path on a 1-GPU box: 2 and 4 ranks sharing cuda:0 over gloo (logic check only)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
for n in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29517 \
    bench.py --gpus $n --steps 3 --warmup 3 --dist-backend gloo > gpurun_out/bench_multi_$n.json 2> gpurun_out/bench_multi_$n.err
  echo "n=$n rc=$?" >> gpurun_out/bench_multi.rc
done
