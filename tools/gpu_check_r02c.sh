mkdir -p gpurun_out
python tools/solve_ab.py 2 5 > gpurun_out/solve_ab_c2.json 2>&1; cat gpurun_out/solve_ab_c2.json
python tools/solve_ab.py 3 6 > gpurun_out/solve_ab_c3.json 2>&1; cat gpurun_out/solve_ab_c3.json
python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29600 bench.py --gpus 2 --steps 5 --warmup 3 --dist-backend gloo --no-cpu > gpurun_out/bench_gloo2.json 2> gpurun_out/bench_gloo2.err; echo "gloo2 rc $?"; tail -c 1500 gpurun_out/bench_gloo2.json
