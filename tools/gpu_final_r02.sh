# round-2 closing evidence: all GPU tests, smoke, default bench line
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -rs > gpurun_out/pytest_gpu_final.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu_final.log
tail -3 gpurun_out/pytest_gpu_final.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?"; tail -1 gpurun_out/smoke.log
python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc $?"
python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_reference.json 2>&1; echo "ref rc $?"
tail -c 400 gpurun_out/bench_reference.json
