# closing evidence on the final build: all GPU tests, smoke, bench line
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/final3_gpu_tests.log 2>&1; echo "rc $?" >> gpurun_out/final3_gpu_tests.log
tail -3 gpurun_out/final3_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final3_smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/final3_smoke.log
tail -2 gpurun_out/final3_smoke.log
python bench.py > gpurun_out/final3_bench.json 2> gpurun_out/final3_bench.err; echo "bench rc $?"
