# closing evidence on the final build (QDB + wide A items at k = 2 fp64): all GPU tests, smoke, bench line,
# A/B against the pre-QDB build (ab/base.so), ncu --set full of the brick kernel
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/final2_gpu_tests.log 2>&1; echo "rc $?" >> gpurun_out/final2_gpu_tests.log
tail -3 gpurun_out/final2_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final2_smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/final2_smoke.log
tail -2 gpurun_out/final2_smoke.log
python bench.py > gpurun_out/final2_bench.json 2> gpurun_out/final2_bench.err; echo "bench rc $?"
python tools/ab_lib.py vmult 2:5 2:4 3:5 | tee gpurun_out/ab_final2.jsonl
bash tools/prof_brick.sh
