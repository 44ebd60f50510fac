# round-2 GPU pass: full GPU tests, default bench line, Table-2 reproduction
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -rs > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $?"
tail -c 3000 gpurun_out/bench.json
python tools/table2.py gpurun_out/table2.json > gpurun_out/table2.log 2>&1; echo "table2 rc $?"
cat gpurun_out/table2.log | tail -4
