# ncu evidence of the QDB build: brick operator --set full (C2 fp64), bench launch list, smoke
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/qdb_smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/qdb_smoke.log
tail -2 gpurun_out/qdb_smoke.log
bash tools/prof_brick.sh
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_qdb.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-solve > /dev/null 2>&1; echo "ncu list rc $?"
