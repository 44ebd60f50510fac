# round-2 closing evidence on the final build: sanitizers, all GPU tests, smoke, bench (C2) + reference
# arm, ncu launch list, Table-2 setting, slow oracle tests and high-degree MG
mkdir -p gpurun_out
for t in racecheck memcheck synccheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_c1.py > gpurun_out/sanitizer_$t.log 2>&1; echo "rc $?" >> gpurun_out/sanitizer_$t.log
done
grep -h "ERROR SUMMARY\|RACECHECK SUMMARY" gpurun_out/sanitizer_*.log
bash tools/gpu_final_r02.sh
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r02.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-solve > /dev/null 2>&1; echo "ncu list rc $?"
python tools/table2.py gpurun_out/table2.json > gpurun_out/table2.log 2>&1; echo "table2 rc $?"
bash tools/gpu_slow_r02.sh
