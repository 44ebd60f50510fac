# round-2 bench evidence: default bench line, C3 line, ncu launch list of the bench command, ncu --set
# full of the dominant kernel (DRAM traffic per launch)
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "bench rc $?"
python bench.py --degree 3 --level 6 --no-cpu --steps 100 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "c3 rc $?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r02.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-solve > /dev/null 2>&1; echo "ncu list rc $?"
ncu --set full --clock-control none -k regex:stokes_vmult_kernel -s 2 -c 1 --csv --page raw \
    python tools/prof_vmult.py 2 5 vmult > gpurun_out/ncu_vmult_raw_r02.csv 2>/dev/null; echo "ncu full rc $?"
tail -c 600 gpurun_out/bench_c2.json
