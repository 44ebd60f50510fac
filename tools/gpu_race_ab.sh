mkdir -p gpurun_out
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_c1.py > gpurun_out/sanitizer_racecheck.log 2>&1; echo "rc $?" >> gpurun_out/sanitizer_racecheck.log
grep -h "RACECHECK SUMMARY\|ERROR SUMMARY" gpurun_out/sanitizer_racecheck.log
AB_CASES="${AB_CASES:-2:5 1:5 3:5}" bash tools/gpu_ab_vmult.sh
