# in-tree candidate: full GPU test suite + smoke; then A/B of each ab/<name>.so in $CANDS against ab/base.so
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x > gpurun_out/${TAG}_gpu_tests.log 2>&1; echo "rc $?" >> gpurun_out/${TAG}_gpu_tests.log
tail -3 gpurun_out/${TAG}_gpu_tests.log
cp paper_2410_09497_b200/libsmg_b200.so ab/_intree.so
for c in $CANDS; do
  cp ab/$c.so paper_2410_09497_b200/libsmg_b200.so
  python tools/ab_lib.py vmult ${AB_CASES:-2:5 3:5} | sed "s/^/{\"cand_lib\": \"$c\", \"r\": /; s/$/}/" | tee -a gpurun_out/ab_$TAG.jsonl
done
cp ab/_intree.so paper_2410_09497_b200/libsmg_b200.so
python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc $?"
tail -c 600 gpurun_out/${TAG}_bench.json
