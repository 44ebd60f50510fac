# brick-shape variants per degree (library built with TUNE=1): KV="k:v1,v2,... k:..." fp64/fp32 apply times
mkdir -p gpurun_out
: > gpurun_out/tune_all.txt
for kv in ${KV:-"1:0,1,2,4,5,6,7,8,0" "3:0,1,3,4,5,6,7,8,0" "4:0,1,2,3,4,5,6,0"}; do
  k=${kv%%:*}; lv=5; [ $k -ge 4 ] && lv=4
  for v in $(echo ${kv#*:} | tr ',' ' '); do
    echo "k $k level $lv variant $v $(SMG_VMULT_VARIANT=$v timeout 300 python tools/zm_check.py --time $k $lv 2>&1 | tail -1)" >> gpurun_out/tune_all.txt
  done
done
cat gpurun_out/tune_all.txt
