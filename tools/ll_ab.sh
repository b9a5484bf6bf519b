mkdir -p gpurun_out
for v in left right; do
TCG_CHOL=$v timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/setup_cfg3_$v.csv python tools/setup_once.py cfg3 > gpurun_out/ncu_$v.log 2>&1
echo $v rc $?
done
