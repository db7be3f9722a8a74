# Round-1 final evidence: launch list of the default bench command and one
# --set full capture per headline kernel (each after its plain run exits 0).
set -x
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extra --no-e2e"
timeout -s KILL 300 $CMD > gpurun_out/plain_final.log 2>&1 && \
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_final.csv $CMD > gpurun_out/ncu_launch_final.log 2>&1
echo LAUNCH=$?
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_pair -s 1 -c 1 -o gpurun_out/final_c5_pair $CMD > gpurun_out/ncu_full_c5.log 2>&1
echo FULL5=$?
CMD3="python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline --no-extra --no-e2e"
timeout -s KILL 300 $CMD3 > gpurun_out/plain_final3.log 2>&1 && \
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_pair -s 1 -c 1 -o gpurun_out/final_c3_pair $CMD3 > gpurun_out/ncu_full_c3.log 2>&1
echo FULL3=$?
CMDC="python tools/conv_once.py"
timeout -s KILL 300 $CMDC > gpurun_out/plain_conv.log 2>&1 && \
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_pair -s 1 -c 1 -o gpurun_out/final_c4_conv $CMDC > gpurun_out/ncu_full_c4.log 2>&1
echo FULLC=$?
