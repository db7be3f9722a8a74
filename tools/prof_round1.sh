set -x
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra --no-e2e"
timeout -s KILL 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c5.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo LAUNCH=$?
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 1 -c 1 -o gpurun_out/prof_tc_c5 $CMD > gpurun_out/ncu_full.log 2>&1
echo FULL=$?
CMD3="python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline --no-extra --no-e2e"
timeout -s KILL 300 $CMD3 > gpurun_out/plain3.log 2>&1 && \
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 1 -c 1 -o gpurun_out/prof_tc_c3 $CMD3 > gpurun_out/ncu_full3.log 2>&1
echo FULL3=$?
CMD4="python bench.py --config c3 --kernel bitserial --steps 2 --warmup 3 --no-cpu-baseline --no-extra --no-e2e"
timeout -s KILL 300 $CMD4 > gpurun_out/plain4.log 2>&1 && \
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:gemm_bitserial -s 1 -c 1 -o gpurun_out/prof_bs_c3 $CMD4 > gpurun_out/ncu_full4.log 2>&1
echo FULL4=$?
tail -3 gpurun_out/plain.log gpurun_out/plain3.log
