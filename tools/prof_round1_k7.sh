# Round-1 evidence after K7: GPU tests, the default bench line, the launch list
# of the bench's headline command, one --set full capture each of K5 (c5) and
# K7 (c4), each after its plain run exits 0.
set -x
timeout -s KILL 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_s2.log 2>&1; echo TESTS=$?
timeout -s KILL 600 python bench.py > gpurun_out/bench_s2.json 2> gpurun_out/bench_s2.err; echo BENCH=$?
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extra --no-e2e"
timeout -s KILL 300 $CMD > gpurun_out/plain_k7.log 2>&1 && \
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_s2.csv $CMD > gpurun_out/ncu_launch_k7.log 2>&1
echo LAUNCH=$?
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:gemm_fp4_pair -s 1 -c 1 -o gpurun_out/k5_full_s2 $CMD > gpurun_out/ncu_full_k5.log 2>&1
echo FULL5=$?
CMDC="python tools/conv_once.py"
timeout -s KILL 300 $CMDC > gpurun_out/plain_conv.log 2>&1 && \
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:conv_fp4_halo -s 2 -c 1 -o gpurun_out/k7_full $CMDC > gpurun_out/ncu_full_k7.log 2>&1
echo FULL7=$?
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4_k7.csv $CMDC > /dev/null 2>&1
echo LAUNCHC=$?
tail -3 gpurun_out/gpu_tests_s2.log
