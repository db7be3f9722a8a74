# Round-2 evidence on the B200: GPU suite, the default bench line, the launch list of the
# same bench command, and one --set full capture each of K5 (c5) and K7 (c4) — every ncu run
# only after its plain command exited 0.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout -s KILL 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2_pytest.log 2>&1
echo PYTEST=$? >> gpurun_out/r2_pytest.log
timeout -s KILL 900 python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err
echo BENCH=$? >> gpurun_out/r2_pytest.log
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extra --no-e2e"
timeout 300 $CMD > gpurun_out/r2_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches_c5.csv $CMD > gpurun_out/r2_ncu_launch.log 2>&1
echo LAUNCH=$? >> gpurun_out/r2_pytest.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_fp4_pair -s 1 -c 1 -o gpurun_out/r2_k5_c5 $CMD > gpurun_out/r2_ncu_k5.log 2>&1
echo FULLK5=$? >> gpurun_out/r2_pytest.log
timeout 120 python tools/conv_once.py > gpurun_out/r2_conv_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_fp4_ -s 2 -c 1 -o gpurun_out/r2_k7_c4 python tools/conv_once.py > gpurun_out/r2_ncu_k7.log 2>&1
echo FULLK7=$? >> gpurun_out/r2_pytest.log
