CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra --no-e2e"
timeout -s KILL 300 $CMD > gpurun_out/plain_p.log 2>&1 && \
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 1 -c 1 -o gpurun_out/prof_pair2_c5 $CMD > gpurun_out/ncu_pair.log 2>&1
echo FULL=$?
