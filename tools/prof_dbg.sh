CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extra --no-e2e"
for d in 0 1 2; do
LOWBIT_DEBUG_PAIR=$d timeout -s KILL 300 $CMD > gpurun_out/plain_d$d.log 2>&1 && \
LOWBIT_DEBUG_PAIR=$d timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__cycles_active.avg,sm__ops_path_tensor_op_utcimma_src_int8_sparsity_off.sum.pct_of_peak_sustained_elapsed,smsp__inst_executed.sum --clock-control none -k regex:gemm_tc -s 2 -c 3 --csv --log-file gpurun_out/dbg$d.csv $CMD > /dev/null 2>&1
echo D$d=$?
done
