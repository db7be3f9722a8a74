cd "$(dirname "$0")/.."
mkdir -p gpurun_out
L=gpurun_out/tsprof.log
rm -f $L
LOWBIT_LIB=paper_2205_09120_b200/build_t/liblowbit_t.so LOWBIT_HALO_DEBUG=32 timeout 120 python tools/ts_trace.py >> $L 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --warp-sampling-interval 0 -k regex:conv_fp4_ts -s 2 -c 1 -o gpurun_out/ts_prof python tools/conv_once.py > gpurun_out/ts_prof_ncu.log 2>&1
echo NCU=$? >> $L
