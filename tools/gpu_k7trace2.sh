# K7 full per-tile traces (TUNING build), plus timing-experiment variants
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
L=gpurun_out/k7_trace2.log
rm -f $L
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv >> $L
for d in 32 160 36 34 544; do
  echo "== dbg $d" >> $L
  LOWBIT_LIB=paper_2205_09120_b200/build_t/liblowbit_t.so LOWBIT_HALO_DEBUG=$d timeout 120 python tools/halo_trace.py >> $L 2>&1
done
LOWBIT_LIB=paper_2205_09120_b200/build_t/liblowbit_t.so KERNELS=2 timeout 300 python tools/conv_c4_time.py >> $L 2>&1
