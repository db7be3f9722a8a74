cd "$(dirname "$0")/.."
mkdir -p gpurun_out
bash tools/ab_conv.sh > gpurun_out/k7_ab.log 2>&1
for d in 0 1 16 17 512 4 516 8 128 2; do
  echo -n "dbg $d: " >> gpurun_out/k7_dbg.log
  LOWBIT_LIB=paper_2205_09120_b200/build_t/liblowbit_t.so LOWBIT_HALO_DEBUG=$d KERNELS=2 timeout 120 python tools/conv_c4_time.py 2>&1 | tail -1 >> gpurun_out/k7_dbg.log
done
