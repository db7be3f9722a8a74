cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for L in 0 2; do echo "== layout $L" >> gpurun_out/fp4stats.log; LAYOUT=$L LOWBIT_LIB=paper_2205_09120_b200/build_t/liblowbit_t.so LOWBIT_DEBUG_FP4=8 timeout 300 python tools/fp4_stats.py >> gpurun_out/fp4stats.log 2>&1; done
