# K7 isolation traces (TUNING build): which role slows the MMA period
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
L=gpurun_out/k7iso.log
rm -f $L
for d in 676 672 548 544 36 160 32; do
  echo "== dbg $d" >> $L
  LOWBIT_LIB=paper_2205_09120_b200/build_t/liblowbit_t.so LOWBIT_HALO_DEBUG=$d timeout 120 python tools/halo_trace.py 2>&1 | grep "phases\|steady\|MMA waits" >> $L
done
