# K7 per-tile trace + phases (TUNING build)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
L=gpurun_out/k7_trace3.log
rm -f $L
for d in ${DBGS:-32}; do
  echo "== dbg $d" >> $L
  LOWBIT_LIB=paper_2205_09120_b200/build_t/liblowbit_t.so LOWBIT_HALO_DEBUG=$d timeout 120 python tools/halo_trace.py >> $L 2>&1
done
