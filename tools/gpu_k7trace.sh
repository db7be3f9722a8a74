# K7 per-tile traces (TUNING build) under timing experiments: LOWBIT_HALO_DEBUG = 32 | extra
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
rm -f gpurun_out/k7_traces.log
for d in 32 36 160 49 34; do
  echo "== dbg $d" >> gpurun_out/k7_traces.log
  LOWBIT_LIB=paper_2205_09120_b200/build_t/liblowbit_t.so LOWBIT_HALO_DEBUG=$d timeout 120 python tools/halo_trace.py 2>&1 | grep "phases\|steady\|MMA waits" >> gpurun_out/k7_traces.log
done
